"""GPU <-> oracle parity for the 2D Sylvester step (S8-S10, Eq. 4.3) through the
C-ABI fde2d_step.  The oracle is the dense Bartels-Stewart solve of oracle/sylvester2d.py
(reading R11: the right-hand side carries dt).  Bar: relative Frobenius error <= 1e-8 per
step with ek_tol 1e-11 and HODLR tol 1e-12 (reading R13)."""
import numpy as np
import pytest
import torch

from oracle.sylvester2d import operators_2d, BartelsStewart
from paper_1804_05522_b200 import workloads as W

gpu = pytest.mark.gpu


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def _stepper(wl, ek_tol=1e-11):
    from paper_1804_05522_b200.hodlr import Fde2dStepper
    return Fde2dStepper(wl.nx, wl.ny, wl.alpha1, wl.alpha2, wl.hx, wl.hy, wl.dt,
                        _t(wl.d1p), _t(wl.d1m), _t(wl.d2p), _t(wl.d2m), wl.tol, ek_tol=ek_tol,
                        leaf=wl.leaf)


def _oracle(wl):
    A1, A2 = operators_2d(wl.alpha1, wl.alpha2, wl.nx, wl.ny, wl.hx, wl.hy, wl.dt,
                          wl.d1p, wl.d1m, wl.d2p, wl.d2m)
    return BartelsStewart(A1, A2)


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _run(wl, K, check_every=True, ek_tol=1e-11):
    st = _stepper(wl, ek_tol=ek_tol)
    bs = _oracle(wl)
    Uo = np.zeros((wl.nx, wl.ny))
    Xu = Xv = None
    errs = []
    for m in range(1, K + 1):
        Fa, Fb = wl.source_factors(m)
        Fu, Fv = _t(Fa.T), _t(Fb.T)
        if Xu is None:
            Xu, Xv, res, its = st.step(Fu, Fv)
        else:
            Xu, Xv, res, its = st.step(Fu, Fv, Xu, Xv)
        Xg = (Xu.cpu().numpy().T @ Xv.cpu().numpy())
        Uo = bs.solve(Uo + wl.dt * Fa @ Fb.T)
        errs.append(_rel(Xg, Uo))
        assert res <= 10 * wl.ek_tol, (m, res, its)    # ek_tol or its rounding floor (R19)
    st.close()
    return errs


@gpu
@pytest.mark.parametrize("n", [64, 200, 512])
def test_cfg5_shape_trajectory(n):
    """cfg5 parameters at reduced size: 3 steps, each side propagating its own state."""
    wl = W.cfg5(n=n)                       # dt = 1/16 as in cfg5
    errs = _run(wl, 3)
    assert max(errs) <= 1e-8, errs


@gpu
def test_cfg5_full_size_first_steps():
    """cfg5 at full size (nx = ny = 2048): two steps against dense Bartels-Stewart."""
    wl = W.cfg5()
    errs = _run(wl, 2)
    assert max(errs) <= 1e-8, errs


@gpu
def test_zero_rhs_gives_zero():
    wl = W.cfg5(n=128, K=1)
    st = _stepper(wl)
    Fu = torch.zeros(2, wl.nx, dtype=torch.float64, device="cuda")
    Fv = torch.zeros(2, wl.ny, dtype=torch.float64, device="cuda")
    Xu, Xv, res, its = st.step(Fu, Fv)
    assert Xu.shape[0] == 0
    st.close()


@gpu
def test_dt_zero_gives_half_identity_solution():
    """dt = 0: A1 = A2 = I/2, so A1 X + X A2^T = C gives X = C (C = U U^T, no source)."""
    wl = W.cfg5(n=150, K=1)
    wl.dt = 0.0
    st = _stepper(wl)
    rng = np.random.default_rng(11)
    Ua, Ub = rng.standard_normal((3, 150)), rng.standard_normal((3, 150))
    Fu = torch.zeros(1, 150, dtype=torch.float64, device="cuda")
    Xu, Xv, res, its = st.step(Fu, Fu.clone(), _t(Ua), _t(Ub))
    Xg = Xu.cpu().numpy().T @ Xv.cpu().numpy()
    assert _rel(Xg, Ua.T @ Ub) <= 1e-12
    st.close()


@gpu
def test_symmetric_data_gives_symmetric_solution():
    """alpha1 = alpha2, same coefficients, symmetric source  =>  X = X^T."""
    wl = W.cfg5(n=256, K=1)
    wl.alpha2 = wl.alpha1
    wl.d2p, wl.d2m = wl.d1p.copy(), wl.d1m.copy()
    st = _stepper(wl)
    Fa, _ = wl.source_factors(1)
    Xu, Xv, res, its = st.step(_t(Fa.T), _t(Fa.T))
    Xg = Xu.cpu().numpy().T @ Xv.cpu().numpy()
    assert _rel(Xg, Xg.T) <= 1e-10
    st.close()


@gpu
def test_rank_cap_and_nonconvergence_are_reported():
    """rmax below the solution rank -> FDE_EDIM; ek_maxit = 1 -> FDE_ENOCONV (best iterate kept)."""
    from paper_1804_05522_b200._lib import FdeError, FDE_EDIM, FDE_ENOCONV
    from paper_1804_05522_b200.hodlr import Fde2dStepper
    wl = W.cfg5(n=256)
    Fa, Fb = wl.source_factors(1)
    st = Fde2dStepper(wl.nx, wl.ny, wl.alpha1, wl.alpha2, wl.hx, wl.hy, wl.dt, _t(wl.d1p), _t(wl.d1m),
                      _t(wl.d2p), _t(wl.d2m), wl.tol, ek_tol=wl.ek_tol, leaf=wl.leaf, rmax=3)
    with pytest.raises(FdeError) as e:
        st.step(_t(Fa.T), _t(Fb.T))
    assert e.value.code == FDE_EDIM
    st.close()
    st = Fde2dStepper(wl.nx, wl.ny, wl.alpha1, wl.alpha2, wl.hx, wl.hy, wl.dt, _t(wl.d1p), _t(wl.d1m),
                      _t(wl.d2p), _t(wl.d2m), wl.tol, ek_tol=wl.ek_tol, ek_maxit=1, leaf=wl.leaf)
    with pytest.raises(FdeError) as e:
        st.step(_t(Fa.T), _t(Fb.T))
    assert e.value.code == FDE_ENOCONV
    st.close()


@gpu
@pytest.mark.parametrize("variable,alphas", [(False, (1.3, 1.7)), (True, (1.7, 1.9))])
def test_paper_2d_protocol_trajectory(variable, alphas):
    """The paper's own 2D problem (Sec. 5.1: rank-2 source with sin(10 t), dt = 1,
    8 steps; constant and Eq. (5.1) coefficients) at n = 192: every step within 1e-8 of the
    Bartels-Stewart trajectory at the parity tolerances (HODLR tol 1e-12, EK tolerance 1e-11).
    This case caught the right-hand side's loss of small-singular-value directions in the Gram-
    based compression (4.4e-8 before the column scaling)."""
    wl = W.paper2d(192, *alphas, variable=variable, tol=1e-12, ek_tol=1e-11, leaf=32)
    errs = _run(wl, wl.K, ek_tol=wl.ek_tol)
    assert max(errs) <= 1e-8, errs
