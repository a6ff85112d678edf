"""Full-size and full-length GPU <-> oracle parity (SURVEY.md §8(c)-(d) parity bars):
* cfg4 (512 x n = 8192) through the timed kept-factor path (factor once; 16 solves with
  coeffs_changed = 0, k_leaf_apply + k_solve_level): dense-oracle trajectories of the 16 §8(d)
  instances (alpha / a + b extremes + 12 rng(40) picks) and the backward error on all 512 at
  every step;
* cfg4 sharding: a 64-instance slice run alone is bitwise equal to the same instances of the
  512 batch (what shard.py's "bitwise equal per instance" claim rests on);
* cfg2: all 64 steps through fde1d_run (the pipelined path bench.py times) and 16 steps through
  fde1d_step (kept factor and fused), each side propagating its own state;
* cfg5 (2D, 2048^2): step 16 with a shared seeded rank-27 state (plus steps 1-2 of the
  trajectory in test_parity_2d.py), and all 16 steps at n = 512."""
import numpy as np
import pytest
import torch

from oracle.fd1d import assemble_A, step_dense, backward_error
from oracle.sylvester2d import operators_2d, BartelsStewart
from paper_1804_05522_b200 import workloads as W

gpu = pytest.mark.gpu
NO_KEEP = 8


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@gpu
def test_cfg4_factor_once_16_steps_vs_dense():
    from paper_1804_05522_b200.hodlr import Fde1dStepper
    wl = W.cfg4()
    picks = W.cfg4_checked_instances(wl)
    dp, dm = wl.coeffs(1)
    f = wl.source(1)
    st = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf, batch=wl.batch)
    DP, DM, F = _t(dp), _t(dm), _t(f)
    u = _t(wl.u0)
    gpu_traj = {b: [] for b in picks}
    prev = wl.u0
    for m in range(1, wl.K + 1):
        u = st.step(wl.dt, DP, DM, F, u, coeffs_changed=(m == 1))   # m > 1: solve with the kept factor
        torch.cuda.synchronize()
        un = u.cpu().numpy()
        for b in picks:
            gpu_traj[b].append(un[b].copy())
        for b in range(wl.batch):                                   # eta on all 512 (own state)
            be = backward_error(float(wl.alpha[b]), wl.h, wl.dt, dp[b], dm[b], un[b], prev[b] + wl.dt * f[b])
            assert be["eta"] <= 1e-12, (m, b, be)
        prev = un
    st.close()
    worst = 0.0
    for b in picks:                                                 # dense trajectory, LU reused
        A = assemble_A(float(wl.alpha[b]), wl.n, wl.h, wl.dt, dp[b], dm[b])
        uo, lu = wl.u0[b], None
        for m in range(1, wl.K + 1):
            uo, lu = step_dense(A, uo, f[b], wl.dt, lu)
            e = _rel(gpu_traj[b][m - 1], uo)
            worst = max(worst, e)
            assert e <= 1e-8, (b, m, float(wl.alpha[b]), e)
        del A, lu
    print("cfg4 factor-once worst relative error over 16 instances x 16 steps: %.3e" % worst)


@gpu
def test_cfg4_slice_bitwise_equal_to_batch():
    from paper_1804_05522_b200.hodlr import Fde1dStepper
    wl = W.cfg4()
    dp, dm = wl.coeffs(1)
    f = wl.source(1)
    sl = slice(128, 192)                        # rank 2 of 8 (shard.shard_range(512, 8, 2))
    outs = []
    for s_ in (slice(0, 512), sl):
        b = s_.stop - s_.start
        st = Fde1dStepper(wl.n, wl.alpha[s_], wl.h, wl.tol, wl.leaf, batch=b)
        u = _t(wl.u0[s_])
        res = []
        for m in (1, 2):
            u = st.step(wl.dt, _t(dp[s_]), _t(dm[s_]), _t(f[s_]), u, coeffs_changed=(m == 1))
            res.append(u.clone())
        run = st.run(wl.dt, _t(dp[s_])[None], _t(dm[s_])[None], _t(f[s_])[None], _t(wl.u0[s_]), K=2)
        torch.cuda.synchronize()
        outs.append((torch.stack(res).cpu().numpy(), run.cpu().numpy()))
        st.close()
    (a_step, a_run), (b_step, b_run) = outs
    np.testing.assert_array_equal(a_step[:, sl], b_step)
    np.testing.assert_array_equal(a_run[:, sl], b_run)


_CFG2 = {}


def _cfg2_oracle():
    """Dense oracle trajectory of cfg2 (64 steps, A_m refactored every step)."""
    if "traj" not in _CFG2:
        wl = W.cfg2()
        u, traj = wl.u0[0], []
        for m in range(1, wl.K + 1):
            dp, dm = wl.coeffs(m)
            A = assemble_A(float(wl.alpha[0]), wl.n, wl.h, wl.dt, dp[0], dm[0])
            u, _ = step_dense(A, u, wl.source(m)[0], wl.dt)
            traj.append(u)
        _CFG2["wl"], _CFG2["traj"] = wl, traj
    return _CFG2["wl"], _CFG2["traj"]


@gpu
def test_cfg2_all_64_steps_pipelined_run():
    from paper_1804_05522_b200.hodlr import Fde1dStepper
    wl, traj = _cfg2_oracle()
    st = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf)
    out = st.run(wl.dt, _t(wl.d_plus), _t(wl.d_minus), _t(wl.f), _t(wl.u0)).cpu().numpy()
    st.close()
    errs = [_rel(out[m, 0], traj[m]) for m in range(wl.K)]
    assert max(errs) <= 1e-8, (int(np.argmax(errs)), max(errs))


@gpu
@pytest.mark.parametrize("flags", [0, NO_KEEP], ids=["keep", "nokeep"])
def test_cfg2_16_steps_per_step_path(flags):
    from paper_1804_05522_b200.hodlr import Fde1dStepper
    wl, traj = _cfg2_oracle()
    st = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf)
    u = _t(wl.u0)
    for m in range(1, 17):
        dp, dm = wl.coeffs(m)
        u = st.step(wl.dt, _t(dp), _t(dm), _t(wl.source(m)), u, flags=flags)
        e = _rel(u.cpu().numpy()[0], traj[m - 1])
        assert e <= 1e-8, (m, e)
    st.close()


def _stepper2d(wl):
    from paper_1804_05522_b200.hodlr import Fde2dStepper
    return Fde2dStepper(wl.nx, wl.ny, wl.alpha1, wl.alpha2, wl.hx, wl.hy, wl.dt,
                        _t(wl.d1p), _t(wl.d1m), _t(wl.d2p), _t(wl.d2m), wl.tol, ek_tol=wl.ek_tol,
                        leaf=wl.leaf)


@gpu
def test_cfg5_step16_shared_input():
    """cfg5 at 2048^2, step m = 16 from a shared seeded rank-27 state U (same bits on both sides):
    X = (A1, A2 Sylvester)^{-1}(U + dt F^(16)) against dense Bartels-Stewart."""
    wl = W.cfg5()
    Su, Sv = W.lowrank_state(wl.nx, wl.ny)
    Fa, Fb = wl.source_factors(16)
    st = _stepper2d(wl)
    Xu, Xv, res, its = st.step(_t(Fa.T), _t(Fb.T), _t(Su.T), _t(Sv.T))
    Xg = Xu.cpu().numpy().T @ Xv.cpu().numpy()
    st.close()
    A1, A2 = operators_2d(wl.alpha1, wl.alpha2, wl.nx, wl.ny, wl.hx, wl.hy, wl.dt,
                          wl.d1p, wl.d1m, wl.d2p, wl.d2m)
    Xo = BartelsStewart(A1, A2).solve(Su @ Sv.T + wl.dt * Fa @ Fb.T)
    assert _rel(Xg, Xo) <= 1e-8, (_rel(Xg, Xo), res, its)


@gpu
def test_cfg5_shape_all_16_steps():
    """cfg5's parameters at n = 512: the whole 16-step trajectory, each side its own state."""
    wl = W.cfg5(n=512)
    st = _stepper2d(wl)
    A1, A2 = operators_2d(wl.alpha1, wl.alpha2, wl.nx, wl.ny, wl.hx, wl.hy, wl.dt,
                          wl.d1p, wl.d1m, wl.d2p, wl.d2m)
    bs = BartelsStewart(A1, A2)
    Uo = np.zeros((wl.nx, wl.ny))
    Xu = Xv = None
    for m in range(1, wl.K + 1):
        Fa, Fb = wl.source_factors(m)
        if Xu is None:
            Xu, Xv, res, its = st.step(_t(Fa.T), _t(Fb.T))
        else:
            Xu, Xv, res, its = st.step(_t(Fa.T), _t(Fb.T), Xu, Xv)
        Uo = bs.solve(Uo + wl.dt * Fa @ Fb.T)
        e = _rel(Xu.cpu().numpy().T @ Xv.cpu().numpy(), Uo)
        assert e <= 1e-8, (m, e, res, its)
    st.close()
