"""Device-side error paths through the C-ABI (GPU): the zero / non-finite pivot latch of the leaf
LU and its report through hodlr_status() / FDE_SYNC (a singular pivot is an error
naming the leaf; the leaves are factorised without pivoting, because A_m is strictly
diagonally dominant for d+- >= 0), the report-once clearing of the latch, and FDE_CHECK
rejecting negative / non-finite coefficients (d+- >= 0) on the device."""
import numpy as np
import pytest
import torch

from paper_1804_05522_b200 import workloads as W

gpu = pytest.mark.gpu
ESINGULAR, EDOMAIN = 3, 1


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def _singular_coeffs(n, row):
    """h = 1, dt = 1, alpha = 2 (c = 1, T diagonal 2): d+[row] = -1/2, d-[row] = 0 makes the
    diagonal entry 1 + 2 d+ + 2 d- of that row exactly 0 -- the first pivot of the leaf starting
    at `row`."""
    dp = np.full(n, 0.25)
    dm = np.full(n, 0.25)
    dp[row], dm[row] = -0.5, 0.0
    return dp, dm


@gpu
@pytest.mark.parametrize("leaf_index", [0, 1, 3])
def test_zero_leaf_pivot_latches_esingular_with_leaf_index(leaf_index):
    from paper_1804_05522_b200.hodlr import Hodlr
    n, leaf = 128, 32                                   # 4 leaves of 32 rows
    dp, dm = _singular_coeffs(n, 32 * leaf_index)
    H = Hodlr(n, 2.0, 1.0, 1.0, _t(dp), _t(dm), 1e-12, leaf)
    H.factor()                                          # asynchronous: no error yet
    code, where = H.status()
    assert code == ESINGULAR
    assert where % 65536 == leaf_index and where // 65536 == 0
    # reported once: the latch is clear afterwards
    assert H.status()[0] == 0
    H.close()


@gpu
def test_sync_flag_reports_singular_pivot_then_recovers():
    from paper_1804_05522_b200.hodlr import Fde1dStepper, FDE_SYNC, FDE_NO_KEEP
    from paper_1804_05522_b200._lib import FdeError
    n, leaf = 256, 32
    st = Fde1dStepper(n, 2.0, 1.0, 1e-12, leaf)
    u = _t(np.ones((1, n)))
    f = _t(np.zeros((1, n)))
    for flags in (FDE_SYNC, FDE_SYNC | FDE_NO_KEEP):
        dp, dm = _singular_coeffs(n, 64)
        with pytest.raises(FdeError) as e:
            st.step(1.0, _t(dp[None]), _t(dm[None]), f, u, flags=flags)
        assert e.value.code == ESINGULAR
        # a regular step on the same handle starts clean
        good = _t(np.full((1, n), 0.25))
        out = st.step(1.0, good, good, f, u, flags=flags)
        assert bool(torch.isfinite(out).all())
    st.close()


@gpu
def test_nonfinite_coefficient_latches_in_pipelined_run():
    from paper_1804_05522_b200.hodlr import Fde1dStepper, FDE_SYNC
    from paper_1804_05522_b200._lib import FdeError
    wl = W.make_1d(1000, 1.6, 64, 1e-12, K=3)
    st = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf)
    dp, dm = wl.coeffs(1)
    dp = dp.copy()
    dp[0, 500] = np.nan
    with pytest.raises(FdeError) as e:
        st.run(wl.dt, _t(dp)[None], _t(dm)[None], _t(wl.source(1))[None], _t(wl.u0), K=3, flags=FDE_SYNC)
    assert e.value.code == ESINGULAR
    st.close()


@gpu
@pytest.mark.parametrize("bad", [-1e-3, np.nan])
def test_check_flag_rejects_bad_coefficients_on_device(bad):
    from paper_1804_05522_b200.hodlr import Hodlr, Fde1dStepper, FDE_CHECK, FDE_HOST_PTRS
    from paper_1804_05522_b200._lib import FdeError
    wl = W.make_1d(600, 1.4, 64, 1e-12, K=1)
    dp, dm = wl.coeffs(1)
    dm = dm.copy()
    dm[0, 123] = bad
    with pytest.raises(FdeError) as e:
        Hodlr(wl.n, wl.alpha, wl.h, wl.dt, _t(dp[0]), _t(dm[0]), wl.tol, wl.leaf, flags=FDE_CHECK)
    assert e.value.code == EDOMAIN
    st = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf)
    with pytest.raises(FdeError) as e:
        st.step(wl.dt, _t(dp), _t(dm), _t(wl.source(1)), _t(wl.u0), flags=FDE_CHECK)
    assert e.value.code == EDOMAIN
    hp = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64)
    with pytest.raises(FdeError) as e:
        st.step(wl.dt, hp(dp), hp(dm), hp(wl.source(1)), hp(wl.u0), u_next=hp(np.zeros((1, wl.n))),
                flags=FDE_CHECK | FDE_HOST_PTRS)
    assert e.value.code == EDOMAIN
    st.close()


@gpu
def test_check_with_host_pointers_matches_device_path():
    """FDE_HOST_PTRS | FDE_CHECK must give the device-pointer result bitwise (the check's flag
    word must not alias the staged d+)."""
    from paper_1804_05522_b200.hodlr import Fde1dStepper, FDE_CHECK, FDE_HOST_PTRS
    wl = W.make_1d(1000, 1.7, 64, 1e-12, K=1)
    dp, dm = wl.coeffs(1)
    a = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf)
    ud = a.step(wl.dt, _t(dp), _t(dm), _t(wl.source(1)), _t(wl.u0)).cpu().numpy()
    b = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf)
    hp = lambda x: torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64)
    uh = hp(np.zeros((1, wl.n)))
    b.step(wl.dt, hp(dp), hp(dm), hp(wl.source(1)), hp(wl.u0), u_next=uh, flags=FDE_CHECK | FDE_HOST_PTRS)
    np.testing.assert_array_equal(uh.numpy(), ud)
    a.close(); b.close()


@gpu
@pytest.mark.parametrize("refactor", [False, True], ids=["factor_once", "refactor"])
def test_run_longer_than_one_launch_chunk(refactor):
    """fde1d_run splits K > RUN_KMAX steps into several launches; a long cheap run (n = 256,
    K = 8193 > 8192) matches the fused per-step path at its last steps -- with the factor formed
    once per launch (stride-0 coefficients) and with FDE_REFACTOR."""
    from paper_1804_05522_b200.hodlr import Fde1dStepper, FDE_NO_KEEP, FDE_REFACTOR
    n, K = 256, 8193
    wl = W.make_1d(n, 1.5, 32, 1e-12, K=1, kind="const")
    dp, dm = wl.coeffs(1)
    f = wl.source(1)
    st = Fde1dStepper(n, wl.alpha, wl.h, wl.tol, wl.leaf)
    out = st.run(1e-3, _t(dp)[None], _t(dm)[None], _t(f)[None], _t(wl.u0), K=K,
                 flags=FDE_REFACTOR if refactor else 0)
    torch.cuda.synchronize()
    ref = Fde1dStepper(n, wl.alpha, wl.h, wl.tol, wl.leaf)
    u = out[K - 3].clone()
    for m in (K - 2, K - 1):
        u = ref.step(1e-3, _t(dp), _t(dm), _t(f), u, flags=FDE_NO_KEEP)
        np.testing.assert_allclose(out[m].cpu().numpy(), u.cpu().numpy(), rtol=1e-12, atol=1e-14)
    st.close(); ref.close()
