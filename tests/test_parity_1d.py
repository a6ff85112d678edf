"""GPU <-> oracle parity for the 1D path (S1-S7) through the C-ABI.

Bar (BASELINE north_star): relative 2-norm error <= 1e-8 per time step at truncation tol
1e-12 against the dense oracle.  At tol 1e-10 / n = 65536 (cfg3) no dense oracle exists
and the forward error is set by conditioning (reading R16): there the bar is the
backward error eta <= 1e-10 from the FFT residual of the exact operator."""
import numpy as np
import pytest
import torch

from oracle.fd1d import assemble_A, step_dense, backward_error, toeplitz_matvec_fft
from oracle.compress import level_ranks, hodlr_levels
from paper_1804_05522_b200 import workloads as W

gpu = pytest.mark.gpu
DEV = "cuda"


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def _stepper(wl):
    from paper_1804_05522_b200.hodlr import Fde1dStepper
    return Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf, batch=wl.batch)


def _gpu_step(st, wl, m, u_prev, coeffs_changed=True, flags=0):
    dp, dm = wl.coeffs(m)
    out = st.step(wl.dt, _t(dp), _t(dm), _t(wl.source(m)), _t(u_prev),
                  coeffs_changed=coeffs_changed, flags=flags)
    torch.cuda.synchronize()
    return out.cpu().numpy().reshape(wl.batch, wl.n)


def _oracle_step(wl, m, u_prev, b=0):
    dp, dm = wl.coeffs(m)
    A = assemble_A(float(wl.alpha[b]), wl.n, wl.h, wl.dt, dp[b], dm[b])
    u, _ = step_dense(A, u_prev[b], wl.source(m)[b], wl.dt)
    return u


def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


CASES = [  # n, alpha, leaf, tol, kind
    (256, 1.5, 32, 1e-12, "smooth"),
    (300, 1.3, 40, 1e-12, "smooth"),       # ragged leaves and segments
    (1000, 1.7, 64, 1e-12, "smooth"),
    (1001, 1.9, 100, 1e-12, "smooth"),
    (513, 1.1, 16, 1e-12, "smooth"),       # deep tree, small leaves
    (2048, 1.6, 128, 1e-12, "smooth"),
    (100, 1.5, 128, 1e-12, "smooth"),      # single leaf (L = 0)
    (1, 1.5, 2, 1e-12, "smooth"),          # n = 1
    (257, 2.0, 32, 1e-12, "smooth"),       # classical limit
]


NO_KEEP = 8   # FDE_NO_KEEP: fused factor + solve through the projected tree (k_leaf Q + k_tree)


@gpu
@pytest.mark.parametrize("flags", [0, NO_KEEP], ids=["keep", "nokeep"])
@pytest.mark.parametrize("n,alpha,leaf,tol,kind", CASES)
def test_one_step_shared_input(n, alpha, leaf, tol, kind, flags):
    wl = W.make_1d(n, alpha, leaf, tol, K=3, kind=kind)
    st = _stepper(wl)
    u = wl.u0
    for m in (1, 2, 3):
        ug = _gpu_step(st, wl, m, u, flags=flags)
        uo = _oracle_step(wl, m, u)
        assert _rel(ug[0], uo) <= 1e-8, (m, _rel(ug[0], uo))
        u = uo[None]                         # shared input for the next step
    st.close()


@gpu
@pytest.mark.parametrize("n,alpha,leaf,tol", [(512, 1.5, 32, 1e-12), (4096, 1.8, 128, 1e-12),
                                               (2048, 1.1, 64, 1e-12), (4096, 1.3, 32, 1e-10),
                                               (1024, 1.9, 16, 1e-8)])
def test_ranks_equal_truncated_svd(n, alpha, leaf, tol):
    """S2: the kept rank per level equals the truncated-SVD rank of the oracle, level by
    level, on trees whose nodes of a level are all equal (n / leaf a power of
    two: every BASELINE config)."""
    wl = W.make_1d(n, alpha, leaf, tol, K=1)
    st = _stepper(wl)
    _gpu_step(st, wl, 1, wl.u0)
    got = st.ranks()
    want = level_ranks(alpha, n, leaf, tol)
    assert len(got) == len(hodlr_levels(n, leaf))
    assert got == want, (got, want)
    st.close()


@gpu
@pytest.mark.parametrize("n,alpha,leaf,tol", [(1000, 1.3, 64, 1e-10), (777, 1.1, 50, 1e-8),
                                               (300, 1.7, 40, 1e-12)])
def test_ranks_ragged_tree_within_one(n, alpha, leaf, tol):
    """Ragged trees (node sizes n1 = n2 - 1 inside a level): one factor per level compresses the
    leading m x m Hankel section (m = largest n2 of the level), which contains every node's
    n2 x n1 block; by singular-value interlacing its truncated rank is >= each node's, and at
    most one higher (one extra column).  The oracle's rank is the max over the level's nodes."""
    wl = W.make_1d(n, alpha, leaf, tol, K=1)
    st = _stepper(wl)
    _gpu_step(st, wl, 1, wl.u0)
    got = st.ranks()
    want = level_ranks(alpha, n, leaf, tol)
    assert all(0 <= g - w <= 1 for g, w in zip(got, want)), (got, want)
    st.close()


@gpu
def test_cfg1_trajectory():
    """cfg1: 8 steps, each side propagating its own state, relative error <= 1e-8 per step."""
    wl = W.cfg1()
    st = _stepper(wl)
    ug, uo = wl.u0, wl.u0
    for m in range(1, wl.K + 1):
        ug = _gpu_step(st, wl, m, ug, coeffs_changed=(m == 1))      # d+- time-invariant
        uo = _oracle_step(wl, m, uo)[None]
        assert _rel(ug[0], uo[0]) <= 1e-8, (m, _rel(ug[0], uo[0]))
    st.close()


@gpu
@pytest.mark.parametrize("flags", [0, NO_KEEP], ids=["keep", "nokeep"])
def test_cfg2_steps(flags):
    """cfg2 (n = 4096, time-dependent d+-, refactor every step): first 4 steps of the trajectory."""
    wl = W.cfg2(K=4)
    st = _stepper(wl)
    ug, uo = wl.u0, wl.u0
    for m in range(1, 5):
        ug = _gpu_step(st, wl, m, ug, flags=flags)
        uo = _oracle_step(wl, m, uo)[None]
        assert _rel(ug[0], uo[0]) <= 1e-8, (m, _rel(ug[0], uo[0]))
    st.close()


@gpu
def test_lu_reuse_matches_refactor():
    wl = W.make_1d(1000, 1.6, 64, 1e-12, K=3, kind="const")
    a, b = _stepper(wl), _stepper(wl)
    ua = ub = wl.u0
    for m in (1, 2, 3):
        ua = _gpu_step(a, wl, m, ua, coeffs_changed=(m == 1))
        ub = _gpu_step(b, wl, m, ub, coeffs_changed=True)
        np.testing.assert_allclose(ua, ub, rtol=1e-13, atol=1e-15)
    a.close(); b.close()


@gpu
@pytest.mark.parametrize("flags", [0, NO_KEEP], ids=["keep", "nokeep"])
def test_deterministic(flags):
    wl = W.make_1d(3000, 1.4, 128, 1e-12, K=1)
    r1 = _gpu_step(_stepper(wl), wl, 1, wl.u0, flags=flags)
    r2 = _gpu_step(_stepper(wl), wl, 1, wl.u0, flags=flags)
    assert np.array_equal(r1, r2)


@gpu
def test_tree_path_matches_level_passes():
    """The projected-tree S5/S6 (FDE_NO_KEEP) and the level-pass S5/S6 compute the same
    SMW solve of the same compressed matrix: equal up to rounding."""
    wl = W.make_1d(5000, 1.7, 100, 1e-12, K=2)
    a, b = _stepper(wl), _stepper(wl)
    ua = _gpu_step(a, wl, 1, wl.u0, flags=0)
    ub = _gpu_step(b, wl, 1, wl.u0, flags=NO_KEEP)
    assert _rel(ub[0], ua[0]) <= 1e-11
    a.close(); b.close()


@gpu
def test_special_cases():
    n = 700
    wl = W.make_1d(n, 1.5, 64, 1e-12, K=1)
    st = _stepper(wl)
    u = wl.u0
    dp, dm = wl.coeffs(1)
    f = wl.source(1)
    # dt = 0  =>  A = I, u_next = u_prev exactly
    out = st.step(0.0, _t(dp), _t(dm), _t(f), _t(u)).cpu().numpy()
    assert np.array_equal(out.reshape(1, n), u)
    # d+- = 0  =>  u_next = u_prev + dt f
    z = np.zeros_like(dp)
    out = st.step(0.25, _t(z), _t(z), _t(f), _t(u)).cpu().numpy()
    np.testing.assert_allclose(out.reshape(1, n), u + 0.25 * f, rtol=1e-15, atol=1e-15)
    # f = 0, u0 = 0  =>  0
    out = st.step(0.25, _t(dp), _t(dm), _t(0 * f), _t(0 * u)).cpu().numpy()
    assert np.all(out == 0)
    st.close()


@gpu
def test_maximum_principle():
    wl = W.make_1d(1500, 1.3, 128, 1e-12, K=4)
    wl.f = np.abs(wl.f)
    st = _stepper(wl)
    u = np.abs(wl.u0)
    for m in range(1, 5):
        u = _gpu_step(st, wl, m, u)
        assert u.min() >= -1e-8 * np.abs(u).max()
    st.close()


@gpu
def test_batched_instances_differ_in_alpha():
    """cfg4 shape: independent instances with their own alpha in one launch."""
    n, batch = 600, 5
    wl = W.make_1d(n, np.linspace(1.1, 1.9, batch), 64, 1e-12, K=1, batch=batch)
    wl.d_plus = wl.d_plus[:1]; wl.d_minus = wl.d_minus[:1]; wl.f = wl.f[:1]
    st = _stepper(wl)
    ug = _gpu_step(st, wl, 1, wl.u0)
    for b in range(batch):
        uo = _oracle_step(wl, 1, wl.u0, b)
        assert _rel(ug[b], uo) <= 1e-8, (b, _rel(ug[b], uo))
    st.close()


@gpu
def test_host_pointer_path_matches_device_path():
    from paper_1804_05522_b200.hodlr import FDE_HOST_PTRS
    wl = W.make_1d(900, 1.6, 64, 1e-12, K=1)
    dp, dm = wl.coeffs(1)
    st = _stepper(wl)
    dev = _gpu_step(st, wl, 1, wl.u0)
    st2 = _stepper(wl)
    c = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64).pin_memory()
    out = torch.empty(900, dtype=torch.float64).pin_memory()
    st2.step(wl.dt, c(dp), c(dm), c(wl.source(1)), c(wl.u0), u_next=out, flags=FDE_HOST_PTRS)
    assert np.array_equal(out.numpy(), dev[0])
    st.close(); st2.close()


@gpu
def test_hodlr_solve_and_matvec_multi_rhs():
    from paper_1804_05522_b200.hodlr import Hodlr
    n, alpha, leaf = 1200, 1.7, 64
    h, dt = 1.0 / (n + 1), 0.05
    x = h * np.arange(1, n + 1)
    dp, dm = 1 + x, 2 - x ** 2
    H = Hodlr(n, alpha, h, dt, _t(dp), _t(dm), 1e-12, leaf)
    H.factor()
    rng = np.random.default_rng(0)
    B = rng.standard_normal((5, n))
    Xg = H.solve(_t(B)[None]).cpu().numpy()[0]          # (batch, nrhs, n)
    A = assemble_A(alpha, n, h, dt, dp, dm)
    Xo = np.linalg.solve(A, B.T).T
    for j in range(5):
        assert _rel(Xg[j], Xo[j]) <= 1e-8
    Yg = H.matvec(_t(B)[None]).cpu().numpy()[0]
    Yo = (A @ B.T).T
    for j in range(5):
        assert _rel(Yg[j], Yo[j]) <= 1e-10
    # aliasing x = b
    Bt = _t(B)[None].contiguous()
    H.solve(Bt, Bt)
    np.testing.assert_array_equal(Bt.cpu().numpy()[0], Xg)
    H.close()


@gpu
@pytest.mark.parametrize("flags", [0, NO_KEEP], ids=["keep", "nokeep"])
def test_cfg3_full_size_backward_error(flags):
    """cfg3 at full size (n = 65536, tol 1e-10, leaf 128): eta <= 1e-10 for two steps
    (NO_KEEP is the launch configuration bench.py times)."""
    wl = W.cfg3(K=2)
    st = _stepper(wl)
    u = wl.u0
    for m in (1, 2):
        un = _gpu_step(st, wl, m, u, flags=flags)
        dp, dm = wl.coeffs(m)
        b = u[0] + wl.dt * wl.source(m)[0]
        be = backward_error(float(wl.alpha[0]), wl.h, wl.dt, dp[0], dm[0], un[0], b)
        assert be["eta"] <= 1e-10, be
        u = un
    st.close()


@gpu
def test_cfg4_sampled_instances():
    """cfg4 shape at full size (batch 512, n = 8192): dense oracle on sampled instances
    (the alpha extremes + 2 seeded picks), eta on all instances."""
    wl = W.cfg4()
    st = _stepper(wl)
    ug = _gpu_step(st, wl, 1, wl.u0)
    picks = [int(np.argmax(wl.alpha)), int(np.argmin(wl.alpha))]
    picks += [int(i) for i in np.random.default_rng(40).choice(512, 2, replace=False)]
    for b in picks:
        uo = _oracle_step(wl, 1, wl.u0, b)
        assert _rel(ug[b], uo) <= 1e-8, (b, wl.alpha[b], _rel(ug[b], uo))
    dp, dm = wl.coeffs(1)
    f = wl.source(1)
    for b in range(0, 512, 7):
        be = backward_error(float(wl.alpha[b]), wl.h, wl.dt, dp[b], dm[b], ug[b], wl.dt * f[b])
        assert be["eta"] <= 1e-12, (b, be)
    st.close()


@gpu
def test_batched_fused_step_matches_oracle():
    """Batched instances through the fused k_step path (FDE_NO_KEEP): each instance vs dense."""
    n, batch = 1500, 6
    wl = W.make_1d(n, np.linspace(1.15, 1.85, batch), 100, 1e-12, K=2, batch=batch)
    st = _stepper(wl)
    u = wl.u0
    for m in (1, 2):
        ug = _gpu_step(st, wl, m, u, flags=NO_KEEP)
        for b in range(batch):
            uo = _oracle_step(wl, m, u, b)
            assert _rel(ug[b], uo) <= 1e-8, (m, b, _rel(ug[b], uo))
        u = ug
    st.close()


@gpu
@pytest.mark.parametrize("n,alpha,leaf,batch", [(2000, 1.6, 100, 1), (1500, 1.3, 64, 3), (300, 1.9, 40, 2)])
def test_pipelined_run_matches_steps_and_oracle(n, alpha, leaf, batch):
    """fde1d_run (K steps in one pipelined launch) = K fused fde1d_step calls (to rounding) and
    each step matches the dense oracle trajectory."""
    wl = W.make_1d(n, np.linspace(alpha, min(alpha + 0.2, 2.0), batch), leaf, 1e-12, K=5, batch=batch)
    st = _stepper(wl)
    K = wl.K
    DP = torch.stack([_t(wl.coeffs(m)[0]) for m in range(1, K + 1)])
    DM = torch.stack([_t(wl.coeffs(m)[1]) for m in range(1, K + 1)])
    F = torch.stack([_t(wl.source(m)) for m in range(1, K + 1)])
    out = st.run(wl.dt, DP, DM, F, _t(wl.u0)).cpu().numpy()
    torch.cuda.synchronize()
    st2 = _stepper(wl)
    u = wl.u0
    uo = wl.u0
    for m in range(1, K + 1):
        u = _gpu_step(st2, wl, m, u, flags=NO_KEEP)
        for b in range(batch):
            assert _rel(out[m - 1, b], u[b]) <= 1e-12, (m, b, _rel(out[m - 1, b], u[b]))
        uo = np.stack([_oracle_step(wl, m, uo, b) for b in range(batch)])
        for b in range(batch):
            assert _rel(out[m - 1, b], uo[b]) <= 1e-8
    st.close(); st2.close()


@gpu
def test_pipelined_run_split_and_unsplit_tree_units_agree():
    """k_run splits every tree unit into a U unit (all columns but the right-hand side) and an R
    unit (the right-hand-side column) while the run has fewer than 2 leaves per SM, and runs whole
    units otherwise (csrc/fdehodlr.cu run_chunk).  The same instance alone (128 leaves: split) and
    inside a batch of 3 (384 leaves: whole units) agree to rounding, and both follow the dense
    oracle trajectory."""
    n, K, batch = 2000, 4, 3
    wl = W.make_1d(n, np.array([1.7, 1.4, 1.55]), 16, 1e-12, K=K, batch=batch)
    from paper_1804_05522_b200.hodlr import Fde1dStepper
    DP = torch.stack([_t(wl.coeffs(m)[0]) for m in range(1, K + 1)])
    DM = torch.stack([_t(wl.coeffs(m)[1]) for m in range(1, K + 1)])
    F = torch.stack([_t(wl.source(m)) for m in range(1, K + 1)])
    st3 = _stepper(wl)
    assert 3 * 128 >= 2 * torch.cuda.get_device_properties(0).multi_processor_count > 128
    out3 = st3.run(wl.dt, DP, DM, F, _t(wl.u0)).cpu().numpy()
    st1 = Fde1dStepper(n, wl.alpha[:1], wl.h, wl.tol, wl.leaf, batch=1)
    out1 = st1.run(wl.dt, DP[:, :1].contiguous(), DM[:, :1].contiguous(), F[:, :1].contiguous(),
                   _t(wl.u0[:1])).cpu().numpy()
    uo = wl.u0
    for m in range(1, K + 1):
        assert _rel(out1[m - 1, 0], out3[m - 1, 0]) <= 1e-12, (m, _rel(out1[m - 1, 0], out3[m - 1, 0]))
        uo = np.stack([_oracle_step(wl, m, uo, b) for b in range(batch)])
        for b in range(batch):
            assert _rel(out3[m - 1, b], uo[b]) <= 1e-8, (m, b)
        assert _rel(out1[m - 1, 0], uo[0]) <= 1e-8, m
    st1.close(); st3.close()


RUN_EDGE = [  # n, alpha, leaf, K, batch
    (300, 1.3, 40, 3, 1),      # ragged leaves, odd leaf offsets
    (1001, 1.9, 100, 4, 2),    # odd n (misaligned row pairs), batch
    (513, 1.1, 16, 3, 1),      # deep tree, small leaves
    (100, 1.5, 128, 3, 1),     # single leaf (L = 0): device fallback to fused steps
    (1, 1.5, 2, 2, 1),         # n = 1
    (257, 2.0, 32, 3, 1),      # classical limit
    (1000, 1.7, 64, 1, 1),     # K = 1 (only the finals of step K after the first step)
]


@gpu
@pytest.mark.parametrize("n,alpha,leaf,K,batch", RUN_EDGE)
def test_pipelined_run_edge_cases(n, alpha, leaf, K, batch):
    """fde1d_run on ragged / odd / degenerate trees and K = 1: every step against the dense
    oracle trajectory (each side propagates its own state)."""
    wl = W.make_1d(n, np.linspace(alpha, min(alpha + 0.1, 2.0), batch), leaf, 1e-12, K=K, batch=batch)
    st = _stepper(wl)
    DP = torch.stack([_t(wl.coeffs(m)[0]) for m in range(1, K + 1)])
    DM = torch.stack([_t(wl.coeffs(m)[1]) for m in range(1, K + 1)])
    F = torch.stack([_t(wl.source(m)) for m in range(1, K + 1)])
    out = st.run(wl.dt, DP, DM, F, _t(wl.u0)).cpu().numpy()
    uo = wl.u0
    for m in range(1, K + 1):
        uo = np.stack([_oracle_step(wl, m, uo, b) for b in range(batch)])
        for b in range(batch):
            assert _rel(out[m - 1, b], uo[b]) <= 1e-8, (m, b, _rel(out[m - 1, b], uo[b]))
    st.close()


@gpu
def test_pipelined_run_invariant_coefficients_and_dt0():
    """Stride-0 coefficients / source (one time level for all K steps) equal the explicit
    K-level arrays bitwise; dt = 0 gives u^(m) = u0 (A = I)."""
    wl = W.make_1d(777, 1.6, 64, 1e-12, K=4)
    st = _stepper(wl)
    dp, dm = wl.coeffs(1)
    f = wl.source(1)
    u0 = _t(np.random.default_rng(11).standard_normal((1, wl.n)))
    one = st.run(wl.dt, _t(dp)[None], _t(dm)[None], _t(f)[None], u0, K=4)
    rep = lambda a: _t(a)[None].repeat(4, 1, 1).contiguous()
    full = st.run(wl.dt, rep(dp), rep(dm), rep(f), u0)
    assert torch.equal(one, full)
    z = st.run(0.0, rep(dp), rep(dm), rep(f), u0)
    assert torch.allclose(z, u0[None].expand_as(z), rtol=0, atol=1e-14)
    st.close()


FACTOR_ONCE = [  # n, alphas, leaf, K, batch
    (777, [1.6], 64, 5, 1),                  # split-unit size: refactor path bitwise equal
    (2000, [1.7, 1.4, 1.55], 16, 4, 3),      # 384 leaves: the refactor run uses whole units
    (300, [1.3, 1.35], 40, 3, 2),            # ragged leaves, batch
    (1000, [1.8], 64, 1, 1),                 # K = 1 (factor step only)
    (513, [1.1], 16, 6, 1),                  # deep tree
]


@gpu
@pytest.mark.parametrize("n,alphas,leaf,K,batch", FACTOR_ONCE)
def test_pipelined_run_factor_once(n, alphas, leaf, K, batch):
    """Time-invariant coefficients (stride 0) make fde1d_run factor once (the LU computed
    only once at the beginning) and run only the rhs column after step 0 (k_run.cuh, inv).  Every
    step matches the dense oracle trajectory with one A for all steps (each side propagating its
    own state), and the FDE_REFACTOR run of the same data to rounding -- bitwise where both runs
    use split tree units."""
    from paper_1804_05522_b200.hodlr import FDE_REFACTOR
    wl = W.make_1d(n, np.array(alphas), leaf, 1e-12, K=K, batch=batch)
    dp, dm = wl.coeffs(1)
    f = wl.source(1)
    st = _stepper(wl)
    once = st.run(wl.dt, _t(dp)[None], _t(dm)[None], _t(f)[None], _t(wl.u0), K=K).cpu().numpy()
    ref = st.run(wl.dt, _t(dp)[None], _t(dm)[None], _t(f)[None], _t(wl.u0), K=K,
                 flags=FDE_REFACTOR).cpu().numpy()
    split_refactor = batch * -(-n // leaf) < 2 * torch.cuda.get_device_properties(0).multi_processor_count
    if split_refactor:
        np.testing.assert_array_equal(once, ref)
    for b in range(batch):
        A = assemble_A(float(wl.alpha[b]), n, wl.h, wl.dt, dp[b], dm[b])
        uo = wl.u0[b]
        for m in range(K):
            uo, _ = step_dense(A, uo, f[b], wl.dt)
            assert _rel(once[m, b], ref[m, b]) <= 1e-12, (m, b, _rel(once[m, b], ref[m, b]))
            assert _rel(once[m, b], uo) <= 1e-8, (m, b, _rel(once[m, b], uo))
    st.close()


@gpu
def test_cfg1_factor_once_pipelined_run():
    """cfg1 (d+- = 1, time-invariant) through fde1d_run: the factor-once launch bench.py times,
    all 8 steps against the dense oracle trajectory."""
    wl = W.cfg1()
    st = _stepper(wl)
    out = st.run(wl.dt, _t(wl.d_plus), _t(wl.d_minus), _t(wl.f), _t(wl.u0)).cpu().numpy()
    assert wl.d_plus.shape[0] == 1 and out.shape[0] == wl.K
    uo = wl.u0
    for m in range(1, wl.K + 1):
        uo = _oracle_step(wl, m, uo)[None]
        assert _rel(out[m - 1, 0], uo[0]) <= 1e-8, (m, _rel(out[m - 1, 0], uo[0]))
    st.close()


@gpu
def test_cfg3_pipelined_run_backward_error():
    """cfg3 at full size through fde1d_run (the launch bench.py times): eta <= 1e-10 per step."""
    wl = W.cfg3(K=4)
    st = _stepper(wl)
    DP = torch.stack([_t(wl.coeffs(m)[0]) for m in range(1, 5)])
    DM = torch.stack([_t(wl.coeffs(m)[1]) for m in range(1, 5)])
    out = st.run(wl.dt, DP, DM, _t(wl.source(1))[None], _t(wl.u0)).cpu().numpy()
    u = wl.u0[0]
    for m in range(1, 5):
        dp, dm = wl.coeffs(m)
        b = u + wl.dt * wl.source(m)[0]
        be = backward_error(float(wl.alpha[0]), wl.h, wl.dt, dp[0], dm[0], out[m - 1, 0], b)
        assert be["eta"] <= 1e-10, (m, be)
        u = out[m - 1, 0]
    st.close()


@gpu
def test_cfg4_pipelined_run_full_size():
    """cfg4 at full size (batch 512, n = 8192) through fde1d_run, 3 steps.  With FDE_REFACTOR the
    pipelined k_run launch refactors every step: dense oracle on the first step of the alpha
    extremes, eta <= 1e-12 on every 7th instance at every step.  Without it (stride-0 coefficients,
    32768 leaves > 16 per SM) the run factors once on the kept-factor path: the same checks, and
    agreement with the refactor run to 1e-9."""
    from paper_1804_05522_b200.hodlr import FDE_REFACTOR
    wl = W.cfg4(K=3)
    st = _stepper(wl)
    dp, dm = wl.coeffs(1)
    f = wl.source(1)
    out = st.run(wl.dt, _t(dp)[None], _t(dm)[None], _t(f)[None], _t(wl.u0), K=3,
                 flags=FDE_REFACTOR).cpu().numpy()
    once = st.run(wl.dt, _t(dp)[None], _t(dm)[None], _t(f)[None], _t(wl.u0), K=3).cpu().numpy()
    for b in (int(np.argmax(wl.alpha)), int(np.argmin(wl.alpha))):
        uo = _oracle_step(wl, 1, wl.u0, b)
        assert _rel(out[0, b], uo) <= 1e-8, (b, wl.alpha[b], _rel(out[0, b], uo))
        assert _rel(once[0, b], uo) <= 1e-8, (b, wl.alpha[b], _rel(once[0, b], uo))
    for res in (out, once):
        u = wl.u0
        for m in range(3):
            for b in range(0, 512, 7):
                be = backward_error(float(wl.alpha[b]), wl.h, wl.dt, dp[b], dm[b], res[m, b], u[b] + wl.dt * f[b])
                assert be["eta"] <= 1e-12, (m, b, be)
                assert _rel(once[m, b], out[m, b]) <= 1e-9, (m, b)
            u = res[m]
    st.close()


@gpu
def test_pipelined_run_host_pointers_match_device():
    """fde1d_run with FDE_HOST_PTRS (host arrays staged by the library, the e2e path bench.py
    times) equals the device-pointer run bitwise."""
    from paper_1804_05522_b200.hodlr import FDE_HOST_PTRS
    wl = W.make_1d(1000, 1.6, 64, 1e-12, K=4)
    st = _stepper(wl)
    DP = np.stack([wl.coeffs(m)[0] for m in range(1, 5)])
    DM = np.stack([wl.coeffs(m)[1] for m in range(1, 5)])
    F = np.stack([wl.source(m) for m in range(1, 5)])
    dev = st.run(wl.dt, _t(DP), _t(DM), _t(F), _t(wl.u0)).cpu().numpy()
    hp = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64).pin_memory()
    host = st.run(wl.dt, hp(DP), hp(DM), hp(F), hp(wl.u0), flags=FDE_HOST_PTRS)
    assert not host.is_cuda
    np.testing.assert_array_equal(host.numpy(), dev)
    st.close()


@gpu
@pytest.mark.parametrize("K,f_invariant", [(24, False), (37, True)])
def test_pipelined_run_host_pointers_overlapped_chunks(K, f_invariant):
    """K >= 24 with per-step coefficients: the host-pointer run is three launches (head, body,
    tail) with the copies overlapped on side streams; bitwise equal to the one-launch
    device-pointer run (also with a time-invariant source, stride 0, and pageable host arrays)."""
    from paper_1804_05522_b200.hodlr import FDE_HOST_PTRS
    wl = W.make_1d(700, 1.4, 32, 1e-12, K=K)
    st = _stepper(wl)
    DP = np.stack([wl.coeffs(m)[0] for m in range(1, K + 1)])
    DM = np.stack([wl.coeffs(m)[1] for m in range(1, K + 1)])
    F = wl.source(1)[None] if f_invariant else np.stack([wl.source(m) for m in range(1, K + 1)])
    dev = st.run(wl.dt, _t(DP), _t(DM), _t(F), _t(wl.u0), K=K).cpu().numpy()
    for pin in (True, False):
        hp = lambda a: (lambda x: x.pin_memory() if pin else x)(
            torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64))
        host = st.run(wl.dt, hp(DP), hp(DM), hp(F), hp(wl.u0), K=K, flags=FDE_HOST_PTRS)
        assert not host.is_cuda
        np.testing.assert_array_equal(host.numpy(), dev)
    st.close()
