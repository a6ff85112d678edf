"""x/y split of the 2D Sylvester step -- split2d.py + the C-ABI
fde2d_step_split.

CPU (gloo, world 2): the exchange layout the library relies on (Xchg in csrc/fde2d.cuh, mirrored
by split2d.side_slot) -- each rank fills its own side's slot, after the all-gather both ranks read
both sides identically -- and a model of the projection exchange: each rank projects only its own
operator (dense, numpy) on its own basis, the projected matrices and right-hand-side factors are
exchanged in the library's slot format, both ranks solve the same projected equation; the 2-rank
result equals the 1-rank result bitwise.
GPU (one device): fde2d_step_split at world 1 with the Python all-gather callback (every exchange
goes through ctypes -> torch as a loopback) is bitwise equal to fde2d_step."""
import os
import socket

import numpy as np
import pytest
import scipy.linalg as sla
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1804_05522_b200.split2d import side_slot, gather_into

gpu = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _model_problem(n=40, s=9, r=3, seed=3):
    rng = np.random.default_rng(seed)
    A1 = np.eye(n) * 3 + rng.standard_normal((n, n)) * 0.1
    A2 = np.eye(n) * 2 + rng.standard_normal((n, n)) * 0.1
    U = np.linalg.qr(rng.standard_normal((n, s)))[0]
    V = np.linalg.qr(rng.standard_normal((n, s)))[0]
    Cu = np.linalg.qr(rng.standard_normal((n, r)))[0]
    Cv = np.linalg.qr(rng.standard_normal((n, r)))[0]
    sig = np.array([3.0, 1.0, 0.25])
    return A1, A2, U, V, Cu, Cv, sig


def _side_message(d, A1, A2, U, V, Cu, Cv, S, smax, rcr):
    """The library's projection slot of side d: [s, A~ (or B^) padded to smax^2, U^T Cu (s x rcr)]."""
    Ub, Ab, Cb = (U, A1, Cu) if d == 0 else (V, A2, Cv)
    s = Ub.shape[1]
    msg = np.zeros(S)
    msg[0] = s
    msg[1:1 + s * s] = (Ub.T @ Ab @ Ub).ravel(order="F")
    msg[1 + smax * smax:1 + smax * smax + s * rcr] = (Ub.T @ Cb).ravel(order="F")
    return msg


def _solve_from(recv, world, S, smax, rcr, sig):
    g0 = side_slot(recv, 0, S, world).numpy()
    g1 = side_slot(recv, 1, S, world).numpy()
    sa, sb = int(g0[0]), int(g1[0])
    At = g0[1:1 + sa * sa].reshape(sa, sa, order="F")
    Bh = g1[1:1 + sb * sb].reshape(sb, sb, order="F")
    UC = g0[1 + smax * smax:1 + smax * smax + sa * rcr].reshape(sa, rcr, order="F")
    VC = g1[1 + smax * smax:1 + smax * smax + sb * rcr].reshape(sb, rcr, order="F")
    Ct = UC @ np.diag(sig) @ VC.T
    return sla.solve_sylvester(At, Bh.T, Ct)           # A~ Y + Y B~ = C~ with B~ = B^^T


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A1, A2, U, V, Cu, Cv, sig = _model_problem()
    smax, rcr = 12, 3
    S = 1 + smax * smax + smax * rcr
    # layout check: rank r fills only its own side's slot with r-tagged data
    send = torch.zeros(2 * S, dtype=torch.float64)
    send[rank * S:(rank + 1) * S] = torch.arange(S, dtype=torch.float64) + 1000.0 * (rank + 1)
    recv = torch.empty(world * 2 * S, dtype=torch.float64)
    gather_into(recv, send)
    for d in (0, 1):
        assert torch.equal(side_slot(recv, d, S, world), torch.arange(S, dtype=torch.float64) + 1000.0 * (d + 1))
    # projection exchange: rank d projects only operator d
    send = torch.zeros(2 * S, dtype=torch.float64)
    send[rank * S:(rank + 1) * S] = torch.as_tensor(_side_message(rank, A1, A2, U, V, Cu, Cv, S, smax, rcr))
    gather_into(recv, send)
    Y = _solve_from(recv, world, S, smax, rcr, sig)
    q.put((rank, Y))
    dist.barrier()
    dist.destroy_process_group()


def test_split_exchange_two_ranks_equals_one_rank():
    A1, A2, U, V, Cu, Cv, sig = _model_problem()
    smax, rcr = 12, 3
    S = 1 + smax * smax + smax * rcr
    send = torch.zeros(2 * S, dtype=torch.float64)
    for d in (0, 1):
        send[d * S:(d + 1) * S] = torch.as_tensor(_side_message(d, A1, A2, U, V, Cu, Cv, S, smax, rcr))
    recv = torch.empty(2 * S, dtype=torch.float64)
    gather_into(recv, send)                             # world 1: loopback
    Y1 = _solve_from(recv, 1, S, smax, rcr, sig)
    # and the model itself: Y solves the Galerkin equation of A1 X + X A2^T = Cu diag(sig) Cv^T
    At, Bt = U.T @ A1 @ U, (V.T @ A2 @ V).T
    Ct = (U.T @ Cu) @ np.diag(sig) @ (V.T @ Cv).T
    assert np.allclose(At @ Y1 + Y1 @ Bt, Ct, atol=1e-12)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(got[0], Y1) and np.array_equal(got[1], Y1)


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


@gpu
def test_split_world1_through_callback_equals_fde2d_step():
    from paper_1804_05522_b200 import workloads as W
    from paper_1804_05522_b200.hodlr import Fde2dStepper
    from paper_1804_05522_b200.split2d import SplitSylvesterStepper
    wl = W.cfg5(n=512)
    args = (wl.nx, wl.ny, wl.alpha1, wl.alpha2, wl.hx, wl.hy, wl.dt, _t(wl.d1p), _t(wl.d1m), _t(wl.d2p),
            _t(wl.d2m), wl.tol)
    a = Fde2dStepper(*args, ek_tol=wl.ek_tol, leaf=wl.leaf)
    b = SplitSylvesterStepper(*args, ek_tol=wl.ek_tol, leaf=wl.leaf, world=1, rank=0)
    Xa = Xb = None
    for m in (1, 2, 3):
        Fa, Fb = wl.source_factors(m)
        ua = a.step(_t(Fa.T), _t(Fb.T), *(Xa if Xa else (None, None)))
        ub = b.step(_t(Fa.T), _t(Fb.T), *(Xb if Xb else (None, None)))
        Xa = (ua[0], ua[1])
        (bu, bv), r, res, its = ub
        Xb = (bu, bv)
        assert torch.equal(ua[0], bu) and torch.equal(ua[1], bv)
        assert ua[2] == res and ua[3] == its
    assert b.calls > 0
    a.close(); b.close()
