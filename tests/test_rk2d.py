"""Multi-shift rational Krylov 2D step (the paper's Galerkin framework,
P:1519-1550, with bases from independent shifted HODLR solves) -- fde2d_step_rk.

GPU: the cfg5 trajectory (n = 512, 8 steps) and cfg5 at full size (2 steps) against dense
Bartels-Stewart within the 1e-8 parity bar; the reported residual against the oracle's true
residual; explicit poles accepted.  CPU (gloo, world 2): the pole-sharded exchange layout (block j
of a round computed by rank j mod pw, read back in pole order by every rank)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.sylvester2d import operators_2d, BartelsStewart
from paper_1804_05522_b200 import workloads as W
from paper_1804_05522_b200.split2d import gather_into, pole_block

gpu = pytest.mark.gpu


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _rk(wl, **kw):
    from paper_1804_05522_b200.split2d import RkSylvesterStepper
    return RkSylvesterStepper(wl.nx, wl.ny, wl.alpha1, wl.alpha2, wl.hx, wl.hy, wl.dt, _t(wl.d1p), _t(wl.d1m),
                              _t(wl.d2p), _t(wl.d2m), wl.tol, rk_tol=wl.ek_tol, leaf=wl.leaf, **kw)


@gpu
@pytest.mark.parametrize("n,K", [(512, 8), (2048, 2)])
def test_rk_trajectory_matches_bartels_stewart(n, K):
    wl = W.cfg5(n=n)
    A1, A2 = operators_2d(wl.alpha1, wl.alpha2, wl.nx, wl.ny, wl.hx, wl.hy, wl.dt, wl.d1p, wl.d1m, wl.d2p, wl.d2m)
    bs = BartelsStewart(A1, A2)
    st = _rk(wl, npole=8, rounds=4)
    Uo = np.zeros((wl.nx, wl.ny))
    Xu = Xv = None
    for m in range(1, K + 1):
        Fa, Fb = wl.source_factors(m)
        Xu, Xv, res, rounds = st.step(_t(Fa.T), _t(Fb.T), Xu, Xv)
        Xg = Xu.cpu().numpy().T @ Xv.cpu().numpy()
        C = Uo + wl.dt * Fa @ Fb.T
        Uo = bs.solve(C)
        assert _rel(Xg, Uo) <= 1e-8, (m, _rel(Xg, Uo), res, rounds)
    st.close()


@gpu
def test_rk_explicit_poles_and_residual():
    wl = W.cfg5(n=256)
    A1, A2 = operators_2d(wl.alpha1, wl.alpha2, wl.nx, wl.ny, wl.hx, wl.hy, wl.dt, wl.d1p, wl.d1m, wl.d2p, wl.d2m)
    Fa, Fb = wl.source_factors(1)
    poles = np.concatenate([np.logspace(np.log10(0.5), 5.5, 12 * 3)] * 2)
    st = _rk(wl, npole=12, rounds=3, poles=poles)
    Xu, Xv, res, rounds = st.step(_t(Fa.T), _t(Fb.T))
    Xg = Xu.cpu().numpy().T @ Xv.cpu().numpy()
    C = wl.dt * Fa @ Fb.T
    true = np.linalg.norm(A1 @ Xg + Xg @ A2.T - C) / np.linalg.norm(C)
    assert res <= 10 * true + 1e-14 and true <= 10 * res + 1e-14, (res, true)
    assert _rel(Xg, BartelsStewart(A1, A2).solve(C)) <= 1e-8
    st.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    K, blk = 5, 3
    per = (K + world - 1) // world
    cnt = per * blk
    send = torch.zeros(cnt, dtype=torch.float64)
    for i, j in enumerate(range(rank, K, world)):        # this rank's poles, packed
        send[i * blk:(i + 1) * blk] = 100.0 * j + torch.arange(blk, dtype=torch.float64)
    recv = torch.empty(world * cnt, dtype=torch.float64)
    gather_into(recv, send)
    got = [pole_block(recv, j, world, cnt, blk).numpy().copy() for j in range(K)]
    q.put((rank, got))
    dist.barrier()
    dist.destroy_process_group()


def test_pole_sharded_exchange_two_ranks():
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
    for r in (0, 1):
        for j in range(5):
            np.testing.assert_array_equal(got[r][j], 100.0 * j + np.arange(3))
