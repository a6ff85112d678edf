"""Top-level split of one 1D problem -- fde1d_step_split.

GPU (one device): every part of a world-2/4/8 split run in this process, one launch after the
other (rank = -1: the launches the ranks run, nothing waits on another part's launch), is bitwise
equal to the unsplit fused step (fde1d_step, FDE_NO_KEEP) and within the parity bar of the dense
oracle; world 1 through the Python all-gather callback (loopback) is bitwise equal too.
CPU (gloo, world 2): the row-block all-gather of u_next the library relies on (rank-major blocks)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1804_05522_b200 import workloads as W
from paper_1804_05522_b200.split2d import gather_into

gpu = pytest.mark.gpu
NO_KEEP = 8


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


@gpu
@pytest.mark.parametrize("n,leaf,worlds", [(4096, 64, (2, 4, 8)), (65536, 128, (2, 8))])
def test_split_parts_equal_unsplit_step(n, leaf, worlds):
    from paper_1804_05522_b200.hodlr import Fde1dStepper
    from paper_1804_05522_b200.split1d import Split1dStepper
    from oracle.fd1d import assemble_A, step_dense, backward_error
    wl = W.cfg3(K=2, n=n) if n == 65536 else W.make_1d(n, 1.6, leaf, 1e-12, K=2)
    ref = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf)
    u = _t(wl.u0)
    outs = []
    for m in (1, 2):
        dp, dm = wl.coeffs(m)
        u = ref.step(wl.dt, _t(dp), _t(dm), _t(wl.source(m)), u, flags=NO_KEEP)
        outs.append(u.clone())
    ref.close()
    for world in worlds:
        sp = Split1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf, world=world, rank=-1)
        u = _t(wl.u0[0])
        for m in (1, 2):
            dp, dm = wl.coeffs(m)
            un = torch.empty_like(u)
            sp.step(wl.dt, _t(dp[0]), _t(dm[0]), _t(wl.source(m)[0]), u, un, use_callback=False)
            assert torch.equal(un, outs[m - 1][0]), (world, m)
            u = un
        sp.close()
    # the unsplit result against the oracle (dense at n = 4096, backward error at cfg3)
    u0 = wl.u0[0]
    dp, dm = wl.coeffs(1)
    if n <= 4096:
        A = assemble_A(float(wl.alpha[0]), wl.n, wl.h, wl.dt, dp[0], dm[0])
        uo, _ = step_dense(A, u0, wl.source(1)[0], wl.dt)
        assert np.linalg.norm(outs[0].cpu().numpy()[0] - uo) <= 1e-8 * np.linalg.norm(uo)
    else:
        be = backward_error(float(wl.alpha[0]), wl.h, wl.dt, dp[0], dm[0], outs[0].cpu().numpy()[0],
                            u0 + wl.dt * wl.source(1)[0])
        assert be["eta"] <= 1e-10


@gpu
def test_split_world1_through_callback():
    from paper_1804_05522_b200.hodlr import Fde1dStepper
    from paper_1804_05522_b200.split1d import Split1dStepper
    wl = W.make_1d(2048, 1.4, 64, 1e-12, K=1)
    dp, dm = wl.coeffs(1)
    ref = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf)
    want = ref.step(wl.dt, _t(dp), _t(dm), _t(wl.source(1)), _t(wl.u0), flags=NO_KEEP)
    sp = Split1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf, world=1, rank=0)
    un = torch.empty(wl.n, dtype=torch.float64, device="cuda")
    sp.step(wl.dt, _t(dp[0]), _t(dm[0]), _t(wl.source(1)[0]), _t(wl.u0[0]), un)
    assert torch.equal(un, want[0])
    ref.close(); sp.close()


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
    n = 24
    rows = n // world
    u = torch.full((n,), -1.0, dtype=torch.float64)
    u[rank * rows:(rank + 1) * rows] = torch.arange(rank * rows, (rank + 1) * rows, dtype=torch.float64)
    send = u[rank * rows:(rank + 1) * rows].clone()          # the library's staging copy
    gather_into(u, send)                                     # recv = u itself (rank-major blocks)
    q.put((rank, u.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_row_block_gather_two_ranks():
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
        np.testing.assert_array_equal(got[r], np.arange(24, dtype=np.float64))
