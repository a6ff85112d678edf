"""Multi-rank sharding of independent instances on CPU with gloo, world 2:
partition arithmetic, and a 2-rank run whose gathered result equals the 1-rank run bitwise.
The per-instance step is the dense oracle (test infrastructure), injected into the same
ShardedRun the GPU driver uses."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1804_05522_b200.shard import shard_range, ShardedRun


def test_shard_range_partitions_exactly():
    for batch in (1, 5, 8, 512, 513):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(batch, world, r) for r in range(world)]
            assert spans[0][0] == 0
            for (s0, c0), (s1, c1) in zip(spans, spans[1:]):
                assert s1 == s0 + c0
                assert abs(c1 - c0) <= 1
            assert spans[-1][0] + spans[-1][1] == batch


def _problem():
    from paper_1804_05522_b200 import workloads as W
    return W.make_1d(96, np.linspace(1.2, 1.9, 5), 32, 1e-12, K=3, batch=5)


def _oracle_step_fn(wl, start):
    from oracle.fd1d import assemble_A, step_dense

    def step(m, u):
        dp, dm = wl.coeffs(m)
        f = wl.source(m)
        out = []
        for j in range(u.shape[0]):
            b = start + j
            A = assemble_A(float(wl.alpha[b]), wl.n, wl.h, wl.dt, dp[b], dm[b])
            out.append(step_dense(A, u[j].numpy(), f[b], wl.dt)[0])
        return torch.as_tensor(np.array(out))
    return step


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = _problem()
    run = ShardedRun(wl.batch)
    u0 = torch.as_tensor(run.local_slice(wl.u0))
    out = run.run(u0, wl.K, _oracle_step_fn(wl, run.start))
    if rank == 0:
        q.put(out.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_gather_matches_single_rank():
    wl = _problem()
    single = ShardedRun(wl.batch, world=1, rank=0).run(torch.as_tensor(wl.u0), wl.K,
                                                       _oracle_step_fn(wl, 0)).numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(got, single)
