"""Multi-GPU sharding of independent 1D problems (BASELINE configs[3]).

The batched workload (512 independent instances) shards naturally: rank r of a world of size G
owns a contiguous slice of the instances, runs the same batched kernels on it (one
fde1d_step launch sequence per step for all its instances), and results are gathered over
NCCL only when they are checked or at the end -- never inside a step (no data-path
collective).  Instance i computed on any rank is bitwise equal to instance i of a 1-GPU run:
every kernel works per instance with a schedule-independent reduction order.

The step function is injected so the partition/gather logic can be tested on CPU with the
gloo backend; the product path passes the CUDA stepper (``Fde1dStepper.step``).
"""
import torch
import torch.distributed as dist


def shard_range(batch, world, rank):
    """Contiguous split of `batch` instances over `world` ranks: (start, count) of `rank`.
    The first batch % world ranks get one extra instance."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def gather_instances(local, batch, world, rank, group=None):
    """All-gather the (count, n) per-rank result slices into a (batch, n) tensor (rank order =
    instance order).  Slices may differ in length by one: pad to the max and trim."""
    n = local.shape[-1]
    counts = [shard_range(batch, world, r)[1] for r in range(world)]
    mx = max(counts)
    buf = torch.zeros((mx, n), dtype=local.dtype, device=local.device)
    buf[:local.shape[0]] = local
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    return torch.cat([o[:c] for o, c in zip(outs, counts)], dim=0)


class ShardedRun:
    """Run K implicit-Euler steps of the local instance slice with an injected step function
    step_fn(m, u_local) -> u_local_next (m = 1..K), gathering only at the end."""

    def __init__(self, batch, world=None, rank=None):
        self.world = world if world is not None else (dist.get_world_size() if dist.is_initialized() else 1)
        self.rank = rank if rank is not None else (dist.get_rank() if dist.is_initialized() else 0)
        self.batch = batch
        self.start, self.count = shard_range(batch, self.world, self.rank)

    def local_slice(self, arr):
        """Rows of a (batch, ...) array owned by this rank."""
        return arr[self.start:self.start + self.count]

    def run(self, u0_local, K, step_fn, gather=True):
        u = u0_local
        for m in range(1, K + 1):
            u = step_fn(m, u)
        if gather and self.world > 1:
            return gather_instances(u, self.batch, self.world, self.rank)
        return u
