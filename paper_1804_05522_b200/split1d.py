"""The top-level split of ONE 1D problem over ranks.

Rank g of world = 2^p owns the rows [g, g+1) * n / world: its leaves and the SMW levels p .. L-1 of
its subtree run locally; the parts exchange only the (xc_p - 1) x xc_p projected matrices of
their subtree roots, then every rank runs the top p levels on the same data and the finals of its
own leaves; u_next's row blocks are all-gathered.  All arithmetic is in the C-ABI call
fde1d_step_split (include/fdehodlr.h); this module supplies its all-gather callback
(torch.distributed: NCCL over NVLink on the GPU box) and marshals arguments.
"""
import ctypes

import numpy as np

from . import _lib
from ._lib import check
from .split2d import as_tensor, gather_into


class Split1dStepper:
    """fde1d_step_split with a cached handle.  world / rank / group: the split; rank = -1 runs every
    part in this process (the same launches, one after the other)."""

    def __init__(self, n, alpha, h, tol, leaf, world=1, rank=0, group=None):
        self.n, self.h, self.tol, self.leaf = n, h, tol, leaf
        self.alpha = float(np.asarray(alpha).reshape(-1)[0])
        self.world, self.rank, self.group = world, rank, group
        self._cache = ctypes.c_void_p()
        self.calls = 0
        self._cb = _lib.ALLGATHER_FN(self._gather)

    def _gather(self, ctx, send, recv, count, stream):
        try:
            gather_into(as_tensor(recv, self.world * count), as_tensor(send, count),
                        self.group if self.world > 1 else None)
            self.calls += 1
            return 0
        except Exception:
            return 1

    def step(self, dt, d_plus, d_minus, f, u_prev, u_next, flags=0, stream=None, use_callback=True):
        from .hodlr import _dev, _stream
        n = self.n
        cb = ctypes.cast(self._cb, ctypes.c_void_p) if use_callback else None
        check(_lib.load().fde1d_step_split(
            self.world, self.rank, cb, None, n, self.alpha, self.h, dt, _dev(d_plus, "d_plus", n),
            _dev(d_minus, "d_minus", n), _dev(f, "f", n), _dev(u_prev, "u_prev", n), _dev(u_next, "u_next", n),
            self.tol, self.leaf, flags, ctypes.byref(self._cache), _stream(stream)))
        return u_next

    def close(self):
        if self._cache:
            _lib.load().hodlr_destroy(self._cache)
            self._cache = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
