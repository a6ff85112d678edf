"""The x/y split of the 2D Sylvester step over a pair of ranks (BASELINE
configs[4]; the extended block Arnoldi processes for A1 and A2 are independent).

Rank 0 of a pair owns A1, its Krylov basis and the factor Xu; rank 1 owns A2, its basis and Xv.
All arithmetic runs in the C-ABI call fde2d_step_split (include/fdehodlr.h); this module only
supplies its all-gather callback -- torch.distributed over NCCL on the GPU box -- and marshals
arguments.  With world > 2 the ranks form independent pairs (2p, 2p+1), each solving its own
problem (replicas of the split; weak scaling).

The exchange layout (mirrors ``Xchg`` in csrc/fde2d.cuh): a send buffer of two slots of S doubles
[side 0 | side 1], of which an owned side fills its own; after the all-gather the receive buffer
is world x send in rank order and side d is read from the slot of its owner (rank d; at world 1,
rank 0).
"""
import ctypes

import torch
import torch.distributed as dist

from . import _lib
from ._lib import check


class _DevPtr:
    """Zero-copy view of a device buffer of doubles for torch (``__cuda_array_interface__``)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def as_tensor(ptr, n):
    return torch.as_tensor(_DevPtr(ptr, n), device="cuda")


def owner(d, world):
    return 0 if world == 1 else d


def side_slot(recv, d, S, world):
    """Side d's slot in a gathered receive buffer (1-D tensor of world * 2 * S)."""
    o = owner(d, world) * 2 * S + d * S
    return recv[o:o + S]


def gather_into(recv, send, group=None):
    """recv (world * count) <- all-gather of every rank's send (count), rank order."""
    if group is None and not dist.is_initialized():
        recv.copy_(send)                 # world 1 loopback
        return
    dist.all_gather_into_tensor(recv, send, group=group)


def pair_group(world, rank):
    """Pairs (2p, 2p+1) of the default group (every rank must call this); (group, pair rank, pair size)."""
    if world == 1:
        return None, 0, 1
    groups = [dist.new_group([2 * p, 2 * p + 1]) if 2 * p + 1 < world else dist.new_group([2 * p])
              for p in range((world + 1) // 2)]
    g = groups[rank // 2]
    size = 2 if 2 * (rank // 2) + 1 < world else 1
    return g, rank % 2, size


class SplitSylvesterStepper:
    """One implicit-Euler step of the 2D FDE as the Sylvester equation of Eq. (4.3) with the x/y
    split over a pair of ranks (pair size 1: both sides local, the exchanges through the same
    callback as a loopback).  step() returns (X_own, rank, resid, iters): X_own = Xu (r, nx) on
    pair rank 0 and Xv (r, ny) on pair rank 1 (both at pair size 1, as (Xu, Xv))."""

    def __init__(self, nx, ny, alpha1, alpha2, hx, hy, dt, d1p, d1m, d2p, d2m, tol, ek_tol=1e-11,
                 ek_maxit=60, leaf=128, rmax=256, group=None, world=1, rank=0):
        from .hodlr import _dev
        self.nx, self.ny, self.world, self.rank, self.group = nx, ny, world, rank, group
        self.alpha1, self.alpha2, self.hx, self.hy, self.dt = alpha1, alpha2, hx, hy, dt
        nul = ctypes.c_void_p()
        own0, own1 = world == 1 or rank == 0, world == 1 or rank == 1
        self.coef = [_dev(d1p, "d1p", nx) if own0 else nul, _dev(d1m, "d1m", nx) if own0 else nul,
                     _dev(d2p, "d2p", ny) if own1 else nul, _dev(d2m, "d2m", ny) if own1 else nul]
        self._keep = (d1p, d1m, d2p, d2m)
        self.own = (own0, own1)
        self.tol, self.ek_tol, self.ek_maxit, self.leaf, self.rmax = tol, ek_tol, ek_maxit, leaf, rmax
        self._cache = (ctypes.c_void_p * 2)()
        self.calls = 0
        self._cb = _lib.ALLGATHER_FN(self._gather)       # (kept alive with the stepper)

    def _gather(self, ctx, send, recv, count, stream):
        try:
            s = as_tensor(send, count)
            r = as_tensor(recv, self.world * count)
            gather_into(r, s, self.group if self.world > 1 else None)
            self.calls += 1
            return 0
        except Exception:                                  # reported by the library as FDE_ECUDA
            return 1

    def step(self, Fu, Fv, Uu=None, Uv=None, flags=0, stream=None):
        """Fu (rf, nx) / Fv (rf, ny), Uu (ru, nx) / Uv (ru, ny): CUDA float64; a rank passes only its
        own side's factors (the other may be None)."""
        from .hodlr import _dev, _stream
        nul = ctypes.c_void_p()
        own0, own1 = self.own
        rf = (Fu if own0 else Fv).shape[0]
        U_own = Uu if own0 else Uv
        ru = 0 if U_own is None else U_own.shape[0]
        dev = (Fu if own0 else Fv).device
        Xu = torch.zeros(self.rmax, self.nx, dtype=torch.float64, device=dev) if own0 else None
        Xv = torch.zeros(self.rmax, self.ny, dtype=torch.float64, device=dev) if own1 else None
        rx, res, its = ctypes.c_int(), ctypes.c_double(), ctypes.c_int()
        p = lambda t, name, cnt, ok: _dev(t, name, cnt) if (ok and t is not None) else nul
        check(_lib.load().fde2d_step_split(
            self.world, self.rank, ctypes.cast(self._cb, ctypes.c_void_p), None,
            self.nx, self.ny, self.alpha1, self.alpha2, self.hx, self.hy, self.dt, *self.coef,
            p(Fu, "Fu", rf * self.nx, own0), p(Fv, "Fv", rf * self.ny, own1), rf,
            p(Uu, "Uu", ru * self.nx, own0 and ru > 0), p(Uv, "Uv", ru * self.ny, own1 and ru > 0), ru,
            p(Xu, "Xu", None, own0), p(Xv, "Xv", None, own1), self.rmax, ctypes.byref(rx), self.tol,
            self.ek_tol, self.ek_maxit, self.leaf, ctypes.cast(self._cache, ctypes.POINTER(ctypes.c_void_p)),
            ctypes.byref(res), ctypes.byref(its), flags, _stream(stream)))
        r = rx.value
        if own0 and own1:
            return (Xu[:r].contiguous(), Xv[:r].contiguous()), r, res.value, its.value
        X = Xu if own0 else Xv
        return X[:r].contiguous(), r, res.value, its.value

    def close(self):
        for i in range(2):
            if self._cache[i]:
                _lib.load().hodlr_destroy(self._cache[i])
                self._cache[i] = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pole_block(recv, j, pw, cnt, blk):
    """Block j of an all-gathered pole exchange (mirrors fde2d.cuh rk_grow): rank j mod pw sent
    its blocks j = pr, pr + pw, ... packed, so block j sits at (j mod pw) * cnt + (j // pw) * blk."""
    o = (j % pw) * cnt + (j // pw) * blk
    return recv[o:o + blk]


class RkSylvesterStepper:
    """fde2d_step_rk: the 2D step with a multi-shift rational Krylov projection (NEXT-1); with
    pw > 1 the shifted solves of a round are sharded over the ranks of `group` (pole j on rank
    j mod pw, blocks all-gathered).  step() returns (Xu, Xv, resid, rounds) on every rank."""

    def __init__(self, nx, ny, alpha1, alpha2, hx, hy, dt, d1p, d1m, d2p, d2m, tol, rk_tol=1e-11,
                 npole=8, rounds=3, poles=None, leaf=128, rmax=256, group=None, pw=1, pr=0):
        import numpy as np
        from .hodlr import _dev
        self.nx, self.ny, self.alpha1, self.alpha2, self.hx, self.hy, self.dt = nx, ny, alpha1, alpha2, hx, hy, dt
        self.coef = [_dev(d1p, "d1p", nx), _dev(d1m, "d1m", nx), _dev(d2p, "d2p", ny), _dev(d2m, "d2m", ny)]
        self._keep = (d1p, d1m, d2p, d2m)
        self.tol, self.rk_tol, self.npole, self.rounds, self.leaf, self.rmax = tol, rk_tol, npole, rounds, leaf, rmax
        self.poles = None if poles is None else np.ascontiguousarray(poles, dtype=np.float64)
        self.group, self.pw, self.pr = group, pw, pr
        self._cache = (ctypes.c_void_p * (2 + 2 * npole * rounds))()
        self.calls = 0
        self._cb = _lib.ALLGATHER_FN(self._gather)

    def _gather(self, ctx, send, recv, count, stream):
        try:
            gather_into(as_tensor(recv, self.pw * count), as_tensor(send, count), self.group if self.pw > 1 else None)
            self.calls += 1
            return 0
        except Exception:
            return 1

    def step(self, Fu, Fv, Uu=None, Uv=None, flags=0, stream=None):
        from .hodlr import _dev, _stream
        nul = ctypes.c_void_p()
        rf = Fu.shape[0]
        ru = 0 if Uu is None else Uu.shape[0]
        Xu = torch.zeros(self.rmax, self.nx, dtype=torch.float64, device=Fu.device)
        Xv = torch.zeros(self.rmax, self.ny, dtype=torch.float64, device=Fu.device)
        rx, res, rnd = ctypes.c_int(), ctypes.c_double(), ctypes.c_int()
        pp = (self.poles.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if self.poles is not None
              else ctypes.POINTER(ctypes.c_double)())
        check(_lib.load().fde2d_step_rk(
            self.pw, self.pr, ctypes.cast(self._cb, ctypes.c_void_p) if self.pw > 1 else None, None,
            self.nx, self.ny, self.alpha1, self.alpha2, self.hx, self.hy, self.dt, *self.coef,
            _dev(Fu, "Fu", rf * self.nx), _dev(Fv, "Fv", rf * self.ny), rf,
            _dev(Uu, "Uu", ru * self.nx) if ru else nul, _dev(Uv, "Uv", ru * self.ny) if ru else nul, ru,
            _dev(Xu, "Xu"), _dev(Xv, "Xv"), self.rmax, ctypes.byref(rx), self.tol, self.rk_tol, self.npole,
            self.rounds, pp, self.leaf, ctypes.cast(self._cache, ctypes.POINTER(ctypes.c_void_p)),
            ctypes.byref(res), ctypes.byref(rnd), flags, _stream(stream)))
        r = rx.value
        return Xu[:r].contiguous(), Xv[:r].contiguous(), res.value, rnd.value

    def close(self):
        for i in range(len(self._cache)):
            if self._cache[i]:
                _lib.load().hodlr_destroy(self._cache[i])
                self._cache[i] = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
