"""Thin Python binding over the C-ABI (include/fdehodlr.h): argument marshalling only.

Tensors supply device pointers (``data_ptr()``) and torch supplies the current CUDA stream;
every step of the method runs in the CUDA kernels of ``csrc/``.  There is no CPU path.
"""
import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import (check, FDE_SYNC, FDE_CHECK, FDE_HOST_PTRS, FDE_NO_KEEP, FDE_RECOMPRESS,  # noqa: F401
                   FDE_COMPRESS_ONLY, FDE_COEFFS_CHANGED, FDE_REFACTOR)


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _dev(t, name, numel=None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64:
        raise TypeError("%s must be a CUDA float64 tensor" % name)
    if not t.is_contiguous():
        raise ValueError("%s must be contiguous" % name)
    if numel is not None and t.numel() != numel:
        raise ValueError("%s has %d elements, expected %d" % (name, t.numel(), numel))
    return ctypes.c_void_p(t.data_ptr())


def _alpha_arr(alpha, batch):
    a = np.ascontiguousarray(np.broadcast_to(np.asarray(alpha, dtype=np.float64), (batch,)))
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class Hodlr:
    """HODLR representation + factor of  A_b = shift I + (dt/h^alpha_b)(D+ T + D- T^T)."""

    def __init__(self, n, alpha, h, dt, d_plus, d_minus, tol, leaf, shift=1.0, batch=1,
                 flags=0, stream=None):
        lib = _lib.load()
        self.n, self.batch = n, batch
        self._alpha, ap = _alpha_arr(alpha, batch)
        self._h = ctypes.c_void_p()
        check(lib.hodlr_build(batch, n, ap, h, dt, _dev(d_plus, "d_plus", batch * n),
                              _dev(d_minus, "d_minus", batch * n), shift, tol, leaf, flags,
                              _stream(stream), ctypes.byref(self._h)))

    def update(self, dt, d_plus=None, d_minus=None, flags=0, stream=None):
        dp = _dev(d_plus, "d_plus", self.batch * self.n) if d_plus is not None else None
        dm = _dev(d_minus, "d_minus", self.batch * self.n) if d_minus is not None else None
        check(_lib.load().hodlr_update(self._h, dt, dp, dm, flags, _stream(stream)))

    def factor(self, flags=0, stream=None):
        check(_lib.load().hodlr_factor(self._h, flags, _stream(stream)))

    def solve(self, b, x=None, flags=0, stream=None):
        """b: (batch, nrhs, n) or (batch, n) CUDA float64; returns x (may be b)."""
        if x is None:
            x = torch.empty_like(b)
        nrhs = 1 if b.dim() <= 2 else b.shape[-2]
        check(_lib.load().hodlr_solve(self._h, _dev(b, "b"), _dev(x, "x", b.numel()), nrhs,
                                      self.n, flags, _stream(stream)))
        return x

    def matvec(self, x, y=None, flags=0, stream=None):
        if y is None:
            y = torch.empty_like(x)
        nrhs = 1 if x.dim() <= 2 else x.shape[-2]
        check(_lib.load().hodlr_matvec(self._h, _dev(x, "x"), _dev(y, "y", x.numel()), nrhs,
                                       self.n, flags, _stream(stream)))
        return y

    def status(self):
        where = ctypes.c_int()
        return _lib.load().hodlr_status(self._h, ctypes.byref(where)), where.value

    def ranks(self, inst=0):
        buf = (ctypes.c_int * 64)()
        levels = ctypes.c_int()
        check(_lib.load().hodlr_ranks(self._h, inst, buf, 64, ctypes.byref(levels)))
        return [buf[i] for i in range(levels.value)]

    def close(self):
        if self._h:
            _lib.load().hodlr_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Fde1dStepper:
    """Implicit-Euler stepper (Eq. 2.5) over fde1d_step with a cached handle."""

    def __init__(self, n, alpha, h, tol, leaf, batch=1):
        self.n, self.batch, self.h, self.tol, self.leaf = n, batch, h, tol, leaf
        self._alpha, self._ap = _alpha_arr(alpha, batch)
        self._cache = ctypes.c_void_p()

    def step(self, dt, d_plus, d_minus, f, u_prev, u_next=None, coeffs_changed=True, flags=0,
             stream=None):
        cnt = self.batch * self.n
        host = bool(flags & FDE_HOST_PTRS)
        if u_next is None:
            u_next = torch.empty_like(u_prev)

        def ptr(t, name):
            if host:
                if t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous() or t.numel() != cnt:
                    raise TypeError("%s must be a contiguous CPU float64 tensor of %d" % (name, cnt))
                return ctypes.c_void_p(t.data_ptr())
            return _dev(t, name, cnt)

        check(_lib.load().fde1d_step(self.batch, self.n, self._ap, self.h, dt,
                                     ptr(d_plus, "d_plus"), ptr(d_minus, "d_minus"), ptr(f, "f"),
                                     ptr(u_prev, "u_prev"), ptr(u_next, "u_next"), self.tol,
                                     self.leaf, int(bool(coeffs_changed)), flags,
                                     ctypes.byref(self._cache), _stream(stream)))
        return u_next

    def run(self, dt, d_plus, d_minus, f, u0, u_out=None, flags=0, stream=None, K=None):
        """K steps in one pipelined launch (fde1d_run).  d_plus, d_minus, f: CUDA float64
        (K, batch, n) -- or (1, batch, n) for time-invariant data (coefficients given once: the
        launch factors once, unless flags has FDE_REFACTOR); u0 (batch, n).  K defaults to the
        largest leading dimension.  Returns u_out (K, batch, n): every step's solution."""
        cnt = self.batch * self.n
        if K is None:
            K = max(d_plus.shape[0], f.shape[0])
        for name, t in (("d_plus", d_plus), ("d_minus", d_minus), ("f", f)):
            if t.shape[0] not in (1, K) or t[0].numel() != cnt:
                raise ValueError("%s must be (K or 1, batch, n)" % name)
        cs = cnt if d_plus.shape[0] > 1 else 0
        if d_minus.shape[0] != d_plus.shape[0]:
            raise ValueError("d_plus and d_minus must have the same number of time levels")
        fs = cnt if f.shape[0] > 1 else 0
        host = bool(flags & FDE_HOST_PTRS)
        if u_out is None:
            u_out = torch.empty((K,) + tuple(u0.shape), dtype=torch.float64, device=u0.device)
            if host:
                u_out = u_out.pin_memory()

        def ptr(t, name, numel=None):
            if not host:
                return _dev(t, name, numel)
            if t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
                raise TypeError("%s must be a contiguous CPU float64 tensor (pinned for async copies)" % name)
            return ctypes.c_void_p(t.data_ptr())
        check(_lib.load().fde1d_run(self.batch, self.n, self._ap, self.h, dt, K, ptr(d_plus, "d_plus"),
                                    ptr(d_minus, "d_minus"), cs, ptr(f, "f"), fs, ptr(u0, "u0", cnt),
                                    ptr(u_out, "u_out", K * cnt), self.tol, self.leaf, flags,
                                    ctypes.byref(self._cache), _stream(stream)))
        return u_out

    def ranks(self, inst=0):
        buf = (ctypes.c_int * 64)()
        levels = ctypes.c_int()
        check(_lib.load().hodlr_ranks(self._cache, inst, buf, 64, ctypes.byref(levels)))
        return [buf[i] for i in range(levels.value)]

    def close(self):
        if self._cache:
            _lib.load().hodlr_destroy(self._cache)
            self._cache = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def launch_count():
    return _lib.load().fde_launch_count()


class Fde2dStepper:
    """One implicit-Euler step of the 2D FDE as the Sylvester equation of Eq. (4.3)
    over fde2d_step, with the two HODLR operator handles cached across steps.

    step(Fu, Fv, Uu, Uv) solves  A1 X + X A2^T = Uu Uv^T + dt Fu Fv^T  and returns
    (Xu, Xv, resid, iters) with X = Xu Xv^T (CUDA float64, column blocks (r, n) row-major =
    column-major (n, r))."""

    def __init__(self, nx, ny, alpha1, alpha2, hx, hy, dt, d1p, d1m, d2p, d2m, tol, ek_tol=1e-11,
                 ek_maxit=60, leaf=128, rmax=256):
        self.nx, self.ny = nx, ny
        self.alpha1, self.alpha2, self.hx, self.hy, self.dt = alpha1, alpha2, hx, hy, dt
        self.coef = [_dev(d1p, "d1p", nx), _dev(d1m, "d1m", nx), _dev(d2p, "d2p", ny), _dev(d2m, "d2m", ny)]
        self._keep = (d1p, d1m, d2p, d2m)
        self.tol, self.ek_tol, self.ek_maxit, self.leaf, self.rmax = tol, ek_tol, ek_maxit, leaf, rmax
        self._cache = (ctypes.c_void_p * 2)()

    def step(self, Fu, Fv, Uu=None, Uv=None, flags=0, stream=None):
        """Fu (rf, nx), Fv (rf, ny), Uu (ru, nx), Uv (ru, ny): CUDA float64, one factor column per row."""
        dev = Fu.device
        rf = Fu.shape[0]
        ru = 0 if Uu is None else Uu.shape[0]
        Xu = torch.zeros(self.rmax, self.nx, dtype=torch.float64, device=dev)
        Xv = torch.zeros(self.rmax, self.ny, dtype=torch.float64, device=dev)
        rx = ctypes.c_int()
        res = ctypes.c_double()
        its = ctypes.c_int()
        nul = ctypes.c_void_p()
        check(_lib.load().fde2d_step(
            self.nx, self.ny, self.alpha1, self.alpha2, self.hx, self.hy, self.dt,
            *self.coef, _dev(Fu, "Fu", rf * self.nx), _dev(Fv, "Fv", rf * self.ny), rf,
            _dev(Uu, "Uu", ru * self.nx) if ru else nul, _dev(Uv, "Uv", ru * self.ny) if ru else nul, ru,
            _dev(Xu, "Xu"), _dev(Xv, "Xv"), self.rmax, ctypes.byref(rx), self.tol, self.ek_tol,
            self.ek_maxit, self.leaf, ctypes.cast(self._cache, ctypes.POINTER(ctypes.c_void_p)),
            ctypes.byref(res), ctypes.byref(its), flags, _stream(stream)))
        r = rx.value
        return Xu[:r].contiguous(), Xv[:r].contiguous(), res.value, its.value

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


def pgmres(n, alpha, h, dt, d_plus, d_minus, b, precond=2, tol=1e-7, maxit=100, x=None, stream=None):
    """fde1d_pgmres: GMRES for A_m x = b with the tridiagonal preconditioner P1 (precond=1) or P2
    (precond=2), or none (0), on the FFT-applied exact operator.  Returns (x, iterations, relres)."""
    if x is None:
        x = torch.empty_like(b)
    its, rel = ctypes.c_int(), ctypes.c_double()
    check(_lib.load().fde1d_pgmres(n, float(alpha), h, dt, _dev(d_plus, "d_plus", n), _dev(d_minus, "d_minus", n),
                                   _dev(b, "b", n), _dev(x, "x", n), precond, tol, maxit, ctypes.byref(its),
                                   ctypes.byref(rel), 0, _stream(stream)))
    return x, its.value, rel.value


def apply_exact(n, alpha, h, dt, d_plus, d_minus, x, y=None, stream=None):
    """fde1d_apply_exact: y = A_m x with the exact operator (FFT circulant embedding)."""
    if y is None:
        y = torch.empty_like(x)
    check(_lib.load().fde1d_apply_exact(n, float(alpha), h, dt, _dev(d_plus, "d_plus", n),
                                        _dev(d_minus, "d_minus", n), _dev(x, "x", n), _dev(y, "y", n),
                                        _stream(stream)))
    return y


class PgmresPlan:
    """fde1d_pgmres_plan / _solve: the operator spectra and preconditioner factors built once,
    then any number of solves (time-invariant coefficients)."""

    def __init__(self, n, alpha, h, dt, d_plus, d_minus, precond=2, maxit=100, stream=None):
        self.n = n
        self._p = ctypes.c_void_p()
        self._keep = (d_plus, d_minus)
        check(_lib.load().fde1d_pgmres_plan(n, float(alpha), h, dt, _dev(d_plus, "d_plus", n),
                                            _dev(d_minus, "d_minus", n), precond, maxit, _stream(stream),
                                            ctypes.byref(self._p)))

    def solve(self, b, x=None, tol=1e-7, stream=None):
        if x is None:
            x = torch.empty_like(b)
        its, rel = ctypes.c_int(), ctypes.c_double()
        check(_lib.load().fde1d_pgmres_solve(self._p, _dev(b, "b", self.n), _dev(x, "x", self.n), tol,
                                             ctypes.byref(its), ctypes.byref(rel), _stream(stream)))
        return x, its.value, rel.value

    def close(self):
        if self._p:
            _lib.load().fde1d_pgmres_destroy(self._p)
            self._p = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
