"""ctypes loader for libfdehodlr.so (the C-ABI of include/fdehodlr.h).

There is no fallback: if the library is missing or fails to load, every call raises.
"""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# the diagnostics build (trace / experiment switches read from the environment) only on request
LIB_PATH = os.path.join(HERE, "libfdehodlr_dbg.so" if os.environ.get("FDE_LIB_DEBUG") == "1"
                        else "libfdehodlr.so")

FDE_OK, FDE_EDOMAIN, FDE_EDIM, FDE_ESINGULAR, FDE_ENOCONV, FDE_ECUDA, FDE_ENOMEM = range(7)
FDE_SYNC, FDE_CHECK, FDE_HOST_PTRS, FDE_NO_KEEP, FDE_RECOMPRESS, FDE_COMPRESS_ONLY = 1, 2, 4, 8, 16, 32
FDE_COEFFS_CHANGED = 64
FDE_REFACTOR = 128
FDE_LEAF_MAX, FDE_RANK_MAX = 128, 47

# every symbol the header declares, with its ctypes signature
_d, _i, _u, _p = ctypes.c_double, ctypes.c_int, ctypes.c_uint, ctypes.c_void_p
_pd = ctypes.POINTER(ctypes.c_double)
_pi = ctypes.POINTER(ctypes.c_int)
_ph = ctypes.POINTER(ctypes.c_void_p)
SIGNATURES = {
    "hodlr_build": (_i, [_i, _i, _pd, _d, _d, _p, _p, _d, _d, _i, _u, _p, _ph]),
    "hodlr_update": (_i, [_p, _d, _p, _p, _u, _p]),
    "hodlr_factor": (_i, [_p, _u, _p]),
    "hodlr_solve": (_i, [_p, _p, _p, _i, _i, _u, _p]),
    "hodlr_matvec": (_i, [_p, _p, _p, _i, _i, _u, _p]),
    "hodlr_status": (_i, [_p, _pi]),
    "hodlr_ranks": (_i, [_p, _i, _pi, _i, _pi]),
    "hodlr_destroy": (None, [_p]),
    "fde1d_step": (_i, [_i, _i, _pd, _d, _d, _p, _p, _p, _p, _p, _d, _i, _i, _u, _ph, _p]),
    "fde1d_run": (_i, [_i, _i, _pd, _d, _d, _i, _p, _p, ctypes.c_longlong, _p, ctypes.c_longlong, _p, _p,
                       _d, _i, _u, _ph, _p]),
    "fde2d_step": (_i, [_i, _i, _d, _d, _d, _d, _d, _p, _p, _p, _p, _p, _p, _i, _p, _p, _i,
                        _p, _p, _i, _pi, _d, _d, _i, _i, _ph, _pd, _pi, _u, _p]),
    "fde1d_step_split": (_i, [_i, _i, _p, _p, _i, _d, _d, _d, _p, _p, _p, _p, _p, _d, _i, _u, _ph, _p]),
    "fde1d_pgmres": (_i, [_i, _d, _d, _d, _p, _p, _p, _p, _i, _d, _i, _pi, _pd, _u, _p]),
    "fde1d_pgmres_plan": (_i, [_i, _d, _d, _d, _p, _p, _i, _i, _p, _ph]),
    "fde1d_pgmres_solve": (_i, [_p, _p, _p, _d, _pi, _pd, _p]),
    "fde1d_pgmres_destroy": (None, [_p]),
    "fde1d_apply_exact": (_i, [_i, _d, _d, _d, _p, _p, _p, _p, _p]),
    "fde2d_step_rk": (_i, [_i, _i, _p, _p, _i, _i, _d, _d, _d, _d, _d, _p, _p, _p, _p, _p, _p, _i, _p, _p, _i,
                           _p, _p, _i, _pi, _d, _d, _i, _i, _pd, _i, _ph, _pd, _pi, _u, _p]),
    "fde2d_step_split": (_i, [_i, _i, _p, _p, _i, _i, _d, _d, _d, _d, _d, _p, _p, _p, _p, _p, _p, _i, _p, _p, _i,
                              _p, _p, _i, _pi, _d, _d, _i, _i, _ph, _pd, _pi, _u, _p]),
    "fde_last_error": (ctypes.c_char_p, []),
    "fde_launch_count": (ctypes.c_longlong, []),
    "fde_profile_enable": (None, [_i]),
    "fde_profile_dump": (_i, [ctypes.c_char_p, _i]),
}

# all-gather callback of fde2d_step_split: (ctx, send, recv, count, stream) -> 0
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_longlong, ctypes.c_void_p)

_lib = None


class FdeError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("fdehodlr error %d: %s" % (code, msg))
        self.code = code


def load():
    """Load (once) and return the ctypes library; raises if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FdeError(FDE_ECUDA, "%s not built (run __graft_entry__.build() or "
                                  "python paper_1804_05522_b200/build.py)" % os.path.basename(LIB_PATH))
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc):
    if rc != FDE_OK:
        raise FdeError(rc, load().fde_last_error().decode())
    return rc
