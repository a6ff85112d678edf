"""C-ABI tests that need no GPU: the library loads, exports every symbol the header
declares, and rejects out-of-domain arguments on the host before any device work."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fdehodlr.h")


@pytest.fixture(scope="module")
def lib():
    from paper_1804_05522_b200 import build as b
    b.build()
    from paper_1804_05522_b200 import _lib
    return _lib.load()


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    src = re.sub(r"^\s*typedef[^;]*;", "", src, flags=re.M | re.S)      # (function-pointer typedefs)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_ ]+\*?\s*\b([a-z0-9_]+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    names = header_functions()
    for need in ("hodlr_build", "hodlr_factor", "hodlr_solve", "fde1d_step", "fde2d_step"):
        assert need in names


def test_every_declared_symbol_is_exported(lib):
    from paper_1804_05522_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (\w+)$", out, flags=re.M))
    for name in header_functions():
        assert name in exported, name
        assert name in _lib.SIGNATURES, name


def test_library_is_sm100a(lib):
    from paper_1804_05522_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _step(lib, **kw):
    a = dict(batch=1, n=64, alpha=1.5, h=1.0 / 65, dt=0.1, tol=1e-12, leaf=16)
    a.update(kw)
    alpha = np.full(max(a["batch"], 1), a["alpha"], dtype=np.float64)
    dummy = ctypes.c_void_p(8)  # never dereferenced: domain checks run first on the host
    cache = ctypes.c_void_p()
    rc = lib.fde1d_step(a["batch"], a["n"], alpha.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                        a["h"], a["dt"], dummy, dummy, dummy, dummy, dummy, a["tol"], a["leaf"], 1, 0,
                        ctypes.byref(cache), None)
    return rc, lib.fde_last_error().decode()


@pytest.mark.parametrize("kw,frag", [
    (dict(alpha=1.0), "alpha"), (dict(alpha=2.5), "alpha"), (dict(n=0), "n="),
    (dict(leaf=1), "leaf"), (dict(leaf=129), "leaf"), (dict(tol=0.0), "tol"), (dict(tol=1.0), "tol"),
    (dict(h=0.0), "h="), (dict(dt=-1.0), "dt"), (dict(batch=0), "batch"),
])
def test_domain_errors(lib, kw, frag):
    from paper_1804_05522_b200._lib import FDE_EDOMAIN
    rc, msg = _step(lib, **kw)
    assert rc == FDE_EDOMAIN and frag in msg


def test_null_handle_errors(lib):
    from paper_1804_05522_b200._lib import FDE_EDOMAIN
    assert lib.hodlr_factor(None, 0, None) == FDE_EDOMAIN
    assert lib.hodlr_solve(None, None, None, 1, 1, 0, None) == FDE_EDOMAIN
    assert lib.hodlr_status(None, None) == FDE_EDOMAIN
    lib.hodlr_destroy(None)


def test_product_path_never_touches_the_oracle():
    """The package must not import oracle/ (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_1804_05522_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", txt, flags=re.M), f


def test_fde2d_rejects_bad_arguments_on_host(lib):
    """fde2d_step validates alpha / sizes / tolerances before any device work (no GPU needed)."""
    import ctypes
    from paper_1804_05522_b200 import _lib
    nul = ctypes.c_void_p()
    rx, res, its = ctypes.c_int(), ctypes.c_double(), ctypes.c_int()
    cache = (ctypes.c_void_p * 2)()
    def call(nx=64, a1=1.3, a2=1.7, tol=1e-12, ek_tol=1e-11, rmax=8):
        return lib.fde2d_step(nx, 64, a1, a2, 1.0 / 65, 1.0 / 65, 0.1, nul, nul, nul, nul, nul, nul, 0,
                              nul, nul, 0, nul, nul, rmax, ctypes.byref(rx), tol, ek_tol, 10, 32,
                              ctypes.cast(cache, ctypes.POINTER(ctypes.c_void_p)), ctypes.byref(res),
                              ctypes.byref(its), 0, nul)
    assert call(a1=2.5) == _lib.FDE_EDOMAIN
    assert call(nx=0) == _lib.FDE_EDOMAIN
    assert call(tol=0.0) == _lib.FDE_EDOMAIN
    assert call() == _lib.FDE_EDOMAIN            # NULL coefficient arrays
    assert "NULL" in lib.fde_last_error().decode() or "coefficient" in lib.fde_last_error().decode()
