"""Build the sm_100a shared libraries in-tree (nvcc, no torch).

libfdehodlr.so      the product library (the C-ABI of include/fdehodlr.h)
libfdehodlr_dbg.so  the same sources with -DFDE_DEBUG: adds the environment-driven trace /
                    experiment switches (FDE_TRACE_RUN, FDE_DEBUG2D, ...) used by tools/ and by
                    bench.py's untimed task profile; never loaded unless FDE_LIB_DEBUG=1
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "fdehodlr.cu")
OUT = os.path.join(HERE, "libfdehodlr.so")
OUT_DBG = os.path.join(HERE, "libfdehodlr_dbg.so")


def _cmd(out, debug, verbose):
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-shared", "-Xcompiler", "-fPIC", "-o", out + ".tmp", SRC]
    if debug:
        cmd.insert(1, "-DFDE_DEBUG")
    cmd[1:1] = os.environ.get("FDE_NVCC_FLAGS", "").split()        # (experiments: -D...)
    if verbose:
        cmd[1:1] = ["-Xptxas", "-v"]
    return cmd


def build(verbose: bool = False, force: bool = False, debug: bool = True) -> str:
    """Compile the product library (and, with debug=True, the diagnostics variant) if any
    source is newer than it; both compile concurrently."""
    deps = [os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "fdehodlr.h"))
    todo = []
    for out, dbg in ((OUT, False), (OUT_DBG, True)):
        if dbg and not debug:
            continue
        if force or not os.path.exists(out) or any(os.path.getmtime(out) < os.path.getmtime(d) for d in deps):
            todo.append((out, dbg))
    procs = [(out, subprocess.Popen(_cmd(out, dbg, verbose and not dbg), stdout=subprocess.PIPE,
                                    stderr=subprocess.PIPE, text=True)) for out, dbg in todo]
    failed = False
    for out, p in procs:
        so, se = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(so + se)
            failed = True
            continue
        if verbose and out == OUT:
            sys.stderr.write(se)
        os.replace(out + ".tmp", out)
    if failed:
        raise RuntimeError("nvcc failed for libfdehodlr")
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True, debug="--no-debug" not in sys.argv))
