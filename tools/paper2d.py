"""The paper's 2D experiment protocol (Sec. 5.1) on the GPU:
8 implicit-Euler steps with dt = 1 of the Sylvester form (Eq. 4.3), HODLR tol 1e-8, EK tolerance
1e-6, alpha = (1.3, 1.7) and (1.7, 1.9), constant and Eq. (5.1) coefficients, for a ladder of N.
Reports the total time of the 8 steps (build + factor of both operators included, as t_HODLR in
the paper's tables), the final rank of X, the operators' top-level ranks and the EK iterations.
usage: python tools/paper2d.py [out.json] [N ...]"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1804_05522_b200 import workloads as W  # noqa: E402
from paper_1804_05522_b200.hodlr import Fde2dStepper, Hodlr, FDE_COMPRESS_ONLY  # noqa: E402


def run(n, alphas, variable):
    wl = W.paper2d(n, *alphas, variable=variable)
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = Fde2dStepper(wl.nx, wl.ny, wl.alpha1, wl.alpha2, wl.hx, wl.hy, wl.dt, t(wl.d1p), t(wl.d1m),
                      t(wl.d2p), t(wl.d2m), wl.tol, ek_tol=wl.ek_tol, ek_maxit=60, leaf=wl.leaf)   # (binding default 30:
    # the first step from u0 = 0 needs 27-31 EK iterations at N >= 32768 with alpha = (1.7, 1.9))
    Xu = Xv = None
    its, ranks, res = [], [], []
    for m in range(1, wl.K + 1):
        Fa, Fb = wl.source_factors(m)
        Fu, Fv = t(Fa.T), t(Fb.T)
        Xu, Xv, r, it = st.step(Fu, Fv) if Xu is None else st.step(Fu, Fv, Xu, Xv)
        its.append(it); ranks.append(int(Xu.shape[0])); res.append(r)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    st.close()
    qs = []
    for a, d in ((wl.alpha1, (wl.d1p, wl.d1m)), (wl.alpha2, (wl.d2p, wl.d2m))):
        H = Hodlr(n, a, wl.hx, wl.dt, t(d[0]), t(d[1]), wl.tol, wl.leaf, shift=0.5, flags=FDE_COMPRESS_ONLY)
        qs.append(max(H.ranks()) + 1 if n > wl.leaf else 0)      # +1: the exact -g_0 term
        H.close()
    return {"n": n, "alpha": list(alphas), "coefficients": "Eq. (5.1)" if variable else "constant 1",
            "t_8_steps_s": el, "final_rank": ranks[-1], "ranks": ranks, "ek_iterations": its,
            "residuals": res, "qsrank_ops": qs}


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02_paper2d.json")
    ns = [int(a) for a in sys.argv[2:]] or [1024, 2048, 4096, 8192, 16384, 32768, 65536]
    run(512, (1.3, 1.7), False)                                  # warm-up (module load, JIT-free)
    rows = []
    for variable in (False, True):
        for alphas in ((1.3, 1.7), (1.7, 1.9)):
            for n in ns:
                r = run(n, alphas, variable)
                rows.append(r)
                print("%s a=%s n=%6d: %.3f s  rank %d  its %s  qs %s" % (r["coefficients"], r["alpha"], n,
                      r["t_8_steps_s"], r["final_rank"], r["ek_iterations"], r["qsrank_ops"]), flush=True)
    with open(out, "w") as fh:
        json.dump({"protocol": "paper Sec. 5.1 (P:1584-1632): dt = 1, 8 steps, HODLR tol 1e-8, "
                               "EK tol 1e-6, leaf 128; time = host wall clock of all 8 steps incl. "
                               "build + factor of both operators", "runs": rows}, fh, indent=1)
    with open(os.path.splitext(out)[0] + ".md", "w") as fh:
        fh.write("# Paper protocol 2D run (Sec. 5.1, P:1584-1632; SURVEY 8(f) NEXT-2)\n\n"
                 "`tools/paper2d.py` on B200: dt = 1, 8 implicit-Euler steps of the Sylvester form, HODLR tol "
                 "1e-8, EK tolerance 1e-6, leaf 128; t = host wall clock of all 8 steps including build + "
                 "factor of both operators; rank = rank of the final X; its = EK iterations per step; "
                 "qs = max compressed rank + 1 of A1, A2; res = largest reported relative residual.\n\n"
                 "| coefficients | alpha | N | t (s) | rank | its | qs | res |\n|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            fh.write("| %s | (%s, %s) | %d | %.3f | %d | %s | %d/%d | %.1e |\n" % (
                r["coefficients"], r["alpha"][0], r["alpha"][1], r["n"], r["t_8_steps_s"], r["final_rank"],
                ",".join(str(i) for i in r["ek_iterations"]), r["qsrank_ops"][0], r["qsrank_ops"][1],
                max(r["residuals"])))
    print("wrote", out)


if __name__ == "__main__":
    main()
