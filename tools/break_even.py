"""The paper's 1D comparison (Sec. 3.6): HODLR (factor once + one back substitution per
time step) against GMRES preconditioned by P1 / P2 per time step, at N = 131072 with the
Sec. 3.6 coefficients, HODLR tolerance 1e-8, GMRES tolerance 1e-7 (alpha 1.2) / 1e-6 (alpha 1.8).
Break-even step count k* = T_factor / (T_pgmres - T_backsub): beyond k* steps the HODLR solver is
faster (the paper: ~13 at alpha = 1.2, ~25 at alpha = 1.8 on a CPU).  Leaf 128 here (the
paper: 256; FDE_LEAF_MAX = 128).  Prints one JSON object."""
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_05522_b200.hodlr import Hodlr, PgmresPlan, apply_exact  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
    out = {"n": n, "leaf": 128, "hodlr_tol": 1e-8}
    for alpha, gtol in ((1.2, 1e-7), (1.8, 1e-6)):
        h = 2.0 / (n + 1)
        dt = h
        x = h * np.arange(1, n + 1)
        g = math.gamma(3.0 - alpha)
        dp = torch.as_tensor(g * x ** alpha, device="cuda")
        dm = torch.as_tensor(g * (2.0 - x) ** alpha, device="cuda")
        b = torch.as_tensor(np.sin(np.pi * x / 2) + 0.3 * x * (2 - x), device="cuda")
        r = {}
        # HODLR: build (S1-S2) + factor once, then back substitutions
        for rep in range(2):
            torch.cuda.synchronize()
            a, e = ev()
            a.record()
            H = Hodlr(n, alpha, h, dt, dp, dm, 1e-8, 128)
            H.factor()
            e.record()
            torch.cuda.synchronize()
            t_fac = a.elapsed_time(e)
            if rep == 0:
                H.close()
        a, e = ev()
        xs = torch.empty_like(b)
        H.solve(b[None], xs[None])
        torch.cuda.synchronize()
        a.record()
        for _ in range(20):
            H.solve(b[None], xs[None])
        e.record()
        torch.cuda.synchronize()
        t_bs = a.elapsed_time(e) / 20
        y = apply_exact(n, alpha, h, dt, dp, dm, xs)
        r["hodlr"] = {"ms_build_factor": t_fac, "ms_backsub": t_bs,
                      "res_over_x": float(torch.linalg.norm(y - b) / torch.linalg.norm(xs)),
                      "res_over_b": float(torch.linalg.norm(y - b) / torch.linalg.norm(b)), "ranks": H.ranks()}
        H.close()
        from paper_1804_05522_b200._lib import FdeError
        for p in (1, 2):
            torch.cuda.synchronize()
            a, e = ev()
            a.record()
            plan = PgmresPlan(n, alpha, h, dt, dp, dm, precond=p, maxit=127)
            e.record()
            torch.cuda.synchronize()
            t_plan = a.elapsed_time(e)
            try:
                plan.solve(b, tol=gtol)
            except FdeError as ex:
                r["P%d" % p] = {"converged": False, "error": str(ex)[:160]}
                plan.close()
                continue
            ts = []
            for _ in range(5):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                xg, its, rel = plan.solve(b, tol=gtol)
                ts.append(1e3 * (time.perf_counter() - t0))
            t_g = min(ts)
            plan.close()
            y = apply_exact(n, alpha, h, dt, dp, dm, xg)
            k = t_fac / (t_g - t_bs) if t_g > t_bs else None
            r["P%d" % p] = {"converged": True, "ms_plan_once": t_plan, "ms_per_solve": t_g, "iterations": its,
                            "prec_relres": rel,
                            "res_over_x": float(torch.linalg.norm(y - b) / torch.linalg.norm(xg)),
                            "res_over_b": float(torch.linalg.norm(y - b) / torch.linalg.norm(b)),
                            "break_even_steps": k}
        out["alpha_%g" % alpha] = r
    out["note"] = ("HODLR times by CUDA events; PGMRES solve by host wall clock around the synchronous call "
                   "(one read-back per iteration, best of 5), its plan (FFT spectra + preconditioner factors, "
                   "once per coefficients) reported apart; break_even_steps = HODLR build+factor / (PGMRES "
                   "solve - HODLR back substitution); Res = ||A x - b|| / ||x|| as in the paper's tables")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
