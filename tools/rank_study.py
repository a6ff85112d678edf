"""GPU rank study: per-level compressed ranks of T_{alpha,N} from the
device compression (S2: pivoted Cholesky of the level Hankel + Jacobi recompression at
tau = tol * 2^alpha) for N = 2^9 .. 2^17, and the S2 build time.  Writes
profiles/r01_rank_study.json; tests/test_rank_study.py checks the ranks against the paper's
bounds (Lemma 3.7 / Cor. 3.8, oracle.compress)."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1804_05522_b200.hodlr import Hodlr, FDE_COMPRESS_ONLY  # noqa: E402


def ranks_gpu(n, alpha, tol, leaf=128):
    ones = torch.ones(n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    H = Hodlr(n, alpha, 1.0 / (n + 1), 1.0 / 32, ones, ones, tol, leaf, flags=FDE_COMPRESS_ONLY)
    r = H.ranks()
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    H.close()
    return r, el


def main():
    out = []
    for tol in (1e-8, 1e-10, 1e-12):
        for alpha in (1.1, 1.3, 1.5, 1.7, 1.9):
            for e in range(9, 18):
                n = 1 << e
                r, el = ranks_gpu(n, alpha, tol)
                out.append({"n": n, "alpha": alpha, "tol": tol, "leaf": 128, "ranks": r,
                            "max_rank": max(r) if r else 0, "build_s": el})
                print(n, alpha, tol, max(r) if r else 0, "%.3f s" % el, flush=True)
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r01_rank_study.json")
    with open(path, "w") as fh:
        json.dump({"what": "per-level ranks of the device compression of T_{alpha,N} "
                           "(tau = tol * 2^alpha, leaf 128, uniform-depth tree)", "runs": out}, fh, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
