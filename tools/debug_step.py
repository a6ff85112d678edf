"""Stage-by-stage GPU debugging harness (ranks, status, factor, solve, matvec vs dense)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_05522_b200.hodlr import Hodlr, Fde1dStepper  # noqa: E402
from oracle.fd1d import assemble_A  # noqa: E402
from oracle.compress import level_ranks  # noqa: E402


def t(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def run(n, alpha, leaf, tol, dt=0.125):
    h = 1.0 / (n + 1)
    x = h * np.arange(1, n + 1)
    dp, dm = 1 + 0.5 * x, 1.5 - x ** 2
    H = Hodlr(n, alpha, h, dt, t(dp), t(dm), tol, leaf)
    torch.cuda.synchronize()
    print("n=%d alpha=%.2f leaf=%d tol=%g" % (n, alpha, leaf, tol))
    print("  status after build", H.status(), "ranks", H.ranks(),
          "svd", level_ranks(alpha, n, leaf, tol) if n <= 4096 else "-")
    A = assemble_A(alpha, n, h, dt, dp, dm)
    b = np.sin(np.pi * x) + x
    y = H.matvec(t(b)).cpu().numpy()
    print("  matvec rel err", np.linalg.norm(y - A @ b) / np.linalg.norm(A @ b), "nan", np.isnan(y).sum())
    H.factor()
    torch.cuda.synchronize()
    print("  status after factor", H.status())
    u = H.solve(t(b)).cpu().numpy()
    ue = np.linalg.solve(A, b)
    print("  solve rel err", np.linalg.norm(u - ue) / np.linalg.norm(ue), "nan", np.isnan(u).sum())
    st = Fde1dStepper(n, alpha, h, tol, leaf)
    z = np.zeros(n)
    un = st.step(dt, t(dp), t(dm), t(z), t(b)).cpu().numpy()
    print("  fused step rel err", np.linalg.norm(un - ue) / np.linalg.norm(ue), "nan", np.isnan(un).sum())
    H.close(); st.close()


if __name__ == "__main__":
    run(100, 1.5, 128, 1e-12)
    run(256, 1.5, 32, 1e-12)
    run(1000, 1.3, 64, 1e-12)
