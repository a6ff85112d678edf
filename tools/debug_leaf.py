"""Targeted checks of the leaf kernel paths (single leaf, ragged leaves, matvec)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_05522_b200.hodlr import Hodlr  # noqa: E402
from oracle.fd1d import assemble_A  # noqa: E402


def t(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


for (n, leaf) in [(64, 64), (63, 64), (40, 64), (128, 64), (127, 64), (100, 128), (200, 128)]:
    h = 1.0 / (n + 1); dt = 0.1; alpha = 1.5
    x = h * np.arange(1, n + 1)
    dp, dm = 1 + x, 2 - x
    H = Hodlr(n, alpha, h, dt, t(dp), t(dm), 1e-12, leaf)
    A = assemble_A(alpha, n, h, dt, dp, dm)
    b = np.sin(3 * x) + x
    y = H.matvec(t(b)).cpu().numpy()
    H.factor()
    u = H.solve(t(b)).cpu().numpy()
    ue = np.linalg.solve(A, b)
    print(n, leaf, "matvec", np.linalg.norm(y - A @ b) / np.linalg.norm(A @ b),
          "solve", np.linalg.norm(u - ue) / np.linalg.norm(ue), H.status())
    H.close()
