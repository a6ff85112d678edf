"""HODLR operator with shift 1/2 (2D operators): matvec / solve vs dense."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_05522_b200.hodlr import Hodlr  # noqa: E402
from oracle.fd1d import assemble_A  # noqa: E402

t = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
for n, leaf in [(64, 128), (512, 128), (2048, 128)]:
    h, dt, alpha = 1.0 / (n + 1), 1.0 / 16, 1.3
    x = h * np.arange(1, n + 1)
    dp, dm = 1 + x, 2 - x
    H = Hodlr(n, alpha, h, dt, t(dp), t(dm), 1e-12, leaf, shift=0.5)
    H.factor()
    A = assemble_A(alpha, n, h, dt, dp, dm, shift=0.5)
    B = np.random.default_rng(0).standard_normal((7, n))
    Y = H.matvec(t(B)[None]).cpu().numpy()[0]
    X = H.solve(t(B)[None]).cpu().numpy()[0]
    print(n, "matvec", np.linalg.norm(Y - B @ A.T) / np.linalg.norm(B @ A.T),
          "solve", np.linalg.norm(X - np.linalg.solve(A, B.T).T) / np.linalg.norm(X), "status", H.status())
    H.close()
