import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_1804_05522_b200 import workloads as W
from paper_1804_05522_b200.hodlr import Fde2dStepper, Hodlr
from oracle.sylvester2d import operators_2d, BartelsStewart
for ek in (1e-11,):
    wl = W.paper2d(192, 1.3, 1.7, variable=False, tol=1e-12, ek_tol=ek, leaf=32)
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
    st = Fde2dStepper(wl.nx, wl.ny, wl.alpha1, wl.alpha2, wl.hx, wl.hy, wl.dt, t(wl.d1p), t(wl.d1m), t(wl.d2p), t(wl.d2m), wl.tol, ek_tol=ek, leaf=wl.leaf)
    A1, A2 = operators_2d(wl.alpha1, wl.alpha2, wl.nx, wl.ny, wl.hx, wl.hy, wl.dt, wl.d1p, wl.d1m, wl.d2p, wl.d2m)
    bs = BartelsStewart(A1, A2)
    H1 = Hodlr(wl.nx, wl.alpha1, wl.hx, wl.dt, t(wl.d1p), t(wl.d1m), wl.tol, wl.leaf, shift=0.5)
    H2 = Hodlr(wl.ny, wl.alpha2, wl.hy, wl.dt, t(wl.d2p), t(wl.d2m), wl.tol, wl.leaf, shift=0.5)
    if os.environ.get("DBG_FACTOR"):
        H1.factor(); H2.factor()
    def hmv(H, M):   # H @ M for M (n, k): k right-hand sides in blocks of 64 (batch 1: (1, k, n))
        out = []
        for c0 in range(0, M.shape[1], 64):
            y = H.matvec(t(np.ascontiguousarray(M[:, c0:c0 + 64].T))[None])
            out.append(y[0].cpu().numpy().T)
        return np.concatenate(out, axis=1)
    Uo = np.zeros((wl.nx, wl.ny)); Xu = Xv = None; Xprev = np.zeros((wl.nx, wl.ny))
    for m in range(1, 9):
        Fa, Fb = wl.source_factors(m)
        Fu, Fv = t(Fa.T), t(Fb.T)
        if os.environ.get("DBG_FRESH"):
            st.close()
            st = Fde2dStepper(wl.nx, wl.ny, wl.alpha1, wl.alpha2, wl.hx, wl.hy, wl.dt, t(wl.d1p), t(wl.d1m), t(wl.d2p), t(wl.d2m), wl.tol, ek_tol=ek, leaf=wl.leaf)
        if Xu is not None and os.environ.get("DBG_ORTHO"):   # hand the step an orthonormal U factor
            Aq, Bq = Xu.cpu().numpy().T, Xv.cpu().numpy().T
            Q, R = np.linalg.qr(Aq)
            Xu, Xv = t(Q.T), t((Bq @ R.T).T)
        Xu, Xv, res, its = st.step(Fu, Fv) if Xu is None else st.step(Fu, Fv, Xu, Xv)
        Xg = Xu.cpu().numpy().T @ Xv.cpu().numpy()
        Uo = bs.solve(Uo + wl.dt * Fa @ Fb.T)
        C = Xprev + wl.dt * Fa @ Fb.T
        R = A1 @ Xg + Xg @ A2.T - C
        tres = np.linalg.norm(R) / np.linalg.norm(C)
        Xl = bs.solve(C)
        lerr = np.linalg.norm(Xg - Xl) / np.linalg.norm(Xl)
        Rh = hmv(H1, Xg) + hmv(H2, Xg.T).T - C
        hres = np.linalg.norm(Rh) / np.linalg.norm(C)
        Xprev = Xg
        # residual of the GPU X against the exact operator with the GPU's own previous state is not tracked here
        print(ek, m, "err %.2e local err %.2e res %.2e true res %.2e hodlr res %.2e its %d rank %d |C|^2 %.6e" % (np.linalg.norm(Xg - Uo) / np.linalg.norm(Uo), lerr, res, tres, hres, its, Xu.shape[0], np.linalg.norm(C) ** 2))
    st.close()
