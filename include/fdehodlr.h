/*
 * fdehodlr.h -- C-ABI of the B200-native HODLR time-stepper for space-fractional
 * diffusion (arXiv 1804.05522).  Citations: P:<n> = /root/reference/PAPER.md line n.
 *
 * Problem (Eq. 1.1; scheme Eq. 2.5-2.6):
 *   A_m u^(m) = u^(m-1) + dt f^(m),
 *   A_m = shift*I + c (D+^(m) T_{alpha,N} + D-^(m) T_{alpha,N}^T),  c = dt / h^alpha,
 *   T_{alpha,N}[i,j] = -g_{i-j+1} (lower Hessenberg Toeplitz), g_k = (-1)^k binom(alpha,k).
 * shift = 1 for the 1D step (Eq. 2.5); shift = 1/2 for the two operators of the
 * 2D Sylvester step (Eq. 4.3).
 *
 * Method (HODLR): GL weights by the recursion of P:1190-1193,
 * per-level compression of the Toeplitz off-diagonal blocks at tolerance tol (P:1145,
 * reading R7: threshold tol*2^alpha on the T-blocks), diagonal scaling + identity shift
 * applied to the compressed factors and leaves, level-by-level factorisation
 * (batched unpivoted leaf LU + Sherman-Morrison-Woodbury updates), tree-ordered solve.
 *
 * Conventions (all entry points):
 *  - Floating point is IEEE double.  Arrays are column-major.  Pointers marked [dev] are
 *    device pointers (e.g. torch.Tensor.data_ptr() of a CUDA tensor), [host] are host
 *    pointers.  Arrays of a batch are stored instance after instance: d_plus[b*n + i].
 *  - Callers own every array they pass.  The library owns only the handle and its
 *    workspaces, released by hodlr_destroy().
 *  - `stream` is a cudaStream_t passed as void*; NULL means the legacy default stream.
 *    Every call only enqueues work on `stream` (asynchronous) unless FDE_SYNC is set in
 *    `flags`, in which case it synchronises the stream and reports device-side errors.
 *  - Return value: FDE_OK or a positive FDE_E* code; fde_last_error() (thread-local)
 *    names the offending argument.  Device-side failures (zero / non-finite leaf pivot,
 *    singular SMW capacitance matrix, rank cap exceeded) are latched in the handle and
 *    returned by hodlr_status() after the stream is synchronised.
 *  - Results are deterministic: every reduction has a fixed order, independent of the
 *    CTA schedule.
 */
#ifndef FDEHODLR_H
#define FDEHODLR_H

#ifdef __cplusplus
extern "C" {
#endif

#define FDE_OK        0
#define FDE_EDOMAIN   1   /* argument outside its domain (alpha, n, h, dt, tol, leaf, batch) */
#define FDE_EDIM      2   /* dimension / leading-dimension / rank-capacity mismatch */
#define FDE_ESINGULAR 3   /* zero or non-finite pivot (leaf LU or SMW capacitance matrix) */
#define FDE_ENOCONV   4   /* compression did not reach tol within the rank cap; EK not converged */
#define FDE_ECUDA     5   /* a CUDA runtime call failed */
#define FDE_ENOMEM    6   /* device allocation failed */

/* flags */
#define FDE_SYNC      1u  /* synchronise `stream` before returning and report device errors */
#define FDE_CHECK     2u  /* also check d_plus, d_minus >= 0 on the device (implies a sync) */
#define FDE_HOST_PTRS 4u  /* fde1d_step: d_plus, d_minus, f, u_prev, u_next are HOST arrays; the
                             library copies them through pinned staging buffers on `stream` */
#define FDE_NO_KEEP   8u  /* fde1d_step: do not keep the factor for reuse (saves HBM traffic when
                             the coefficients change every step) */
#define FDE_RECOMPRESS 16u /* fde1d_step: recompute S1 (GL weights) and S2 (compression of T)
                             even when the cached handle already holds them */

#define FDE_COMPRESS_ONLY 32u /* hodlr_build: stop after S1-S2 (GL weights + compression); the handle
                                 serves hodlr_ranks / hodlr_status / hodlr_destroy only (rank
                                 studies beyond the factorisation's width limits) */
#define FDE_COEFFS_CHANGED 64u /* fde2d_step: the coefficient arrays were rewritten in place since the
                                 operators were factorised: refactorise them (the cache otherwise
                                 refactorises only when dt or the coefficient pointers change) */
#define FDE_REFACTOR  128u /* fde1d_run: refactorise every step even when coef_stride is 0 (timing and
                                 checking of the refactor path; the default then factors once) */

/* Compile-time capacities of this build. */
#define FDE_LEAF_MAX  128 /* largest leaf (dense diagonal block) held in shared memory */
#define FDE_RANK_MAX  47  /* largest compressed rank of one level's T-block */

typedef struct fde_hodlr* fde_hodlr_t;   /* opaque; one per (operator family, batch) */

/* All-gather callback of the split entry points (fde1d_step_split, fde2d_step_split):
 * gather(ctx, send, recv, count, stream) gathers `count` doubles of every rank's `send` (device)
 * into `recv` (device, world * count, rank order), ordered on `stream`; returns 0 on success.
 * The Python binding implements it with torch.distributed (NCCL over NVLink on the GPU box). */
typedef int (*fde_allgather_fn)(void* ctx, const double* send, double* recv, long long count, void* stream);

/* Build the HODLR representation of `batch` operators
 *     A_b = shift*I + (dt/h^alpha_b)(D+_b T_{alpha_b} + D-_b T_{alpha_b}^T),  b < batch,
 * i.e. steps S1 (GL weights) and S2 (per-level compression of the Toeplitz
 * off-diagonal blocks) on the device, and records dt and copies of
 * d_plus/d_minus for the next hodlr_factor().
 *   batch >= 1; n >= 1; alpha[host, batch] in (1, 2]; h > 0; dt >= 0; shift > 0;
 *   d_plus, d_minus [dev, batch*n] (>= 0, checked only under FDE_CHECK);
 *   tol in (0, 1): truncation tolerance (relative to ||T||_2 <= 2^alpha, reading R7);
 *   2 <= leaf <= FDE_LEAF_MAX: leaf size (every level is split while its largest node
 *   exceeds leaf, reading R10).
 * On success *out receives a new handle (caller releases it with hodlr_destroy). */
int hodlr_build(int batch, int n, const double* alpha, double h, double dt,
                const double* d_plus, const double* d_minus, double shift,
                double tol, int leaf, unsigned flags, void* stream, fde_hodlr_t* out);

/* Replace dt and the diffusion coefficients (copied from [dev, batch*n]) of a built handle;
 * the compression of T (which depends on alpha, n, leaf, tol only) is reused.
 * d_plus / d_minus may be NULL to keep the current values.  Invalidates the factor. */
int hodlr_update(fde_hodlr_t H, double dt, const double* d_plus, const double* d_minus,
                 unsigned flags, void* stream);

/* Factorise A (S3 diagonal scaling + shift fused into S4 batched leaf LU; S5
 * Sherman-Morrison-Woodbury level updates, leaves to root).  The factor is kept in the
 * handle for any number of hodlr_solve() calls (LU reuse). */
int hodlr_factor(fde_hodlr_t H, unsigned flags, void* stream);

/* Solve A X = B with the kept factor (S6 tree-ordered solve).
 *   b, x [dev]: nrhs columns of length n per instance, leading dimension ld >= n,
 *   instance stride ld*nrhs: element (i, j) of instance q at [q*ld*nrhs + j*ld + i].
 *   x may alias b.  1 <= nrhs <= 64. */
int hodlr_solve(fde_hodlr_t H, const double* b, double* x, int nrhs, int ld,
                unsigned flags, void* stream);

/* y = A x with the HODLR representation (leaf blocks + scaled low-rank factors),
 * same layout conventions as hodlr_solve; y must not alias x. */
int hodlr_matvec(fde_hodlr_t H, const double* x, double* y, int nrhs, int ld,
                 unsigned flags, void* stream);

/* Device-side status latched by the kernels (synchronises the handle's last stream):
 * returns FDE_OK / FDE_ESINGULAR / FDE_ENOCONV; *where (may be NULL) gets the instance*
 * 65536 + index of the first failure (leaf LU pivot: the leaf index; SMW capacitance
 * pivot: 32768 + the node index 2^l - 1 + j; compression: the level).  A latched failure is reported once: returning it here
 * (or from any call given FDE_SYNC) clears the word, so later calls on the handle start clean. */
int hodlr_status(fde_hodlr_t H, int* where);

/* Per-level compressed ranks of instance `inst` (host copy; synchronises the handle's
 * last stream).  ranks[host, levels]; returns the number of levels L in *levels. */
int hodlr_ranks(fde_hodlr_t H, int inst, int* ranks, int max_levels, int* levels);

void hodlr_destroy(fde_hodlr_t H);

/* One implicit-Euler step of Eq. (2.5) for `batch` independent 1D problems:
 *     u_next = A_m^{-1} (u_prev + dt f_m)          (S1-S7)
 * d_plus_m, d_minus_m, f_m, u_prev, u_next: [dev, batch*n] (or [host] with FDE_HOST_PTRS);
 * u_next may alias u_prev.  alpha [host, batch].
 * `cache` (may be NULL): in/out handle.  If *cache is NULL or was built for different
 * (batch, n, alpha, h, leaf, tol), a new handle is built (and the old one destroyed).
 * coeffs_changed != 0 (or no factor kept): the step refactorises with the new d+-, dt and
 * the right-hand side is carried through the factorisation as an extra column (fused
 * factor+solve); coeffs_changed == 0 reuses the kept factor (solve only).
 * With cache == NULL a temporary handle is built and destroyed inside the call. */
int fde1d_step(int batch, int n, const double* alpha, double h, double dt,
               const double* d_plus_m, const double* d_minus_m, const double* f_m,
               const double* u_prev, double* u_next, double tol, int leaf,
               int coeffs_changed, unsigned flags, fde_hodlr_t* cache, void* stream);

/* One implicit-Euler step of ONE problem (batch 1) split over `world` ranks at the top of the HODLR
 * tree (every lower off-diagonal block is a sub-block of
 * the top-level ones).  world = 2^p; rank g owns the leaves [g, g+1) * nleaf/world, i.e. the rows
 * [g, g+1) * n/world, and runs the leaf work (assembly, LU, panel, projection) and the SMW levels
 * p .. L-1 of its subtree; the parts then exchange the level-p projected matrices of their subtree
 * roots ((xc_p - 1) x xc_p doubles each), every rank runs the top levels 0 .. p-1 on the same data
 * and the finals u = X v of its own leaves, and u_next's row blocks are all-gathered, so every rank
 * returns the full u_next.  Same arithmetic as fde1d_step with FDE_NO_KEEP (d+- new every step).
 *   gather: as fde2d_step_split (all-gather of `count` doubles per rank, rank order) -- NULL only
 *   at world 1; rank = -1: run every part in this process, one launch after the other (the
 *   launches of a world-rank split, for checking and per-part timing).
 *   Needs the tree path with L >= p and equal leaves (n = number of leaves x leaf size): FDE_EDIM
 *   otherwise.  u_next must not alias u_prev.  d_plus_m, d_minus_m, f_m, u_prev [dev, n] on every
 *   rank (each reads its rows); cache as fde1d_step. */
int fde1d_step_split(int world, int rank, fde_allgather_fn gather, void* ctx, int n, double alpha, double h,
                     double dt, const double* d_plus_m, const double* d_minus_m, const double* f_m,
                     const double* u_prev, double* u_next, double tol, int leaf, unsigned flags,
                     fde_hodlr_t* cache, void* stream);

/* K implicit-Euler steps of Eq. (2.5) in one pipelined launch (fused factor + solve every step,
 * P:1310-1315):  u^(m) = A_m^{-1}(u^(m-1) + dt f^(m)),  m = 1..K.  The coefficient-dependent
 * leaf work of step m+1 (LU, U columns of the panel, their projection) overlaps the tree levels
 * of step m; only the rhs column waits for u^(m).  Same factorisation as fde1d_step; the rhs
 * column's leaf solve uses the stored LU (results agree with fde1d_step to rounding).
 *   d_plus, d_minus [dev]: step m at d_plus + m * coef_stride (batch*n each; coef_stride = 0:
 *   the same coefficients every step, so A_m = A for all m and the launch factors once -- leaf
 *   LUs, U-column panel, projections and the non-rhs tree work at step 0 only; every later step
 *   is the rhs column alone against that factor ("the LU can be computed only once at
 *   the beginning"); FDE_REFACTOR in flags refactors every step instead, with bitwise-equal
 *   results when the run uses split tree units); f [dev] likewise with f_stride; u0 [dev, batch*n];
 *   u_out [dev, K * batch*n] receives every step's solution (step m at u_out + m*batch*n);
 *   u_out must not alias u0 or the coefficient arrays.
 *   `cache`, alpha, h, tol, leaf, stream as in fde1d_step.  Asynchronous unless FDE_SYNC.
 * FDE_HOST_PTRS: d_plus, d_minus, f, u0 and u_out are HOST arrays (pinned for asynchronous copies;
 * strides 0 or batch*n): the library stages them on the device on `stream`, runs, copies every
 * step's solution back and synchronises (the copies are part of the call).  With per-step
 * coefficients and K >= 24 the run is three launches (head, body, tail of max(4, K/16) | rest |
 * max(4, K/16) steps) and the copies overlap them on two internal streams: only the head's H2D
 * and the tail's D2H are exposed; results are bitwise those of the one-launch run.
 * The handle owns a second panel/projection buffer set, two stored leaf LUs and per-step
 * counters sized for K: the first call (and any call with a larger K) allocates them, which
 * synchronises the stream.  Without the tree path (L = 0 or a panel too wide for it) the call
 * falls back to K fde1d_step calls on the device. */
int fde1d_run(int batch, int n, const double* alpha, double h, double dt, int K,
              const double* d_plus, const double* d_minus, long long coef_stride,
              const double* f, long long f_stride, const double* u0, double* u_out,
              double tol, int leaf, unsigned flags, fde_hodlr_t* cache, void* stream);

/* One step of the 2D scheme as a Sylvester equation (Eq. 4.3, reading R11):
 *     A1 X + X A2^T = Uu Uv^T + dt Fu Fv^T,
 *     A1 = 1/2 I + (dt/hx^alpha1)(D1+ T1 + D1- T1^T),  A2 likewise in y,
 * solved by the extended Krylov method on the HODLR factors of A1 and A2; the
 * right-hand side is compressed by Householder QR of both factors + an SVD and the
 * solution truncated at tol relative to its largest singular value.
 *   d1p, d1m [dev, nx]; d2p, d2m [dev, ny]; Fu [dev, nx*rf], Fv [dev, ny*rf];
 *   Uu [dev, nx*ru], Uv [dev, ny*ru] (ru may be 0); Xu [dev, nx*rmax], Xv [dev, ny*rmax].
 *   *rx receives the rank of X = Xu Xv^T; resid_out (host, may be NULL) the relative residual
 *   ||A1 X + X A2^T - C||_F / ||C||_F of the RETURNED (truncated) X against the input C, with
 *   A1, A2 the HODLR operators; iters_out (host, may be NULL) the EK iterations.  cache[2]
 *   holds the two operator handles: built and factorised on first use, rebuilt when (n, alpha,
 *   h, tol, leaf) change, refactorised when dt or the coefficient pointers change or flags has
 *   FDE_COEFFS_CHANGED.  Device-side failures of either operator are reported (and cleared).
 *   Synchronous: the EK iteration reads back the small quantities that steer it.
 *   Returns FDE_ENOCONV with the best iterate if ek_maxit is reached, FDE_EDIM if the
 *   truncated rank exceeds rmax. */
int fde2d_step(int nx, int ny, double alpha1, double alpha2, double hx, double hy, double dt,
               const double* d1p, const double* d1m, const double* d2p, const double* d2m,
               const double* Fu, const double* Fv, int rf,
               const double* Uu, const double* Uv, int ru,
               double* Xu, double* Xv, int rmax, int* rx,
               double tol, double ek_tol, int ek_maxit, int leaf,
               fde_hodlr_t* cache, double* resid_out, int* iters_out,
               unsigned flags, void* stream);

/* The x/y split of the 2D step over two processes (the two extended block
 * Arnoldi processes are independent): rank 0 owns A1, its Krylov basis and Xu; rank 1
 * owns A2, its basis and Xv.  The sides couple only through four small exchanges per projected
 * solve (the right-hand side's R factors, the projected matrices, the basis sizes, the residual
 * parts), which the library hands to `gather`:
 *   gather(ctx, send, recv, count, stream): all-gather `count` doubles of every rank's `send`
 *   (device) into `recv` (device, world * count, rank order) ordered on `stream`; returns 0 on
 *   success.  (The Python binding implements it with torch.distributed over NCCL.)
 * The small dense work is repeated on both ranks on identical data, so both take the same
 * decisions and return the same rank, residual and status.  world = 1 is fde2d_step (both sides
 * local, the exchanges local copies; gather may be NULL).  Arguments as fde2d_step; a rank reads
 * only its own side's arrays (d1p, d1m, Fu, Uu, Xu on rank 0; d2p, d2m, Fv, Uv, Xv on rank 1) and
 * builds only its own operator in cache. */
int fde2d_step_split(int world, int rank, fde_allgather_fn gather, void* ctx,
                     int nx, int ny, double alpha1, double alpha2, double hx, double hy, double dt,
                     const double* d1p, const double* d1m, const double* d2p, const double* d2m,
                     const double* Fu, const double* Fv, int rf,
                     const double* Uu, const double* Uv, int ru,
                     double* Xu, double* Xv, int rmax, int* rx,
                     double tol, double ek_tol, int ek_maxit, int leaf,
                     fde_hodlr_t* cache, double* resid_out, int* iters_out,
                     unsigned flags, void* stream);

/* The 2D step with a multi-shift rational Krylov projection: the same
 * Galerkin framework as fde2d_step with the bases grown by rounds of `npole`
 * independent shifted solves per side -- W_j = (A1 + p_j I)^{-1} Cu, (A2 + q_j I)^{-1} Cv, each
 * shifted operator its own HODLR factorisation (shift 1/2 + p_j), kept in cache -- until the
 * residual is below rk_tol or `rounds` rounds are used.  poles [host, 2 * npole * rounds]: side 0
 * (A1) then side 1, round-major, all > 0; NULL = automatic (log-spaced in the other operator's
 * spectral range [1/2, 1/2 + c 2^alpha (max|d+| + max|d-|)], round r offset).  The shifted solves of
 * a round are independent: with pw > 1, rank pr solves poles j = pr mod pw and the blocks are
 * all-gathered through `gather` (as fde2d_step_split); the rest runs on every rank.
 *   cache [2 + 2 * npole * rounds]: the two operators, then the shifted factorisations (required).
 *   *rounds_out (host, may be NULL): rounds used.  Other arguments, outputs and errors as fde2d_step
 *   (FDE_ENOCONV when rk_tol is not reached).  npole in 1..16, rounds in 1..6. */
int fde2d_step_rk(int pw, int pr, fde_allgather_fn gather, void* ctx,
                  int nx, int ny, double alpha1, double alpha2, double hx, double hy, double dt,
                  const double* d1p, const double* d1m, const double* d2p, const double* d2m,
                  const double* Fu, const double* Fv, int rf,
                  const double* Uu, const double* Uv, int ru,
                  double* Xu, double* Xv, int rmax, int* rx,
                  double tol, double rk_tol, int npole, int rounds, const double* poles, int leaf,
                  fde_hodlr_t* cache, double* resid_out, int* rounds_out, unsigned flags, void* stream);

/* The paper's 1D comparison method: GMRES (full, x0 = 0)
 * for A_m x = b, left-preconditioned by a tridiagonal structure-preserving preconditioner of [DMS]
 * -- A_m with T_{alpha,N} replaced by T_{1,N} (precond = 1, P1: Eq. 2.6 at alpha = 1) or by
 * tridiag(-1, 2, -1) = T_{2,N} (precond = 2, P2); precond = 0: no preconditioner -- with the exact
 * operator applied by FFT circulant embedding.  Stops when the preconditioned relative
 * residual ||P^{-1}(b - A x)|| / ||P^{-1} b|| <= tol (*relres, host) or after maxit (1..127)
 * iterations (*iters, host; FDE_ENOCONV with the best iterate).  d_plus, d_minus, b, x [dev, n];
 * n <= 2^19.  Synchronous (one read-back per iteration). */
int fde1d_pgmres(int n, double alpha, double h, double dt, const double* d_plus, const double* d_minus,
                 const double* b, double* x, int precond, double tol, int maxit, int* iters,
                 double* relres, unsigned flags, void* stream);

/* The same solver split into a plan (FFT spectra of T and T^T, the preconditioner's block factors,
 * the Krylov workspace: built once for time-invariant coefficients) and solves. */
typedef struct fde_pgmres* fde_pgmres_t;
int fde1d_pgmres_plan(int n, double alpha, double h, double dt, const double* d_plus, const double* d_minus,
                      int precond, int maxit, void* stream, fde_pgmres_t* out);
int fde1d_pgmres_solve(fde_pgmres_t plan, const double* b, double* x, double tol, int* iters, double* relres,
                       void* stream);
void fde1d_pgmres_destroy(fde_pgmres_t plan);

/* y = A_m x with the exact (uncompressed) operator of Eq. (2.5) (shift 1), T x and T^T x by FFT
 * circulant embedding; for residual checks.  [dev, n] arrays; y must not alias x. */
int fde1d_apply_exact(int n, double alpha, double h, double dt, const double* d_plus, const double* d_minus,
                      const double* x, double* y, void* stream);

/* Thread-local description of the last error returned on this thread ("" if none). */
const char* fde_last_error(void);

/* Number of kernels this library has launched in this process (for launch accounting). */
long long fde_launch_count(void);

/* Tracing: when enabled, every kernel launch is bracketed by a pair of CUDA events on its
 * stream.  fde_profile_dump() synchronises those events, writes a JSON object
 * {"kernel": [launches, total_ms], ...} into buf (NUL terminated), clears the records and
 * returns the string length (or -(needed+1) if len is too small).  Disabling drops them. */
void fde_profile_enable(int on);
int fde_profile_dump(char* buf, int len);

#ifdef __cplusplus
}
#endif
#endif /* FDEHODLR_H */
