// fde2d.cuh -- S8-S10: one implicit-Euler step of the 2D FDE as a Sylvester equation
// (Eq. 4.3, reading R11/R12):
//     A1 X + X A2^T = C,   C = Uu Uv^T + dt Fu Fv^T,
//     A_i = 1/2 I + (dt/h_i^alpha_i)(D_i+ T_i + D_i- T_i^T),
// solved by the extended Krylov subspace method: orthonormal bases U of
// EK(A1, C_u) and V of EK(A2, C_v) grown by one HODLR solve (A^{-1} N) and one HODLR matvec
// (A P) per iteration and side, the projected equation  A~ Y + Y B~ = C~  (A~ = U^T A1 U,
// B~ = (V^T A2 V)^T, C~ = U^T C V) solved with dense linear algebra (here the
// Newton iteration for the matrix sign function, which only needs inverses and products,
// safe because Sym(A_i) > 0 puts the spectra of A~, B~ in the open right half plane), the
// true residual from the exact splitting  R = Ra Y V^T + U Y Rb^T  (Ra = A1 U - U A~ is
// orthogonal to U):  ||R||_F^2 = ||Ra Y||_F^2 + ||Rb Y^T||_F^2,  and the solution truncated
// to X = Xu Xv^T by an SVD of Y.  The right-hand side is compressed first (QR of
// both factors + small SVD).  All arithmetic runs in the kernels of
// k_dense.cuh and the HODLR kernels; the host only sequences them and reads back the small
// quantities that steer the iteration (ranks kept, residual, iteration count).
#pragma once
#include <algorithm>
#include <initializer_list>
#include "k_dense.cuh"

#define EK_SMAX 320                    // cap on the projected size per side

struct Fde2dCtx {
  cudaStream_t s;
  DevStatus* st;
  double* scratch;                     // device scratch (small matrices)
  double* hbuf;                        // pinned-free host staging (std::vector managed)
};

static int dn_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(FDE_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return FDE_OK;
}

// C (m x n) = alpha A^T B + beta C  (A: K x m, B: K x n; K tall)
static double* g_dn_part = nullptr;     // split-K partials (device, grown on demand)
static size_t g_dn_part_cap = 0;

static int ts_tn(cudaStream_t s, int m, int n, int K, double alpha, const double* A, int lda,
                 const double* B, int ldb, double beta, double* C, int ldc) {
  if (m <= 0 || n <= 0) return FDE_OK;
  const int nz = std::min(32, std::max(1, K / 128));
  if (nz > 1) {
    const size_t need = (size_t)nz * m * n;
    if (need > g_dn_part_cap) {
      if (g_dn_part) { cudaStreamSynchronize(s); cudaFree(g_dn_part); }
      CU(cudaMalloc(&g_dn_part, need * sizeof(double)));
      g_dn_part_cap = need;
    }
    const int kchunk = round_up((K + nz - 1) / nz, 64);
    const int nzz = (K + kchunk - 1) / kchunk;
    { PROF("k_ts_gemm_tn"); k_ts_gemm_tn_split<<<dim3((m + TS_TILE - 1) / TS_TILE, (n + TS_TILE - 1) / TS_TILE, nzz), DN_THREADS, 0, s>>>(
        m, n, K, kchunk, A, lda, B, ldb, g_dn_part); }
    TRY(dn_check("k_ts_gemm_tn_split"));
    { PROF("k_reduce_partials"); k_reduce_partials<<<(m * n + 255) / 256, 256, 0, s>>>(m, n, nzz, g_dn_part, alpha, beta, C, ldc); }
    return dn_check("k_reduce_partials");
  }
  { PROF("k_ts_gemm_tn"); k_ts_gemm_tn<<<dim3((m + TS_TILE - 1) / TS_TILE, (n + TS_TILE - 1) / TS_TILE), DN_THREADS, 0, s>>>(
      m, n, K, alpha, A, lda, B, ldb, beta, C, ldc); }
  return dn_check("k_ts_gemm_tn");
}

// C (M x n) = alpha A B + beta C  (A: M x K tall, B: K x n small)
static int ts_nn(cudaStream_t s, int M, int n, int K, double alpha, const double* A, int lda,
                 const double* B, int ldb, double beta, double* C, int ldc) {
  if (M <= 0 || n <= 0) return FDE_OK;
  { PROF("k_ts_gemm_nn"); k_ts_gemm_nn<<<dim3((M + DN_THREADS - 1) / DN_THREADS, n), DN_THREADS, 0, s>>>(
      M, n, K, alpha, A, lda, B, ldb, beta, C, ldc); }
  return dn_check("k_ts_gemm_nn");
}

static int transpose(cudaStream_t s, int m, int n, const double* X, int ldx, double* Y, int ldy) {
  if (m <= 0 || n <= 0) return FDE_OK;
  { PROF("k_transpose"); k_transpose<<<dim3((m + 31) / 32, (n + 31) / 32), dim3(32, 8), 0, s>>>(m, n, X, ldx, Y, ldy); }
  return dn_check("k_transpose");
}

static bool g_dn_attr = false;
static int dn_attrs() {
  if (g_dn_attr) return FDE_OK;
  CU(cudaFuncSetAttribute(k_sym_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, DN_SMEM_MAX + 4096));
  CU(cudaFuncSetAttribute(k_osj_svd, cudaFuncAttributeMaxDynamicSharedMemorySize, DN_SMEM_MAX + 4096));
  CU(cudaFuncSetAttribute(k_gj_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, DN_SMEM_MAX + 4096));
  // the per-step workspace comes from the device's default stream-ordered pool: keep freed
  // blocks mapped across synchronisations (release threshold 0 would unmap and re-map ~50 MB
  // every fde2d_step)
  int dev = 0;
  cudaMemPool_t pool;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetDefaultMemPool(&pool, dev));
  unsigned long long keep_bytes = 1ULL << 30;
  CU(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep_bytes));
  g_dn_attr = true;
  return FDE_OK;
}
static size_t dn_smem(long long resident_doubles, int ints) {
  const long long b = resident_doubles * 8 + ints * 4;
  return (size_t)(b <= DN_SMEM_MAX ? b + 16 : ints * 4 + 16);
}

static int scale_copy(cudaStream_t s, int m, int n, double alpha, const double* X, int ldx, double* Y, int ldy) {
  const long long tot = (long long)m * n;
  if (tot <= 0) return FDE_OK;
  { PROF("k_scale_copy"); k_scale_copy<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(m, n, alpha, X, ldx, Y, ldy); }
  return dn_check("k_scale_copy");
}

static int sumsq(cudaStream_t s, int m, int n, const double* X, int ldx, double* dout, double* hout) {
  { PROF("k_sumsq"); k_sumsq<<<1, DN_BIG, 0, s>>>(m, n, X, ldx, dout); }
  TRY(dn_check("k_sumsq"));
  CU(cudaMemcpyAsync(hout, dout, sizeof(double), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return FDE_OK;
}

// Build S (b x nk) = V[:, idx] diag(lam[idx])^{-1/2}  (SVQB scaling)
__global__ void k_svqb_scale(int b, const double* __restrict__ V, const double* __restrict__ lam,
                             const int* __restrict__ idx, int nk, double* __restrict__ S) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= b * nk) return;
  const int i = e % b, j = e / b, c = idx[j];
  S[(long long)j * b + i] = V[(long long)c * b + i] / sqrt(lam[c]);
}

// gather columns: Y[:, j] = alpha_j X[:, idx[j]]  (alpha_j = sc ? 1/sc[idx[j]] : 1)
__global__ void k_gather_cols(int m, int nk, const double* __restrict__ X, int ldx, const int* __restrict__ idx,
                              const double* __restrict__ sc, double* __restrict__ Y, int ldy) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)m * nk) return;
  const int i = (int)(e % m), j = (int)(e / m), c = idx[j];
  Y[(long long)j * ldy + i] = X[(long long)c * ldx + i] * (sc ? 1.0 / sc[c] : 1.0);
}

// Rank-revealing Householder QR with column pivoting (one CTA), truncation step of S10: W (m x n,
// ld m, overwritten) <- H_k .. H_1 W, stopping at the first step k whose largest remaining column
// norm is <= rtol * the largest initial column norm (the dropped block then has Frobenius norm
// <= sqrt(n) rtol |W|_max-col).  Pivoting is by index (no column swaps), so rows 0..k-1 are
// Q_k^T W in the original column order; they are written transposed to AT (n x k, ld n) and k
// to *kout.  Residual column norms are recomputed every step (no downdating).
__global__ void __launch_bounds__(DN_BIG)
k_qrcp_rows(int m, int n, double* __restrict__ W, double rtol, double* __restrict__ AT, int* __restrict__ kout) {
  __shared__ double v[EK_SMAX], nrm[EK_SMAX];
  __shared__ double s_tau, s_n0;
  __shared__ int s_jp, s_stop;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31, nw = DN_BIG / 32;
  const int kmax = min(m, n);
  int k = 0;
  for (int step = 0; step < kmax; ++step) {
    for (int j = warp; j < n; j += nw) {               // residual column norms, rows step..m-1
      double a = 0.0;
      for (int i = step + lane; i < m; i += 32) { const double x = W[(long long)j * m + i]; a = fma(x, x, a); }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (lane == 0) nrm[j] = a;
    }
    __syncthreads();
    if (warp == 0) {                                   // argmax (smallest index on ties)
      double best = -1.0; int bj = 0;
      for (int j = lane; j < n; j += 32) if (nrm[j] > best) { best = nrm[j]; bj = j; }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
        if (ob > best || (ob == best && oj < bj)) { best = ob; bj = oj; }
      }
      if (lane == 0) {
        if (step == 0) s_n0 = best;
        s_jp = bj;
        s_stop = !(best > 0.0) || best <= rtol * rtol * s_n0;
        if (!s_stop) {
          const double x0 = W[(long long)bj * m + step], nx = sqrt(best);
          const double al = x0 >= 0.0 ? -nx : nx;
          v[0] = x0 - al;
          s_tau = 1.0 / (nx * (nx + fabs(x0)));           // 2 / (v^T v)
        }
      }
    }
    __syncthreads();
    if (s_stop) break;
    const int jp = s_jp;
    for (int i = step + 1 + t; i < m; i += DN_BIG) v[i - step] = W[(long long)jp * m + i];
    __syncthreads();
    const double tau = s_tau;
    for (int j = warp; j < n; j += nw) {               // W[step:, j] -= tau v (v^T W[step:, j])
      double* wc = W + (long long)j * m + step;
      double a = 0.0;
      for (int i = lane; i < m - step; i += 32) a = fma(v[i], wc[i], a);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      a *= tau;
      for (int i = lane; i < m - step; i += 32) wc[i] = fma(-a, v[i], wc[i]);
    }
    __syncthreads();
    k = step + 1;
  }
  for (long long e = t; e < (long long)n * k; e += DN_BIG) {
    const int j = (int)(e % n), i = (int)(e / n);
    AT[(long long)i * n + j] = W[(long long)j * m + i];
  }
  if (t == 0) *kout = k;
}

// Newton sign iteration update (one CTA):  with mu = scaling,
//   A <- (mu A + Ainv/mu)/2,  B <- (mu B + Binv/mu)/2,  C <- (mu C + (Ainv C Binv)/mu)/2 where
//   T = Ainv C Binv is given; out[0] = ||A_new - A_old||_1-ish change measure.
__global__ void __launch_bounds__(DN_BIG)
k_sign_update(int sa, int sb, double* __restrict__ A, const double* __restrict__ Ai, double* __restrict__ B,
              const double* __restrict__ Bi, double* __restrict__ C, const double* __restrict__ T,
              double* __restrict__ out) {
  __shared__ double red[4][DN_BIG];
  const int t = threadIdx.x;
  // norms for the scaling mu = sqrt(||Z^-1||_F / ||Z||_F) of Z = [[A, -C], [0, -B]]
  double na = 0, nai = 0, nb = 0, nbi = 0;
  for (int e = t; e < sa * sa; e += DN_BIG) { na = fma(A[e], A[e], na); nai = fma(Ai[e], Ai[e], nai); }
  for (int e = t; e < sb * sb; e += DN_BIG) { nb = fma(B[e], B[e], nb); nbi = fma(Bi[e], Bi[e], nbi); }
  red[0][t] = na + nb; red[1][t] = nai + nbi;
  __syncthreads();
  for (int w = DN_BIG / 2; w > 0; w >>= 1) {
    if (t < w) { red[0][t] += red[0][t + w]; red[1][t] += red[1][t + w]; }
    __syncthreads();
  }
  const double mu = sqrt(sqrt(red[1][0] / red[0][0]));
  __syncthreads();
  double dch = 0, dnm = 0;
  for (int e = t; e < sa * sa; e += DN_BIG) {
    const double o = A[e], nw = 0.5 * (mu * o + Ai[e] / mu);
    A[e] = nw; dch += fabs(nw - o); dnm += fabs(nw);
  }
  for (int e = t; e < sb * sb; e += DN_BIG) {
    const double o = B[e], nw = 0.5 * (mu * o + Bi[e] / mu);
    B[e] = nw; dch += fabs(nw - o); dnm += fabs(nw);
  }
  for (int e = t; e < sa * sb; e += DN_BIG) C[e] = 0.5 * (mu * C[e] + T[e] / mu);
  red[2][t] = dch; red[3][t] = dnm;
  __syncthreads();
  for (int w = DN_BIG / 2; w > 0; w >>= 1) {
    if (t < w) { red[2][t] += red[2][t + w]; red[3][t] += red[3][t + w]; }
    __syncthreads();
  }
  if (t == 0) { out[0] = red[2][0] / red[3][0]; out[1] = mu; }
}

struct DenseWs {                        // device scratch for the small dense operations
  double *G, *V, *lam, *S, *M1, *M2, *M3, *M4, *M5, *M6, *dv;
  int* idx;
  InvJob* jobs;
};

// Orthonormalise the n x b block W (ld n, destroyed) against the orthonormal basis
// Ub[:, 0:s] (ld n) -- block Gram-Schmidt twice -- then by SVQB twice (Gram eigen-
// decomposition; directions with singular value below dtol * ref are deflated).  The new
// orthonormal columns are written to Ub[:, s:s+nb]; returns nb in *nb.  Optionally
// (coef != null) coef (nb x b, ld ldcoef) = Q^T W_original for the RHS compression (s == 0).
static int orth_append(cudaStream_t s, const DenseWs& w, int n, double* W, int b, double* Ub, int sb,
                       int smax, double dtol, int* nb, double* coef, int ldcoef, double* W0) {
  *nb = 0;
  if (b <= 0) return FDE_OK;
  std::vector<double> h((size_t)b * 2 + 8);
  // reference scale: largest column norm of W before the projection
  TRY(ts_tn(s, b, b, n, 1.0, W, n, W, n, 0.0, w.G, b));
  CU(cudaMemcpy2DAsync(h.data(), sizeof(double), w.G, (b + 1) * sizeof(double), sizeof(double), b,
                       cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  double ref = 0.0;
  for (int i = 0; i < b; ++i) ref = std::max(ref, h[i]);
  ref = std::sqrt(ref);
  if (!(ref > 0.0)) return FDE_OK;
  if (W0) CU(cudaMemcpyAsync(W0, W, (size_t)n * b * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if (coef && W0 && sb == 0) {
    // right-hand-side compression: unit columns before the Gram-based steps.  The Gram matrix
    // resolves directions only down to ~1e-8 of its largest column, and [U_u, dt F_u] mixes a
    // low-rank factor whose columns carry the singular values (1e2 .. 1e-10) with dt F_u; after
    // the scaling its conditioning reflects angles only (coef is taken from the unscaled W0).
    std::vector<double> sc(b);
    for (int i = 0; i < b; ++i) sc[i] = h[i] > 0.0 ? 1.0 / std::sqrt(h[i]) : 0.0;
    CU(cudaMemcpyAsync(w.lam, sc.data(), b * sizeof(double), cudaMemcpyHostToDevice, s));
    { PROF("k_scale_cols"); k_scale_cols<<<(unsigned)(((long long)n * b + 255) / 256), 256, 0, s>>>(n, b, W, n, w.lam); }
    TRY(dn_check("k_scale_cols"));
    CU(cudaStreamSynchronize(s));                      // (sc is a host temporary)
    ref = 1.0;
  }
  // (project, normalise) twice: "twice is enough" block Gram-Schmidt with SVQB normalisation;
  // pass 0 deflates directions below dtol * ref, pass 1 drops any that lost half their norm
  int cur = b;
  double* src = W;
  for (int pass = 0; pass < 2; ++pass) {
    if (sb > 0) {
      TRY(ts_tn(s, sb, cur, n, 1.0, Ub, n, src, n, 0.0, w.M1, sb));      // H = U^T W
      TRY(ts_nn(s, n, cur, sb, -1.0, Ub, n, w.M1, sb, 1.0, src, n));      // W -= U H
    }
    TRY(ts_tn(s, cur, cur, n, 1.0, src, n, src, n, 0.0, w.G, cur));
    { PROF("k_sym_jacobi"); k_sym_jacobi<<<1, DN_BIG, dn_smem(2LL * cur * cur, cur + 2), s>>>(cur, w.G, cur, w.V, w.lam, 60); }
    TRY(dn_check("k_sym_jacobi"));
    CU(cudaMemcpyAsync(h.data(), w.lam, cur * sizeof(double), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    std::vector<int> order(cur);
    for (int i = 0; i < cur; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int a, int c) { return h[a] > h[c] || (h[a] == h[c] && a < c); });
    std::vector<int> keep;
    const double thr = pass == 0 ? (dtol * ref) * (dtol * ref) : 0.25;
    for (int i : order)
      if (h[i] > thr && (int)keep.size() < smax - sb) keep.push_back(i);
    if (keep.empty()) return FDE_OK;
    const int nk = (int)keep.size();
    CU(cudaMemcpyAsync(w.idx, keep.data(), nk * sizeof(int), cudaMemcpyHostToDevice, s));
    { PROF("k_svqb_scale"); k_svqb_scale<<<(cur * nk + 255) / 256, 256, 0, s>>>(cur, w.V, w.lam, w.idx, nk, w.S); }
    TRY(dn_check("k_svqb_scale"));
    double* dst = pass == 0 ? w.M2 : Ub + (size_t)sb * n;                 // M2 holds n x b (sized)
    TRY(ts_nn(s, n, nk, cur, 1.0, src, n, w.S, cur, 0.0, dst, n));
    CU(cudaStreamSynchronize(s));                                        // idx reused next pass
    src = dst;
    cur = nk;
  }
  *nb = cur;
  if (coef && W0) TRY(ts_tn(s, cur, b, n, 1.0, Ub + (size_t)sb * n, n, W0, n, 0.0, coef, ldcoef));
  return FDE_OK;
}

// Solve A~ Y + Y B~ = C~ (sa x sa, sb x sb, sa x sb, all ld = own rows) by the scaled Newton
// sign iteration; Y is returned in C (overwritten).  A, B are destroyed.
static int proj_sylvester(cudaStream_t s, const DenseWs& w, int sa, int sb, double* A, double* B, double* C,
                          DevStatus* st, int* iters) {
  double* Ai = w.M3;
  double* Bi = w.M4;
  double* T = w.M5;
  double* T2 = w.M6;
  InvJob hj[2] = {{Ai, sa, sa}, {Bi, sb, sb}};
  CU(cudaMemcpyAsync(w.jobs, hj, sizeof(hj), cudaMemcpyHostToDevice, s));
  double hout[2] = {1, 1};
  int it = 0;
  for (; it < 60; ++it) {
    CU(cudaMemcpyAsync(Ai, A, (size_t)sa * sa * sizeof(double), cudaMemcpyDeviceToDevice, s));
    CU(cudaMemcpyAsync(Bi, B, (size_t)sb * sb * sizeof(double), cudaMemcpyDeviceToDevice, s));
    { PROF("k_gj_inverse"); k_gj_inverse<<<2, DN_BIG, std::max(dn_smem((long long)sa * sa, sa), dn_smem((long long)sb * sb, sb)), s>>>(w.jobs, st); }
    TRY(dn_check("k_gj_inverse"));
    // T2 = Ai C Bi
    TRY(ts_nn(s, sa, sb, sa, 1.0, Ai, sa, C, sa, 0.0, T, sa));
    TRY(ts_nn(s, sa, sb, sb, 1.0, T, sa, Bi, sb, 0.0, T2, sa));
    { PROF("k_sign_update"); k_sign_update<<<1, DN_BIG, 0, s>>>(sa, sb, A, Ai, B, Bi, C, T2, w.dv); }
    TRY(dn_check("k_sign_update"));
    CU(cudaMemcpyAsync(hout, w.dv, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (fde_dbg_env("FDE_DEBUG2D") && fde_dbg_env("FDE_DEBUG2D")[0] == '2')
      fprintf(stderr, "  sign it %d change %.3e mu %.3e\n", it, hout[0], hout[1]);
    if (hout[0] < 1e-14) { ++it; break; }
  }
  // sign(Z) = [[I, 2Y'], [0, -I]] for Z = [[A, -C], [0, -B]]: the C block carries -(2Y)...
  // with the update above C_k -> C_inf = 2Y  (verified against the oracle in the tests)
  TRY(scale_copy(s, sa, sb, 0.5, C, sa, C, sa));
  *iters = it;
  return FDE_OK;
}

// y = A x for nrhs columns (chunks of NRHS_MAX)
static int hodlr_mv_cols(fde_hodlr* H, const double* X, double* Y, int ncol, cudaStream_t s) {
  for (int c = 0; c < ncol; c += NRHS_MAX) {
    const int nc = std::min(NRHS_MAX, ncol - c);
    TRY(matvec_impl(H, X + (size_t)c * H->n, Y + (size_t)c * H->n, nc, H->n, s));
  }
  return FDE_OK;
}
static int hodlr_solve_cols(fde_hodlr* H, const double* B, double* X, int ncol, cudaStream_t s) {
  for (int c = 0; c < ncol; c += NRHS_MAX) {
    const int nc = std::min(NRHS_MAX, ncol - c);
    TRY(solve_impl(H, B + (size_t)c * H->n, nullptr, X + (size_t)c * H->n, nc, H->n, s));
  }
  return FDE_OK;
}

struct EkSide {
  fde_hodlr* H;
  int n;
  double *U, *AU;                      // basis (n x EK_SMAX) and A * basis
  int s;                               // basis size
  int p0, np, n0, nn;                  // last blocks: positive (A^j) and negative (A^-j) parts
};

// Grow one side by one extended-Krylov step: P' = orth(A P), N' = orth(A^{-1} N).
static int ek_grow(cudaStream_t s, const DenseWs& w, EkSide& e, double* Wtmp, double dtol) {
  const int n = e.n;
  int nbp = 0, nbn = 0;
  const int oldp = e.p0, oldnp = e.np, oldn = e.n0, oldnn = e.nn;
  // A P_j is already in AU
  if (oldnp > 0) {
    CU(cudaMemcpyAsync(Wtmp, e.AU + (size_t)oldp * n, (size_t)n * oldnp * sizeof(double), cudaMemcpyDeviceToDevice, s));
    TRY(orth_append(s, w, n, Wtmp, oldnp, e.U, e.s, EK_SMAX, dtol, &nbp, nullptr, 0, nullptr));
    if (nbp) TRY(hodlr_mv_cols(e.H, e.U + (size_t)e.s * n, e.AU + (size_t)e.s * n, nbp, s));
    e.p0 = e.s; e.np = nbp; e.s += nbp;
  } else { e.np = 0; }
  if (oldnn > 0) {
    TRY(hodlr_solve_cols(e.H, e.U + (size_t)oldn * n, Wtmp, oldnn, s));
    TRY(orth_append(s, w, n, Wtmp, oldnn, e.U, e.s, EK_SMAX, dtol, &nbn, nullptr, 0, nullptr));
    if (nbn) TRY(hodlr_mv_cols(e.H, e.U + (size_t)e.s * n, e.AU + (size_t)e.s * n, nbn, s));
    e.n0 = e.s; e.nn = nbn; e.s += nbn;
  } else { e.nn = 0; }
  return FDE_OK;
}

static int build_op_2d(int n, double alpha, double h, double dt, const double* dp, const double* dm, double tol,
                       int leaf, cudaStream_t s, fde_hodlr** out) {
  TRY(build_impl(1, n, &alpha, h, dt, dp, dm, 0.5, tol, leaf, 0, s, out));
  fde_hodlr* H = *out;
  const int rc = factor_impl(H, H->d_dp, H->d_dm, 0, nullptr, nullptr, nullptr, 1, s);
  if (rc != FDE_OK) { free_handle(H); *out = nullptr; return rc; }
  H->factored = true;
  H->last_stream = s;
  return FDE_OK;
}

static bool op_matches(const fde_hodlr* H, int n, double alpha, double h, double dt, double tol, int leaf) {
  return H && H->batch == 1 && H->n == n && H->alpha[0] == alpha && H->h == h && H->dt == dt &&
         H->tol == tol && H->leaf == leaf && H->shift == 0.5 && H->factored;
}

extern "C" int fde2d_step(int nx, int ny, double alpha1, double alpha2, double hx, double hy, double dt,
                          const double* d1p, const double* d1m, const double* d2p, const double* d2m,
                          const double* Fu, const double* Fv, int rf, const double* Uu, const double* Uv,
                          int ru, double* Xu, double* Xv, int rmax, int* rx, double tol, double ek_tol,
                          int ek_maxit, int leaf, fde_hodlr_t* cache, double* resid_out, int* iters_out,
                          unsigned flags, void* stream) {
  g_last_error.clear();
  TRY(check_common(1, nx, &alpha1, hx, dt, tol, leaf));
  TRY(check_common(1, ny, &alpha2, hy, dt, tol, leaf));
  if (!d1p || !d1m || !d2p || !d2m) return set_err(FDE_EDOMAIN, "NULL coefficient array");
  if (rf < 0 || ru < 0 || (rf > 0 && (!Fu || !Fv)) || (ru > 0 && (!Uu || !Uv)))
    return set_err(FDE_EDOMAIN, "bad right-hand-side factors (rf=%d, ru=%d)", rf, ru);
  if (!Xu || !Xv || !rx || rmax < 1) return set_err(FDE_EDOMAIN, "bad output factors (rmax=%d)", rmax);
  if (!(ek_tol > 0.0 && ek_tol < 1.0) || ek_maxit < 1) return set_err(FDE_EDOMAIN, "ek_tol / ek_maxit out of range");
  if (rf + ru > NRHS_MAX) return set_err(FDE_EDIM, "rf + ru = %d exceeds %d", rf + ru, NRHS_MAX);
  cudaStream_t s = (cudaStream_t)stream;
  TRY(dn_attrs());
  // operators (built and factorised once, reused while the arguments match)
  fde_hodlr* tmp[2] = {nullptr, nullptr};
  fde_hodlr** ops = cache ? reinterpret_cast<fde_hodlr**>(cache) : tmp;
  if (!op_matches(ops[0], nx, alpha1, hx, dt, tol, leaf)) {
    if (ops[0]) hodlr_destroy(ops[0]);
    ops[0] = nullptr;
    TRY(build_op_2d(nx, alpha1, hx, dt, d1p, d1m, tol, leaf, s, &ops[0]));
  }
  if (!op_matches(ops[1], ny, alpha2, hy, dt, tol, leaf)) {
    if (ops[1]) hodlr_destroy(ops[1]);
    ops[1] = nullptr;
    const int rc = build_op_2d(ny, alpha2, hy, dt, d2p, d2m, tol, leaf, s, &ops[1]);
    if (rc != FDE_OK) { if (!cache) hodlr_destroy(ops[0]); return rc; }
  }
  auto cleanup = [&]() { if (!cache) { hodlr_destroy(ops[0]); hodlr_destroy(ops[1]); } };
  int rc = FDE_OK;
  // workspace
  const int nmax = std::max(nx, ny), r0 = ru + rf;
  const size_t big = (size_t)nmax * EK_SMAX;
  const size_t sm2 = (size_t)EK_SMAX * EK_SMAX;
  std::vector<void*> mem;
  auto dm_alloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (cudaMallocAsync(&p, std::max<size_t>(bytes, 16), s) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    mem.push_back(p);
    return p;
  };
  auto release = [&]() { for (void* p : mem) cudaFreeAsync(p, s); mem.clear(); };
  double* Ux = (double*)dm_alloc(big * 8);
  double* AUx = (double*)dm_alloc(big * 8);
  double* Vy = (double*)dm_alloc(big * 8);
  double* AVy = (double*)dm_alloc(big * 8);
  double* Wt = (double*)dm_alloc(big * 8);
  double* W0 = (double*)dm_alloc(big * 8);
  DenseWs w{};
  w.G = (double*)dm_alloc(sm2 * 8); w.V = (double*)dm_alloc(sm2 * 8); w.lam = (double*)dm_alloc(EK_SMAX * 8);
  w.S = (double*)dm_alloc(sm2 * 8); w.M1 = (double*)dm_alloc(sm2 * 8); w.M2 = (double*)dm_alloc(big * 8);
  w.M3 = (double*)dm_alloc(sm2 * 8); w.M4 = (double*)dm_alloc(sm2 * 8); w.M5 = (double*)dm_alloc(sm2 * 8);
  w.M6 = (double*)dm_alloc(sm2 * 8); w.dv = (double*)dm_alloc(64 * 8);
  w.idx = (int*)dm_alloc(EK_SMAX * 4); w.jobs = (InvJob*)dm_alloc(2 * sizeof(InvJob));
  double* Am = (double*)dm_alloc(sm2 * 8);
  double* Bm = (double*)dm_alloc(sm2 * 8);
  double* Cm = (double*)dm_alloc(sm2 * 8);
  double* Ym = (double*)dm_alloc(sm2 * 8);
  double* Zm = (double*)dm_alloc(sm2 * 8);
  double* sig = (double*)dm_alloc(EK_SMAX * 8);
  double* Lc = (double*)dm_alloc(sm2 * 8);   // coefficient matrices of the RHS compression
  double* Rc = (double*)dm_alloc(sm2 * 8);
  for (void* p : mem) if (!p) { release(); cleanup(); return set_err(FDE_ENOMEM, "fde2d workspace allocation failed"); }
  DevStatus* st = ops[0]->d_status;
  auto fail = [&](int code) { release(); cudaStreamSynchronize(s); cleanup(); return code; };
  std::vector<double> hs(EK_SMAX + 8);
  double hsum = 0.0;
  *rx = 0;
  if (resid_out) *resid_out = 0.0;
  if (iters_out) *iters_out = 0;
  // ---- S8: right-hand side C = [Uu, dt Fu] [Uv, Fv]^T, compressed
  int bl = 0, br = 0;
  if (r0 > 0) {
    if (ru) CU(cudaMemcpyAsync(Wt, Uu, (size_t)nx * ru * 8, cudaMemcpyDeviceToDevice, s));
    if (rf && (rc = scale_copy(s, nx, rf, dt, Fu, nx, Wt + (size_t)ru * nx, nx)) != FDE_OK) return fail(rc);
    if ((rc = orth_append(s, w, nx, Wt, r0, Ux, 0, EK_SMAX, 1e-15, &bl, Lc, EK_SMAX, W0)) != FDE_OK) return fail(rc);
    if (ru) CU(cudaMemcpyAsync(Wt, Uv, (size_t)ny * ru * 8, cudaMemcpyDeviceToDevice, s));
    if (rf) CU(cudaMemcpyAsync(Wt + (size_t)ru * ny, Fv, (size_t)ny * rf * 8, cudaMemcpyDeviceToDevice, s));
    if ((rc = orth_append(s, w, ny, Wt, r0, Vy, 0, EK_SMAX, 1e-15, &br, Rc, EK_SMAX, W0)) != FDE_OK) return fail(rc);
  }
  if (bl == 0 || br == 0) {                        // C = 0  =>  X = 0
    release();
    CU(cudaStreamSynchronize(s));
    cleanup();
    return FDE_OK;
  }
  // M = Lc Rc^T (bl x br) ; one-sided Jacobi SVD: M Z = W Sigma
  // Lc is (bl x r0) with ld EK_SMAX (column q at Lc + q*EK_SMAX); Lc^T as "A^T" operand:
  // M = Lc Rc^T = (Lc^T)^T (Rc^T): need A = Lc^T (r0 x bl) stored column-major ld r0.
  {
    double* LcT = w.M3;
    double* RcT = w.M4;
    // transpose via k_scale_copy row/col swap: write element (q, i) of LcT = Lc(i, q)
    if ((rc = transpose(s, bl, r0, Lc, EK_SMAX, LcT, r0)) != FDE_OK) return fail(rc);
    if ((rc = transpose(s, br, r0, Rc, EK_SMAX, RcT, r0)) != FDE_OK) return fail(rc);
    if ((rc = ts_tn(s, bl, br, r0, 1.0, LcT, r0, RcT, r0, 0.0, Ym, bl)) != FDE_OK) return fail(rc);
  }
  { PROF("k_osj_svd"); k_osj_svd<<<1, DN_BIG, dn_smem((long long)bl * br, br + 2), s>>>(bl, br, Ym, bl, Zm, sig, 60); }
  if ((rc = dn_check("k_osj_svd")) != FDE_OK) return fail(rc);
  CU(cudaMemcpyAsync(hs.data(), sig, br * sizeof(double), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  std::vector<int> ord(br);
  for (int i = 0; i < br; ++i) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](int a, int c) { return hs[a] > hs[c] || (hs[a] == hs[c] && a < c); });
  std::vector<int> keep;
  for (int i : ord) if (hs[i] > tol * hs[ord[0]] && hs[i] > 0.0) keep.push_back(i);
  const int rcr = (int)keep.size();
  std::vector<double> sigc(rcr);
  for (int i = 0; i < rcr; ++i) sigc[i] = hs[keep[i]];
  // Cu = Ql (M Z)[:, keep] / sigma ; Cv = Qr Z[:, keep]   (C = Cu diag(sigc) Cv^T)
  double* Cu = W0;                                  // nx x rcr
  double* Cv = W0 + (size_t)nmax * 64;              // ny x rcr
  CU(cudaMemcpyAsync(w.idx, keep.data(), rcr * sizeof(int), cudaMemcpyHostToDevice, s));
  { PROF("k_gather_cols"); k_gather_cols<<<(bl * rcr + 255) / 256, 256, 0, s>>>(bl, rcr, Ym, bl, w.idx, sig, w.M5, bl); }
  { PROF("k_gather_cols"); k_gather_cols<<<(br * rcr + 255) / 256, 256, 0, s>>>(br, rcr, Zm, br, w.idx, nullptr, w.M6, br); }
  if ((rc = dn_check("k_gather_cols")) != FDE_OK) return fail(rc);
  if ((rc = ts_nn(s, nx, rcr, bl, 1.0, Ux, nx, w.M5, bl, 0.0, Cu, nx)) != FDE_OK) return fail(rc);
  if ((rc = ts_nn(s, ny, rcr, br, 1.0, Vy, ny, w.M6, br, 0.0, Cv, ny)) != FDE_OK) return fail(rc);
  double cnorm2 = 0.0;
  for (double v : sigc) cnorm2 += v * v;
  // ---- S9: extended Krylov bases, first block orth([C, A^{-1} C])
  EkSide sx{ops[0], nx, Ux, AUx, 0, 0, 0, 0, 0}, sy{ops[1], ny, Vy, AVy, 0, 0, 0, 0, 0};
  const double dtol = 1e-11;
  for (EkSide* e : {&sx, &sy}) {
    const double* Cs = (e == &sx) ? Cu : Cv;
    int nb = 0;
    CU(cudaMemcpyAsync(Wt, Cs, (size_t)e->n * rcr * 8, cudaMemcpyDeviceToDevice, s));
    if ((rc = orth_append(s, w, e->n, Wt, rcr, e->U, 0, EK_SMAX, dtol, &nb, nullptr, 0, nullptr)) != FDE_OK) return fail(rc);
    if ((rc = hodlr_mv_cols(e->H, e->U, e->AU, nb, s)) != FDE_OK) return fail(rc);
    e->p0 = 0; e->np = nb; e->s = nb;
    if ((rc = hodlr_solve_cols(e->H, Cs, Wt, rcr, s)) != FDE_OK) return fail(rc);
    int nn = 0;
    if ((rc = orth_append(s, w, e->n, Wt, rcr, e->U, e->s, EK_SMAX, dtol, &nn, nullptr, 0, nullptr)) != FDE_OK) return fail(rc);
    if (nn && (rc = hodlr_mv_cols(e->H, e->U + (size_t)e->s * e->n, e->AU + (size_t)e->s * e->n, nn, s)) != FDE_OK) return fail(rc);
    e->n0 = e->s; e->nn = nn; e->s += nn;
  }
  // ---- S10: projected solves until the true residual is below ek_tol (relative to ||C||_F)
  int it = 0, sit = 0;
  double rel = 1.0, prev_rel = 1e300;
  bool conv = false;
  int solved_x = -1, solved_y = -1;
  // one projected solve on the current bases + the true residual (returns rc; sets rel)
  auto solve_and_check = [&]() -> int {
    const int sa = sx.s, sbb = sy.s;
    // A~ = U^T A1 U ; Bh = V^T A2 V ; B~ = Bh^T ; C~ = (U^T Cu) diag(sig) (V^T Cv)^T
    if ((rc = ts_tn(s, sa, sa, nx, 1.0, Ux, nx, AUx, nx, 0.0, Am, sa)) != FDE_OK) return rc;
    if ((rc = ts_tn(s, sbb, sbb, ny, 1.0, AVy, ny, Vy, ny, 0.0, Bm, sbb)) != FDE_OK) return rc;  // (A2 V)^T V = B~
    if ((rc = ts_tn(s, sa, rcr, nx, 1.0, Ux, nx, Cu, nx, 0.0, w.M1, sa)) != FDE_OK) return rc;
    if ((rc = ts_tn(s, rcr, sbb, ny, 1.0, Cv, ny, Vy, ny, 0.0, w.S, rcr)) != FDE_OK) return rc;   // (V^T Cv)^T
    CU(cudaMemcpyAsync(w.lam, sigc.data(), rcr * 8, cudaMemcpyHostToDevice, s));
    {
      // scale the rows of (V^T Cv)^T by sigma: use a diagonal via k_ts_gemm_nn with a diag matrix
      std::vector<double> dg((size_t)rcr * rcr, 0.0);
      for (int i = 0; i < rcr; ++i) dg[(size_t)i * rcr + i] = sigc[i];
      CU(cudaMemcpyAsync(w.G, dg.data(), dg.size() * 8, cudaMemcpyHostToDevice, s));
      if ((rc = ts_nn(s, sa, rcr, rcr, 1.0, w.M1, sa, w.G, rcr, 0.0, w.M2, sa)) != FDE_OK) return rc;
      if ((rc = ts_nn(s, sa, sbb, rcr, 1.0, w.M2, sa, w.S, rcr, 0.0, Cm, sa)) != FDE_OK) return rc;
      CU(cudaStreamSynchronize(s));
    }
    CU(cudaMemcpyAsync(Ym, Cm, (size_t)sa * sbb * 8, cudaMemcpyDeviceToDevice, s));
    // keep copies of A~ and B~ (the sign iteration destroys them): Lc <- A~, Rc <- Bh = B~^T
    CU(cudaMemcpyAsync(Lc, Am, (size_t)sa * sa * 8, cudaMemcpyDeviceToDevice, s));
    if ((rc = ts_tn(s, sbb, sbb, ny, 1.0, Vy, ny, AVy, ny, 0.0, Rc, sbb)) != FDE_OK) return rc;
    if ((rc = proj_sylvester(s, w, sa, sbb, Am, Bm, Ym, st, &sit)) != FDE_OK) return rc;
    // residual: Ra = A1 U - U A~ (nx x sa) ; ||Ra Y|| ; Rb = A2 V - V Bh ; ||Rb Y^T||
    CU(cudaMemcpyAsync(Wt, AUx, (size_t)nx * sa * 8, cudaMemcpyDeviceToDevice, s));
    if ((rc = ts_nn(s, nx, sa, sa, -1.0, Ux, nx, Lc, sa, 1.0, Wt, nx)) != FDE_OK) return rc;
    if ((rc = ts_nn(s, nx, sbb, sa, 1.0, Wt, nx, Ym, sa, 0.0, w.M2, nx)) != FDE_OK) return rc;
    double ra2 = 0.0, rb2 = 0.0;
    if ((rc = sumsq(s, nx, sbb, w.M2, nx, w.dv + 8, &ra2)) != FDE_OK) return rc;
    CU(cudaMemcpyAsync(Wt, AVy, (size_t)ny * sbb * 8, cudaMemcpyDeviceToDevice, s));
    if ((rc = ts_nn(s, ny, sbb, sbb, -1.0, Vy, ny, Rc, sbb, 1.0, Wt, ny)) != FDE_OK) return rc;
    // Y^T (sbb x sa) for Rb Y^T: transpose Y into Zm
    if ((rc = transpose(s, sa, sbb, Ym, sa, Zm, sbb)) != FDE_OK) return rc;
    if ((rc = ts_nn(s, ny, sa, sbb, 1.0, Wt, ny, Zm, sbb, 0.0, w.M2, ny)) != FDE_OK) return rc;
    if ((rc = sumsq(s, ny, sa, w.M2, ny, w.dv + 8, &rb2)) != FDE_OK) return rc;
    // the projected equation's own residual P = A~ Y + Y B~ - C~ (the splitting assumes P = 0;
    // the sign iteration leaves a rounding-level P, which is added here, not assumed away)
    CU(cudaMemcpyAsync(w.M1, Cm, (size_t)sa * sbb * 8, cudaMemcpyDeviceToDevice, s));
    if ((rc = ts_nn(s, sa, sbb, sa, 1.0, Lc, sa, Ym, sa, -1.0, w.M1, sa)) != FDE_OK) return rc;
    if ((rc = transpose(s, sbb, sbb, Rc, sbb, w.G, sbb)) != FDE_OK) return rc;
    if ((rc = ts_nn(s, sa, sbb, sbb, 1.0, Ym, sa, w.G, sbb, 1.0, w.M1, sa)) != FDE_OK) return rc;
    double rp2 = 0.0;
    if ((rc = sumsq(s, sa, sbb, w.M1, sa, w.dv + 8, &rp2)) != FDE_OK) return rc;
    rel = std::sqrt((ra2 + rb2 + rp2) / cnorm2);
    if (fde_dbg_env("FDE_DEBUG2D")) {
      double oe[2] = {0.0, 0.0};
      for (int side = 0; side < 2; ++side) {
        const int ss = side ? sbb : sa, nn2 = side ? ny : nx;
        const double* Ub = side ? Vy : Ux;
        std::vector<double> g((size_t)ss * ss);
        if ((rc = ts_tn(s, ss, ss, nn2, 1.0, Ub, nn2, Ub, nn2, 0.0, w.G, ss)) != FDE_OK) return rc;
        CU(cudaMemcpy(g.data(), w.G, g.size() * 8, cudaMemcpyDeviceToHost));
        for (int i = 0; i < ss; ++i) for (int j = 0; j < ss; ++j) oe[side] = std::max(oe[side], std::fabs(g[(size_t)i * ss + j] - (i == j)));
      }
      double yy2 = 0.0;
      if ((rc = sumsq(s, sa, sbb, Ym, sa, w.dv + 8, &yy2)) != FDE_OK) return rc;
      fprintf(stderr, "fde2d it %d: |U^T U - I| %.3e |V^T V - I| %.3e |Y| %.6e\n", it, oe[0], oe[1], std::sqrt(yy2));
      double ct2 = 0.0;
      if ((rc = sumsq(s, sa, sbb, Cm, sa, w.dv + 8, &ct2)) != FDE_OK) return rc;
      fprintf(stderr, "fde2d it %d: sa %d sb %d rc %d sign-its %d rel %.3e (ra2 %.3e rb2 %.3e rp2 %.3e c2 %.3e "
              "|C~|^2 - c2 %.3e)\n", it, sa, sbb, rcr, sit, rel, ra2, rb2, rp2, cnorm2, ct2 - cnorm2);
    }
    solved_x = sx.s; solved_y = sy.s;
    return FDE_OK;
  };
  bool solve_now = true;
  for (it = 1; it <= ek_maxit; ++it) {
    if (solve_now || it == ek_maxit) {
      if ((rc = solve_and_check()) != FDE_OK) return fail(rc);
      // converged: below ek_tol, or stagnated at the rounding floor of the residual evaluation
      // (reading R19: ||Rb|| carries eps ||A2 V||; cfg5's floor is ~1.2e-11 relative) within 10x
      if (rel <= ek_tol || (rel <= 10.0 * ek_tol && rel >= 0.9 * prev_rel)) { conv = true; break; }
      prev_rel = rel;
      // far from converged: grow twice before the next projected solve (the residual of the
      // extended Krylov method falls by well under 1e3 per iteration)
      solve_now = rel <= 1e3 * ek_tol;
    } else {
      solve_now = true;
    }
    if (it == ek_maxit) break;
    const int s0x = sx.s, s0y = sy.s;
    if ((rc = ek_grow(s, w, sx, Wt, dtol)) != FDE_OK) return fail(rc);
    if ((rc = ek_grow(s, w, sy, Wt, dtol)) != FDE_OK) return fail(rc);
    if (sx.s == s0x && sy.s == s0y) break;         // no new directions (EK_SMAX or exhausted)
  }
  if (!conv && (solved_x != sx.s || solved_y != sy.s)) {   // Y must belong to the final bases
    if ((rc = solve_and_check()) != FDE_OK) return fail(rc);
    conv = rel <= 10.0 * ek_tol;
  }
  (void)hsum;
  if (resid_out) *resid_out = rel;
  if (iters_out) *iters_out = std::min(it, ek_maxit);
  // ---- truncation: X = U_s Y V_s^T with Y = sum sigma_i u_i w_i^T, keep sigma > tol sigma_1
  const int sa = sx.s, sbb = sy.s;
  const bool dbg2 = fde_dbg_env("FDE_DEBUG2D") != nullptr;
  if (dbg2) {                                       // stored A U vs a fresh product, both sides
    for (EkSide* e : {&sx, &sy}) {
      if ((rc = hodlr_mv_cols(e->H, e->U, Wt, e->s, s)) != FDE_OK) return fail(rc);
      std::vector<double> h1((size_t)e->n * e->s), h2((size_t)e->n * e->s);
      CU(cudaMemcpy(h1.data(), Wt, h1.size() * 8, cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(h2.data(), e->AU, h2.size() * 8, cudaMemcpyDeviceToHost));
      double dmax = 0.0, amax = 0.0;
      int worst = -1;
      for (int j = 0; j < e->s; ++j)
        for (int i = 0; i < e->n; ++i) {
          const double d = std::fabs(h1[(size_t)j * e->n + i] - h2[(size_t)j * e->n + i]);
          if (d > dmax) { dmax = d; worst = j; }
          amax = std::max(amax, std::fabs(h1[(size_t)j * e->n + i]));
        }
      fprintf(stderr, "fde2d AU check side %d: s %d max|AU - A U| %.3e (col %d) max|A U| %.3e\n",
              e == &sx ? 0 : 1, e->s, dmax, worst, amax);
    }
  }
  if (dbg2) CU(cudaMemcpyAsync(w.M3, Ym, (size_t)sa * sbb * 8, cudaMemcpyDeviceToDevice, s));
  // Y (sa x sbb) is numerically low-rank: rank-revealing QR with column pivoting first
  // (Q_k^T Y, k ~ final rank), then the one-sided Jacobi SVD of (Q_k^T Y)^T (sbb x k) gives Y's
  // right singular vectors W and sigma; the left factor is Y W (exact product, no Q_k needed).
  // (A Jacobi SVD of the whole sa x sbb Y cost ~50 ms per step at cfg5.)
  int kq = 0;
  {
    int* kdev = reinterpret_cast<int*>(w.dv + 32);
    CU(cudaMemcpyAsync(w.M4, Ym, (size_t)sa * sbb * 8, cudaMemcpyDeviceToDevice, s));
    { PROF("k_qrcp_rows"); k_qrcp_rows<<<1, DN_BIG, 0, s>>>(sa, sbb, w.M4, 1e-2 * tol, w.V, kdev); }
    if ((rc = dn_check("k_qrcp_rows")) != FDE_OK) return fail(rc);
    CU(cudaMemcpyAsync(&kq, kdev, sizeof(int), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
  }
  if (kq > 0) {
    { PROF("k_osj_svd"); k_osj_svd<<<1, DN_BIG, dn_smem((long long)sbb * kq, kq + 2), s>>>(sbb, kq, w.V, sbb, Zm, sig, 60); }
    if ((rc = dn_check("k_osj_svd")) != FDE_OK) return fail(rc);
    CU(cudaMemcpyAsync(hs.data(), sig, kq * sizeof(double), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
  }
  if (fde_dbg_env("FDE_DEBUG2D") && kq > 0) {            // orthogonality of the Jacobi rotations
    std::vector<double> g((size_t)kq * kq);
    if ((rc = ts_tn(s, kq, kq, kq, 1.0, Zm, kq, Zm, kq, 0.0, w.G, kq)) != FDE_OK) return fail(rc);
    CU(cudaMemcpy(g.data(), w.G, g.size() * 8, cudaMemcpyDeviceToHost));
    double e = 0.0;
    for (int i = 0; i < kq; ++i) for (int j = 0; j < kq; ++j) e = std::max(e, std::fabs(g[(size_t)i * kq + j] - (i == j)));
    fprintf(stderr, "fde2d svd: sa %d sb %d qr rank %d |Z^T Z - I|max %.3e sig1 %.3e\n", sa, sbb, kq, e, hs[0]);
  }
  ord.assign(kq, 0);
  for (int i = 0; i < kq; ++i) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](int a, int c) { return hs[a] > hs[c] || (hs[a] == hs[c] && a < c); });
  keep.clear();
  for (int i : ord) if (hs[i] > tol * hs[ord[0]] && hs[i] > 0.0) keep.push_back(i);
  const int rk = (int)keep.size();
  if (rk > rmax) { fail(FDE_OK); return set_err(FDE_EDIM, "solution rank %d exceeds rmax=%d", rk, rmax); }
  if (rk > 0) {
    CU(cudaMemcpyAsync(w.idx, keep.data(), rk * sizeof(int), cudaMemcpyHostToDevice, s));
    // right vectors M6 = (AT Z)[:, keep] / sigma, left factor M5 = Y M6 (= U_k Sigma_k)
    { PROF("k_gather_cols"); k_gather_cols<<<(sbb * rk + 255) / 256, 256, 0, s>>>(sbb, rk, w.V, sbb, w.idx, sig, w.M6, sbb); }
    if ((rc = dn_check("k_gather_cols")) != FDE_OK) return fail(rc);
    if ((rc = ts_nn(s, sa, rk, sbb, 1.0, Ym, sa, w.M6, sbb, 0.0, w.M5, sa)) != FDE_OK) return fail(rc);
    if (dbg2) {                                     // |M5 M6^T - Y| / |Y|: the truncated assembly
      if ((rc = transpose(s, sbb, rk, w.M6, sbb, w.G, rk)) != FDE_OK) return fail(rc);
      if ((rc = ts_nn(s, sa, sbb, rk, 1.0, w.M5, sa, w.G, rk, -1.0, w.M3, sa)) != FDE_OK) return fail(rc);
      double d2 = 0.0, y2 = 0.0;
      if ((rc = sumsq(s, sa, sbb, w.M3, sa, w.dv + 8, &d2)) != FDE_OK) return fail(rc);
      for (int i = 0; i < kq; ++i) y2 += hs[i] * hs[i];
      fprintf(stderr, "fde2d assembly: rk %d of %d, |M5 M6^T - Y|/|Y| %.3e, |Y| %.6e sig max %.3e min kept %.3e\n", rk, sbb,
              std::sqrt(d2 / y2), std::sqrt(y2), hs[ord[0]], hs[keep[rk - 1]]);
    }
    if ((rc = ts_nn(s, nx, rk, sa, 1.0, Ux, nx, w.M5, sa, 0.0, Xu, nx)) != FDE_OK) return fail(rc);
    if ((rc = ts_nn(s, ny, rk, sbb, 1.0, Vy, ny, w.M6, sbb, 0.0, Xv, ny)) != FDE_OK) return fail(rc);
  }
  *rx = rk;
  release();
  CU(cudaStreamSynchronize(s));
  DevStatus dst{};
  CU(cudaMemcpy(&dst, st, sizeof(dst), cudaMemcpyDeviceToHost));
  cleanup();
  if (dst.code != FDE_OK) return set_err(dst.code, "device status %d in fde2d_step", dst.code);
  if (!conv) return set_err(FDE_ENOCONV, "extended Krylov: relative residual %.3e > ek_tol %.1e after %d iterations",
                            rel, ek_tol, ek_maxit);
  (void)flags;
  return FDE_OK;
}
