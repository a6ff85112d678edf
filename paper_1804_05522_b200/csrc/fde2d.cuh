// fde2d.cuh -- S8-S10: one implicit-Euler step of the 2D FDE as a Sylvester equation
// (Eq. 4.3, readings R11/R12):
//     A1 X + X A2^T = C,   C = Uu Uv^T + dt Fu Fv^T,
//     A_i = 1/2 I + (dt/h_i^alpha_i)(D_i+ T_i + D_i- T_i^T),
// solved by the extended Krylov subspace method on the HODLR factors of A1, A2.
//
//  S8  right-hand side: Householder QR of both factors, W_u = [Uu, dt Fu] = Q_u R_u,
//      W_v = [Uv, Fv] = Q_v R_v, SVD of the small R_u R_v^T, truncation below tol * sigma_1:
//      C ~ Cu diag(sig) Cv^T with orthonormal Cu = Q_u P, Cv = Q_v Z ("QR of the factors + small
//      SVD").  Householder, not a Gram matrix: the columns of [Uu, dt Fu] span ~12
//      decades (the singular values of the previous X next to dt F) and a Gram-based
//      orthogonalisation loses the directions below ~1e-8 of the largest column -- exactly the
//      component of C the Krylov bases would then miss (round 1's open residual discrepancy).
//  S9  bases U of EK(A1, Cu) and V of EK(A2, Cv): first block [Cu | orth(A^{-1} Cu)], then per
//      iteration and side one HODLR matvec (A P) and one HODLR solve (A^{-1} N), each new block
//      orthonormalised against the basis by block Gram-Schmidt twice with a pivoted-Cholesky
//      normalisation (k_pchol_orth: deflation of directions below dtol).  The products A U are
//      kept (one matvec per new column).
//  S10 projected equation A~ Y + Y B~ = C~ (A~ = U^T A1 U, B~ = (V^T A2 V)^T, C~ = U^T C V) by the
//      scaled Newton iteration for the matrix sign function (inverses by k_gj_inv_cl: Gauss-Jordan
//      with partial pivoting on a thread-block cluster); since Sym(A_i) > 0 the spectra of A~, B~
//      lie in the open right half plane and the iteration converges.
//      Residual from the exact splitting (U orthonormal, C inside span(U) x span(V), Ra = A1 U -
//      U A~ orthogonal to U):  ||R||^2 = ||Ra Y||^2 + ||Rb Y^T||^2 + ||A~ Y + Y B~ - C~||^2.
//      Truncation of X = U Y V^T: rank-revealing QR of Y + one-sided Jacobi SVD; the
//      reported residual is the splitting evaluated at the TRUNCATED Y (plus the dropped part of
//      C), i.e. the residual of the returned X against the input C and the HODLR operators.
#pragma once
#include <algorithm>
#include <initializer_list>
#include "k_dense.cuh"
#include "k_small.cuh"

#define EK_SMAX 320                    // cap on the projected size per side
#define GJ_SMEM_MAX (220 * 1024)       // dynamic shared memory of one inverse CTA

static int dn_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(FDE_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return FDE_OK;
}

// ---- per-device one-time attributes (cudaFuncSetAttribute applies to the current device)
static std::atomic<unsigned long long> g_dn_attr_mask{0};
static int dn_attrs() {
  int dev = 0;
  CU(cudaGetDevice(&dev));
  const unsigned long long bit = 1ULL << (dev & 63);
  if (g_dn_attr_mask.load() & bit) return FDE_OK;
  CU(cudaFuncSetAttribute(k_osj_svd, cudaFuncAttributeMaxDynamicSharedMemorySize, DN_SMEM_MAX + 4096));
  CU(cudaFuncSetAttribute(k_pchol_orth, cudaFuncAttributeMaxDynamicSharedMemorySize, PO_SMEM));
  CU(cudaFuncSetAttribute(k_gj_inv_cl<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, GJ_SMEM_MAX));
  CU(cudaFuncSetAttribute(k_gj_inv_cl<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, GJ_SMEM_MAX));
  CU(cudaFuncSetAttribute(k_gj_inv_cl<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, GJ_SMEM_MAX));
  CU(cudaFuncSetAttribute(k_gj_inv_cl<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, GJ_SMEM_MAX));
  // the per-step workspace comes from the device's default stream-ordered pool: keep freed
  // blocks mapped across synchronisations (a release threshold of 0 would unmap and re-map the
  // workspace every fde2d_step)
  cudaMemPool_t pool;
  CU(cudaDeviceGetDefaultMemPool(&pool, dev));
  unsigned long long keep_bytes = 1ULL << 30;
  CU(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep_bytes));
  g_dn_attr_mask.fetch_or(bit);
  return FDE_OK;
}

// ---- step workspace: one stream-ordered allocation, carved (split-K partials included)
struct Ws2d {
  double* part; size_t part_cap;       // split-K partials of k_gemm_tn
  double *G, *S, *M1, *M2, *M3, *M4, *M5, *M6, *dv;
  int* iv;                             // small device ints (counts, index lists)
  InvJob* jobs;
  QrJob* qjobs;
  QJob* qqjobs;
};

// C (m x n) = alpha A^T B + beta C  (A: K x m, B: K x n; K tall), DMMA with split-K partials
static int ts_tn(cudaStream_t s, const Ws2d& w, int m, int n, int K, double alpha, const double* A, int lda,
                 const double* B, int ldb, double beta, double* C, int ldc) {
  if (m <= 0 || n <= 0) return FDE_OK;
  const int tiles = ((m + SG_TILE - 1) / SG_TILE) * ((n + SG_TILE - 1) / SG_TILE);
  int nz = std::max(1, std::min(64, (296 + tiles - 1) / tiles));      // ~2 CTAs per SM
  int kchunk = round_up(std::max(1, (K + nz - 1) / nz), SG_TILE);
  nz = (K + kchunk - 1) / kchunk;
  while (nz > 1 && (size_t)nz * m * n > w.part_cap) { kchunk *= 2; nz = (K + kchunk - 1) / kchunk; }
  const dim3 grid((m + SG_TILE - 1) / SG_TILE, (n + SG_TILE - 1) / SG_TILE, std::max(nz, 1));
  if (nz <= 1) {
    { PROF("k_gemm_tn"); k_gemm_tn<<<grid, SG_THREADS, 0, s>>>(m, n, K, std::max(K, 1), A, lda, B, ldb, nullptr, alpha, beta, C, ldc); }
    return dn_check("k_gemm_tn");
  }
  { PROF("k_gemm_tn"); k_gemm_tn<<<grid, SG_THREADS, 0, s>>>(m, n, K, kchunk, A, lda, B, ldb, w.part, 0.0, 0.0, nullptr, 0); }
  TRY(dn_check("k_gemm_tn"));
  { PROF("k_sum_partials"); k_sum_partials<<<(m * n + 255) / 256, 256, 0, s>>>(m, n, nz, w.part, alpha, beta, C, ldc); }
  return dn_check("k_sum_partials");
}

// C (M x n) = alpha A B + beta C  (A: M x K, B: K x n)
static int ts_nn(cudaStream_t s, int M, int n, int K, double alpha, const double* A, int lda,
                 const double* B, int ldb, double beta, double* C, int ldc) {
  if (M <= 0 || n <= 0) return FDE_OK;
  { PROF("k_gemm_nn"); k_gemm_nn<<<dim3((M + 63) / 64, (n + 31) / 32), SG_THREADS, 0, s>>>(M, n, K, alpha, A, lda, B, ldb, beta, C, ldc); }
  return dn_check("k_gemm_nn");
}

static int transpose(cudaStream_t s, int m, int n, const double* X, int ldx, double* Y, int ldy) {
  if (m <= 0 || n <= 0) return FDE_OK;
  { PROF("k_transpose"); k_transpose<<<dim3((m + 31) / 32, (n + 31) / 32), dim3(32, 8), 0, s>>>(m, n, X, ldx, Y, ldy); }
  return dn_check("k_transpose");
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

// out[0] = sum of squares of X (m x n); one CTA (fixed order)
static int sumsq_dev(cudaStream_t s, int m, int n, const double* X, int ldx, double* out) {
  { PROF("k_sumsq"); k_sumsq<<<1, DN_BIG, 0, s>>>(m, n, X, ldx, out); }
  return dn_check("k_sumsq");
}

// gather columns: Y[:, j] = alpha_j X[:, idx[j]]  (alpha_j = sc ? 1/sc[idx[j]] : 1)
__global__ void k_gather_cols(int m, int nk, const double* __restrict__ X, int ldx, const int* __restrict__ idx,
                              const double* __restrict__ sc, double* __restrict__ Y, int ldy) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)m * nk) return;
  const int i = (int)(e % m), j = (int)(e / m), c = idx[j];
  Y[(long long)j * ldy + i] = X[(long long)c * ldx + i] * (sc ? 1.0 / sc[c] : 1.0);
}

// M (k1 x k2) = R1 R2^T with R1 = upper triangle of W1[0:k1, 0:r], R2 likewise (W ld n1 / n2)
__global__ void k_rrt(int k1, int k2, int r, const double* __restrict__ W1, int ld1, const double* __restrict__ W2,
                      int ld2, double* __restrict__ M) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= k1 * k2) return;
  const int i = e % k1, j = e / k1;
  double a = 0.0;
  for (int q = max(i, j); q < r; ++q) a = fma(W1[(long long)q * ld1 + i], W2[(long long)q * ld2 + j], a);
  M[(long long)j * k1 + i] = a;
}

// Y (m x n, ld m) = X (m x n, ld ldx) with row i scaled by d[i]
__global__ void k_scale_rows(int m, int n, const double* __restrict__ X, int ldx, const double* __restrict__ d,
                             double* __restrict__ Y) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)m * n) return;
  const int i = (int)(e % m), j = (int)(e / m);
  Y[(long long)j * m + i] = d[i] * X[(long long)j * ldx + i];
}

// Rank-revealing Householder QR with column pivoting (one CTA), truncation step of S10: W (m x n,
// ld m, overwritten) <- H_k .. H_1 W, stopping at the first step k whose largest remaining column
// norm is <= rtol * the largest initial column norm.  Pivoting is by index (no column swaps), so
// rows 0..k-1 are Q_k^T W in the original column order; they are written transposed to AT (n x k,
// ld n) and k to *kout.  Residual column norms are recomputed every step (no downdating).
__global__ void __launch_bounds__(DN_BIG)
k_qrcp_rows(int m, int n, double* __restrict__ W, double rtol, double* __restrict__ AT, int* __restrict__ kout) {
  __shared__ double v[EK_SMAX], nrm[EK_SMAX];
  __shared__ double s_tau, s_n0;
  __shared__ int s_jp, s_stop;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31, nw = DN_BIG / 32;
  const int kmax = min(m, n);
  int k = 0;
  for (int step = 0; step < kmax; ++step) {
    for (int j = warp; j < n; j += nw) {
      double a = 0.0;
      for (int i = step + lane; i < m; i += 32) { const double x = W[(long long)j * m + i]; a = fma(x, x, a); }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (lane == 0) nrm[j] = a;
    }
    __syncthreads();
    if (warp == 0) {
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
          s_tau = 1.0 / (nx * (nx + fabs(x0)));
        }
      }
    }
    __syncthreads();
    if (s_stop) break;
    const int jp = s_jp;
    for (int i = step + 1 + t; i < m; i += DN_BIG) v[i - step] = W[(long long)jp * m + i];
    __syncthreads();
    const double tau = s_tau;
    for (int j = warp; j < n; j += nw) {
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

// Newton sign iteration update (one CTA):  with mu = sqrt(||Z^-1||_F / ||Z||_F) for
// Z = [[A, -C], [0, -B]]:  A <- (mu A + Ainv/mu)/2,  B <- (mu B + Binv/mu)/2,
// C <- (mu C + (Ainv C Binv)/mu)/2 (T = Ainv C Binv given); out[0] = relative change of A, B.
__global__ void __launch_bounds__(DN_BIG)
k_sign_update(int sa, int sb, double* __restrict__ A, const double* __restrict__ Ai, double* __restrict__ B,
              const double* __restrict__ Bi, double* __restrict__ C, const double* __restrict__ T,
              double* __restrict__ out) {
  __shared__ double red[4][DN_BIG];
  const int t = threadIdx.x;
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

// ---------------------------------------------------------------------------------------
// Orthonormalise the n x b block W (ld n, destroyed) against the orthonormal basis Ub[:, 0:sb]
// (ld n): (project, normalise) twice -- block Gram-Schmidt then a pivoted-Cholesky normalisation
// (k_pchol_orth).  Pass 0 deflates directions below dtol * (largest column norm), pass 1 drops
// any that lost more than half their norm.  New columns -> Ub[:, sb:sb+nb]; *nb = their count.
static int orth_append(cudaStream_t s, const Ws2d& w, int n, double* W, int b, double* Ub, int sb,
                       int smax, double dtol, int* nb) {
  *nb = 0;
  if (b <= 0 || sb >= smax) return FDE_OK;
  if (b > PO_MAX) return set_err(FDE_EDIM, "block of %d columns exceeds %d", b, PO_MAX);
  // ref = largest squared column norm of the block, kept on the device (w.dv[30]): pass 0's
  // threshold is dtol^2 * ref inside k_pchol_orth (a zero block keeps no column: nk = 0)
  TRY(ts_tn(s, w, b, b, n, 1.0, W, n, W, n, 0.0, w.G, b));
  { PROF("k_diag_max"); k_diag_max<<<1, 32, 0, s>>>(b, w.G, w.dv + 30); }
  TRY(dn_check("k_diag_max"));
  int cur = b;
  double* src = W;
  for (int pass = 0; pass < 2; ++pass) {
    if (sb > 0) {
      TRY(ts_tn(s, w, sb, cur, n, 1.0, Ub, n, src, n, 0.0, w.M1, sb));      // H = U^T W
      TRY(ts_nn(s, n, cur, sb, -1.0, Ub, n, w.M1, sb, 1.0, src, n));      // W -= U H
    }
    TRY(ts_tn(s, w, cur, cur, n, 1.0, src, n, src, n, 0.0, w.G, cur));
    const double thr = pass == 0 ? dtol * dtol : 0.25;
    { PROF("k_pchol_orth"); k_pchol_orth<<<1, 256, PO_SMEM, s>>>(cur, w.G, thr, std::min(cur, smax - sb), w.S, w.iv,
                                                                  pass == 0 ? w.dv + 30 : nullptr); }
    TRY(dn_check("k_pchol_orth"));
    int nk = 0;
    CU(cudaMemcpyAsync(&nk, w.iv, sizeof(int), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (nk == 0) return FDE_OK;
    double* dst = pass == 0 ? w.M2 : Ub + (size_t)sb * n;               // M2 holds n x PO_MAX
    TRY(ts_nn(s, n, nk, cur, 1.0, src, n, w.S, cur, 0.0, dst, n));
    src = dst;
    cur = nk;
  }
  *nb = cur;
  return FDE_OK;
}

// Solve A~ Y + Y B~ = C~ (sa x sa, sb x sb, sa x sb, all ld = own rows) by the scaled Newton sign
// iteration; Y is returned in C (overwritten).  A, B are destroyed.
static int proj_sylvester(cudaStream_t s, const Ws2d& w, int sa, int sb, double* A, double* B, double* C,
                          DevStatus* st, int* iters) {
  double* Ai = w.M3;
  double* Bi = w.M4;
  double* T = w.M5;
  double* T2 = w.M6;
  InvJob hj[2] = {{Ai, sa, sa}, {Bi, sb, sb}};
  CU(cudaMemcpyAsync(w.jobs, hj, sizeof(hj), cudaMemcpyHostToDevice, s));
  const int smx = std::max(sa, sb);
  int CL = 1;
  while (CL < 8 && gj_smem(smx, CL) > GJ_SMEM_MAX) CL *= 2;
  const size_t smem = gj_smem(smx, CL);
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  cfg.gridDim = dim3(2 * CL);
  cfg.blockDim = dim3(GJ_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  double hout[2] = {1, 1};
  int it = 0;
  for (; it < 60; ++it) {
    CU(cudaMemcpyAsync(Ai, A, (size_t)sa * sa * sizeof(double), cudaMemcpyDeviceToDevice, s));
    CU(cudaMemcpyAsync(Bi, B, (size_t)sb * sb * sizeof(double), cudaMemcpyDeviceToDevice, s));
    {
      PROF("k_gj_inv_cl");
      const InvJob* jp = w.jobs;
      if (CL == 1) CU(cudaLaunchKernelEx(&cfg, k_gj_inv_cl<1>, jp, st));
      else if (CL == 2) CU(cudaLaunchKernelEx(&cfg, k_gj_inv_cl<2>, jp, st));
      else if (CL == 4) CU(cudaLaunchKernelEx(&cfg, k_gj_inv_cl<4>, jp, st));
      else CU(cudaLaunchKernelEx(&cfg, k_gj_inv_cl<8>, jp, st));
    }
    TRY(dn_check("k_gj_inv_cl"));
    TRY(ts_nn(s, sa, sb, sa, 1.0, Ai, sa, C, sa, 0.0, T, sa));            // T2 = Ai C Bi
    TRY(ts_nn(s, sa, sb, sb, 1.0, T, sa, Bi, sb, 0.0, T2, sa));
    { PROF("k_sign_update"); k_sign_update<<<1, DN_BIG, 0, s>>>(sa, sb, A, Ai, B, Bi, C, T2, w.dv); }
    TRY(dn_check("k_sign_update"));
    // (the iteration needs ~log2 of the spectrum's spread before it contracts: 9-11 iterations on
    //  the projected EK operators, so the first four are queued without reading the change back)
    if (it < 4) continue;
    CU(cudaMemcpyAsync(hout, w.dv, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (fde_dbg_env("FDE_DEBUG2D") && fde_dbg_env("FDE_DEBUG2D")[0] == '2')
      fprintf(stderr, "  sign it %d change %.3e mu %.3e\n", it, hout[0], hout[1]);
    if (hout[0] < 1e-14) { ++it; break; }
  }
  // sign(Z) = [[I, 2Y], [0, -I]] for Z = [[A, -C], [0, -B]]: the iterated C block tends to 2Y
  TRY(scale_copy(s, sa, sb, 0.5, C, sa, C, sa));
  *iters = it;
  return FDE_OK;
}

// y = A x for ncol columns (chunks of NRHS_MAX)
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
static int ek_grow(cudaStream_t s, const Ws2d& w, EkSide& e, double* Wtmp, double dtol) {
  const int n = e.n;
  int nbp = 0, nbn = 0;
  const int oldp = e.p0, oldnp = e.np, oldn = e.n0, oldnn = e.nn;
  if (oldnp > 0) {                     // A P_j is already in AU
    CU(cudaMemcpyAsync(Wtmp, e.AU + (size_t)oldp * n, (size_t)n * oldnp * sizeof(double), cudaMemcpyDeviceToDevice, s));
    TRY(orth_append(s, w, n, Wtmp, oldnp, e.U, e.s, EK_SMAX, dtol, &nbp));
    if (nbp) TRY(hodlr_mv_cols(e.H, e.U + (size_t)e.s * n, e.AU + (size_t)e.s * n, nbp, s));
    e.p0 = e.s; e.np = nbp; e.s += nbp;
  } else { e.np = 0; }
  if (oldnn > 0) {
    TRY(hodlr_solve_cols(e.H, e.U + (size_t)oldn * n, Wtmp, oldnn, s));
    TRY(orth_append(s, w, n, Wtmp, oldnn, e.U, e.s, EK_SMAX, dtol, &nbn));
    if (nbn) TRY(hodlr_mv_cols(e.H, e.U + (size_t)e.s * n, e.AU + (size_t)e.s * n, nbn, s));
    e.n0 = e.s; e.nn = nbn; e.s += nbn;
  } else { e.nn = 0; }
  return FDE_OK;
}

// ---- the two operators (built and factorised once, reused while the arguments match)
static int build_op_2d(int n, double alpha, double h, double dt, const double* dp, const double* dm, double tol,
                       int leaf, cudaStream_t s, fde_hodlr** out, double shift = 0.5) {
  TRY(build_impl(1, n, &alpha, h, dt, dp, dm, shift, tol, leaf, 0, s, out));
  fde_hodlr* H = *out;
  const int rc = factor_impl(H, H->d_dp, H->d_dm, 0, nullptr, nullptr, nullptr, 1, s);
  if (rc != FDE_OK) { free_handle(H); *out = nullptr; return rc; }
  H->factored = true;
  H->src_dp = dp; H->src_dm = dm;
  H->last_stream = s;
  return FDE_OK;
}

// Ensure *op is the factorised operator 1/2 I + (dt/h^alpha)(D+ T + D- T^T) for these arguments:
// rebuild when (n, alpha, h, tol, leaf) differ; re-copy the coefficients, set dt and refactorise
// when only dt, the coefficient pointers or FDE_COEFFS_CHANGED differ (compression reused).
static int ensure_op_2d(fde_hodlr** op, int n, double alpha, double h, double dt, const double* dp,
                        const double* dm, double tol, int leaf, unsigned flags, cudaStream_t s, double shift = 0.5) {
  fde_hodlr* H = *op;
  const bool same = H && H->batch == 1 && H->n == n && H->alpha[0] == alpha && H->h == h && H->tol == tol &&
                    H->leaf == leaf && H->shift == shift && !H->compress_only;
  if (!same) {
    if (H) hodlr_destroy(H);
    *op = nullptr;
    return build_op_2d(n, alpha, h, dt, dp, dm, tol, leaf, s, op, shift);
  }
  if (H->factored && H->dt == dt && H->src_dp == dp && H->src_dm == dm && !(flags & FDE_COEFFS_CHANGED))
    return FDE_OK;
  const size_t bytes = (size_t)n * sizeof(double);
  CU(cudaMemcpyAsync(H->d_dp, dp, bytes, cudaMemcpyDeviceToDevice, s));
  CU(cudaMemcpyAsync(H->d_dm, dm, bytes, cudaMemcpyDeviceToDevice, s));
  TRY(set_dt(H, dt, s));
  TRY(factor_impl(H, H->d_dp, H->d_dm, 0, nullptr, nullptr, nullptr, 1, s));
  H->factored = true;
  H->src_dp = dp; H->src_dm = dm;
  H->last_stream = s;
  return FDE_OK;
}

// ---------------------------------------------------------------------------------------
// Multi-shift rational Krylov mode (the paper's projection framework,
// P:1519-1550, with rational instead of extended Krylov bases).  The bases grow by rounds of
// npole independent shifted solves per side, W_j = (A1 + p_j I)^{-1} Cu and (A2 + q_j I)^{-1} Cv,
// each shifted operator an independent HODLR factorisation (hodlr_build with shift 1/2 + p_j).
// Poles: the A1 side takes p_j in the spectral range of A2 and the A2 side q_j in that of A1 (the
// poles of the solution X = int e^{-t A1} C e^{-t A2^T} dt seen from either side), log-spaced in
// [1/2, 1/2 + c 2^alpha (max d+ + max d-)] (reading R7's norm bound), round r offset by phi_r;
// or given.  The poles of a round are independent: with pw > 1 ranks, pole j is solved by rank
// j mod pw and the blocks are all-gathered (one exchange per round and side); everything else
// runs on every rank on the same data.
struct RkSpec {
  int npole;                    // poles per round and side
  int rounds;                   // maximum number of rounds
  const double* poles;          // host [2 * npole * rounds] (side 0 then side 1, round-major) or NULL
  int pw, pr;                   // pole sharding: world, rank
  fde_allgather_fn gather; void* ctx;
  fde_hodlr** shifted;          // cache [2 * npole * rounds] of the shifted factorisations
};

__global__ void k_absmax2(int n, const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out) {
  __shared__ double red[2][1024];
  double ma = 0.0, mb = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) { ma = fmax(ma, fabs(a[i])); mb = fmax(mb, fabs(b[i])); }
  red[0][threadIdx.x] = ma; red[1][threadIdx.x] = mb;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      red[0][threadIdx.x] = fmax(red[0][threadIdx.x], red[0][threadIdx.x + w]);
      red[1][threadIdx.x] = fmax(red[1][threadIdx.x], red[1][threadIdx.x + w]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { out[0] = red[0][0]; out[1] = red[1][0]; }
}

// ---------------------------------------------------------------------------------------
// The step on one or two processes.  world = 1: this process owns both sides.  world = 2 (the
// x/y split of SURVEY §8(e), the two EK processes being independent): rank 0 owns
// A1, the basis U and the factor Xu; rank 1 owns A2, V and Xv.  Everything that couples the
// sides goes through four exchanges of small device buffers -- the R factors of the
// right-hand side, the projected matrices (A~ or B^ and U^T Cu or V^T Cv), the basis sizes
// after growth, and the residual parts -- each an all-gather over the pair (`gather`; at
// world = 1 a local copy).  The small dense work (SVDs, the projected Sylvester equation, the
// convergence decisions) is repeated on both ranks on identical data, so both take the same
// decisions.  Layout of an exchange with slot size S: send = [side-0 slot | side-1 slot] (an
// owned side fills its slot), recv = world x send (rank order); side d is read from the slot of
// its owner.
struct Xchg {
  int world, rank;
  fde_allgather_fn gather;
  void* ctx;
  double *send, *recv;
  int owner(int d) const { return world == 1 ? 0 : d; }
  bool own(int d) const { return world == 1 || rank == d; }
  double* slot(int d, long long S) { return send + (long long)d * S; }
  const double* got(int d, long long S) const { return recv + (long long)owner(d) * 2 * S + (long long)d * S; }
  int run(long long S, cudaStream_t s) {
    if (world == 1 && !gather) {
      if (cudaMemcpyAsync(recv, send, (size_t)(2 * S) * sizeof(double), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return set_err(FDE_ECUDA, "exchange copy failed");
      return FDE_OK;
    }
    const int rc = gather(ctx, send, recv, 2 * S, s);
    if (rc != 0) return set_err(FDE_ECUDA, "exchange callback failed (%d)", rc);
    return FDE_OK;
  }
};

static int step_2d_impl(Xchg& xc, int nx, int ny, double alpha1, double alpha2, double hx, double hy, double dt,
                        const double* d1p, const double* d1m, const double* d2p, const double* d2m,
                        const double* Fu, const double* Fv, int rf, const double* Uu, const double* Uv,
                        int ru, double* Xu, double* Xv, int rmax, int* rx, double tol, double ek_tol,
                        int ek_maxit, int leaf, fde_hodlr_t* cache, double* resid_out, int* iters_out,
                        unsigned flags, cudaStream_t s, const RkSpec* rk = nullptr) {
  const bool own0 = xc.own(0), own1 = xc.own(1);
  TRY(check_common(1, nx, &alpha1, hx, dt, tol, leaf));
  TRY(check_common(1, ny, &alpha2, hy, dt, tol, leaf));
  if ((own0 && (!d1p || !d1m)) || (own1 && (!d2p || !d2m))) return set_err(FDE_EDOMAIN, "NULL coefficient array");
  if (rf < 0 || ru < 0 || (rf > 0 && ((own0 && !Fu) || (own1 && !Fv))) || (ru > 0 && ((own0 && !Uu) || (own1 && !Uv))))
    return set_err(FDE_EDOMAIN, "bad right-hand-side factors (rf=%d, ru=%d)", rf, ru);
  if ((own0 && !Xu) || (own1 && !Xv) || !rx || rmax < 1) return set_err(FDE_EDOMAIN, "bad output factors (rmax=%d)", rmax);
  if (!(ek_tol > 0.0 && ek_tol < 1.0) || ek_maxit < 1) return set_err(FDE_EDOMAIN, "ek_tol / ek_maxit out of range");
  if (rf + ru > NRHS_MAX) return set_err(FDE_EDIM, "rf + ru = %d exceeds %d", rf + ru, NRHS_MAX);
  if (rf + ru > std::min(nx, ny)) return set_err(FDE_EDIM, "rf + ru = %d exceeds n", rf + ru);
  TRY(dn_attrs());
  fde_hodlr* tmp[2] = {nullptr, nullptr};
  fde_hodlr** ops = cache ? reinterpret_cast<fde_hodlr**>(cache) : tmp;
  auto cleanup = [&]() { if (!cache) { hodlr_destroy(ops[0]); hodlr_destroy(ops[1]); ops[0] = ops[1] = nullptr; } };
  int rc = FDE_OK;
  if (own0) rc = ensure_op_2d(&ops[0], nx, alpha1, hx, dt, d1p, d1m, tol, leaf, flags, s);
  if (rc == FDE_OK && own1) rc = ensure_op_2d(&ops[1], ny, alpha2, hy, dt, d2p, d2m, tol, leaf, flags, s);
  if (rc != FDE_OK) { cleanup(); return rc; }
  // the owned handles' device status words start clean (any earlier failure was reported)
  for (int i = 0; i < 2; ++i)
    if (xc.own(i) && cudaMemsetAsync(ops[i]->d_status, 0, sizeof(DevStatus), s) != cudaSuccess) {
      cleanup(); return set_err(FDE_ECUDA, "status reset failed");
    }
  DevStatus* st = ops[own0 ? 0 : 1]->d_status;
  // ---- workspace: one stream-ordered allocation (kept mapped by the pool between steps)
  const int nmax = std::max(nx, ny), r0 = ru + rf;
  const size_t big = (size_t)nmax * EK_SMAX, sm2 = (size_t)EK_SMAX * EK_SMAX;
  const size_t part_cap = (size_t)16 * sm2;
  const long long SS = 1 + (long long)sm2 + (long long)EK_SMAX * NRHS_MAX;      // projection slot
  size_t o = 0;
  auto carve = [&](size_t doubles) { const size_t r = o; o += (doubles + 31) & ~(size_t)31; return r; };
  const size_t oUx = carve(big), oAUx = carve(big), oVy = carve(big), oAVy = carve(big), oWt = carve(big);
  const size_t oQu = carve((size_t)nx * NRHS_MAX), oQv = carve((size_t)ny * NRHS_MAX), oTau = carve(2 * NRHS_MAX);
  const size_t oCu = carve((size_t)nx * NRHS_MAX), oCv = carve((size_t)ny * NRHS_MAX);
  const size_t oPart = carve(part_cap), oG = carve(sm2), oS = carve(sm2), oM1 = carve(sm2);
  const size_t oM2 = carve(std::max(big, sm2)), oM3 = carve(sm2), oM4 = carve(sm2), oM5 = carve(sm2), oM6 = carve(sm2);
  const size_t oDv = carve(64), oIv = carve(EK_SMAX), oJobs = carve(64), oAm = carve(sm2), oBm = carve(sm2);
  const size_t oCm = carve(sm2), oYm = carve(sm2), oZm = carve(sm2), oSig = carve(EK_SMAX), oLc = carve(sm2), oRc = carve(sm2);
  const size_t oSg = carve(NRHS_MAX), oXs = carve(2 * SS), oXr = carve((size_t)xc.world * 2 * SS);
  const int rk_np = rk ? rk->npole : 0, rk_pw = rk ? std::max(1, rk->pw) : 1;
  const size_t rk_cnt = (size_t)((rk_np + rk_pw - 1) / rk_pw) * nmax * NRHS_MAX;     // blocks per rank
  const size_t oWs = carve(rk ? rk_cnt : 0), oWr = carve(rk && rk_pw > 1 ? rk_pw * rk_cnt : 0);
  double* base = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&base), o * sizeof(double), s) != cudaSuccess) {
    cudaGetLastError(); cleanup(); return set_err(FDE_ENOMEM, "fde2d workspace allocation failed (%zu MB)", o * 8 >> 20);
  }
  bool failed = false;                             // (fail() may be reached twice: inner + outer)
  auto fail = [&](int code) {
    if (!failed) { failed = true; cudaFreeAsync(base, s); cudaStreamSynchronize(s); cleanup(); }
    return code;
  };
#define CK(call) do { cudaError_t e_ = (call); if (e_ != cudaSuccess) return fail(set_err(FDE_ECUDA, "%s: %s", #call, cudaGetErrorString(e_))); } while (0)
#define TK(call) do { const int r_ = (call); if (r_ != FDE_OK) return fail(r_); } while (0)
  double *Ux = base + oUx, *AUx = base + oAUx, *Vy = base + oVy, *AVy = base + oAVy, *Wt = base + oWt;
  double *Qu = base + oQu, *Qv = base + oQv, *tau = base + oTau, *Cu = base + oCu, *Cv = base + oCv;
  double *Am = base + oAm, *Bm = base + oBm, *Cm = base + oCm, *Ym = base + oYm, *Zm = base + oZm;
  double *sig = base + oSig, *Lc = base + oLc, *Rc = base + oRc, *sgd = base + oSg;
  xc.send = base + oXs; xc.recv = base + oXr;
  Ws2d w{};
  w.part = base + oPart; w.part_cap = part_cap;
  w.G = base + oG; w.S = base + oS; w.M1 = base + oM1; w.M2 = base + oM2; w.M3 = base + oM3; w.M4 = base + oM4;
  w.M5 = base + oM5; w.M6 = base + oM6; w.dv = base + oDv;
  w.iv = reinterpret_cast<int*>(base + oIv);
  w.jobs = reinterpret_cast<InvJob*>(base + oJobs);
  w.qjobs = reinterpret_cast<QrJob*>(base + oJobs + 16);
  w.qqjobs = reinterpret_cast<QJob*>(base + oJobs + 32);
  *rx = 0;
  if (resid_out) *resid_out = 0.0;
  if (iters_out) *iters_out = 0;
  std::vector<double> hs(EK_SMAX + 8);
  // ---- S8: right-hand side C = [Uu, dt Fu] [Uv, Fv]^T, compressed
  if (r0 == 0) { cudaFreeAsync(base, s); CU(cudaStreamSynchronize(s)); cleanup(); return FDE_OK; }
  {
    std::vector<QrJob> qj;
    if (own0) {
      if (ru) CK(cudaMemcpyAsync(Qu, Uu, (size_t)nx * ru * 8, cudaMemcpyDeviceToDevice, s));
      if (rf) TK(scale_copy(s, nx, rf, dt, Fu, nx, Qu + (size_t)ru * nx, nx));
      qj.push_back({Qu, nx, r0, tau});
    }
    if (own1) {
      if (ru) CK(cudaMemcpyAsync(Qv, Uv, (size_t)ny * ru * 8, cudaMemcpyDeviceToDevice, s));
      if (rf) CK(cudaMemcpyAsync(Qv + (size_t)ru * ny, Fv, (size_t)ny * rf * 8, cudaMemcpyDeviceToDevice, s));
      qj.push_back({Qv, ny, r0, tau + NRHS_MAX});
    }
    CK(cudaMemcpyAsync(w.qjobs, qj.data(), qj.size() * sizeof(QrJob), cudaMemcpyHostToDevice, s));
    { PROF("k_hqr"); k_hqr<<<(int)qj.size(), QR_THREADS, 0, s>>>(w.qjobs); }
    TK(dn_check("k_hqr"));
    CK(cudaStreamSynchronize(s));                                 // (qj is a host temporary)
  }
  // exchange 1: the R factors (r0 x r0, ld r0)
  const long long S1 = (long long)r0 * r0;
  if (own0) CK(cudaMemcpy2DAsync(xc.slot(0, S1), r0 * 8, Qu, (size_t)nx * 8, r0 * 8, r0, cudaMemcpyDeviceToDevice, s));
  if (own1) CK(cudaMemcpy2DAsync(xc.slot(1, S1), r0 * 8, Qv, (size_t)ny * 8, r0 * 8, r0, cudaMemcpyDeviceToDevice, s));
  TK(xc.run(S1, s));
  // M = R_u R_v^T (r0 x r0); one-sided Jacobi SVD: M Z = W Sigma
  { PROF("k_rrt"); k_rrt<<<(r0 * r0 + 255) / 256, 256, 0, s>>>(r0, r0, r0, xc.got(0, S1), r0, xc.got(1, S1), r0, Ym); }
  TK(dn_check("k_rrt"));
  const int ku = r0, kv = r0;
  { PROF("k_osj_svd"); k_osj_svd<<<1, DN_BIG, dn_smem((long long)ku * kv, kv + 2), s>>>(ku, kv, Ym, ku, Zm, sig, 60); }
  TK(dn_check("k_osj_svd"));
  CK(cudaMemcpyAsync(hs.data(), sig, kv * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  std::vector<int> ord(kv);
  for (int i = 0; i < kv; ++i) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](int a, int c) { return hs[a] > hs[c] || (hs[a] == hs[c] && a < c); });
  std::vector<int> keep;
  double cnorm2 = 0.0, cdrop2 = 0.0;
  for (int i : ord) {
    if (hs[i] > tol * hs[ord[0]] && hs[i] > 0.0) keep.push_back(i);
    else cdrop2 += hs[i] * hs[i];
    cnorm2 += hs[i] * hs[i];
  }
  const int rcr = (int)keep.size();
  if (rcr == 0) {                                    // C = 0  =>  X = 0
    cudaFreeAsync(base, s); CU(cudaStreamSynchronize(s)); cleanup(); return FDE_OK;
  }
  std::vector<double> sigc(rcr);
  for (int i = 0; i < rcr; ++i) sigc[i] = hs[keep[i]];
  CK(cudaMemcpyAsync(sgd, sigc.data(), rcr * sizeof(double), cudaMemcpyHostToDevice, s));
  // P = (M Z)[:, keep] / sigma (left singular vectors), Zk = Z[:, keep]; Cu = Q_u [P; 0], Cv = Q_v [Zk; 0]
  CK(cudaMemcpyAsync(w.iv, keep.data(), rcr * sizeof(int), cudaMemcpyHostToDevice, s));
  { PROF("k_gather_cols"); k_gather_cols<<<(ku * rcr + 255) / 256, 256, 0, s>>>(ku, rcr, Ym, ku, w.iv, sig, w.M5, ku); }
  { PROF("k_gather_cols"); k_gather_cols<<<(kv * rcr + 255) / 256, 256, 0, s>>>(kv, rcr, Zm, kv, w.iv, nullptr, w.M6, kv); }
  TK(dn_check("k_gather_cols"));
  {
    std::vector<QJob> qq;
    if (own0) qq.push_back({Qu, nx, ku, tau, w.M5, ku, rcr, Cu});
    if (own1) qq.push_back({Qv, ny, kv, tau + NRHS_MAX, w.M6, kv, rcr, Cv});
    CK(cudaMemcpyAsync(w.qqjobs, qq.data(), qq.size() * sizeof(QJob), cudaMemcpyHostToDevice, s));
    { PROF("k_hqr_q"); k_hqr_q<<<(int)qq.size(), QR_THREADS, 0, s>>>(w.qqjobs); }
    TK(dn_check("k_hqr_q"));
    CK(cudaStreamSynchronize(s));
  }
  // ---- S9: extended Krylov bases, first block [C_s | orth(A^{-1} C_s)]
  EkSide sx{ops[0], nx, Ux, AUx, 0, 0, 0, 0, 0}, sy{ops[1], ny, Vy, AVy, 0, 0, 0, 0, 0};
  EkSide* sides[2] = {&sx, &sy};
  const double dtol = 1e-11;
  // ---- rational Krylov mode: poles, and one round of shifted solves + orthogonalisation
  std::vector<double> poles;
  int rk_round = 0;
  if (rk) {
    const int K = rk->npole, R = rk->rounds;
    poles.assign((size_t)2 * K * R, 0.0);
    if (rk->poles) std::copy(rk->poles, rk->poles + 2 * K * R, poles.begin());
    else {
      // spectral range of A_d (real parts in [1/2, 1/2 + c_d 2^alpha_d (max|d+| + max|d-|)])
      double hm[4] = {0, 0, 0, 0};
      { PROF("k_absmax2"); k_absmax2<<<1, 1024, 0, s>>>(nx, d1p, d1m, w.dv + 20); }
      { PROF("k_absmax2"); k_absmax2<<<1, 1024, 0, s>>>(ny, d2p, d2m, w.dv + 22); }
      TK(dn_check("k_absmax2"));
      CK(cudaMemcpyAsync(hm, w.dv + 20, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      const double hi[2] = {0.5 + dt / std::pow(hx, alpha1) * std::exp2(alpha1) * (hm[0] + hm[1]),
                            0.5 + dt / std::pow(hy, alpha2) * std::exp2(alpha2) * (hm[2] + hm[3])};
      const double phi[6] = {0.5, 0.0, 1.0, 0.25, 0.75, 0.125};
      for (int d = 0; d < 2; ++d)
        for (int r = 0; r < R; ++r)
          for (int j = 0; j < K; ++j) {
            const double e = (j + phi[r % 6]) / K, lo = 0.5, h_ = hi[1 - d];   // the other side's range
            poles[((size_t)d * R + r) * K + j] = lo * std::pow(h_ / lo, e);
          }
    }
  }
  auto rk_grow = [&](int r) -> int {
    const int K = rk->npole, R = rk->rounds, pw = rk_pw, pr = rk->pr;
    for (int d = 0; d < 2; ++d) {
      EkSide* e = sides[d];
      const double* Cs = d == 0 ? Cu : Cv;
      const long long blk = (long long)e->n * rcr;
      double* Ws = base + oWs;
      for (int j = pr; j < K; j += pw) {                // this rank's poles of the round
        const size_t idx = ((size_t)d * R + r) * K + j;
        const double pole = poles[idx];
        TRY(ensure_op_2d(&rk->shifted[idx], e->n, d == 0 ? alpha1 : alpha2, d == 0 ? hx : hy, dt,
                         d == 0 ? d1p : d2p, d == 0 ? d1m : d2m, tol, leaf, flags, s, 0.5 + pole));
        TRY(hodlr_solve_cols(rk->shifted[idx], Cs, Ws + (size_t)(j / pw) * blk, rcr, s));
      }
      const double* Wall = Ws;
      const long long cnt = (long long)((K + pw - 1) / pw) * blk;
      if (pw > 1) {                                     // blocks of every rank (rank-major)
        double* Wr = base + oWr;
        if (rk->gather(rk->ctx, Ws, Wr, cnt, s) != 0) return set_err(FDE_ECUDA, "pole exchange callback failed");
        Wall = Wr;
      }
      for (int j = 0; j < K; ++j) {                     // orthogonalise in pole order (every rank)
        const double* Wj = Wall + (size_t)(j % pw) * cnt + (size_t)(j / pw) * blk;
        CK(cudaMemcpyAsync(Wt, Wj, (size_t)blk * 8, cudaMemcpyDeviceToDevice, s));
        int nb = 0;
        TRY(orth_append(s, w, e->n, Wt, rcr, e->U, e->s, EK_SMAX, dtol, &nb));
        if (nb) TRY(hodlr_mv_cols(e->H, e->U + (size_t)e->s * e->n, e->AU + (size_t)e->s * e->n, nb, s));
        e->s += nb;
      }
    }
    return FDE_OK;
  };
  for (int d = 0; d < 2; ++d) {
    if (!xc.own(d)) continue;
    if (rk) {                                           // first block C_s; then round 0 of the poles
      EkSide* e = sides[d];
      const double* Cs = d == 0 ? Cu : Cv;
      CK(cudaMemcpyAsync(e->U, Cs, (size_t)e->n * rcr * 8, cudaMemcpyDeviceToDevice, s));
      TK(hodlr_mv_cols(e->H, e->U, e->AU, rcr, s));
      e->s = rcr;
      continue;
    }
    EkSide* e = sides[d];
    const double* Cs = d == 0 ? Cu : Cv;
    CK(cudaMemcpyAsync(e->U, Cs, (size_t)e->n * rcr * 8, cudaMemcpyDeviceToDevice, s));   // orthonormal
    TK(hodlr_mv_cols(e->H, e->U, e->AU, rcr, s));
    e->p0 = 0; e->np = rcr; e->s = rcr;
    TK(hodlr_solve_cols(e->H, Cs, Wt, rcr, s));
    int nn = 0;
    TK(orth_append(s, w, e->n, Wt, rcr, e->U, e->s, EK_SMAX, dtol, &nn));
    if (nn) TK(hodlr_mv_cols(e->H, e->U + (size_t)e->s * e->n, e->AU + (size_t)e->s * e->n, nn, s));
    e->n0 = e->s; e->nn = nn; e->s += nn;
  }
  // basis sizes of both sides (exchange of one value per side)
  std::vector<double> hsz(2);
  auto sizes = [&](int* sa_out, int* sb_out) -> int {
    hsz[0] = sx.s; hsz[1] = sy.s;
    for (int d = 0; d < 2; ++d)
      if (xc.own(d)) CK(cudaMemcpyAsync(xc.slot(d, 1), &hsz[d], sizeof(double), cudaMemcpyHostToDevice, s));
    TRY(xc.run(1, s));
    double v0 = 0, v1 = 0;
    CK(cudaMemcpyAsync(&v0, xc.got(0, 1), sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&v1, xc.got(1, 1), sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *sa_out = (int)v0; *sb_out = (int)v1;
    return FDE_OK;
  };
  if (rk) { TK(rk_grow(0)); rk_round = 1; }
  int sa = 0, sbb = 0;
  TK(sizes(&sa, &sbb));
  // ---- S10: projected solves until the residual is below ek_tol (relative to ||C||_F)
  int it = 0, sit = 0;
  double rel = 1.0, prev_rel = 1e300;
  bool conv = false;
  int solved_x = -1, solved_y = -1;
  // residual splitting at a projected solution Y0 (sa x sb, ld sa): ||Ra Y0||^2 on the owner of
  // side 0, ||Rb Y0^T||^2 on the owner of side 1 (exchanged), ||P||^2 on every rank
  auto resid_at = [&](const double* Y0, double* out3) -> int {
    if (own0) {
      CK(cudaMemcpyAsync(Wt, AUx, (size_t)nx * sa * 8, cudaMemcpyDeviceToDevice, s));
      TRY(ts_nn(s, nx, sa, sa, -1.0, Ux, nx, Lc, sa, 1.0, Wt, nx));         // Ra = A1 U - U A~
      TRY(ts_nn(s, nx, sbb, sa, 1.0, Wt, nx, Y0, sa, 0.0, w.M2, nx));
      TRY(sumsq_dev(s, nx, sbb, w.M2, nx, xc.slot(0, 1)));
    }
    if (own1) {
      CK(cudaMemcpyAsync(Wt, AVy, (size_t)ny * sbb * 8, cudaMemcpyDeviceToDevice, s));
      TRY(ts_nn(s, ny, sbb, sbb, -1.0, Vy, ny, Rc, sbb, 1.0, Wt, ny));      // Rb = A2 V - V B^
      TRY(transpose(s, sa, sbb, Y0, sa, Zm, sbb));
      TRY(ts_nn(s, ny, sa, sbb, 1.0, Wt, ny, Zm, sbb, 0.0, w.M2, ny));
      TRY(sumsq_dev(s, ny, sa, w.M2, ny, xc.slot(1, 1)));
    }
    TRY(xc.run(1, s));
    CK(cudaMemcpyAsync(w.M1, Cm, (size_t)sa * sbb * 8, cudaMemcpyDeviceToDevice, s));   // P = A~ Y + Y B~ - C~
    TRY(ts_nn(s, sa, sbb, sa, 1.0, Lc, sa, Y0, sa, -1.0, w.M1, sa));
    TRY(ts_nn(s, sa, sbb, sbb, 1.0, Y0, sa, Bm, sbb, 1.0, w.M1, sa));
    TRY(sumsq_dev(s, sa, sbb, w.M1, sa, w.dv + 10));
    CK(cudaMemcpyAsync(out3, xc.got(0, 1), sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(out3 + 1, xc.got(1, 1), sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(out3 + 2, w.dv + 10, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return FDE_OK;
  };
  auto solve_and_check = [&]() -> int {
    // exchange 2: side 0 -> A~ = U^T A1 U and U^T Cu; side 1 -> B^ = V^T A2 V and V^T Cv
    if (own0) {
      double* sl = xc.slot(0, SS);
      TRY(ts_tn(s, w, sa, sa, nx, 1.0, Ux, nx, AUx, nx, 0.0, sl, sa));
      TRY(ts_tn(s, w, sa, rcr, nx, 1.0, Ux, nx, Cu, nx, 0.0, sl + sm2, sa));
    }
    if (own1) {
      double* sl = xc.slot(1, SS);
      TRY(ts_tn(s, w, sbb, sbb, ny, 1.0, Vy, ny, AVy, ny, 0.0, sl, sbb));
      TRY(ts_tn(s, w, sbb, rcr, ny, 1.0, Vy, ny, Cv, ny, 0.0, sl + sm2, sbb));
    }
    TRY(xc.run(SS, s));
    const double* g0 = xc.got(0, SS);
    const double* g1 = xc.got(1, SS);
    CK(cudaMemcpyAsync(Am, g0, (size_t)sa * sa * 8, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(Lc, g0, (size_t)sa * sa * 8, cudaMemcpyDeviceToDevice, s));      // keep A~
    CK(cudaMemcpyAsync(Rc, g1, (size_t)sbb * sbb * 8, cudaMemcpyDeviceToDevice, s));    // keep B^
    TRY(transpose(s, sbb, sbb, g1, sbb, Bm, sbb));                                       // B~ = B^T
    // C~ = (U^T Cu) diag(sig) (V^T Cv)^T
    TRY(transpose(s, sbb, rcr, g1 + sm2, sbb, w.M2, rcr));
    { PROF("k_scale_rows"); k_scale_rows<<<(rcr * sbb + 255) / 256, 256, 0, s>>>(rcr, sbb, w.M2, rcr, sgd, w.S); }
    TRY(dn_check("k_scale_rows"));
    TRY(ts_nn(s, sa, sbb, rcr, 1.0, g0 + sm2, sa, w.S, rcr, 0.0, Cm, sa));
    CK(cudaMemcpyAsync(Ym, Cm, (size_t)sa * sbb * 8, cudaMemcpyDeviceToDevice, s));
    double* Bw = w.G;                                  // the sign iteration destroys its B
    CK(cudaMemcpyAsync(Bw, Bm, (size_t)sbb * sbb * 8, cudaMemcpyDeviceToDevice, s));
    TRY(proj_sylvester(s, w, sa, sbb, Am, Bw, Ym, st, &sit));
    double r3[3];
    TRY(resid_at(Ym, r3));
    rel = std::sqrt((r3[0] + r3[1] + r3[2] + cdrop2) / cnorm2);
    if (fde_dbg_env("FDE_DEBUG2D"))
      fprintf(stderr, "fde2d it %d: sa %d sb %d rc %d sign-its %d rel %.3e (ra2 %.3e rb2 %.3e rp2 %.3e drop2 %.3e c2 %.3e)\n",
              it, sa, sbb, rcr, sit, rel, r3[0], r3[1], r3[2], cdrop2, cnorm2);
    solved_x = sa; solved_y = sbb;
    return FDE_OK;
  };
  bool solve_now = true;
  for (it = 1; it <= ek_maxit; ++it) {
    if (solve_now || it == ek_maxit) {
      TK(solve_and_check());
      // converged: below ek_tol, or stagnated at the rounding floor of the residual evaluation
      // (reading R19: ||Rb|| carries eps ||A2 V||; cfg5's floor is ~1.2e-11 relative) within 10x
      if (rel <= ek_tol || (rel <= 10.0 * ek_tol && rel >= 0.9 * prev_rel)) { conv = true; break; }
      prev_rel = rel;
      // far from converged: grow twice before the next projected solve
      solve_now = rel <= 1e3 * ek_tol;
    } else {
      solve_now = true;
    }
    if (it == ek_maxit) break;
    const int s0x = sa, s0y = sbb;
    if (rk) {
      if (rk_round >= rk->rounds) break;
      TK(rk_grow(rk_round));
      ++rk_round;
      solve_now = true;
    } else {
      if (own0) TK(ek_grow(s, w, sx, Wt, dtol));
      if (own1) TK(ek_grow(s, w, sy, Wt, dtol));
    }
    TK(sizes(&sa, &sbb));
    if (sa == s0x && sbb == s0y) break;              // no new directions (EK_SMAX or exhausted)
  }
  if (!conv && (solved_x != sa || solved_y != sbb)) {   // Y must belong to the final bases
    TK(solve_and_check());
    conv = rel <= 10.0 * ek_tol;
  }
  if (iters_out) *iters_out = rk ? rk_round : std::min(it, ek_maxit);
  // ---- truncation: X = U_s Y V_s^T with Y = sum sigma_i u_i w_i^T, keep sigma > tol sigma_1.
  // Rank-revealing QR of Y first (Q_k^T Y, k ~ final rank), then the one-sided Jacobi SVD of
  // (Q_k^T Y)^T (sbb x k): right singular vectors W and sigma; the left factor is Y W.
  int kq = 0;
  {
    CK(cudaMemcpyAsync(w.M4, Ym, (size_t)sa * sbb * 8, cudaMemcpyDeviceToDevice, s));
    { PROF("k_qrcp_rows"); k_qrcp_rows<<<1, DN_BIG, 0, s>>>(sa, sbb, w.M4, 1e-2 * tol, w.M3, w.iv); }
    TK(dn_check("k_qrcp_rows"));
    CK(cudaMemcpyAsync(&kq, w.iv, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  if (kq > 0) {
    { PROF("k_osj_svd"); k_osj_svd<<<1, DN_BIG, dn_smem((long long)sbb * kq, kq + 2), s>>>(sbb, kq, w.M3, sbb, Zm, sig, 60); }
    TK(dn_check("k_osj_svd"));
    CK(cudaMemcpyAsync(hs.data(), sig, kq * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  ord.assign(kq, 0);
  for (int i = 0; i < kq; ++i) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](int a, int c) { return hs[a] > hs[c] || (hs[a] == hs[c] && a < c); });
  keep.clear();
  for (int i : ord) if (hs[i] > tol * hs[ord[0]] && hs[i] > 0.0) keep.push_back(i);
  const int rkt = (int)keep.size();
  if (rkt > rmax) { fail(FDE_OK); return set_err(FDE_EDIM, "solution rank %d exceeds rmax=%d", rkt, rmax); }
  double rel_t = rel;
  if (rkt > 0) {
    CK(cudaMemcpyAsync(w.iv, keep.data(), rkt * sizeof(int), cudaMemcpyHostToDevice, s));
    // right vectors M6 = (AT Z)[:, keep] / sigma, left factor M5 = Y M6 (= U_k Sigma_k)
    { PROF("k_gather_cols"); k_gather_cols<<<(sbb * rkt + 255) / 256, 256, 0, s>>>(sbb, rkt, w.M3, sbb, w.iv, sig, w.M6, sbb); }
    TK(dn_check("k_gather_cols"));
    TK(ts_nn(s, sa, rkt, sbb, 1.0, Ym, sa, w.M6, sbb, 0.0, w.M5, sa));
    // the returned X's residual: the splitting at Yt = M5 M6^T (plus the dropped part of C)
    double* Yt = w.M4;
    TK(transpose(s, sbb, rkt, w.M6, sbb, w.S, rkt));
    TK(ts_nn(s, sa, sbb, rkt, 1.0, w.M5, sa, w.S, rkt, 0.0, Yt, sa));
    double r3[3];
    TK(resid_at(Yt, r3));
    rel_t = std::sqrt((r3[0] + r3[1] + r3[2] + cdrop2) / cnorm2);
    if (own0) TK(ts_nn(s, nx, rkt, sa, 1.0, Ux, nx, w.M5, sa, 0.0, Xu, nx));
    if (own1) TK(ts_nn(s, ny, rkt, sbb, 1.0, Vy, ny, w.M6, sbb, 0.0, Xv, ny));
  }
  if (resid_out) *resid_out = rel_t;
  *rx = rkt;
  // device status of the owned operators; exchanged so that both ranks report a failure
  CK(cudaStreamSynchronize(s));
  DevStatus dd[2] = {{0, 0}, {0, 0}};
  for (int d = 0; d < 2; ++d) if (xc.own(d)) TK(read_status(ops[d], &dd[d]));
  if (rk)
    for (int d = 0; d < 2; ++d)
      for (int i = 0; i < rk->npole * rk->rounds && dd[d].code == FDE_OK; ++i) {
        fde_hodlr* Hs = rk->shifted[(size_t)d * rk->npole * rk->rounds + i];
        if (Hs) TK(read_status(Hs, &dd[d]));
      }
  std::vector<double> hst(2);
  for (int d = 0; d < 2; ++d) {
    hst[d] = (double)dd[d].code * 4294967296.0 + (double)(unsigned)dd[d].where;
    if (xc.own(d)) CK(cudaMemcpyAsync(xc.slot(d, 1), &hst[d], sizeof(double), cudaMemcpyHostToDevice, s));
  }
  TK(xc.run(1, s));
  CK(cudaMemcpyAsync(&hst[0], xc.got(0, 1), sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&hst[1], xc.got(1, 1), sizeof(double), cudaMemcpyDeviceToHost, s));
  cudaFreeAsync(base, s);
  CU(cudaStreamSynchronize(s));
  cleanup();
  for (int d = 0; d < 2; ++d) {
    const int code = (int)(hst[d] / 4294967296.0);
    if (code != FDE_OK)
      return set_err(code, "device status %d in fde2d_step (operator %d, index %d)", code, d + 1,
                     (int)(unsigned)(hst[d] - (double)code * 4294967296.0));
  }
  if (!conv) return set_err(FDE_ENOCONV, "extended Krylov: relative residual %.3e > ek_tol %.1e after %d iterations",
                            rel, ek_tol, ek_maxit);
#undef CK
#undef TK
  return FDE_OK;
}

extern "C" int fde2d_step(int nx, int ny, double alpha1, double alpha2, double hx, double hy, double dt,
                          const double* d1p, const double* d1m, const double* d2p, const double* d2m,
                          const double* Fu, const double* Fv, int rf, const double* Uu, const double* Uv,
                          int ru, double* Xu, double* Xv, int rmax, int* rx, double tol, double ek_tol,
                          int ek_maxit, int leaf, fde_hodlr_t* cache, double* resid_out, int* iters_out,
                          unsigned flags, void* stream) {
  g_last_error.clear();
  Xchg xc{1, 0, nullptr, nullptr, nullptr, nullptr};
  return step_2d_impl(xc, nx, ny, alpha1, alpha2, hx, hy, dt, d1p, d1m, d2p, d2m, Fu, Fv, rf, Uu, Uv, ru, Xu, Xv,
                      rmax, rx, tol, ek_tol, ek_maxit, leaf, cache, resid_out, iters_out, flags, (cudaStream_t)stream);
}

extern "C" int fde2d_step_split(int world, int rank, fde_allgather_fn gather, void* ctx, int nx, int ny,
                                double alpha1, double alpha2, double hx, double hy, double dt,
                                const double* d1p, const double* d1m, const double* d2p, const double* d2m,
                                const double* Fu, const double* Fv, int rf, const double* Uu, const double* Uv,
                                int ru, double* Xu, double* Xv, int rmax, int* rx, double tol, double ek_tol,
                                int ek_maxit, int leaf, fde_hodlr_t* cache, double* resid_out, int* iters_out,
                                unsigned flags, void* stream) {
  g_last_error.clear();
  if (world != 1 && world != 2) return set_err(FDE_EDOMAIN, "world=%d: the x/y split runs on 1 or 2 ranks", world);
  if (rank < 0 || rank >= world) return set_err(FDE_EDOMAIN, "rank=%d outside [0, %d)", rank, world);
  if (world == 2 && !gather) return set_err(FDE_EDOMAIN, "world=2 needs an all-gather callback");
  // (world = 1 with a callback: the exchanges still go through it -- a loopback test of the path)
  Xchg xc{world, rank, gather, ctx, nullptr, nullptr};
  return step_2d_impl(xc, nx, ny, alpha1, alpha2, hx, hy, dt, d1p, d1m, d2p, d2m, Fu, Fv, rf, Uu, Uv, ru, Xu, Xv,
                      rmax, rx, tol, ek_tol, ek_maxit, leaf, cache, resid_out, iters_out, flags, (cudaStream_t)stream);
}

extern "C" int fde2d_step_rk(int pw, int pr, fde_allgather_fn gather, void* ctx, int nx, int ny, double alpha1,
                             double alpha2, double hx, double hy, double dt, const double* d1p, const double* d1m,
                             const double* d2p, const double* d2m, const double* Fu, const double* Fv, int rf,
                             const double* Uu, const double* Uv, int ru, double* Xu, double* Xv, int rmax, int* rx,
                             double tol, double rk_tol, int npole, int rounds, const double* poles, int leaf,
                             fde_hodlr_t* cache, double* resid_out, int* rounds_out, unsigned flags, void* stream) {
  g_last_error.clear();
  if (npole < 1 || npole > 16 || rounds < 1 || rounds > 6)
    return set_err(FDE_EDOMAIN, "npole=%d (1..16), rounds=%d (1..6)", npole, rounds);
  if (pw < 1 || pr < 0 || pr >= pw) return set_err(FDE_EDOMAIN, "pole sharding pw=%d pr=%d", pw, pr);
  if (pw > 1 && !gather) return set_err(FDE_EDOMAIN, "pw > 1 needs an all-gather callback");
  if (!cache) return set_err(FDE_EDOMAIN, "cache is required (2 + 2 npole rounds handles)");
  if (poles)
    for (int i = 0; i < 2 * npole * rounds; ++i)
      if (!(poles[i] > 0.0) || !std::isfinite(poles[i])) return set_err(FDE_EDOMAIN, "poles[%d]=%g must be > 0", i, poles[i]);
  RkSpec rk{npole, rounds, poles, pw, pr, gather, ctx, reinterpret_cast<fde_hodlr**>(cache) + 2};
  Xchg xc{1, 0, nullptr, nullptr, nullptr, nullptr};
  return step_2d_impl(xc, nx, ny, alpha1, alpha2, hx, hy, dt, d1p, d1m, d2p, d2m, Fu, Fv, rf, Uu, Uv, ru, Xu, Xv,
                      rmax, rx, tol, rk_tol, rounds + 1, leaf, cache, resid_out, rounds_out, flags,
                      (cudaStream_t)stream, &rk);
}
