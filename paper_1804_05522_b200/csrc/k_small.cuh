// k_small.cuh -- dense FP64 kernels of the 2D Sylvester step (S8-S10, fde2d.cuh), round 2:
//   * k_gemm_tn / k_gemm_nn: tall-skinny products of the Krylov bases on the FP64 tensor cores
//     (DMMA m8n8k4), split-K partials reduced in a fixed order (deterministic);
//   * k_hqr / k_hqr_q: Householder QR of a tall n x k factor (one CTA per factor, reflectors kept
//     in place, LAPACK dgeqr2 convention) and the product Q [P; 0] -- the right-hand-side
//     compression "QR of the factors + small SVD" needs an orthogonalisation that
//     resolves directions down to eps of the column norms, which a Gram matrix cannot;
//   * k_gj_inv_cl<CL>: blocked Gauss-Jordan inverse with partial pivoting of an s x s matrix held
//     in the shared memory of a CL-CTA thread-block cluster (column slabs; per block of 8 pivots
//     the owner's panel goes to every CTA through distributed shared memory, then a rank-8 DMMA
//     update): the inverses of the Newton sign iteration for the projected Sylvester equation
//     (P:1541-1547);
//   * k_pchol_orth: diagonally pivoted Cholesky of a small Gram matrix with deflation, giving
//     S = P R^{-1} so that W S has orthonormal columns (Cholesky-QR with column selection; used
//     twice per block by the extended Krylov orthogonalisation).
// Column-major throughout; every reduction has a fixed order.
#pragma once
#include <cooperative_groups.h>
#include "fde_common.cuh"
#include "fde_dmma.cuh"

#define SG_THREADS 256
#define SG_TILE 32                // k_gemm_tn output tile (32 x 32), K chunk 32
#define SG_LD 36                  // = 4 mod 16: conflict-free DMMA fragments

// P[z] (m x n, ld m) = A[kb:ke, :]^T B[kb:ke, :]   (A: K x m, ld lda; B: K x n, ld ldb)
// or, with P == nullptr, C = alpha A^T B + beta C directly (one K chunk).
__global__ void __launch_bounds__(SG_THREADS)
k_gemm_tn(int m, int n, int K, int kchunk, const double* __restrict__ A, int lda,
          const double* __restrict__ B, int ldb, double* __restrict__ P, double alpha, double beta,
          double* __restrict__ C, int ldc) {
  __shared__ double As[SG_TILE * SG_LD], Bs[SG_TILE * SG_LD];
  const int i0 = blockIdx.x * SG_TILE, j0 = blockIdx.y * SG_TILE;
  const int kb = blockIdx.z * kchunk, ke = min(K, kb + kchunk);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31, gid = lane >> 2, tig = lane & 3;
  const int mt = warp & 3, nt = 2 * (warp >> 2);
  double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int k0 = kb; k0 < ke; k0 += SG_TILE) {
    for (int e = t; e < SG_TILE * SG_TILE; e += SG_THREADS) {
      const int kk = e & 31, c = e >> 5, k = k0 + kk;
      As[c * SG_LD + kk] = (k < ke && i0 + c < m) ? A[(long long)(i0 + c) * lda + k] : 0.0;
      Bs[c * SG_LD + kk] = (k < ke && j0 + c < n) ? B[(long long)(j0 + c) * ldb + k] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k4 = 0; k4 < SG_TILE; k4 += 4) {
      const double a = As[(8 * mt + gid) * SG_LD + k4 + tig];
      dmma884(d[0][0], d[0][1], a, Bs[(8 * nt + gid) * SG_LD + k4 + tig]);
      dmma884(d[1][0], d[1][1], a, Bs[(8 * nt + 8 + gid) * SG_LD + k4 + tig]);
    }
    __syncthreads();
  }
  const int i = i0 + 8 * mt + gid;
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = j0 + 8 * (nt + u) + 2 * tig + h;
      if (i < m && j < n) {
        if (P) P[(long long)blockIdx.z * m * n + (long long)j * m + i] = d[u][h];
        else {
          double* c = C + (long long)j * ldc + i;
          *c = alpha * d[u][h] + (beta == 0.0 ? 0.0 : beta * *c);
        }
      }
    }
}

__global__ void k_sum_partials(int m, int n, int nz, const double* __restrict__ P, double alpha, double beta,
                               double* __restrict__ C, int ldc) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)m * n) return;
  double s = 0.0;
  for (int z = 0; z < nz; ++z) s += P[(long long)z * m * n + e];
  const int i = (int)(e % m), j = (int)(e / m);
  double* c = C + (long long)j * ldc + i;
  *c = alpha * s + (beta == 0.0 ? 0.0 : beta * *c);
}

// C (M x n) = alpha A B + beta C   (A: M x K, ld lda; B: K x n, ld ldb).  CTA tile 64 x 32,
// K chunks of 16; warp w: m-tile w, 4 n-tiles.
#define NN_LDA 68                 // = 4 mod 16
#define NN_LDB 20
__global__ void __launch_bounds__(SG_THREADS)
k_gemm_nn(int M, int n, int K, double alpha, const double* __restrict__ A, int lda,
          const double* __restrict__ B, int ldb, double beta, double* __restrict__ C, int ldc) {
  __shared__ double As[16 * NN_LDA], Bs[32 * NN_LDB];
  const int i0 = blockIdx.x * 64, j0 = blockIdx.y * 32;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31, gid = lane >> 2, tig = lane & 3;
  double d[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int e = t; e < 16 * 64; e += SG_THREADS) {
      const int i = e & 63, kk = e >> 6;
      As[kk * NN_LDA + i] = (i0 + i < M && k0 + kk < K) ? A[(long long)(k0 + kk) * lda + i0 + i] : 0.0;
    }
    for (int e = t; e < 16 * 32; e += SG_THREADS) {
      const int kk = e & 15, j = e >> 4;
      Bs[j * NN_LDB + kk] = (j0 + j < n && k0 + kk < K) ? B[(long long)(j0 + j) * ldb + k0 + kk] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k4 = 0; k4 < 16; k4 += 4) {
      const double a = As[(k4 + tig) * NN_LDA + 8 * warp + gid];
#pragma unroll
      for (int u = 0; u < 4; ++u) dmma884(d[u][0], d[u][1], a, Bs[(8 * u + gid) * NN_LDB + k4 + tig]);
    }
    __syncthreads();
  }
  const int i = i0 + 8 * warp + gid;
  if (i >= M) return;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = j0 + 8 * u + 2 * tig + h;
      if (j < n) {
        double* c = C + (long long)j * ldc + i;
        *c = alpha * d[u][h] + (beta == 0.0 ? 0.0 : beta * *c);
      }
    }
}

// ---------------------------------------------------------------------------------------
// Householder QR (one CTA of 1024 threads per job): W (n x k, ld n) is overwritten with R in
// its upper triangle and the reflectors below the diagonal (v_j[0] = 1 implicit), tau[k].
//   H_j = I - tau_j v_j v_j^T,  Q = H_0 H_1 .. H_{k-1},  W = Q R   (LAPACK dgeqr2)
struct QrJob { double* W; int n, k; double* tau; };
#define QR_THREADS 1024

__device__ __forceinline__ double qr_block_sum(double v, double* red) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = red[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[32] = v;
  }
  __syncthreads();
  return red[32];
}

__global__ void __launch_bounds__(QR_THREADS)
k_hqr(const QrJob* __restrict__ jobs) {
  const QrJob jb = jobs[blockIdx.x];
  __shared__ double red[33];
  __shared__ double s_tau, s_beta, s_v0inv;
  __shared__ double dots[64];
  const int n = jb.n, k = jb.k, t = threadIdx.x, warp = t >> 5, lane = t & 31;
  double* W = jb.W;
  for (int j = 0; j < k && j < n; ++j) {
    double* wj = W + (long long)j * n;
    double s = 0.0;
    for (int i = j + 1 + t; i < n; i += QR_THREADS) s = fma(wj[i], wj[i], s);
    s = qr_block_sum(s, red);
    if (t == 0) {
      const double x0 = wj[j];
      if (s == 0.0) { s_tau = 0.0; s_beta = x0; s_v0inv = 0.0; }
      else {
        const double nrm = sqrt(fma(x0, x0, s));
        const double beta = x0 >= 0.0 ? -nrm : nrm;
        s_tau = (beta - x0) / beta;
        s_v0inv = 1.0 / (x0 - beta);
        s_beta = beta;
      }
    }
    __syncthreads();
    const double tau = s_tau, v0i = s_v0inv;
    if (tau != 0.0)
      for (int i = j + 1 + t; i < n; i += QR_THREADS) wj[i] *= v0i;
    __syncthreads();
    if (t == 0) wj[j] = s_beta;
    if (tau != 0.0) {
      // dots[c] = v^T W[j:, c] for c > j (warp per column, fixed-order lane sums)
      for (int c = j + 1 + warp; c < k; c += QR_THREADS / 32) {
        const double* wc = W + (long long)c * n;
        double a = lane == 0 ? wc[j] : 0.0;
        for (int i = j + 1 + lane; i < n; i += 32) a = fma(wj[i], wc[i], a);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) dots[c - j - 1] = a * tau;
      }
      __syncthreads();
      for (int c = j + 1 + warp; c < k; c += QR_THREADS / 32) {
        double* wc = W + (long long)c * n;
        const double f = dots[c - j - 1];
        if (lane == 0) wc[j] -= f;
        for (int i = j + 1 + lane; i < n; i += 32) wc[i] = fma(-f, wj[i], wc[i]);
      }
    }
    __syncthreads();
    if (t == 0) jb.tau[j] = tau;
  }
}

// Z (n x c, ld n) = Q [P; 0],  Q from k_hqr (reflectors of W, tau), P (k x c, ld ldp).
struct QJob { const double* W; int n, k; const double* tau; const double* P; int ldp, c; double* Z; };
__global__ void __launch_bounds__(QR_THREADS)
k_hqr_q(const QJob* __restrict__ jobs) {
  const QJob jb = jobs[blockIdx.x];
  __shared__ double dots[64];
  const int n = jb.n, k = jb.k, t = threadIdx.x, warp = t >> 5, lane = t & 31;
  for (long long e = t; e < (long long)n * jb.c; e += QR_THREADS) {
    const int i = (int)(e % n), col = (int)(e / n);
    jb.Z[(long long)col * n + i] = i < k ? jb.P[(long long)col * jb.ldp + i] : 0.0;
  }
  __syncthreads();
  for (int j = min(k, n) - 1; j >= 0; --j) {
    const double tau = jb.tau[j];
    if (tau == 0.0) continue;
    const double* v = jb.W + (long long)j * n;
    for (int col = warp; col < jb.c; col += QR_THREADS / 32) {
      const double* z = jb.Z + (long long)col * n;
      double a = lane == 0 ? z[j] : 0.0;
      for (int i = j + 1 + lane; i < n; i += 32) a = fma(v[i], z[i], a);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (lane == 0) dots[col] = a * tau;
    }
    __syncthreads();
    for (int col = warp; col < jb.c; col += QR_THREADS / 32) {
      double* z = jb.Z + (long long)col * n;
      const double f = dots[col];
      if (lane == 0) z[j] -= f;
      for (int i = j + 1 + lane; i < n; i += 32) z[i] = fma(-f, v[i], z[i]);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------
// Blocked Gauss-Jordan inverse with partial pivoting on a CL-CTA cluster (one cluster per job).
// CTA r of the cluster holds the column slab [r*cw, min(s, (r+1)*cw)) of A in shared memory
// (column-major, ld GJ_LD(s)); cw is a multiple of GJ_NB so a block of GJ_NB pivot columns lives
// in one CTA.  Per block K = [k0, k0+nb):
//   1. the owner CTA runs nb Gauss-Jordan pivots on its panel A[:, K] alone (pivot = largest
//      |a_ik|, i >= k, smallest index on ties; row swap and elimination inside the panel), which
//      leaves the panel's final in-place values  [A11^{-1} ; -A21 A11^{-1}]  (rows K / the others,
//      rows permuted);
//   2. it writes the panel and the nb pivot rows into every CTA's shared memory (distributed
//      shared memory); one cluster barrier;
//   3. every CTA updates its other columns j:  swap rows (k, p_k) for k in K, X = rows K of
//      column j, rows K <- 0, column j += Panel X  -- a rank-nb update on the FP64 tensor cores.
// The row interchanges are undone at write-out as a column permutation.  In-place Gauss-Jordan:
// the same arithmetic as the unblocked sweep, reassociated by blocks.
struct InvJob { double* A; int s; int lda; };
#define GJ_THREADS 512
#define GJ_NB 8
__host__ __device__ __forceinline__ int gj_ld(int s) { return round_up(s, 16) + 4; }   // = 4 mod 16
__host__ __device__ __forceinline__ int gj_cw(int s, int cl) { return round_up((s + cl - 1) / cl, GJ_NB); }
__host__ __forceinline__ size_t gj_smem(int s, int cl) {
  const int ld = gj_ld(s), cw = gj_cw(s, cl);
  return ((size_t)cw * ld + (size_t)GJ_NB * ld + (size_t)GJ_NB * cw) * 8 + (size_t)(2 * s + 2 * GJ_NB) * 4;
}

template <int CL>
__global__ void __launch_bounds__(GJ_THREADS)
k_gj_inv_cl(const InvJob* __restrict__ jobs, DevStatus* st) {
  namespace cg = cooperative_groups;
  extern __shared__ double gsm[];
  const int job = blockIdx.x / CL;
  const unsigned rank = CL > 1 ? cg::this_cluster().block_rank() : 0;
  const InvJob jb = jobs[job];
  const int s = jb.s, ld = gj_ld(s), cw = gj_cw(s, CL);
  const int c0 = (int)rank * cw, c1 = min(s, c0 + cw), nc = max(0, c1 - c0);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31, nw = GJ_THREADS / 32, gid = lane >> 2, tig = lane & 3;
  double* A = gsm;                                    // [cw][ld] own slab
  double* Pn = A + (long long)cw * ld;                // [GJ_NB][ld] the current block's panel
  double* Xs = Pn + (long long)GJ_NB * ld;            // [cw][GJ_NB] rows K of the own columns
  int* pivs = reinterpret_cast<int*>(Xs + (long long)GJ_NB * cw);   // [s] pivot rows
  int* perm = pivs + s;                               // [s] write-out permutation
  int* bpiv = perm + s;                               // [GJ_NB] the current block's pivots
  __shared__ int s_bad, s_p;
  __shared__ double s_rp;
  if (t == 0) s_bad = 0;
  for (long long e = t; e < (long long)nc * s; e += GJ_THREADS) {
    const int i = (int)(e % s), c = (int)(e / s);
    A[(long long)c * ld + i] = jb.A[(long long)(c0 + c) * jb.lda + i];
  }
  for (long long e = t; e < (long long)cw * ld; e += GJ_THREADS) {   // padding rows / columns: 0
    const int i = (int)(e % ld), c = (int)(e / ld);
    if (i >= s || c >= nc) A[e] = 0.0;
  }
  for (int e = t; e < GJ_NB * ld; e += GJ_THREADS) Pn[e] = 0.0;     // (0 x 0 in the rank-nb update)
  __syncthreads();
  for (int k0 = 0; k0 < s; k0 += GJ_NB) {
    const int nb = min(GJ_NB, s - k0);
    const bool owner = k0 >= c0 && k0 < c1;
    if (owner) {
      double* P = A + (long long)(k0 - c0) * ld;      // the panel, in place
      for (int kk = 0; kk < nb; ++kk) {
        const int k = k0 + kk;
        double* pc = P + (long long)kk * ld;
        if (warp == 0) {
          double bv = -1.0; int bi = s;
          for (int i = k + lane; i < s; i += 32) {
            const double v = fabs(pc[i]);
            if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
          }
          const int p = bi < s ? bi : k;
          // swap rows k, p of the panel (lanes < nb: one column each)
          if (lane < nb && p != k) { double* c = P + (long long)lane * ld; const double x = c[k]; c[k] = c[p]; c[p] = x; }
          if (lane == 0) {
            if (!(bv > 0.0 && isfinite(bv))) s_bad = 1;
            s_p = p; bpiv[kk] = p;
          }
          __syncwarp();
          if (lane == 0) s_rp = 1.0 / pc[k];
        }
        __syncthreads();
        const double rp = s_rp;
        // Gauss-Jordan step on the panel columns (row k read unscaled, then scaled)
        for (int e = t; e < nb * s; e += GJ_THREADS) {
          const int cc = e / s, i = e - cc * s;
          if (cc == kk || i == k) continue;
          double* c = P + (long long)cc * ld;
          c[i] = fma(-pc[i] * rp, c[k], c[i]);
        }
        __syncthreads();
        if (t < nb && t != kk) P[(long long)t * ld + k] *= rp;
        for (int i = t; i < s; i += GJ_THREADS) pc[i] = i == k ? rp : -pc[i] * rp;
        __syncthreads();
      }
      // publish: panel + pivots to every CTA of the cluster
      for (int r = 0; r < CL; ++r) {
        double* dst = Pn;
        int* dpv = pivs;
        if (CL > 1) {
          dst = cg::this_cluster().map_shared_rank(Pn, r);
          dpv = cg::this_cluster().map_shared_rank(pivs, r);
        }
        for (int e = t; e < nb * s; e += GJ_THREADS) {
          const int cc = e / s, i = e - cc * s;
          dst[(long long)cc * ld + i] = P[(long long)cc * ld + i];
        }
        if (t < nb) dpv[k0 + t] = bpiv[t];
      }
    }
    if (CL > 1) cg::this_cluster().sync();
    else __syncthreads();
    // update the own columns outside K: swaps, X = rows K, rows K <- 0, column += Pn X
    for (int cc = t; cc < nc; cc += GJ_THREADS) {                // one column per thread
      const int j = c0 + cc;
      double* xs = Xs + cc * GJ_NB;
      if (j >= k0 && j < k0 + nb) {                                // panel-owned: X = 0
#pragma unroll
        for (int kk = 0; kk < GJ_NB; ++kk) xs[kk] = 0.0;
        continue;
      }
      double* cj = A + (long long)cc * ld;
      for (int kk = 0; kk < nb; ++kk) {
        const int k = k0 + kk, p = pivs[k];
        if (p != k) { const double x = cj[k]; cj[k] = cj[p]; cj[p] = x; }
      }
#pragma unroll
      for (int kk = 0; kk < GJ_NB; ++kk) {
        xs[kk] = kk < nb ? cj[k0 + kk] : 0.0;
        if (kk < nb) cj[k0 + kk] = 0.0;
      }
    }
    __syncthreads();
    {
      // C (rows 0..s, own columns) += Pn (s x 8) X (8 x nc): warp item = m-tile x 2 n-tiles
      const int MT = (s + 7) >> 3, NT = (nc + 7) >> 3, NP = (NT + 1) >> 1;
      for (int it = warp; it < MT * NP; it += nw) {
        const int mt = it % MT, np2 = it / MT;
        const int r = 8 * mt + gid;
        double d[2][2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int c = 8 * (2 * np2 + u) + 2 * tig;
          d[u][0] = c < nc ? A[(long long)c * ld + r] : 0.0;
          d[u][1] = c + 1 < nc ? A[(long long)(c + 1) * ld + r] : 0.0;
        }
#pragma unroll
        for (int k4 = 0; k4 < GJ_NB; k4 += 4) {
          const double a = Pn[(long long)(k4 + tig) * ld + r];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int c = 8 * (2 * np2 + u) + gid;
            dmma884(d[u][0], d[u][1], a, c < nc ? Xs[c * GJ_NB + k4 + tig] : 0.0);
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int c = 8 * (2 * np2 + u) + 2 * tig;
          const bool skip0 = c >= nc || (c0 + c >= k0 && c0 + c < k0 + nb);
          const bool skip1 = c + 1 >= nc || (c0 + c + 1 >= k0 && c0 + c + 1 < k0 + nb);
          if (r < s && !skip0) A[(long long)c * ld + r] = d[u][0];
          if (r < s && !skip1) A[(long long)(c + 1) * ld + r] = d[u][1];
        }
      }
    }
    __syncthreads();
    if (CL > 1) cg::this_cluster().sync();           // (Pn / pivs reused by the next block)
  }
  if (s_bad && t == 0) latch_status(st, FDE_ESINGULAR, job);
  // undo the interchanges: result[:, q] = A[:, idx[q]] with idx = swaps (k, piv[k]) applied for
  // k = s-1 .. 0 to the identity; the CTA writes its column j to every q with idx[q] = j
  if (t == 0) {
    for (int q = 0; q < s; ++q) perm[q] = q;
    for (int k = s - 1; k >= 0; --k) { const int p = pivs[k]; const int x = perm[k]; perm[k] = perm[p]; perm[p] = x; }
  }
  __syncthreads();
  for (long long e = t; e < (long long)s * s; e += GJ_THREADS) {
    const int i = (int)(e % s), q = (int)(e / s), j = perm[q];
    if (j >= c0 && j < c1) jb.A[(long long)q * jb.lda + i] = A[(long long)(j - c0) * ld + i];
  }
}

// ---------------------------------------------------------------------------------------
// Diagonally pivoted Cholesky of the b x b Gram matrix G = W^T W (ld b) with deflation: pivots
// are taken while the largest residual diagonal exceeds thr and fewer than nmax are kept.  With
// the kept columns S (in pivot order) and G[S, S] = R^T R, writes Sm (b x nk, ld b) = rows S of
// R^{-1} (other rows zero), so that W Sm = W[:, S] R^{-1} has orthonormal columns (to the
// rounding of G), and *nk_out.  One CTA; b <= PO_MAX.  Dynamic shared memory PO_SMEM.
#define PO_MAX 64
#define PO_SMEM (2 * PO_MAX * PO_MAX * 8)
// thr_ref (optional, device): the threshold is thr * *thr_ref (a reference norm left on the device
// by k_diag_max, so the host does not read it back).
__global__ void k_diag_max(int b, const double* __restrict__ G, double* __restrict__ out) {
  double v = 0.0;                                      // (one warp; fixed order)
  for (int i = threadIdx.x; i < b; i += 32) v = fmax(v, G[(long long)i * b + i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (threadIdx.x == 0) *out = v;
}

__global__ void __launch_bounds__(256)
k_pchol_orth(int b, const double* __restrict__ G, double thr, int nmax, double* __restrict__ Sm,
             int* __restrict__ nk_out, const double* __restrict__ thr_ref = nullptr) {
  if (thr_ref) thr *= *thr_ref;
  extern __shared__ double po_sm[];
  double* L = po_sm;                                  // L[q * b + i]: column q of the factor
  double* X = po_sm + PO_MAX * PO_MAX;                // X[r * PO_MAX + c] = (R^{-1})[r][c]
  __shared__ double d[PO_MAX];
  __shared__ int piv[PO_MAX], s_p, s_stop;
  __shared__ double s_sp;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (t < b) d[t] = G[(long long)t * b + t];
  __syncthreads();
  int q = 0;
  for (;; ++q) {
    if (warp == 0) {                                  // argmax of the residual diagonal (fixed order)
      double bv = -1.0; int bi = b;
      for (int i = lane; i < b; i += 32) if (d[i] > bv) { bv = d[i]; bi = i; }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (lane == 0) {
        s_stop = !(bv > thr) || q >= nmax || q >= b;
        s_p = bi;
        s_sp = s_stop ? 0.0 : sqrt(bv);
        if (!s_stop) piv[q] = bi;
      }
    }
    __syncthreads();
    if (s_stop) break;
    const int p = s_p;
    const double sp = s_sp;
    // L[:, q] = (G[:, p] - sum_{r<q} L[:, r] L[p, r]) / sp ; d -= L[:, q]^2 ; d[p] = -1 (taken)
    for (int i = t; i < b; i += 256) {
      double a = G[(long long)p * b + i];
      for (int r = 0; r < q; ++r) a = fma(-L[r * b + i], L[r * b + p], a);
      L[q * b + i] = a / sp;
    }
    __syncthreads();
    for (int i = t; i < b; i += 256) d[i] = (i == p || d[i] < 0.0) ? -1.0 : d[i] - L[q * b + i] * L[q * b + i];
    __syncthreads();
  }
  const int nk = q;
  // G[S, S] = Lt Lt^T with Lt[r][c] = L[c * b + piv[r]] (lower triangular in pivot order);
  // R = Lt^T: R[r][c] = L[r * b + piv[c]].  Column c of R^{-1} by back substitution (warp per c).
  for (int c = warp; c < nk; c += 8) {
    for (int r = c; r >= 0; --r) {
      double a = 0.0;
      for (int j = r + 1 + lane; j <= c; j += 32) a = fma(L[r * b + piv[j]], X[j * PO_MAX + c], a);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (lane == 0) X[r * PO_MAX + c] = ((r == c ? 1.0 : 0.0) - a) / L[r * b + piv[r]];
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = t; e < b * nk; e += 256) {
    const int i = e % b, c = e / b;
    double v = 0.0;
    for (int r = 0; r <= c; ++r) if (piv[r] == i) v = X[r * PO_MAX + c];
    Sm[(long long)c * b + i] = v;
  }
  if (t == 0) *nk_out = nk;
}
