// k_dense.cuh -- dense FP64 building blocks of the 2D Sylvester step (S8-S10, fde2d.cuh):
// tall-skinny products of Krylov bases, symmetric Jacobi eigensolver (Gram matrices of the
// SVQB orthonormalisation), one-sided Jacobi SVD (truncation of the low-rank factors),
// Gauss-Jordan inverse with partial pivoting (Newton sign iteration of the projected
// Sylvester equation).  The small matrices live in global memory (L2 resident); the single-CTA
// kernels are latency-bound by design: cfg5's projected problems are <= a few hundred wide.
// All reductions use a fixed order (deterministic).  Column-major throughout.
#pragma once
#include "fde_common.cuh"

#define DN_THREADS 256
#define DN_BIG 1024                    // threads of the single-CTA kernels
#define TS_TILE 16
#define DN_SMEM_MAX (206 * 1024)       // dynamic shared memory of the single-CTA kernels

// C (m x n) = alpha * A^T B + beta * C;  A: K x m (lda), B: K x n (ldb); K is the tall dim.
// One CTA per 16 x 16 tile of C; the K loop is staged through shared memory.
__global__ void __launch_bounds__(DN_THREADS)
k_ts_gemm_tn(int m, int n, int K, double alpha, const double* __restrict__ A, int lda,
             const double* __restrict__ B, int ldb, double beta, double* __restrict__ C, int ldc) {
  __shared__ double As[64][TS_TILE + 1], Bs[64][TS_TILE + 1];
  const int i0 = blockIdx.x * TS_TILE, j0 = blockIdx.y * TS_TILE;
  const int t = threadIdx.x, ti = t % TS_TILE, tj = t / TS_TILE;
  double acc = 0.0;
  for (int k0 = 0; k0 < K; k0 += 64) {
    for (int e = t; e < 64 * TS_TILE; e += DN_THREADS) {
      const int kk = e % 64, c = e / 64;
      As[kk][c] = (k0 + kk < K && i0 + c < m) ? A[(long long)(i0 + c) * lda + k0 + kk] : 0.0;
      Bs[kk][c] = (k0 + kk < K && j0 + c < n) ? B[(long long)(j0 + c) * ldb + k0 + kk] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 64; ++kk) acc = fma(As[kk][ti], Bs[kk][tj], acc);
    __syncthreads();
  }
  if (i0 + ti < m && j0 + tj < n) {
    double* c = C + (long long)(j0 + tj) * ldc + i0 + ti;
    *c = alpha * acc + (beta == 0.0 ? 0.0 : beta * *c);
  }
}

// Split-K variant: partial tile sums of the K chunk blockIdx.z go to P[z][n][m] (column-major
// m x n per chunk); k_reduce_partials adds the chunks in a fixed order.
__global__ void __launch_bounds__(DN_THREADS)
k_ts_gemm_tn_split(int m, int n, int K, int kchunk, const double* __restrict__ A, int lda,
                   const double* __restrict__ B, int ldb, double* __restrict__ P) {
  __shared__ double As[64][TS_TILE + 1], Bs[64][TS_TILE + 1];
  const int i0 = blockIdx.x * TS_TILE, j0 = blockIdx.y * TS_TILE;
  const int kb = blockIdx.z * kchunk, ke = min(K, kb + kchunk);
  const int t = threadIdx.x, ti = t % TS_TILE, tj = t / TS_TILE;
  double acc = 0.0;
  for (int k0 = kb; k0 < ke; k0 += 64) {
    for (int e = t; e < 64 * TS_TILE; e += DN_THREADS) {
      const int kk = e % 64, c = e / 64;
      As[kk][c] = (k0 + kk < ke && i0 + c < m) ? A[(long long)(i0 + c) * lda + k0 + kk] : 0.0;
      Bs[kk][c] = (k0 + kk < ke && j0 + c < n) ? B[(long long)(j0 + c) * ldb + k0 + kk] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 64; ++kk) acc = fma(As[kk][ti], Bs[kk][tj], acc);
    __syncthreads();
  }
  if (i0 + ti < m && j0 + tj < n) P[(long long)blockIdx.z * m * n + (long long)(j0 + tj) * m + i0 + ti] = acc;
}

__global__ void k_reduce_partials(int m, int n, int nz, const double* __restrict__ P, double alpha, double beta,
                                  double* __restrict__ C, int ldc) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)m * n) return;
  double s = 0.0;
  for (int z = 0; z < nz; ++z) s += P[(long long)z * m * n + e];
  const int i = (int)(e % m), j = (int)(e / m);
  double* c = C + (long long)j * ldc + i;
  *c = alpha * s + (beta == 0.0 ? 0.0 : beta * *c);
}

// Y (n x m, ld ldy) = X^T (X: m x n, ld ldx)
__global__ void k_transpose(int m, int n, const double* __restrict__ X, int ldx, double* __restrict__ Y, int ldy) {
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;          // bx over rows of X, by over cols
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = bx + threadIdx.x, j = by + r;
    if (i < m && j < n) tile[r][threadIdx.x] = X[(long long)j * ldx + i];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int j = by + threadIdx.x, i = bx + r;                 // Y[j][i] column i of Y^T... Y(j, i)
    if (i < m && j < n) Y[(long long)i * ldy + j] = tile[threadIdx.x][r];
  }
}

// C (M x n) = alpha * A B + beta * C;  A: M x K (lda, tall), B: K x n (ldb, small).
__global__ void __launch_bounds__(DN_THREADS)
k_ts_gemm_nn(int M, int n, int K, double alpha, const double* __restrict__ A, int lda,
             const double* __restrict__ B, int ldb, double beta, double* __restrict__ C, int ldc) {
  const int i = blockIdx.x * DN_THREADS + threadIdx.x, j = blockIdx.y;
  if (i >= M) return;
  double acc = 0.0;
  const double* bj = B + (long long)j * ldb;
  for (int k = 0; k < K; ++k) acc = fma(A[(long long)k * lda + i], bj[k], acc);
  double* c = C + (long long)j * ldc + i;
  *c = alpha * acc + (beta == 0.0 ? 0.0 : beta * *c);
}

// Y (m x n) = alpha X (m x n), column-major with leading dims (copy / scale).
// X[:, j] *= sc[j] (column scaling, m x n, ld ldx)
__global__ void k_scale_cols(int m, int n, double* __restrict__ X, int ldx, const double* __restrict__ sc) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e < (long long)m * n) {
    const int j = (int)(e / m), i = (int)(e - (long long)j * m);
    X[(long long)j * ldx + i] *= sc[j];
  }
}

__global__ void k_scale_copy(int m, int n, double alpha, const double* __restrict__ X, int ldx,
                             double* __restrict__ Y, int ldy) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)m * n) return;
  const int i = (int)(e % m), j = (int)(e / m);
  Y[(long long)j * ldy + i] = alpha * X[(long long)j * ldx + i];
}

// out[0] = sum of squares of X (m x n); fixed-order two-level reduction in one CTA.
__global__ void __launch_bounds__(DN_BIG)
k_sumsq(int m, int n, const double* __restrict__ X, int ldx, double* __restrict__ out) {
  __shared__ double red[DN_BIG];
  double s = 0.0;
  for (long long e = threadIdx.x; e < (long long)m * n; e += DN_BIG) {
    const double v = X[(e / m) * ldx + e % m];
    s = fma(v, v, s);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = DN_BIG / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

// ---------------------------------------------------------------------------------------
// Cyclic Jacobi eigen-decomposition of a symmetric b x b matrix G (overwritten): on exit
// lam[i] = eigenvalues (unsorted), V (b x b, ld b) the eigenvectors.  Round-robin ordering:
// b/2 disjoint rotations per round run in parallel (one warp each), b-1 rounds per sweep.
__global__ void __launch_bounds__(DN_BIG)
k_sym_jacobi(int b, double* __restrict__ Gg, int ldgg, double* __restrict__ Vg, double* __restrict__ lam,
             int max_sweeps) {
  extern __shared__ double sh_dn[];                  // [G | V | pairs] when resident, else [pairs]
  const bool res = 2LL * b * b * 8 + (b + 2) * 4 <= DN_SMEM_MAX;
  double* G = res ? sh_dn : Gg;
  double* V = res ? sh_dn + b * b : Vg;
  const int ldg = res ? b : ldgg;
  int* sh_pairs = reinterpret_cast<int*>(res ? sh_dn + 2 * b * b : sh_dn);
  if (res) {
    for (int e = threadIdx.x; e < b * b; e += DN_BIG) G[e] = Gg[(long long)(e / b) * ldgg + e % b];
    __syncthreads();
  }
  __shared__ double cs[512], sn[512];
  __shared__ int done;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31, nw = DN_BIG / 32;
  for (long long e = t; e < (long long)b * b; e += DN_BIG) V[e] = ((e % b) == (e / b)) ? 1.0 : 0.0;
  const int bb = b + (b & 1);                        // even player count (dummy = b)
  int* pl = sh_pairs;
  for (int i = t; i < bb; i += DN_BIG) pl[i] = i;
  __syncthreads();
  double off0 = 0.0;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (t == 0) done = 1;
    __syncthreads();
    for (int r = 0; r < bb - 1; ++r) {
      // rotation angles for the pairs (pl[i], pl[bb-1-i])
      for (int pi = warp; pi < bb / 2; pi += nw) {
        int p = pl[pi], q = pl[bb - 1 - pi];
        if (p > q) { const int x = p; p = q; q = x; }
        double c = 1.0, s = 0.0;
        if (q < b) {
          const double apq = G[(long long)q * ldg + p], app = G[(long long)p * ldg + p], aqq = G[(long long)q * ldg + q];
          if (fabs(apq) > 1e-300 && fabs(apq) > 4e-15 * sqrt(fabs(app * aqq))) {
            const double tau = (aqq - app) / (2.0 * apq);
            const double tt = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + tt * tt);
            s = tt * c;
            if (lane == 0) done = 0;
          }
        }
        if (lane == 0) { cs[pi] = c; sn[pi] = s; }
      }
      __syncthreads();
      // apply: G <- J^T G J  (columns then rows), V <- V J
      for (int pi = warp; pi < bb / 2; pi += nw) {
        int p = pl[pi], q = pl[bb - 1 - pi];
        if (p > q) { const int x = p; p = q; q = x; }
        if (q >= b) continue;
        const double c = cs[pi], s = sn[pi];
        for (int i = lane; i < b; i += 32) {          // columns p, q of G and V
          const double gp = G[(long long)p * ldg + i], gq = G[(long long)q * ldg + i];
          G[(long long)p * ldg + i] = c * gp - s * gq;
          G[(long long)q * ldg + i] = s * gp + c * gq;
          const double vp = V[(long long)p * b + i], vq = V[(long long)q * b + i];
          V[(long long)p * b + i] = c * vp - s * vq;
          V[(long long)q * b + i] = s * vp + c * vq;
        }
      }
      __syncthreads();
      for (int pi = warp; pi < bb / 2; pi += nw) {
        int p = pl[pi], q = pl[bb - 1 - pi];
        if (p > q) { const int x = p; p = q; q = x; }
        if (q >= b) continue;
        const double c = cs[pi], s = sn[pi];
        for (int j = lane; j < b; j += 32) {          // rows p, q of G
          const double gp = G[(long long)j * ldg + p], gq = G[(long long)j * ldg + q];
          G[(long long)j * ldg + p] = c * gp - s * gq;
          G[(long long)j * ldg + q] = s * gp + c * gq;
        }
      }
      __syncthreads();
      // rotate the tournament (player 0 fixed)
      if (t == 0) {
        const int last = pl[bb - 1];
        for (int i = bb - 1; i > 1; --i) pl[i] = pl[i - 1];
        pl[1] = last;
      }
      __syncthreads();
    }
    if (done) break;
    (void)off0;
  }
  for (int i = t; i < b; i += DN_BIG) lam[i] = G[(long long)i * ldg + i];
  if (res) {
    __syncthreads();
    for (int e = t; e < b * b; e += DN_BIG) { Vg[e] = V[e]; Gg[(long long)(e / b) * ldgg + e % b] = G[e]; }
  }
}

// ---------------------------------------------------------------------------------------
// One-sided Jacobi SVD of Y (m x n, ld ldy; overwritten by W Sigma): on exit the columns of Y
// are mutually orthogonal (Y_out = Y_in Z), Z (n x n) orthogonal, sig[j] = ||Y_out[:, j]||.
__global__ void __launch_bounds__(DN_BIG)
k_osj_svd(int m, int n, double* __restrict__ Yg, int ldyg, double* __restrict__ Z, double* __restrict__ sig,
          int max_sweeps) {
  extern __shared__ double sh_dn[];                  // [Y | pairs] when resident, else [pairs]
  const bool res = (long long)m * n * 8 + (n + 2) * 4 <= DN_SMEM_MAX;
  double* Y = res ? sh_dn : Yg;
  const int ldy = res ? m : ldyg;
  int* sh_pairs = reinterpret_cast<int*>(res ? sh_dn + (long long)m * n : sh_dn);
  if (res) {
    for (long long e = threadIdx.x; e < (long long)m * n; e += DN_BIG) Y[e] = Yg[(e / m) * ldyg + e % m];
    __syncthreads();
  }
  __shared__ double cs[512], sn[512];
  __shared__ int done;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31, nw = DN_BIG / 32;
  for (long long e = t; e < (long long)n * n; e += DN_BIG) Z[e] = ((e % n) == (e / n)) ? 1.0 : 0.0;
  const int bb = n + (n & 1);
  int* pl = sh_pairs;
  for (int i = t; i < bb; i += DN_BIG) pl[i] = i;
  __syncthreads();
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (t == 0) done = 1;
    __syncthreads();
    for (int r = 0; r < bb - 1; ++r) {
      for (int pi = warp; pi < bb / 2; pi += nw) {
        int p = pl[pi], q = pl[bb - 1 - pi];
        if (p > q) { const int x = p; p = q; q = x; }
        double c = 1.0, s = 0.0;
        if (q < n) {
          double al = 0.0, be = 0.0, ga = 0.0;
          for (int i = lane; i < m; i += 32) {
            const double yp = Y[(long long)p * ldy + i], yq = Y[(long long)q * ldy + i];
            al = fma(yp, yp, al); be = fma(yq, yq, be); ga = fma(yp, yq, ga);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            al += __shfl_xor_sync(0xffffffffu, al, o);
            be += __shfl_xor_sync(0xffffffffu, be, o);
            ga += __shfl_xor_sync(0xffffffffu, ga, o);
          }
          if (fabs(ga) > 4e-15 * sqrt(al * be) && fabs(ga) > 1e-300) {
            const double zeta = (be - al) / (2.0 * ga);
            const double tt = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            c = 1.0 / sqrt(1.0 + tt * tt);
            s = c * tt;
            if (lane == 0) done = 0;
          }
          for (int i = lane; i < m; i += 32) {
            const double yp = Y[(long long)p * ldy + i], yq = Y[(long long)q * ldy + i];
            Y[(long long)p * ldy + i] = c * yp - s * yq;
            Y[(long long)q * ldy + i] = s * yp + c * yq;
          }
          for (int i = lane; i < n; i += 32) {
            const double zp = Z[(long long)p * n + i], zq = Z[(long long)q * n + i];
            Z[(long long)p * n + i] = c * zp - s * zq;
            Z[(long long)q * n + i] = s * zp + c * zq;
          }
        }
        (void)cs; (void)sn;
      }
      __syncthreads();
      if (t == 0) {
        const int last = pl[bb - 1];
        for (int i = bb - 1; i > 1; --i) pl[i] = pl[i - 1];
        pl[1] = last;
      }
      __syncthreads();
    }
    if (done) break;
  }
  for (int j = warp; j < n; j += nw) {
    double s2 = 0.0;
    for (int i = lane; i < m; i += 32) { const double y = Y[(long long)j * ldy + i]; s2 = fma(y, y, s2); }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if (lane == 0) sig[j] = sqrt(s2);
  }
  if (res) {
    __syncthreads();
    for (long long e = t; e < (long long)m * n; e += DN_BIG) Yg[(e / m) * ldyg + e % m] = Y[e];
  }
}

// ---------------------------------------------------------------------------------------
// In-place inverse of blockIdx.x-th matrix (s x s, ld lda) by Gauss-Jordan with partial
// pivoting (the projected matrices of the sign iteration are not diagonally dominant).
// One CTA per matrix; ptrs[b] selects the matrix, piv scratch [s] ints per matrix in smem.
struct InvJob { double* A; int s; int lda; };

__global__ void __launch_bounds__(DN_BIG)
k_gj_inverse(const InvJob* __restrict__ jobs, DevStatus* st) {
  extern __shared__ double sh_dn[];                  // [A | piv] when resident, else [piv]
  __shared__ double colk[1024], rowk[1024];
  __shared__ double red_v[DN_BIG / 32];
  __shared__ int red_i[DN_BIG / 32];
  __shared__ int prow;
  const InvJob jb = jobs[blockIdx.x];
  const int s = jb.s, t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const bool res = (long long)s * s * 8 + s * 4 <= DN_SMEM_MAX;
  double* A = res ? sh_dn : jb.A;
  const int lda = res ? s : jb.lda;
  int* sh_piv = reinterpret_cast<int*>(res ? sh_dn + (long long)s * s : sh_dn);
  if (res) {
    for (int e = t; e < s * s; e += DN_BIG) A[e] = jb.A[(long long)(e / s) * jb.lda + e % s];
    __syncthreads();
  }

  for (int k = 0; k < s; ++k) {
    // pivot search in column k, rows k..s-1 (fixed-order argmax: largest |a|, smallest index)
    double bv = -1.0; int bi = s;
    for (int i = k + t; i < s; i += DN_BIG) {
      const double v = fabs(A[(long long)k * lda + i]);
      if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { red_v[warp] = bv; red_i[warp] = bi; }
    __syncthreads();
    if (warp == 0) {                                 // fixed-order warp reduction of the partials
      double v = red_v[lane];
      int ii = red_i[lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, ii, o);
        if (ov > v || (ov == v && oi < ii)) { v = ov; ii = oi; }
      }
      if (lane == 0) {
        prow = ii;
        if (!(v > 0.0) || !isfinite(v)) latch_status(st, FDE_ESINGULAR, k);
      }
    }
    __syncthreads();
    const int p = prow;
    if (t == 0) sh_piv[k] = p;
    if (p != k) {                                    // swap rows k and p (all columns)
      for (int j = t; j < s; j += DN_BIG) {
        const double x = A[(long long)j * lda + k];
        A[(long long)j * lda + k] = A[(long long)j * lda + p];
        A[(long long)j * lda + p] = x;
      }

    }
    __syncthreads();
    const double rp = 1.0 / A[(long long)k * lda + k];
    for (int i = t; i < s; i += DN_BIG) { colk[i] = A[(long long)k * lda + i]; rowk[i] = A[(long long)i * lda + k]; }
    __syncthreads();
    // Gauss-Jordan update: row k scaled, other rows eliminated; column k becomes -a_ik / p
    // (pivot row and column are read from the shared snapshots: no read-write race)
    // (warp per column, lane per row: no 64-bit index division in the per-pivot sweep)
    for (int j = warp; j < s; j += DN_BIG / 32) {
      if (j == k) continue;
      const double akj = rowk[j];
      double* Aj = A + (long long)j * lda;
      for (int i = lane; i < s; i += 32)
        Aj[i] = (i == k) ? akj * rp : fma(-colk[i] * rp, akj, Aj[i]);
    }
    __syncthreads();
    for (int i = t; i < s; i += DN_BIG) A[(long long)k * lda + i] = (i == k) ? rp : -colk[i] * rp;
    __syncthreads();
  }
  // undo the row interchanges: column swaps in reverse order (in-place Gauss-Jordan)
  for (int k = s - 1; k >= 0; --k) {
    const int p = sh_piv[k];
    if (p != k)
      for (int i = t; i < s; i += DN_BIG) {
        const double x = A[(long long)k * lda + i];
        A[(long long)k * lda + i] = A[(long long)p * lda + i];
        A[(long long)p * lda + i] = x;
      }
    __syncthreads();
  }
  if (res)
    for (int e = t; e < s * s; e += DN_BIG) jb.A[(long long)(e / s) * jb.lda + e % s] = A[e];
}
