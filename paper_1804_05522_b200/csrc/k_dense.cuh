// k_dense.cuh -- small dense FP64 helpers of the 2D Sylvester step (S8-S10, fde2d.cuh):
// transpose, scaled copy, sum of squares, and the one-sided Jacobi SVD (right-hand-side
// compression and truncation of the low-rank factors).  The products, QR, inverses and the
// pivoted-Cholesky orthonormalisation are in k_small.cuh.
// All reductions use a fixed order (deterministic).  Column-major throughout.
#pragma once
#include "fde_common.cuh"

#define DN_THREADS 256
#define DN_BIG 1024                    // threads of the single-CTA kernels
#define TS_TILE 16
#define DN_SMEM_MAX (206 * 1024)       // dynamic shared memory of the single-CTA kernels

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

// Y (m x n) = alpha X (m x n), column-major with leading dims (copy / scale).
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
