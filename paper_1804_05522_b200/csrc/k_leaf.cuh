// k_leaf.cuh -- S3 + S4: fused leaf assembly, unpivoted blocked LU and blocked TRSM.
//
// One CTA per (leaf, instance).  The leaf block of
//   A_m = shift I + c (D+ T + D- T^T),  T[i,j] = -g_{i-j+1}            (Eq. 2.5-2.6)
// is generated from g and d+- straight into shared memory (the identity shift and the
// diagonal scaling touch only the leaves and the factors), factorised without
// pivoting (A_m and all its principal sub-blocks are strictly diagonally dominant),
// and applied to the leaf's rows of the right-hand-side panel:
//   factor mode: X = [b | U_0 | U_1 | ... | U_{L-1}] where b = u_prev + dt f (fused solve,
//     optional) and U_l is the column factor of the level-l off-diagonal block containing
//     the leaf's rows, generated from the level factor L_l and d+- (S3):
//       first child  rows: U12 = [-c D-  J L_l[:n1],  -c d+[r0+n1-1] e_{n1-1}]
//       second child rows: U21 = [-c D+  L_l[:n2],    -c d-[r0+n1]   e_0      ]
//     X <- A_leaf^{-1} X  is written to HBM for the level passes (k_level.cuh);
//   solve mode: y <- A_leaf^{-1} b with the LU kept from the factorisation.
// Blocking: 32 x 32 diagonal blocks (one warp, row per lane), panel triangular solves
// (row/column per thread) and the trailing updates as shared-memory GEMMs.
#pragma once
#include "fde_common.cuh"

#define LEAF_THREADS 256
#define LDA_LEAF (LEAF_MAX + 1)
#define NCHUNK 64
#define LDP_LEAF (LEAF_MAX + 1)

struct LeafArgs {
  TreeDev tree;
  int mode;                 // 0 = factor, 1 = solve
  double shift;
  const double* cfac;       // [batch] c = dt / h^alpha
  double dt;
  const double* g; long long gstride;
  const double* dp; const double* dm;        // [batch*n]
  const double* Lf; long long lf_stride;
  const int* rank;                           // [batch*L] actual ranks
  int kl[LMAX];                              // columns per level (max rank over batch + 1)
  int xcol[LMAX + 1];                        // first X column of each level block; xcol[L] = end
  double* X; long long xstride;              // X[inst*xstride + col*n + row]
  double* LU; long long lustride; int keep;  // leaf LU storage
  int nf;                                    // fused RHS columns (0/1), factor mode
  const double* u_prev; const double* f;     // [batch*n], factor mode with nf = 1
  const double* b; double* y; int nrhs; int ld;   // solve mode
  DevStatus* st;
};

// C[m x n] -= A[m x kk] * B[kk x n]; column-major smem; m <= 128.  Warp w takes column
// groups of 4, lane takes rows lane + 32 r (r < 4): conflict-free A loads, broadcast B.
__device__ __forceinline__ void smem_gemm_sub(double* C, int ldc, const double* A, int lda,
                                              const double* B, int ldb, int m, int n, int kk) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int cg = w; cg * 4 < n; cg += nw) {
    const int j0 = cg * 4;
    double acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
    for (int k = 0; k < kk; ++k) {
      double a[4], bb[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) { const int i = lane + 32 * r; a[r] = (i < m) ? A[i + k * lda] : 0.0; }
#pragma unroll
      for (int c = 0; c < 4; ++c) { const int j = j0 + c; bb[c] = (j < n) ? B[k + j * ldb] : 0.0; }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = fma(a[r], bb[c], acc[r][c]);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = lane + 32 * r;
      if (i >= m) continue;
#pragma unroll
      for (int c = 0; c < 4; ++c) { const int j = j0 + c; if (j < n) C[i + j * ldc] -= acc[r][c]; }
    }
  }
}

// Unpivoted blocked LU of A (s x s, lda) in shared memory.
__device__ void leaf_lu(double* A, int s, DevStatus* st, int where) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  for (int k0 = 0; k0 < s; k0 += PB) {
    const int kw = min(PB, s - k0);
    // (1) diagonal block, warp 0, lane = row
    if (w == 0) {
      for (int k = 0; k < kw; ++k) {
        __syncwarp();
        const double piv = A[(k0 + k) + (k0 + k) * LDA_LEAF];
        if (lane == 0 && !(isfinite(piv) && piv != 0.0)) latch_status(st, FDE_ESINGULAR, where);
        if (lane > k && lane < kw) {
          const double l = A[(k0 + lane) + (k0 + k) * LDA_LEAF] / piv;
          A[(k0 + lane) + (k0 + k) * LDA_LEAF] = l;
          for (int j = k + 1; j < kw; ++j)
            A[(k0 + lane) + (k0 + j) * LDA_LEAF] -= l * A[(k0 + k) + (k0 + j) * LDA_LEAF];
        }
      }
    }
    __syncthreads();
    const int rest = s - k0 - kw;
    if (rest > 0) {
      // (2) panels: rows below <- A U_kk^{-1};  columns right <- L_kk^{-1} A
      if (t < rest) {
        const int i = k0 + kw + t;
        for (int j = 0; j < kw; ++j) {
          double x0 = A[i + (k0 + j) * LDA_LEAF], x1 = 0.0;
          int q = 0;
          for (; q + 1 < j; q += 2) {
            x0 -= A[i + (k0 + q) * LDA_LEAF] * A[(k0 + q) + (k0 + j) * LDA_LEAF];
            x1 -= A[i + (k0 + q + 1) * LDA_LEAF] * A[(k0 + q + 1) + (k0 + j) * LDA_LEAF];
          }
          if (q < j) x0 -= A[i + (k0 + q) * LDA_LEAF] * A[(k0 + q) + (k0 + j) * LDA_LEAF];
          A[i + (k0 + j) * LDA_LEAF] = (x0 + x1) / A[(k0 + j) + (k0 + j) * LDA_LEAF];
        }
      } else if (t < 2 * rest) {
        const int j = k0 + kw + (t - rest);
        for (int i = 1; i < kw; ++i) {
          double x0 = A[(k0 + i) + j * LDA_LEAF], x1 = 0.0;
          int q = 0;
          for (; q + 1 < i; q += 2) {
            x0 -= A[(k0 + i) + (k0 + q) * LDA_LEAF] * A[(k0 + q) + j * LDA_LEAF];
            x1 -= A[(k0 + i) + (k0 + q + 1) * LDA_LEAF] * A[(k0 + q + 1) + j * LDA_LEAF];
          }
          if (q < i) x0 -= A[(k0 + i) + (k0 + q) * LDA_LEAF] * A[(k0 + q) + j * LDA_LEAF];
          A[(k0 + i) + j * LDA_LEAF] = x0 + x1;
        }
      }
      __syncthreads();
      // (3) trailing update
      double* A22 = A + (k0 + kw) + (k0 + kw) * LDA_LEAF;
      smem_gemm_sub(A22, LDA_LEAF, A + (k0 + kw) + k0 * LDA_LEAF, LDA_LEAF,
                    A + k0 + (k0 + kw) * LDA_LEAF, LDA_LEAF, rest, rest, kw);
      __syncthreads();
    }
  }
}

// P <- U^{-1} L^{-1} P for a panel of nc <= NCHUNK columns (ldp), LU in A.
__device__ void leaf_trsm(const double* A, int s, double* P, int nc) {
  const int t = threadIdx.x;
  // forward, unit lower
  for (int k0 = 0; k0 < s; k0 += PB) {
    const int kw = min(PB, s - k0);
    if (t < nc) {
      double pv[PB];
#pragma unroll
      for (int i = 0; i < PB; ++i) pv[i] = (i < kw) ? P[k0 + i + t * LDP_LEAF] : 0.0;
#pragma unroll
      for (int i = 1; i < PB; ++i) {
        if (i < kw) {
          double x = pv[i];
#pragma unroll
          for (int q = 0; q < i; ++q) x -= A[(k0 + i) + (k0 + q) * LDA_LEAF] * pv[q];
          pv[i] = x;
        }
      }
#pragma unroll
      for (int i = 0; i < PB; ++i) if (i < kw) P[k0 + i + t * LDP_LEAF] = pv[i];
    }
    __syncthreads();
    const int rest = s - k0 - kw;
    if (rest > 0) {
      smem_gemm_sub(P + k0 + kw, LDP_LEAF, A + (k0 + kw) + k0 * LDA_LEAF, LDA_LEAF,
                    P + k0, LDP_LEAF, rest, nc, kw);
      __syncthreads();
    }
  }
  // backward, upper
  const int nb = (s + PB - 1) / PB;
  for (int kb = nb - 1; kb >= 0; --kb) {
    const int k0 = kb * PB;
    const int kw = min(PB, s - k0);
    if (t < nc) {
      double pv[PB];
#pragma unroll
      for (int i = 0; i < PB; ++i) pv[i] = (i < kw) ? P[k0 + i + t * LDP_LEAF] : 0.0;
#pragma unroll
      for (int i = PB - 1; i >= 0; --i) {
        if (i < kw) {
          double x = pv[i];
#pragma unroll
          for (int q = i + 1; q < PB; ++q)
            if (q < kw) x -= A[(k0 + i) + (k0 + q) * LDA_LEAF] * pv[q];
          pv[i] = x / A[(k0 + i) + (k0 + i) * LDA_LEAF];
        }
      }
#pragma unroll
      for (int i = 0; i < PB; ++i) if (i < kw) P[k0 + i + t * LDP_LEAF] = pv[i];
    }
    __syncthreads();
    if (k0 > 0) {
      smem_gemm_sub(P, LDP_LEAF, A + k0 * LDA_LEAF, LDA_LEAF, P + k0, LDP_LEAF, k0, nc, kw);
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(LEAF_THREADS)
k_leaf(const LeafArgs a) {
  extern __shared__ double smem[];
  double* A = smem;                               // [LEAF_MAX][LDA_LEAF]
  double* P = smem + LEAF_MAX * LDA_LEAF;         // [NCHUNK][LDP_LEAF]
  const TreeDev& tr = a.tree;
  const int leaf = blockIdx.x, inst = blockIdx.y, t = threadIdx.x;
  const int n = tr.n, L = tr.L;
  const int r0 = tr.leaf_r0[leaf], s = tr.leaf_n[leaf];
  const int where = inst * 65536 + leaf;
  double* LUg = a.LU + (long long)inst * a.lustride + (long long)r0 * LEAF_MAX;

  if (a.mode == 0) {
    // ---- S3: generate the leaf block from g and d+- (never stored unscaled)
    const double c = a.cfac[inst];
    const double* gi = a.g + (long long)inst * a.gstride;
    const double* dpi = a.dp + (long long)inst * n + r0;
    const double* dmi = a.dm + (long long)inst * n + r0;
    for (int e = t; e < s * s; e += LEAF_THREADS) {
      const int i = e % s, j = e / s;
      const int k1 = i - j + 1, k2 = j - i + 1;         // T[i,j] = -g_{i-j+1}, T^T[i,j] = T[j,i]
      const double tij = (k1 >= 0) ? -gi[k1] : 0.0;
      const double tji = (k2 >= 0) ? -gi[k2] : 0.0;
      A[i + j * LDA_LEAF] = (i == j ? a.shift : 0.0) + c * (dpi[i] * tij + dmi[i] * tji);
    }
    __syncthreads();
    leaf_lu(A, s, a.st, where);
    if (a.keep)
      for (int e = t; e < s * s; e += LEAF_THREADS) LUg[e] = A[(e % s) + (e / s) * LDA_LEAF];
    // ---- panel of X columns [1 - nf, 1 + W)
    const int* rk = a.rank + inst * L;
    const int c_end = a.xcol[L];
    const double* Lfi = a.Lf + (long long)inst * a.lf_stride;
    double* Xi = a.X + (long long)inst * a.xstride;
    const double* dpg = a.dp + (long long)inst * n;
    const double* dmg = a.dm + (long long)inst * n;
    for (int c0 = 1 - a.nf; c0 < c_end; c0 += NCHUNK) {
      const int nc = min(NCHUNK, c_end - c0);
      for (int e = t; e < s * nc; e += LEAF_THREADS) {
        const int i = e % s, cc = e / s;
        const int cg = c0 + cc, R = r0 + i;
        double v;
        if (cg == 0) {
          v = a.u_prev[(long long)inst * n + R] + a.dt * a.f[(long long)inst * n + R];
        } else {
          int l = 0;
          while (l + 1 < L && a.xcol[l + 1] <= cg) ++l;
          // q < r: scaled low-rank column; r <= q < k-1: zero padding; q = k-1: exact column
          const int q = cg - a.xcol[l], r = rk[l], kq = a.kl[l];
          const int jn = leaf >> (L - l), child = (leaf >> (L - l - 1)) & 1;
          const int nd = node_index(l, jn);
          const int r0n = tr.node_r0[nd], n1 = tr.node_n1[nd];
          const int m = tr.lev_m[l];
          const double* Ll = Lfi + tr.lev_lofs[l];
          if (child == 0) {
            const int j1 = R - r0n;
            v = (q == kq - 1) ? ((j1 == n1 - 1) ? -c * dpg[R] : 0.0)
                : (q < r ? -c * dmg[R] * Ll[(n1 - 1 - j1) + (long long)q * m] : 0.0);
          } else {
            const int i2 = R - r0n - n1;
            v = (q == kq - 1) ? ((i2 == 0) ? -c * dmg[R] : 0.0)
                : (q < r ? -c * dpg[R] * Ll[i2 + (long long)q * m] : 0.0);
          }
        }
        P[i + cc * LDP_LEAF] = v;
      }
      __syncthreads();
      leaf_trsm(A, s, P, nc);
      for (int e = t; e < s * nc; e += LEAF_THREADS) {
        const int i = e % s, cc = e / s;
        Xi[(long long)(c0 + cc) * n + r0 + i] = P[i + cc * LDP_LEAF];
      }
      __syncthreads();
    }
  } else {
    // ---- solve mode: LU from HBM, right-hand sides b -> y (y may alias b)
    for (int e = t; e < s * s; e += LEAF_THREADS) A[(e % s) + (e / s) * LDA_LEAF] = LUg[e];
    const long long ib = (long long)inst * a.ld * a.nrhs;
    for (int c0 = 0; c0 < a.nrhs; c0 += NCHUNK) {
      const int nc = min(NCHUNK, a.nrhs - c0);
      for (int e = t; e < s * nc; e += LEAF_THREADS) {
        const int i = e % s, cc = e / s;
        double v = a.b[ib + (long long)(c0 + cc) * a.ld + r0 + i];
        if (a.f) v += a.dt * a.f[ib + (long long)(c0 + cc) * a.ld + r0 + i];   // b = u + dt f (S7)
        P[i + cc * LDP_LEAF] = v;
      }
      __syncthreads();
      leaf_trsm(A, s, P, nc);
      for (int e = t; e < s * nc; e += LEAF_THREADS) {
        const int i = e % s, cc = e / s;
        a.y[ib + (long long)(c0 + cc) * a.ld + r0 + i] = P[i + cc * LDP_LEAF];
      }
      __syncthreads();
    }
  }
}
