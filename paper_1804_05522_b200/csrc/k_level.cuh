// k_level.cuh -- level-pass helpers: the per-segment reduction V^T Y of one HODLR level
// (k_lvl_reduce, used by the HODLR matvec k_matvec.cuh) and the copy of the fused rhs column.
// The SMW algebra these passes serve:
//
// At a node of level l with rows [r0, r0+n1+n2):
//   A = blkdiag(A11, A22) + [[0, U12 V12^T], [U21 V21^T, 0]]
//     = blkdiag(A11, A22) (I + blkdiag(W1, W2) Z^T),   W1 = A11^{-1} U12,  W2 = A22^{-1} U21,
//   Z^T = [[0, V12^T], [V21^T, 0]],  V12 = [L_l[:n2], e_0],  V21 = [J L_l[:n1], e_{n1-1}]
// (the V factors do not depend on d+-; the diagonal scaling lives in U), so
//   A^{-1} = (I - W K^{-1} Z^T) blkdiag(A11, A22)^{-1},   K = [[I, V12^T W2], [V21^T W1, I]].
// Processing levels from the leaves up (the paper's "structured LU ... then back
// substitution", realised in this SMW form) applies these factors to the
// ancestor columns of X (and to the fused right-hand side) and keeps W, K for solves.
// K is solved by block elimination: Sc = I - C B (C = V21^T W1, B = V12^T W2), partial
// pivoting LU of Sc; K^{-1}[a; b] = [a - B y; y],  y = Sc^{-1}(b - C a).
//
// The factorisation itself runs in k_levels.cuh (kept factor) and k_tree.cuh (projected tree).
//   k_lvl_reduce: per segment (<= SEG rows of one child) the partial products V^T X
#pragma once
#include "fde_common.cuh"

#define LVL_THREADS 256
#define XCH 32                     // column chunk of the reduce / update passes
#define SLD (2 * KCAP)             // leading dimension of S
#define KLD KCAP                   // leading dimension of the kept K pieces
#define SMEM_REDUCE ((KCAP * (SEG + 1) + XCH * (SEG + 1)) * 8)

struct LevelArgs {
  TreeDev tree;
  int level, mode;                 // mode 0 = factor, 1 = solve
  const double* Lf; long long lf_stride;
  const int* rank; const int* colofs;
  double* X; long long xstride;    // factor: targets + W live here
  double* Y; int ld; int nrhs; long long ystride;   // solve: targets
  int nf;                          // factor mode: fused rhs columns (0/1)
  double* Ppart; long long pstride_seg; long long pstride_inst;   // [inst][seg][KCAP x ncap]
  DevStatus* st;
};

// column range helpers ------------------------------------------------------------------
// factor mode: P columns = X columns [tb, wb + k); targets [tb, wb); W = [wb, wb + k)
// solve  mode: P columns = Y columns [0, nrhs); targets = all.
struct ColRange { int tb, wb, k, r, ncols, ntgt; };

__device__ __forceinline__ ColRange col_range(const LevelArgs& a, int inst) {
  ColRange cr;
  const int L = a.tree.L;
  cr.r = a.rank[inst * L + a.level];
  cr.k = cr.r + 1;
  cr.wb = 1 + a.colofs[inst * (L + 1) + a.level];   // X column of W (both modes)
  if (a.mode == 0) {
    cr.tb = 1 - a.nf;
    cr.ncols = cr.wb + cr.k - cr.tb;
    cr.ntgt = cr.wb - cr.tb;
  } else {
    cr.tb = 0;
    cr.ncols = a.nrhs;
    cr.ntgt = a.nrhs;
  }
  return cr;
}

// V row value of global row R (child c of node (r0n, n1)), column q < k.
__device__ __forceinline__ double vrow(const double* Ll, int m, int r, int c, int R,
                                       int r0n, int n1, int q) {
  if (c == 1) {
    const int i2 = R - r0n - n1;
    return (q < r) ? Ll[i2 + (long long)q * m] : (i2 == 0 ? 1.0 : 0.0);
  } else {
    const int j1 = R - r0n;
    return (q < r) ? Ll[(n1 - 1 - j1) + (long long)q * m] : (j1 == n1 - 1 ? 1.0 : 0.0);
  }
}

// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(LVL_THREADS)
k_lvl_reduce(const LevelArgs a) {
  extern __shared__ double lvl_smem[];
  double* Vs = lvl_smem;                       // V[row][q] at q*(SEG+1) + row
  double* Xs = lvl_smem + KCAP * (SEG + 1);    // X[row][col]
  const TreeDev& tr = a.tree;
  const int seg = blockIdx.x, inst = blockIdx.y, t = threadIdx.x;
  const int l = a.level, n = tr.n;
  const int sg = tr.seg_ofs[l] + seg;
  const int jn = tr.seg_node[sg], c = tr.seg_child[sg];
  const int row0 = tr.seg_row0[sg], len = tr.seg_len[sg];
  const int nd = node_index(l, jn);
  const int r0n = tr.node_r0[nd], n1 = tr.node_n1[nd];
  const ColRange cr = col_range(a, inst);
  const int k = cr.k, m = tr.lev_m[l];
  const double* Ll = a.Lf + (long long)inst * a.lf_stride + tr.lev_lofs[l];
  for (int e = t; e < len * k; e += LVL_THREADS) {
    const int i = e % len, q = e / len;
    Vs[q * (SEG + 1) + i] = vrow(Ll, m, cr.r, c, row0 + i, r0n, n1, q);
  }
  const double* src;
  long long cstride;
  if (a.mode == 0) { src = a.X + (long long)inst * a.xstride + (long long)cr.tb * n; cstride = n; }
  else { src = a.Y + (long long)inst * a.ystride; cstride = a.ld; }
  double* Po = a.Ppart + (long long)inst * a.pstride_inst + (long long)seg * a.pstride_seg;
  for (int c0 = 0; c0 < cr.ncols; c0 += XCH) {
    const int nc = min(XCH, cr.ncols - c0);
    __syncthreads();
    for (int e = t; e < len * nc; e += LVL_THREADS) {
      const int i = e % len, cc = e / len;
      Xs[cc * (SEG + 1) + i] = src[(long long)(c0 + cc) * cstride + row0 + i];
    }
    __syncthreads();
    for (int o = t; o < k * nc; o += LVL_THREADS) {
      const int q = o % k, cc = o / k;
      const double* vq = Vs + q * (SEG + 1);
      const double* xc = Xs + cc * (SEG + 1);
      double s0 = 0.0, s1 = 0.0;
      int i = 0;
      for (; i + 1 < len; i += 2) { s0 = fma(vq[i], xc[i], s0); s1 = fma(vq[i + 1], xc[i + 1], s1); }
      if (i < len) s0 = fma(vq[i], xc[i], s0);
      Po[q + (long long)(c0 + cc) * KCAP] = s0 + s1;
    }
  }
}

// u_next = X[:, 0] (fused right-hand side after the root level)
__global__ void k_copy_col0(const double* __restrict__ X, long long xstride, int n,
                            double* __restrict__ out, int batch) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long tot = (long long)batch * n;
  if (idx >= tot) return;
  const int inst = (int)(idx / n), i = (int)(idx % n);
  out[idx] = X[(long long)inst * xstride + i];
}
