// k_level.cuh -- S5 (Sherman-Morrison-Woodbury level factorisation) and S6 (tree solve).
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
// Per level three launches:
//   k_lvl_reduce: per segment (<= SEG rows of one child) the partial products V^T X
//   k_lvl_node  : per node, fixed-order sum of the segment partials, K (factor mode),
//                 S = K^{-1} Z^T X for the target columns
//   k_lvl_update: per segment, X_target -= W S_half
#pragma once
#include "fde_common.cuh"

#define LVL_THREADS 256
#define XCH 32                     // column chunk of the reduce / update passes
#define SLD (2 * KCAP)             // leading dimension of S
#define KLD KCAP                   // leading dimension of the kept K pieces
#define SMEM_REDUCE ((KCAP * (SEG + 1) + XCH * (SEG + 1)) * 8)
#define SMEM_NODE   (3 * KCAP * KCAP * 8)
#define SMEM_UPDATE ((KCAP * (SEG + 1) + KCAP * XCH) * 8)

struct LevelArgs {
  TreeDev tree;
  int level, mode;                 // mode 0 = factor, 1 = solve
  const double* Lf; long long lf_stride;
  const int* rank; const int* colofs;
  double* X; long long xstride;    // factor: targets + W live here
  double* Y; int ld; int nrhs; long long ystride;   // solve: targets
  int nf;                          // factor mode: fused rhs columns (0/1)
  double* Ppart; long long pstride_seg; long long pstride_inst;   // [inst][seg][KCAP x ncap]
  double* Sbuf; long long sstride_node; long long sstride_inst;   // [inst][node][SLD x ncap]
  double* Kst; long long kstride_node; long long kstride_inst;    // kept B, C, LU(Sc)
  int* Kpiv; long long pivstride_inst;
  int keep;
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

// ---------------------------------------------------------------------------------------
// One CTA per node.  smem: P_top / P_bot column sums are produced column by column.
__global__ void __launch_bounds__(LVL_THREADS)
k_lvl_node(const LevelArgs a) {
  extern __shared__ double lvl_smem[];
  double* Bm = lvl_smem;
  double* Cm = Bm + KCAP * KCAP;
  double* Sc = Cm + KCAP * KCAP;
  __shared__ int piv[KCAP];
  __shared__ double red[32];
  __shared__ int s_p;
  const TreeDev& tr = a.tree;
  const int jn = blockIdx.x, inst = blockIdx.y, t = threadIdx.x;
  const int l = a.level;
  const int nd = node_index(l, jn);
  const ColRange cr = col_range(a, inst);
  const int k = cr.k;
  const int* nseg = tr.node_seg + 3 * nd;
  const int s0 = nseg[0], s1 = nseg[1], s2 = nseg[2];   // child0 segs [s0,s1), child1 [s1,s2)
  const double* Pi = a.Ppart + (long long)inst * a.pstride_inst;
  double* Ks = a.Kst + (long long)inst * a.kstride_inst + (long long)nd * a.kstride_node;
  int* Kp = a.Kpiv + (long long)inst * a.pivstride_inst + (long long)nd * KCAP;
  // sum of segment partials, fixed order.  top = V12^T X2 (child 1), bot = V21^T X1 (child 0)
  auto psum = [&](int sa, int sb, int q, int col) -> double {
    double s = 0.0;
    for (int sg = sa; sg < sb; ++sg) s += Pi[(long long)sg * a.pstride_seg + q + (long long)col * KCAP];
    return s;
  };
  if (a.mode == 0) {
    const int wc = cr.wb - cr.tb;                          // P column of W's first column
    for (int e = t; e < k * k; e += LVL_THREADS) {
      const int q = e % k, j = e / k;
      Bm[q + j * KCAP] = psum(s1, s2, q, wc + j);          // V12^T W2
      Cm[q + j * KCAP] = psum(s0, s1, q, wc + j);          // V21^T W1
    }
    __syncthreads();
    // Sc = I - C B
    for (int e = t; e < k * k; e += LVL_THREADS) {
      const int i = e % k, j = e / k;
      double s = (i == j) ? 1.0 : 0.0;
      for (int q = 0; q < k; ++q) s -= Cm[i + q * KCAP] * Bm[q + j * KCAP];
      Sc[i + j * KCAP] = s;
    }
    __syncthreads();
    // LU with partial pivoting (row interchanges recorded in piv)
    for (int j = 0; j < k; ++j) {
      if (t < 32) {
        double bv = -1.0; int bi = j;
        for (int i = j + t; i < k; i += 32) {
          const double v = fabs(Sc[i + j * KCAP]);
          if (v > bv) { bv = v; bi = i; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double v2 = __shfl_down_sync(0xffffffffu, bv, o);
          const int i2 = __shfl_down_sync(0xffffffffu, bi, o);
          if (v2 > bv || (v2 == bv && i2 < bi)) { bv = v2; bi = i2; }
        }
        if (t == 0) {
          s_p = bi; piv[j] = bi;
          if (!(bv > 0.0) || !isfinite(bv)) latch_status(a.st, FDE_ESINGULAR, inst * 65536 + 32768 + nd);
        }
      }
      __syncthreads();
      const int p = s_p;
      if (p != j && t < k) {
        const double x = Sc[j + t * KCAP]; Sc[j + t * KCAP] = Sc[p + t * KCAP]; Sc[p + t * KCAP] = x;
      }
      __syncthreads();
      const double pv = Sc[j + j * KCAP];
      for (int i = j + 1 + t; i < k; i += LVL_THREADS) Sc[i + j * KCAP] /= pv;
      __syncthreads();
      for (int e = t; e < (k - j - 1) * (k - j - 1); e += LVL_THREADS) {
        const int i = j + 1 + e % (k - j - 1), jj = j + 1 + e / (k - j - 1);
        Sc[i + jj * KCAP] -= Sc[i + j * KCAP] * Sc[j + jj * KCAP];
      }
      __syncthreads();
    }
    if (a.keep) {
      for (int e = t; e < k * k; e += LVL_THREADS) {
        const int i = e % k, j = e / k;
        Ks[i + j * KLD] = Bm[i + j * KCAP];
        Ks[KLD * KCAP + i + j * KLD] = Cm[i + j * KCAP];
        Ks[2 * KLD * KCAP + i + j * KLD] = Sc[i + j * KCAP];
      }
      if (t < k) Kp[t] = piv[t];
    }
  } else {
    for (int e = t; e < k * k; e += LVL_THREADS) {
      const int i = e % k, j = e / k;
      Bm[i + j * KCAP] = Ks[i + j * KLD];
      Cm[i + j * KCAP] = Ks[KLD * KCAP + i + j * KLD];
      Sc[i + j * KCAP] = Ks[2 * KLD * KCAP + i + j * KLD];
    }
    if (t < k) piv[t] = Kp[t];
  }
  __syncthreads();
  // S = K^{-1} [top; bot] for every target column, one thread per column.
  double* So = a.Sbuf + (long long)inst * a.sstride_inst + (long long)jn * a.sstride_node;
  for (int col = t; col < cr.ntgt; col += LVL_THREADS) {
    double av[KCAP], zv[KCAP];
    for (int q = 0; q < k; ++q) { av[q] = psum(s1, s2, q, col); zv[q] = psum(s0, s1, q, col); }
    // z = b - C a
    for (int i = 0; i < k; ++i) {
      double s = zv[i];
      for (int q = 0; q < k; ++q) s -= Cm[i + q * KCAP] * av[q];
      zv[i] = s;
    }
    // y = Sc^{-1} z : apply row interchanges, unit-lower forward, upper backward
    for (int j = 0; j < k; ++j) { const int p = piv[j]; if (p != j) { double x = zv[j]; zv[j] = zv[p]; zv[p] = x; } }
    for (int i = 1; i < k; ++i) { double s = zv[i]; for (int q = 0; q < i; ++q) s -= Sc[i + q * KCAP] * zv[q]; zv[i] = s; }
    for (int i = k - 1; i >= 0; --i) {
      double s = zv[i];
      for (int q = i + 1; q < k; ++q) s -= Sc[i + q * KCAP] * zv[q];
      zv[i] = s / Sc[i + i * KCAP];
    }
    // top = a - B y
    for (int i = 0; i < k; ++i) {
      double s = av[i];
      for (int q = 0; q < k; ++q) s -= Bm[i + q * KCAP] * zv[q];
      So[i + (long long)col * SLD] = s;
      So[k + i + (long long)col * SLD] = zv[i];
    }
  }
}

// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(LVL_THREADS)
k_lvl_update(const LevelArgs a) {
  extern __shared__ double lvl_smem[];
  double* Ws = lvl_smem;                       // W[row][q]
  double* Ss = lvl_smem + KCAP * (SEG + 1);    // S_half[q][col]
  const TreeDev& tr = a.tree;
  const int seg = blockIdx.x, inst = blockIdx.y, t = threadIdx.x;
  const int l = a.level, n = tr.n;
  const int sg = tr.seg_ofs[l] + seg;
  const int jn = tr.seg_node[sg], c = tr.seg_child[sg];
  const int row0 = tr.seg_row0[sg], len = tr.seg_len[sg];
  const ColRange cr = col_range(a, inst);
  if (cr.ntgt <= 0) return;
  const int k = cr.k;
  const double* Xi = a.X + (long long)inst * a.xstride;
  for (int e = t; e < len * k; e += LVL_THREADS) {
    const int i = e % len, q = e / len;
    Ws[q * (SEG + 1) + i] = Xi[(long long)(cr.wb + q) * n + row0 + i];
  }
  const double* Si = a.Sbuf + (long long)inst * a.sstride_inst + (long long)jn * a.sstride_node
                   + (c == 0 ? 0 : k);                      // child 0 uses S_top, child 1 S_bot
  double* dst;
  long long cstride;
  if (a.mode == 0) { dst = a.X + (long long)inst * a.xstride + (long long)cr.tb * n; cstride = n; }
  else { dst = a.Y + (long long)inst * a.ystride; cstride = a.ld; }
  const int rloc = t & (SEG - 1);                 // row handled by this thread
  const int half = t >> 7;                        // 2 groups of 16 columns
  for (int c0 = 0; c0 < cr.ntgt; c0 += XCH) {
    const int nc = min(XCH, cr.ntgt - c0);
    __syncthreads();
    for (int e = t; e < k * nc; e += LVL_THREADS) {
      const int q = e % k, cc = e / k;
      Ss[q * XCH + cc] = Si[q + (long long)(c0 + cc) * SLD];
    }
    __syncthreads();
    if (rloc < len) {
      double acc[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = 0.0;
      for (int q = 0; q < k; ++q) {
        const double w = Ws[q * (SEG + 1) + rloc];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = fma(w, Ss[q * XCH + half * 16 + j], acc[j]);
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int cc = half * 16 + j;
        if (cc < nc) dst[(long long)(c0 + cc) * cstride + row0 + rloc] -= acc[j];
      }
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
