// k_matvec.cuh -- y = A x with the HODLR representation of
//   A = shift I + c (D+ T + D- T^T)                        (Eq. 2.5)
// (O(k N log N) product).  Leaves: dense blocks regenerated from g, d+-;
// off-diagonal blocks: y1 += U12 (V12^T x2), y2 += U21 (V21^T x1) level by level, with
// U12 = [-c D- J L_l, -c d+[r0+n1-1] e_{n1-1}], U21 = [-c D+ L_l, -c d-[r0+n1] e_0]
// (the same factors the factorisation uses, see k_leaf.cuh / k_level.cuh).
// Used by the extended Krylov method of the 2D solver (A U products) and
// for residual monitoring.
#pragma once
#include "fde_common.cuh"
#include "k_leaf.cuh"

#define MV_THREADS 256
#define MV_NC 32
#define MV_LEAF_SMEM ((LEAF_MAX * LDA_LEAF + 2 * MV_NC * LDP_LEAF) * 8)
#define SMEM_MV_UPDATE ((KCAP * NRHS_MAX) * 8)

struct MvArgs {
  TreeDev tree;
  int level;
  double shift;
  const double* cfac;
  const double* g; long long gstride;
  const double* dp; const double* dm;
  const double* Lf; long long lf_stride;
  const int* rank;
  const double* x; double* y; int nrhs; int ld; long long ystride;
  const double* Ppart; long long pstride_seg; long long pstride_inst;
};

// y_leaf = A_leaf x_leaf (overwrites y)
__global__ void __launch_bounds__(MV_THREADS)
k_mv_leaf(const MvArgs a) {
  extern __shared__ double smem[];
  double* A = smem;
  double* Xs = smem + LEAF_MAX * LDA_LEAF;
  double* Ys = Xs + MV_NC * LDP_LEAF;
  const TreeDev& tr = a.tree;
  const int leaf = blockIdx.x, inst = blockIdx.y, t = threadIdx.x, n = tr.n;
  const int r0 = tr.leaf_r0[leaf], s = tr.leaf_n[leaf];
  const double c = a.cfac[inst];
  const double* gi = a.g + (long long)inst * a.gstride;
  const double* dpi = a.dp + (long long)inst * n + r0;
  const double* dmi = a.dm + (long long)inst * n + r0;
  const int sp = round_up(s, 8);                  // zero padded for the DMMA tiles
  for (int e = t; e < sp * sp; e += MV_THREADS) {
    const int i = e % sp, j = e / sp;
    double v = 0.0;
    if (i < s && j < s) {
      const int k1 = i - j + 1, k2 = j - i + 1;
      const double tij = (k1 >= 0) ? -gi[k1] : 0.0;
      const double tji = (k2 >= 0) ? -gi[k2] : 0.0;
      // stored negated: cm_gemm_sub accumulates C -= A B, so C = (-A) x = A x
      v = -((i == j ? a.shift : 0.0) + c * (dpi[i] * tij + dmi[i] * tji));
    }
    A[i + j * LDA_LEAF] = v;
  }
  const long long ib = (long long)inst * a.ystride;
  for (int c0 = 0; c0 < a.nrhs; c0 += MV_NC) {
    const int nc = min(MV_NC, a.nrhs - c0), ncp = round_up(nc, 8);
    __syncthreads();
    for (int e = t; e < sp * ncp; e += MV_THREADS) {
      const int i = e % sp, cc = e / sp;
      Xs[i + cc * LDP_LEAF] = (i < s && cc < nc) ? a.x[ib + (long long)(c0 + cc) * a.ld + r0 + i] : 0.0;
      Ys[i + cc * LDP_LEAF] = 0.0;
    }
    __syncthreads();
    cm_gemm_sub(Ys, LDP_LEAF, A, LDA_LEAF, Xs, LDP_LEAF, sp, ncp, sp, 0, MV_THREADS / 32);   // Ys = A x
    __syncthreads();
    for (int e = t; e < s * nc; e += MV_THREADS) {
      const int i = e % s, cc = e / s;
      a.y[ib + (long long)(c0 + cc) * a.ld + r0 + i] = Ys[i + cc * LDP_LEAF];
    }
  }
}

// y[rows of a segment] += U_child (V_other^T x_other) at level a.level
__global__ void __launch_bounds__(MV_THREADS)
k_mv_update(const MvArgs a) {
  extern __shared__ double zs[];                 // [KCAP][nrhs]
  const TreeDev& tr = a.tree;
  const int seg = blockIdx.x, inst = blockIdx.y, t = threadIdx.x, n = tr.n, L = tr.L;
  const int l = a.level;
  const int sg = tr.seg_ofs[l] + seg;
  const int jn = tr.seg_node[sg], ch = tr.seg_child[sg];
  const int row0 = tr.seg_row0[sg], len = tr.seg_len[sg];
  const int nd = node_index(l, jn);
  const int r0n = tr.node_r0[nd], n1 = tr.node_n1[nd];
  const int r = a.rank[inst * L + l], k = r + 1, m = tr.lev_m[l];
  const int* ns = tr.node_seg + 3 * nd;
  const int sa = ch == 0 ? ns[1] : ns[0], sb = ch == 0 ? ns[2] : ns[1];  // the other child
  const double* Pi = a.Ppart + (long long)inst * a.pstride_inst;
  for (int e = t; e < k * a.nrhs; e += MV_THREADS) {
    const int q = e % k, col = e / k;
    double s = 0.0;
    for (int g2 = sa; g2 < sb; ++g2) s += Pi[(long long)g2 * a.pstride_seg + q + (long long)col * KCAP];
    zs[q + col * KCAP] = s;
  }
  __syncthreads();
  const double c = a.cfac[inst];
  const double* Ll = a.Lf + (long long)inst * a.lf_stride + tr.lev_lofs[l];
  const double* dpg = a.dp + (long long)inst * n;
  const double* dmg = a.dm + (long long)inst * n;
  const long long ib = (long long)inst * a.ystride;
  for (int e = t; e < len * a.nrhs; e += MV_THREADS) {
    const int i = e % len, col = e / len;
    const int R = row0 + i;
    double acc = 0.0;
    if (ch == 0) {
      const int j1 = R - r0n;
      const double sc = -c * dmg[R];
      for (int q = 0; q < r; ++q) acc += sc * Ll[(n1 - 1 - j1) + (long long)q * m] * zs[q + col * KCAP];
      if (j1 == n1 - 1) acc += -c * dpg[R] * zs[r + col * KCAP];
    } else {
      const int i2 = R - r0n - n1;
      const double sc = -c * dpg[R];
      for (int q = 0; q < r; ++q) acc += sc * Ll[i2 + (long long)q * m] * zs[q + col * KCAP];
      if (i2 == 0) acc += -c * dmg[R] * zs[r + col * KCAP];
    }
    a.y[ib + (long long)col * a.ld + R] += acc;
  }
}
