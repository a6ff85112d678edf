// k_solve.cuh -- S6 with a kept factor (LU reuse; hodlr_solve and fde1d_step with
// coeffs_changed == 0): the tree-ordered solve as streaming passes.
//
//  k_leaf_apply : y[leaf rows] = A_leaf^{-1} (b + dt f)  with the kept explicit leaf inverse
//                 (k_leaf keep mode stores A_leaf^{-1}, computed by stripe solves of the
//                 identity): one pass over the 128 x 128 inverse, no sequential sweep.
//  k_solve_level: one launch per level l = L-1 .. 0, one CTA per (node, instance):
//                 a = V12^T y2, b = V21^T y1 (fixed-order warp reductions),
//                 y_v = Sc^{-1}(b - C a), top = a - B y_v   (kept B, C, Sc^{-1}, k_levels.cuh),
//                 y1 -= W1 top, y2 -= W2 y_v   (W = the level's panel columns kept in X).
// Per step the factor data are streamed once: HBM-bound by design.
#pragma once
#include "fde_common.cuh"
#include "fde_dmma.cuh"

#define SA_THREADS 256
#define SL_THREADS 256
#define SA_COLS 4                      // right-hand sides per pass of k_leaf_apply
#define SL_WQ 3                        // (q, side) reductions per warp at once (k_solve_level)

struct SaArgs {
  TreeDev tree;
  const double* Ainv; long long lustride;    // [inst][leaf][sp x sp] column-major
  const double* b; const double* f; double dt;
  double* y; int nrhs; int ld;
};

__global__ void __launch_bounds__(SA_THREADS)
k_leaf_apply(const SaArgs a) {
  __shared__ double xs[LEAF_MAX * SA_COLS];
  __shared__ double part[SA_THREADS * SA_COLS];
  const int leaf = blockIdx.x, inst = blockIdx.y, t = threadIdx.x;
  const int r0 = a.tree.leaf_r0[leaf], s = a.tree.leaf_n[leaf], sp = round_up(s, 32);
  const double* Ai = a.Ainv + (long long)inst * a.lustride + (long long)leaf * LEAF_MAX * LEAF_MAX;
  const long long ib = (long long)inst * a.ld * a.nrhs + r0;
  const int i = t % 128, h = t / 128;            // row, half of the j range
  for (int c0 = blockIdx.z * SA_COLS; c0 < a.nrhs; c0 += gridDim.z * SA_COLS) {   // (column groups over grid.z)
    const int nc = min(SA_COLS, a.nrhs - c0);
    for (int e = t; e < s * nc; e += SA_THREADS) {
      const int j = e % s, cc = e / s;
      const long long o = ib + (long long)(c0 + cc) * a.ld + j;
      xs[cc * LEAF_MAX + j] = a.b[o] + (a.f ? a.dt * a.f[o] : 0.0);
    }
    __syncthreads();
    double acc[SA_COLS] = {0.0, 0.0, 0.0, 0.0};
    if (i < s) {
      const int j0 = h * (s / 2), j1 = h ? s : s / 2;
      for (int j = j0; j < j1; ++j) {
        const double av = Ai[(long long)j * sp + i];
#pragma unroll
        for (int cc = 0; cc < SA_COLS; ++cc) acc[cc] = fma(av, xs[cc * LEAF_MAX + j], acc[cc]);
      }
    }
#pragma unroll
    for (int cc = 0; cc < SA_COLS; ++cc) part[cc * SA_THREADS + t] = acc[cc];
    __syncthreads();
    for (int e = t; e < s * nc; e += SA_THREADS) {
      const int r = e % s, cc = e / s;
      a.y[ib + (long long)(c0 + cc) * a.ld + r] = part[cc * SA_THREADS + r] + part[cc * SA_THREADS + 128 + r];
    }
    __syncthreads();
  }
}

// sum_q W[q * n] s[q] for one row of the level's panel columns: 4 loads in flight per step,
// two FMA chains (fixed order; measured: 8 in flight is slower for k_solve_update)
__device__ __forceinline__ double sl_wdot(const double* wr, int n, const double* s, int k) {
  double a0 = 0.0, a1 = 0.0;
  int q = 0;
  for (; q + 3 < k; q += 4) {
    const double w0 = wr[(long long)q * n], w1 = wr[(long long)(q + 1) * n];
    const double w2 = wr[(long long)(q + 2) * n], w3 = wr[(long long)(q + 3) * n];
    a0 = fma(w0, s[q], a0); a1 = fma(w1, s[q + 1], a1);
    a0 = fma(w2, s[q + 2], a0); a1 = fma(w3, s[q + 3], a1);
  }
  for (; q < k; ++q) a0 = fma(wr[(long long)q * n], s[q], a0);
  return a0 + a1;
}

struct SlArgs {
  TreeDev tree;
  int level, k, xcol;                  // level, columns per level (max rank + 1), first X column
  const double* Lf; long long lf_stride;
  const int* rank;
  const double* X; long long xstride;
  const double* Kst; long long kstride_inst, kofs;
  double* Y; int nrhs, ld;
};

// dynamic shared memory: the node's kept B, C, Sc^{-1} (3 k^2 doubles, prefetched by cp.async
// while the dot products run)
__global__ void __launch_bounds__(SL_THREADS, 4)   // (4 CTAs per SM: the right-hand-side loop over grid.z must not raise the register count)
k_solve_level(const SlArgs a) {
  __shared__ double z[2 * KCAP];                 // [a (k) | b (k)]
  __shared__ double sv[2 * KCAP];                // [top (k) | y_v (k)]
  extern __shared__ double Ks[];                 // [B | C | Sc^{-1}] (k x k row-major each)
  const TreeDev& tr = a.tree;
  const int j = blockIdx.x, inst = blockIdx.y, t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int l = a.level, n = tr.n, L = tr.L, k = a.k;
  const int nd = node_index(l, j);
  const int r0 = tr.node_r0[nd], n1 = tr.node_n1[nd], n2 = tr.node_n2[nd];
  const int m = tr.lev_m[l], r = a.rank[inst * L + l];
  const double* Ll = a.Lf + (long long)inst * a.lf_stride + tr.lev_lofs[l];
  const double* Kn = a.Kst + (long long)inst * a.kstride_inst + a.kofs + (long long)j * 3 * k * k;
  const double* W = a.X + (long long)inst * a.xstride + (long long)a.xcol * n;
  FDE_ASSERT(r0 >= 0 && r0 + n1 + n2 <= n && k >= 1 && k <= KCAP && r <= k - 1);
  for (int e = t; e < 3 * k * k; e += SL_THREADS) cp_async8(Ks + e, Kn + e);
  cp_async_commit();
  const double* Bk = Ks;
  const double* Ck = Ks + k * k;
  const double* Si = Ks + 2 * k * k;
  for (int c = blockIdx.z; c < a.nrhs; c += gridDim.z) {   // (right-hand sides over grid.z)
    double* y = a.Y + (long long)inst * a.ld * a.nrhs + (long long)c * a.ld;
    // a_q = V12[:, q]^T y2 (child 2 rows), b_q = V21[:, q]^T y1 (child 1 rows): a warp per
    // SL_WQ items w = (q, side) at once (independent chains, interleaved reductions)
    for (int w0 = warp; w0 < 2 * k; w0 += SL_WQ * (SL_THREADS / 32)) {
      double acc[SL_WQ];
#pragma unroll
      for (int u = 0; u < SL_WQ; ++u) {
        const int w = w0 + u * (SL_THREADS / 32);
        acc[u] = 0.0;
        if (w >= 2 * k) continue;
        const int q = w % k, side = w / k;     // side 0: a (child 2), 1: b (child 1)
        if (q == k - 1) {                      // exact column: single row
          if (lane == 0) acc[u] = side == 0 ? y[r0 + n1] : y[r0 + n1 - 1];
        } else if (q < r) {
          const double* Lq = Ll + (long long)q * m;
          if (side == 0)
            for (int i2 = lane; i2 < n2; i2 += 32) acc[u] = fma(Lq[i2], y[r0 + n1 + i2], acc[u]);
          else
            for (int j1 = lane; j1 < n1; j1 += 32) acc[u] = fma(Lq[n1 - 1 - j1], y[r0 + j1], acc[u]);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int u = 0; u < SL_WQ; ++u) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
      if (lane == 0)
#pragma unroll
        for (int u = 0; u < SL_WQ; ++u) {
          const int w = w0 + u * (SL_THREADS / 32);
          if (w < 2 * k) z[(w / k) * k + w % k] = acc[u];
        }
    }
    cp_async_wait_all();
    __syncthreads();
    if (warp == 0) {                           // y_v = Sc^{-1}(b - C a) ; top = a - B y_v
      for (int q = lane; q < k; q += 32) {
        double acc = z[k + q];
        for (int p = 0; p < k; ++p) acc = fma(-Ck[q * k + p], z[p], acc);
        sv[k + q] = acc;                       // (temporarily b - C a)
      }
      __syncwarp();
      double yv0 = 0.0, yv1 = 0.0;
      {
        const int q0 = lane, q1 = lane + 32;
        if (q0 < k) for (int p = 0; p < k; ++p) yv0 = fma(Si[q0 * k + p], sv[k + p], yv0);
        if (q1 < k) for (int p = 0; p < k; ++p) yv1 = fma(Si[q1 * k + p], sv[k + p], yv1);
        __syncwarp();
        if (q0 < k) sv[k + q0] = yv0;
        if (q1 < k) sv[k + q1] = yv1;
      }
      __syncwarp();
      for (int q = lane; q < k; q += 32) {
        double acc = z[q];
        for (int p = 0; p < k; ++p) acc = fma(-Bk[q * k + p], sv[k + p], acc);
        sv[q] = acc;
      }
    }
    __syncthreads();
    // y1 -= W1 top (child 1 rows), y2 -= W2 y_v (child 2 rows): 4 W loads in flight per step
    for (int R = r0 + t; R < r0 + n1 + n2; R += SL_THREADS) {
      const double* s = R < r0 + n1 ? sv : sv + k;
      y[R] -= sl_wdot(W + R, n, s, k);
    }
    __syncthreads();
  }
}

// ---- the same level step split over several CTAs per node (levels with fewer nodes than SMs):
//   k_solve_dots  : CTA (node, chunk) -> partial a, b over its rows of the node   [2k per CTA]
//   k_solve_small : CTA per node -> fixed-order sum of the chunks, the K solve -> sv [2k]
//   k_solve_update: CTA (node, chunk) -> y1 -= W1 top, y2 -= W2 y_v on its rows
// Rows of a node [r0, r0 + n1 + n2) are cut into `nch` equal chunks; a chunk may straddle the
// child boundary (each row uses its own child's factor).  Right-hand side c = blockIdx.z.
struct SlSplitArgs {
  SlArgs a;
  int nch;
  double* part;      // [inst][node][chunk][2 KCAP] per rhs slice (c handled sequentially by grid.z)
  double* sv;        // [inst][node][2 KCAP] per rhs
  int c;             // current right-hand side
};

__global__ void __launch_bounds__(SL_THREADS)
k_solve_dots(const SlSplitArgs sp) {
  const SlArgs& a = sp.a;
  const TreeDev& tr = a.tree;
  const int j = blockIdx.x / sp.nch, ch = blockIdx.x % sp.nch, inst = blockIdx.y, t = threadIdx.x;
  const int warp = t >> 5, lane = t & 31;
  const int l = a.level, L = tr.L, k = a.k;
  const int nd = node_index(l, j);
  const int r0 = tr.node_r0[nd], n1 = tr.node_n1[nd], n2 = tr.node_n2[nd], nn = n1 + n2;
  const int m = tr.lev_m[l], r = a.rank[inst * L + l];
  const double* Ll = a.Lf + (long long)inst * a.lf_stride + tr.lev_lofs[l];
  const double* y = a.Y + (long long)inst * a.ld * a.nrhs + (long long)sp.c * a.ld;
  const int cs = (int)((long long)nn * ch / sp.nch), ce = (int)((long long)nn * (ch + 1) / sp.nch);
  double* P = sp.part + (((long long)inst * (1 << l) + j) * sp.nch + ch) * 2 * KCAP;
  // warp per (q, side) as k_solve_level, over this chunk's rows of the side's child
  for (int w = warp; w < 2 * k; w += SL_THREADS / 32) {
    const int q = w % k, side = w / k;         // side 0: a (child 2 rows), 1: b (child 1 rows)
    double acc = 0.0;
    if (side == 0) {
      const int lo = max(cs, n1), hi = ce;     // node-local rows of child 2 in the chunk
      if (q == k - 1) { if (lane == 0 && lo <= n1 && n1 < hi) acc = y[r0 + n1]; }
      else if (q < r) {
        const double* Lq = Ll + (long long)q * m;
        for (int i = lo + lane; i < hi; i += 32) acc = fma(Lq[i - n1], y[r0 + i], acc);
      }
    } else {
      const int lo = cs, hi = min(ce, n1);     // rows of child 1 in the chunk
      if (q == k - 1) { if (lane == 0 && lo <= n1 - 1 && n1 - 1 < hi) acc = y[r0 + n1 - 1]; }
      else if (q < r) {
        const double* Lq = Ll + (long long)q * m;
        for (int i = lo + lane; i < hi; i += 32) acc = fma(Lq[n1 - 1 - i], y[r0 + i], acc);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) P[side * k + q] = acc;
  }
}

__global__ void k_solve_small(const SlSplitArgs sp) {
  const SlArgs& a = sp.a;
  __shared__ double z[2 * KCAP], sv[2 * KCAP];
  const int j = blockIdx.x, inst = blockIdx.y, lane = threadIdx.x, k = a.k;
  const double* P = sp.part + ((long long)inst * (1 << a.level) + j) * sp.nch * 2 * KCAP;
  for (int q = lane; q < 2 * k; q += 32) {
    double v = 0.0;
    for (int c = 0; c < sp.nch; ++c) v += P[(long long)c * 2 * KCAP + q];
    z[q] = v;
  }
  __syncwarp();
  const double* Kn = a.Kst + (long long)inst * a.kstride_inst + a.kofs + (long long)j * 3 * k * k;
  const double* Bk = Kn;
  const double* Ck = Kn + k * k;
  const double* Si = Kn + 2 * k * k;
  for (int q = lane; q < k; q += 32) {
    double acc = z[k + q];
    for (int p = 0; p < k; ++p) acc = fma(-Ck[q * k + p], z[p], acc);
    sv[k + q] = acc;
  }
  __syncwarp();
  double yv0 = 0.0, yv1 = 0.0;
  const int q0 = lane, q1 = lane + 32;
  if (q0 < k) for (int p = 0; p < k; ++p) yv0 = fma(Si[q0 * k + p], sv[k + p], yv0);
  if (q1 < k) for (int p = 0; p < k; ++p) yv1 = fma(Si[q1 * k + p], sv[k + p], yv1);
  __syncwarp();
  if (q0 < k) sv[k + q0] = yv0;
  if (q1 < k) sv[k + q1] = yv1;
  __syncwarp();
  for (int q = lane; q < k; q += 32) {
    double acc = z[q];
    for (int p = 0; p < k; ++p) acc = fma(-Bk[q * k + p], sv[k + p], acc);
    sv[q] = acc;
  }
  __syncwarp();
  double* S = sp.sv + ((long long)inst * (1 << a.level) + j) * 2 * KCAP;
  for (int q = lane; q < 2 * k; q += 32) S[q] = sv[q];
}

__global__ void __launch_bounds__(SL_THREADS)
k_solve_update(const SlSplitArgs sp) {
  const SlArgs& a = sp.a;
  __shared__ double sv[2 * KCAP];
  const TreeDev& tr = a.tree;
  const int j = blockIdx.x / sp.nch, ch = blockIdx.x % sp.nch, inst = blockIdx.y, t = threadIdx.x;
  const int l = a.level, n = tr.n, k = a.k;
  const int nd = node_index(l, j);
  const int r0 = tr.node_r0[nd], n1 = tr.node_n1[nd], n2 = tr.node_n2[nd], nn = n1 + n2;
  const double* S = sp.sv + ((long long)inst * (1 << l) + j) * 2 * KCAP;
  for (int q = t; q < 2 * k; q += SL_THREADS) sv[q] = S[q];
  __syncthreads();
  const double* W = a.X + (long long)inst * a.xstride + (long long)a.xcol * n;
  double* y = a.Y + (long long)inst * a.ld * a.nrhs + (long long)sp.c * a.ld;
  const int cs = (int)((long long)nn * ch / sp.nch), ce = (int)((long long)nn * (ch + 1) / sp.nch);
  for (int i = cs + t; i < ce; i += SL_THREADS) {
    const int R = r0 + i;
    const double* s = i < n1 ? sv : sv + k;
    y[R] -= sl_wdot(W + R, n, s, k);
  }
}
