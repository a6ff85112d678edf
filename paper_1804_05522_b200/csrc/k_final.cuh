// k_final.cuh -- the per-leaf "final" u = X v (v = M_{L-1} .. M_0 e_0 from the kept S blocks of
// every ancestor, k_tree.cuh) and, for the pipelined run (k_run.cuh), the deferred right-hand-side
// column of the next step in the same task: x0 = A_leaf^{-1}(u + dt f) with the stored leaf LU,
// X[:, 0] = x0, Q[:, 0] = V_all^T x0.  Used by k_step (final only) and k_run (B' tasks).
#pragma once
#include "k_leaf.cuh"
#include "k_tree.cuh"


// Block copy of an argument struct into shared memory (whole CTA; ends with a barrier).
template <class T>
__device__ __forceinline__ void rn_copy(T* dst, const T* src) {
  static_assert(sizeof(T) % 8 == 0, "argument block size");
  for (int i = threadIdx.x; i < (int)(sizeof(T) / 8); i += blockDim.x)
    reinterpret_cast<unsigned long long*>(dst)[i] = reinterpret_cast<const unsigned long long*>(src)[i];
  __syncthreads();
}

// v-recursion rows of one level m for the leaf side given by `leaf`: stage S_side(m) (k x xm,
// row-major in HBM) transposed with an odd pitch into Ss, then v[xm + q] = -S_side(m)[q, :] v[:xm]
// (lane = row q, warp = column slice, partial sums through `part`).  Whole CTA.
__device__ __forceinline__ void rn_v_level(const TrArgs& a, const double* Sg, int m, int leaf,
                                           double* Ss, double* v, double* part) {
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31, L = a.L;
  const int xm = a.xc[m], k = a.xc[m + 1] - xm, kp = k | 1;
  const int cw = (xm + LEAF_WARPS - 1) / LEAF_WARPS, c0 = warp * cw, c1 = min(xm, c0 + cw);
  (void)L;
  for (int q0 = 0; q0 < k; q0 += 32) {
    const int q = q0 + lane;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (q < k) {
      int c = c0;
#pragma unroll 2
      for (; c + 3 < c1; c += 4) {
        a0 = fma(Ss[c * kp + q], v[c], a0); a1 = fma(Ss[(c + 1) * kp + q], v[c + 1], a1);
        a2 = fma(Ss[(c + 2) * kp + q], v[c + 2], a2); a3 = fma(Ss[(c + 3) * kp + q], v[c + 3], a3);
      }
      for (; c < c1; ++c) a0 = fma(Ss[c * kp + q], v[c], a0);
    }
    part[warp * 32 + lane] = (a0 + a1) + (a2 + a3);
    __syncthreads();
    if (t < 32 && q0 + t < k) {
      double w = 0.0;
#pragma unroll
      for (int ww = 0; ww < LEAF_WARPS; ++ww) w += part[ww * 32 + t];
      v[xm + q0 + t] = -w;
    }
    __syncthreads();
  }
}

// Issue the transposed copies of S_side(m) for `leaf` into Ss (odd pitch); returns the size.
__device__ __forceinline__ int rn_issue_s(const TrArgs& a, const double* Sg, int m, int leaf, double* Ss) {
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31, L = a.L;
  const int xm = a.xc[m], k = a.xc[m + 1] - xm;
  const int jn = leaf >> (L - m), side = (leaf >> (L - m - 1)) & 1;
  const double* gp = Sg + a.slev[m] + (long long)jn * 2 * k * xm + (long long)side * k * xm;
  (void)t;
  for (int q = warp; q < k; q += LEAF_WARPS)
    for (int c = lane; c < xm; c += 32) cp_async8(Ss + c * (k | 1) + q, gp + q * xm + c);
  return (k | 1) * xm;
}

// B' for a PAIR of sibling leaves (leaf0, leaf0 + 1) -- and the finals of step K.  The two
// leaves share every ancestor below their level-(L-1) parent, so the S blocks and the
// v recursion of levels 0 .. L-2 are staged and computed once; level L-1 differs only in the
// side.  geo: tree geometry; tp = step m-1's tree arguments (X^(m-1), S^(m-1), u^(m-1) output)
// or null at m = 0; la = step m's leaf arguments or null at m = K.
#define RN_FRONT (LEAF_MAX + 2 * NCOL_MAX + 4 * LEAF_MAX + 32)   // b | v0 | v1 | part[4] | z
__device__ void leaf_rhs_final_pair(const TrArgs& geo, const TrArgs* tp, const LeafArgs* la, double* sm,
                                    int smem_doubles, int inst, int leaf0, unsigned long long* prof = nullptr) {
  const TrArgs& a = geo;
  long long ph_t = clock64();
#define RN_PH(i) do { if (prof && threadIdx.x == 0) { const long long t_ = clock64(); \
    atomicAdd(prof + (la ? 0 : 8) + (i), (unsigned long long)(t_ - ph_t)); ph_t = t_; } } while (0)
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int L = a.L, n = a.n, NC = a.xc[L];
  double* bs = sm;                                    // b, then x0
  double* vv2[2] = {bs + LEAF_MAX, bs + LEAF_MAX + NCOL_MAX};   // v of the two sides
  double* part = bs + LEAF_MAX + 2 * NCOL_MAX;        // [4][128]
  double* zs = part + 4 * LEAF_MAX;                   // [32]
  double* LUs = sm + RN_FRONT;                        // [sp x sp] column-major, ld = sp
  double* Ss = LUs + LEAF_MAX * LEAF_MAX;             // S blocks of a batch of levels
  PanelCol* pcd = reinterpret_cast<PanelCol*>(Ss);   // then: V-column descriptors (NC - 1)
  const int scap = smem_doubles - RN_FRONT - LEAF_MAX * LEAF_MAX;
  auto issue_lu = [&](int leaf) {
    const int sp = round_up(a.leaf_n[leaf], 32);
    const double* LUg = la->LU + (long long)inst * la->lustride + (long long)leaf * LEAF_SLOT;
    for (int e = 2 * t; e < sp * sp; e += 2 * LEAF_THREADS) cp_async16(LUs + e, LUg + e);
    cp_async_commit();
  };
  bool lu_pending = false;
  if (tp) {
    // ---- shared levels 0 .. L-2 (batched by shared-memory capacity), then the two sides of L-1
    double* v0 = vv2[0];
    for (int c = t; c < NC; c += LEAF_THREADS) v0[c] = c == 0 ? 1.0 : 0.0;
    const double* Sg = tp->Sst + (long long)inst * tp->sinst;
    int m0 = 0;
    while (m0 < L - 1) {
      int m1 = m0, used = 0;
      while (m1 < L - 1) {
        const int sz = ((a.xc[m1 + 1] - a.xc[m1]) | 1) * a.xc[m1];
        if (m1 > m0 && used + sz > scap) break;
        used += sz; ++m1;
      }
      int o = 0;
      for (int m = m0; m < m1; ++m) o += rn_issue_s(a, Sg, m, leaf0, Ss + o);
      cp_async_commit();
      RN_PH(6);
      cp_async_wait_all();
      __syncthreads();
      RN_PH(1);
      o = 0;
      for (int m = m0; m < m1; ++m) {
        rn_v_level(a, Sg, m, leaf0, Ss + o, v0, part);
        o += ((a.xc[m + 1] - a.xc[m]) | 1) * a.xc[m];
      }
      RN_PH(2);
      m0 = m1;
    }
    {                                                 // level L-1: one block per side
      const int m = L - 1, szl = ((a.xc[m + 1] - a.xc[m]) | 1) * a.xc[m];
      rn_issue_s(a, Sg, m, leaf0, Ss);
      rn_issue_s(a, Sg, m, leaf0 + 1, Ss + szl);
      cp_async_commit();
      if (la) { issue_lu(leaf0); lu_pending = true; cp_async_wait_group1(); }   // (LU stays in flight)
      else cp_async_wait_all();
      for (int c = t; c < a.xc[m]; c += LEAF_THREADS) vv2[1][c] = v0[c];
      __syncthreads();
      rn_v_level(a, Sg, m, leaf0, Ss, v0, part);
      rn_v_level(a, Sg, m, leaf0 + 1, Ss + szl, vv2[1], part);
      RN_PH(2);
    }
  } else if (la) {
    issue_lu(leaf0);
    lu_pending = true;
  }
  for (int side = 0; side < 2; ++side) {
    const int leaf = leaf0 + side;
    const int r0 = a.leaf_r0[leaf], s = a.leaf_n[leaf], sp = round_up(s, 32), nb = sp >> 5;
    const double* vs = vv2[side];
    if (tp) {
      // ---- u^(m-1) = X^(m-1) v on the leaf rows: 2 rows per thread (16-byte loads, 24 in
      //      flight), 4 column quarters, fixed-order sums
      const int i2 = 2 * (t & 63), h = t >> 6;
      const double* Xi = tp->X + (long long)inst * tp->xstride + r0 + i2;
      const bool vec = ((r0 | n | tp->xstride) & 1) == 0;   // 16-byte aligned row pairs
      double ac0[4] = {0.0, 0.0, 0.0, 0.0}, ac1[4] = {0.0, 0.0, 0.0, 0.0};
      if (i2 < s) {                                   // (X is written in this launch: coherent loads)
        int c = h;
        if (vec && i2 + 1 < s) {
          for (; c < NC; c += 4 * 24) {
            double2 x[24];
#pragma unroll
            for (int u = 0; u < 24; ++u)
              x[u] = c + 4 * u < NC ? *reinterpret_cast<const double2*>(Xi + (long long)(c + 4 * u) * n)
                                    : make_double2(0.0, 0.0);
#pragma unroll
            for (int u = 0; u < 24; ++u) {
              const double w = c + 4 * u < NC ? vs[c + 4 * u] : 0.0;
              ac0[u & 3] = fma(x[u].x, w, ac0[u & 3]);
              ac1[u & 3] = fma(x[u].y, w, ac1[u & 3]);
            }
          }
        } else {
          for (; c < NC; c += 4) {
            ac0[0] = fma(Xi[(long long)c * n], vs[c], ac0[0]);
            if (i2 + 1 < s) ac1[0] = fma(Xi[(long long)c * n + 1], vs[c], ac1[0]);
          }
        }
      }
      part[h * LEAF_MAX + i2] = (ac0[0] + ac0[1]) + (ac0[2] + ac0[3]);
      part[h * LEAF_MAX + i2 + 1] = (ac1[0] + ac1[1]) + (ac1[2] + ac1[3]);
      __syncthreads();
      RN_PH(3);
      if (t < s) {
        const double u = (part[t] + part[LEAF_MAX + t]) + (part[2 * LEAF_MAX + t] + part[3 * LEAF_MAX + t]);
        tp->u[(long long)inst * n + r0 + t] = u;
        if (la) bs[t] = u + la->dt * la->f[(long long)inst * n + r0 + t];
      }
    } else if (la && t < s) {
      bs[t] = la->u_prev[(long long)inst * n + r0 + t] + la->dt * la->f[(long long)inst * n + r0 + t];
    }
    if (!la) { __syncthreads(); continue; }
    if (t >= s && t < sp) bs[t] = 0.0;
    cp_async_wait_all();
    __syncthreads();
    RN_PH(4);
    // ---- x0 = A_leaf^{-1} b with the stored LU (k_leaf.cuh inverse-diagonal form: off-diagonal
    //      blocks hold -Lt / -Ut, diagonal blocks D_k = A_kk^{-1}); 2 column halves per row
    const int i = t & 127, h = t >> 7;
    for (int kb = 0; kb + 1 < nb; ++kb) {            // forward: y_i += (-Lt_ik) y_k
      const int c0 = 32 * kb + 16 * h;
      double acc = 0.0;
      if (i >= 32 * (kb + 1) && i < sp)
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) acc = fma(LUs[i + (c0 + jj) * sp], bs[c0 + jj], acc);
      part[h * LEAF_MAX + i] = acc;
      __syncthreads();
      if (t < sp && t >= 32 * (kb + 1)) bs[t] += part[t] + part[LEAF_MAX + t];
      __syncthreads();
    }
    for (int kb = nb - 1; kb >= 0; --kb) {           // backward: x_k = D_k y_k, y_j += (-Ut_jk) y_k
      if (t < 32) zs[t] = bs[32 * kb + t];
      __syncthreads();
      const int c0 = 32 * kb + 16 * h;
      double acc = 0.0;
      if (i < 32 * (kb + 1))
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) acc = fma(LUs[i + (c0 + jj) * sp], zs[16 * h + jj], acc);
      part[h * LEAF_MAX + i] = acc;
      __syncthreads();
      if (t < 32 * (kb + 1)) {
        const double v = part[t] + part[LEAF_MAX + t];
        bs[t] = t >= 32 * kb ? v : bs[t] + v;
      }
      __syncthreads();
    }
    RN_PH(5);
    if (side == 0) issue_lu(leaf0 + 1);               // (the LU region is free again)
    double* X0 = la->X + (long long)inst * la->xstride + r0;
    if (t < s) X0[t] = bs[t];
    for (int j = t; j < NC - 1; j += LEAF_THREADS) pcd[j] = panel_col(*la, inst, leaf, r0, 1 + j, NC);
    __syncthreads();
    // ---- Q[j][0] = V_all[:, j]^T x0: a warp per 6 V columns, lanes over rows (fixed order)
    double* Qo = la->Q + (long long)inst * la->qinst + (long long)leaf * la->qstride;
    double xr[LEAF_MAX / 32];
#pragma unroll
    for (int q = 0; q < LEAF_MAX / 32; ++q) xr[q] = lane + 32 * q < s ? bs[lane + 32 * q] : 0.0;
    constexpr int QG = 6;
    for (int j0 = QG * warp; j0 < NC - 1; j0 += QG * LEAF_WARPS) {
      double vq[QG][LEAF_MAX / 32];
#pragma unroll
      for (int jj = 0; jj < QG; ++jj) {
        const PanelCol pc = j0 + jj < NC - 1 ? pcd[j0 + jj] : PanelCol{la->Lf, 0, 0, 0, 0, 0};
#pragma unroll
        for (int q = 0; q < LEAF_MAX / 32; ++q) {
          const int r = lane + 32 * q, rc = r < s ? r : s - 1;
          const double x = __ldg(pc.Lq + pc.li0 + pc.lstep * rc);   // (valid address for any kind)
          vq[jj][q] = pc.kind == 2 ? x : (pc.kind == 3 && pc.li0 + pc.lstep * r == 0 ? 1.0 : 0.0);
        }
      }
#pragma unroll
      for (int jj = 0; jj < QG; ++jj) {
        double v = 0.0;
#pragma unroll
        for (int q = 0; q < LEAF_MAX / 32; ++q) v = fma(vq[jj][q], xr[q], v);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && j0 + jj < NC - 1) Qo[(long long)(j0 + jj) * NC] = v;
      }
    }
    __syncthreads();                                  // (bs, pcd reused by the next side)
  }
#undef RN_PH
}
