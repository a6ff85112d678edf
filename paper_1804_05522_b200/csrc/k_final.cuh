// k_final.cuh -- the per-leaf "final" u = X v (v = M_{L-1} .. M_0 e_0 from the kept S blocks of
// every ancestor, k_tree.cuh) and, for the pipelined run (k_run.cuh), the deferred right-hand-side
// column of the next step in the same task: x0 = A_leaf^{-1}(u + dt f) with the stored leaf LU,
// X[:, 0] = x0, Q[:, 0] = V_all^T x0.  Used by k_step (final only) and k_run (B' tasks).
#pragma once
#include "k_leaf.cuh"
#include "k_tree.cuh"

#define RN_FRONT (LEAF_MAX + NCOL_MAX + 4 * LEAF_MAX + 32)   // b | v | part[4] | z

// Block copy of an argument struct into shared memory (whole CTA; ends with a barrier).
template <class T>
__device__ __forceinline__ void rn_copy(T* dst, const T* src) {
  static_assert(sizeof(T) % 8 == 0, "argument block size");
  for (int i = threadIdx.x; i < (int)(sizeof(T) / 8); i += blockDim.x)
    reinterpret_cast<unsigned long long*>(dst)[i] = reinterpret_cast<const unsigned long long*>(src)[i];
  __syncthreads();
}

// B' (and the finals of step K; the k_step finals).  geo: tree geometry; tp = step m-1's tree
// arguments (X^(m-1), S^(m-1), u^(m-1) output) or null at m = 0; la = step m's leaf arguments
// or null at m = K.
// q0 = false (k_run fused BB' task): stop after x0 (left in sm[0, s) and X[:, 0]); the projection
// that follows computes Q[:, 0] with its staged V.
__device__ void leaf_rhs_final(const TrArgs& geo, const TrArgs* tp, const LeafArgs* la, double* sm,
                               int smem_doubles, int inst, int leaf, unsigned long long* prof = nullptr,
                               bool q0 = true) {
  const TrArgs& a = geo;
  long long ph_t = clock64();
#define RN_PH(i) do { if (prof && threadIdx.x == 0) { const long long t_ = clock64(); \
    atomicAdd(prof + (la ? 0 : 8) + (i), (unsigned long long)(t_ - ph_t)); ph_t = t_; } } while (0)
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int L = a.L, n = a.n, NC = a.xc[L];
  const int r0 = a.leaf_r0[leaf], s = a.leaf_n[leaf], sp = round_up(s, 32), nb = sp >> 5;
  double* bs = sm;                                    // b, then x0
  double* vs = bs + LEAF_MAX;                         // v (NC)
  double* part = vs + NCOL_MAX;                       // [4][128]
  double* zs = part + 4 * LEAF_MAX;                   // [32]
  double* LUs = sm + RN_FRONT;                        // [sp cols] column-major, ld = LDA_LEAF
  double* Ss = LUs + LEAF_RSLOT;                      // S_side blocks of a batch of levels
  const int scap = smem_doubles - RN_FRONT - LEAF_RSLOT;
  FDE_ASSERT(s >= 1 && s <= LEAF_MAX && NC <= NCOL_MAX && scap > 0 && r0 + s <= n);
  // ---- the first batch of S blocks, then the stored LU, in flight while the final is formed.
  //      The LU (one contiguous 8 sp^2-byte run) is one bulk copy of the TMA engine (mbarrier
  //      rn_bar[0]) when the run is 16-byte aligned, else cp.async.
  __shared__ unsigned long long rn_bar[1];
  const double* LUg = la ? la->LU + (long long)inst * la->lustride + (long long)leaf * LEAF_RSLOT : nullptr;
  const bool lu_bulk = la && (reinterpret_cast<unsigned long long>(LUg) & 15) == 0;
  if (la && t == 0) {
    mbar_init(rn_bar, 1u);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  auto issue_lu = [&]() {
    if (lu_bulk) {
      if (t == 0) {
        // the previous task's generic accesses of this shared memory, and the LU (written by
        // another CTA, acquired by the scheduler), ordered before the async-proxy copy
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("fence.proxy.async.global;" ::: "memory");
        mbar_expect_tx(rn_bar, (unsigned)(sp * LDA_LEAF * 8));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(LUs)), "l"(LUg), "r"((unsigned)(sp * LDA_LEAF * 8)), "r"(smem_u32(rn_bar)) : "memory");
      }
    } else {
      for (int e = 2 * t; e < sp * LDA_LEAF; e += 2 * LEAF_THREADS) cp_async16(LUs + e, LUg + e);
    }
    cp_async_commit();
  };
  if (tp) {
    // X^(m-1) of the leaf rows (read by u = X v below, after the v recursion) is mostly out of L2
    // by now (written a step earlier): L2 prefetch of its 132 x 16 boxes through the TMA engine
    // (no registers, no shared memory), in flight over the S staging and the v recursion
#ifndef FDE_NO_XPF
    if (tp->xmap && t == 0) {
      for (int c0 = 0; c0 < NC; c0 += 16)
        asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];"
                     ::"l"(tp->xmap), "r"(r0), "r"(c0), "r"(inst) : "memory");
    }
#endif
    // ---- v = M_{L-1} .. M_0 e_0,  M_m: v[m-cols] = -S_side(m) v[< xc_m]   (k_tree.cuh);
    //      S_side(m) (k x xm, row-major in HBM) is staged transposed: lane q reads row q
    //      conflict-free while the warp walks the columns
    for (int c = t; c < NC; c += LEAF_THREADS) vs[c] = c == 0 ? 1.0 : 0.0;
    const double* Sg = tp->Sst + (long long)inst * tp->sinst;
    int m0 = 0;
    bool lu_issued = la == nullptr;
    while (m0 < L) {
      // a batch of levels whose S_side blocks (k x xm row-major, one contiguous run each in HBM)
      // fit behind the LU; staged with 16-byte copies
      int m1 = m0, used = 0;
      while (m1 < L) {
        const int sz = round_up((a.xc[m1 + 1] - a.xc[m1]) * a.xc[m1] + 2, 2);
        if (m1 > m0 && used + sz > scap) break;
        used += sz; ++m1;
      }
      auto S_src = [&](int m) {
        const int xm = a.xc[m], k = a.xc[m + 1] - xm;
        const int jn = leaf >> (L - m), side = (leaf >> (L - m - 1)) & 1;
        return Sg + a.slev[m] + (long long)jn * 2 * k * xm + (long long)side * k * xm;
      };
      int o = 0;
      for (int m = m0; m < m1; ++m) {
        const int xm = a.xc[m], k = a.xc[m + 1] - xm;
        cp_contig(Ss + o, S_src(m), k * xm, t, LEAF_THREADS);
        o += round_up(k * xm + 2, 2);
      }
      FDE_ASSERT(o <= scap);
      cp_async_commit();
      if (!lu_issued) { issue_lu(); lu_issued = true; RN_PH(6); cp_async_wait_group1(); } else { RN_PH(6); cp_async_wait_all(); }
      __syncthreads();
      RN_PH(1);
      {                                               // lane = row q of S_side, warp = column slice
        int o2 = 0;
        double* vp = part;                            // [8 warps][32 rows] partial sums
        for (int m = m0; m < m1; ++m) {
          const int xm = a.xc[m], k = a.xc[m + 1] - xm;
          const double* St = cp_contig_dst(Ss + o2, S_src(m));   // [k][xm]
          const int cw = (xm + LEAF_WARPS - 1) / LEAF_WARPS, c0 = warp * cw, c1 = min(xm, c0 + cw);
          for (int q0 = 0; q0 < k; q0 += 32) {
            const int q = q0 + lane;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            if (q < k) {
              const double* sr = St + q * xm;
              int c = c0;
#pragma unroll 2
              for (; c + 3 < c1; c += 4) {
                a0 = fma(sr[c], vs[c], a0); a1 = fma(sr[c + 1], vs[c + 1], a1);
                a2 = fma(sr[c + 2], vs[c + 2], a2); a3 = fma(sr[c + 3], vs[c + 3], a3);
              }
              for (; c < c1; ++c) a0 = fma(sr[c], vs[c], a0);
            }
            vp[warp * 32 + lane] = (a0 + a1) + (a2 + a3);
            __syncthreads();
            if (t < 32 && q0 + t < k) {
              double v = 0.0;
#pragma unroll
              for (int w = 0; w < LEAF_WARPS; ++w) v += vp[w * 32 + t];
              vs[xm + q0 + t] = -v;
            }
            __syncthreads();
          }
          o2 += round_up(k * xm + 2, 2);
        }
      }
      __syncthreads();
      RN_PH(2);
      m0 = m1;
    }
    // ---- u^(m-1) = X^(m-1) v on the leaf rows: 2 rows per thread (16-byte loads, 16 in flight),
    //      4 column quarters, fixed-order sums
    {
      const int i2 = 2 * (t & 63), h = t >> 6;
      const double* Xi = tp->X + (long long)inst * tp->xstride + r0 + i2;
      const bool vec = ((r0 | n | tp->xstride) & 1) == 0;   // 16-byte aligned row pairs
      double ac0[4] = {0.0, 0.0, 0.0, 0.0}, ac1[4] = {0.0, 0.0, 0.0, 0.0};
      if (i2 < s) {                                   // (X is written in this launch: coherent loads)
        int c = h;
        if (vec && i2 + 1 < s) {
          for (; c < NC; c += 4 * 24) {               // 24 x 16-byte loads in flight per thread
            double2 x[24];
#pragma unroll
            for (int u = 0; u < 24; ++u)
              x[u] = c + 4 * u < NC ? *reinterpret_cast<const double2*>(Xi + (long long)(c + 4 * u) * n)
                                    : make_double2(0.0, 0.0);
#pragma unroll
            for (int u = 0; u < 24; ++u) {
              const double vv = c + 4 * u < NC ? vs[c + 4 * u] : 0.0;
              ac0[u & 3] = fma(x[u].x, vv, ac0[u & 3]);
              ac1[u & 3] = fma(x[u].y, vv, ac1[u & 3]);
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
    }
    __syncthreads();
    RN_PH(3);
    if (t < s) {
      const double u = (part[t] + part[LEAF_MAX + t]) + (part[2 * LEAF_MAX + t] + part[3 * LEAF_MAX + t]);
      tp->u[(long long)inst * n + r0 + t] = u;
      if (la) bs[t] = u + la->dt * la->f[(long long)inst * n + r0 + t];
    }
  } else {
    if (la) issue_lu();
    if (t < s) bs[t] = la->u_prev[(long long)inst * n + r0 + t] + la->dt * la->f[(long long)inst * n + r0 + t];
  }
  if (!la) return;
  if (t >= s && t < sp) bs[t] = 0.0;
  cp_async_wait_all();
  if (lu_bulk) mbar_wait(rn_bar, 0);
  __syncthreads();
  RN_PH(4);
  // ---- x0 = A_leaf^{-1} b with the stored LU (k_leaf.cuh inverse-diagonal form, ld LDA_LEAF: off-diagonal
  //      blocks hold -Lt / -Ut, diagonal blocks D_k = A_kk^{-1}); 2 column halves per row
  const int i = t & 127, h = t >> 7;
  for (int kb = 0; kb + 1 < nb; ++kb) {              // forward: y_i += (-Lt_ik) y_k
    const int c0 = 32 * kb + 16 * h;
    double acc = 0.0;
    if (i >= 32 * (kb + 1) && i < sp)
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) acc = fma(LUs[i + (c0 + jj) * LDA_LEAF], bs[c0 + jj], acc);
    part[h * LEAF_MAX + i] = acc;
    __syncthreads();
    if (t < sp && t >= 32 * (kb + 1)) bs[t] += part[t] + part[LEAF_MAX + t];
    __syncthreads();
  }
  for (int kb = nb - 1; kb >= 0; --kb) {             // backward: x_k = D_k y_k, y_j += (-Ut_jk) y_k
    if (t < 32) zs[t] = bs[32 * kb + t];
    __syncthreads();
    const int c0 = 32 * kb + 16 * h;
    double acc = 0.0;
    if (i < 32 * (kb + 1))
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) acc = fma(LUs[i + (c0 + jj) * LDA_LEAF], zs[16 * h + jj], acc);
    part[h * LEAF_MAX + i] = acc;
    __syncthreads();
    if (t < 32 * (kb + 1)) {
      const double v = part[t] + part[LEAF_MAX + t];
      bs[t] = t >= 32 * kb ? v : bs[t] + v;
    }
    __syncthreads();
  }
  RN_PH(5);
  double* X0 = la->X + (long long)inst * la->xstride + r0;
  if (t < s) X0[t] = bs[t];
  if (!q0) {
    if (prof) { __syncthreads(); RN_PH(0); }
    __syncthreads();                                  // (barriers free; x0 stays in bs = sm[0, s))
    if (t == 0) mbar_inval(rn_bar);
    return;
  }
  PanelCol* pcq = reinterpret_cast<PanelCol*>(Ss);   // V-column descriptors (NC - 1)
  for (int j = t; j < NC - 1; j += LEAF_THREADS) pcq[j] = panel_col(*la, inst, leaf, r0, 1 + j, NC);
  __syncthreads();
  // ---- Q[j][0] = V_all[:, j]^T x0: a warp per QG V columns, lanes over rows (fixed order)
  double* Qo = la->Q + (long long)inst * la->qinst + (long long)leaf * la->qstride;
  double xr[LEAF_MAX / 32];
#pragma unroll
  for (int q = 0; q < LEAF_MAX / 32; ++q) xr[q] = lane + 32 * q < s ? bs[lane + 32 * q] : 0.0;
  constexpr int QG = 9;                               // V columns per warp pass (36 loads in flight)
  for (int j0 = QG * warp; j0 < NC - 1; j0 += QG * LEAF_WARPS) {
    double vv[QG][LEAF_MAX / 32];
#pragma unroll
    for (int jj = 0; jj < QG; ++jj) {
      const PanelCol pc = j0 + jj < NC - 1 ? pcq[j0 + jj] : PanelCol{la->Lf, 0, 0, 0, 0, 0};
#pragma unroll
      for (int q = 0; q < LEAF_MAX / 32; ++q) {
        const int r = lane + 32 * q, rc = r < s ? r : s - 1;
        const double x = __ldg(pc.Lq + pc.li0 + pc.lstep * rc);   // (valid address for any kind)
        vv[jj][q] = pc.kind == 2 ? x : (pc.kind == 3 && pc.li0 + pc.lstep * r == 0 ? 1.0 : 0.0);
      }
    }
#pragma unroll
    for (int jj = 0; jj < QG; ++jj) {
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < LEAF_MAX / 32; ++q) v = fma(vv[jj][q], xr[q], v);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && j0 + jj < NC - 1) Qo[(long long)(j0 + jj) * NC] = v;
    }
  }
  __syncthreads();                                    // (barriers and shared memory free)
  if (t == 0) mbar_inval(rn_bar);
  if (prof) { __syncthreads(); RN_PH(0); }
}

