// k_tree.cuh -- S5 + S6 for the fused factor + solve step: the Sherman-Morrison-Woodbury
// level recursion carried out on small projected matrices instead of passes over the panel.
//
// Notation (k_levels.cuh): X^(L) = the leaf-solved panel
// [A_leaf^{-1} b | A_leaf^{-1} U_0 .. U_{L-1}] (k_leaf), X^(m) = the panel after the SMW updates
// of levels L-1 .. m; xc[l] = first panel column of level l (xc[0] = 1: column 0 is the rhs),
// k_l = xc[l+1] - xc[l].  V_l(row) is the level-l V factor row of a row (V21 on child 1 rows,
// V12 on child 2 rows).  For a node mu of level m (or a leaf, m = L):
//     Q_mu = V_{<m}[mu rows]^T X^(m)[mu rows, 0:xc[m]]        ((xc[m]-1) x xc[m]).
// At a node mu of level m with children c1, c2 (level m+1), the level-m rows of Q_c are
//     B = Q_c2[lvl m, m-cols] = V12^T W2,  C = Q_c1[lvl m, m-cols] = V21^T W1,
//     R_top = Q_c2[lvl m, <xc[m]] = V12^T X2,  R_bot = Q_c1[lvl m, <xc[m]] = V21^T X1,
// so the node's K system (K = [[I, B], [C, I]], Sc = I - C B) gives
//     S_bot = Sc^{-1}(R_bot - C R_top),  S_top = R_top - B S_bot,
// the update X1 -= W1 S_top, X2 -= W2 S_bot becomes, projected on the ancestors' V,
//     Q_mu = Q_c1[<, <] + Q_c2[<, <] - Q_c1[<, m-cols] S_top - Q_c2[<, m-cols] S_bot,
// and the solution is  u[leaf rows] = X^(L)[leaf rows, :] v_leaf,  v = M_{L-1} .. M_0 e_0 with
// M_m v: v[m-cols] = -S_side(m) v[<xc[m]]  (side = the child of the level-m node holding the
// leaf).  All arithmetic on (xc x xc)-sized matrices: no pass over the n rows except the
// final u = X v.  Sc is inverted by unpivoted Gauss-Jordan (reading R17).
//
// One persistent cooperative launch: levels L-1 .. 0 separated by grid barriers (work unit
// = node x row chunk of Q_mu; S is recomputed per chunk, stored by chunk 0), then the per-leaf
// v recursion and u = X v.  Every reduction has a fixed order (deterministic).
#pragma once
#include "fde_common.cuh"
#include "fde_dmma.cuh"

#define TR_THREADS 256
#define TR_WARPS (TR_THREADS / 32)

struct TrArgs {
  int L, NC, nleaf, batch, kmaxc;
  int xc[LMAX + 1];
  int rc[LMAX];                  // row chunks per node of level m
  long long qlev[LMAX + 1];      // per-instance offset of level m's Q store (m = 1..L)
  long long slev[LMAX];          // per-instance offset of level m's S store
  long long qinst, sinst;
  const double* Qleaf;           // level-L (leaf) Q store: Q + qlev[L] == Qleaf
  double* Q;                     // Q store of all levels 1..L
  double* Sst;                   // S store: node (m, j): [S_top (k x xc[m]) | S_bot]
  const double* X; long long xstride; int n;
  const void* xmap;              // k_run: TMA map of this X buffer (L2 prefetch of X^(m-1) in B'), or null
  const int* leaf_r0; const int* leaf_n;
  double* u;                     // [batch * n] output
  unsigned* bar;
  DevStatus* st;
  unsigned long long* trace;     // optional: globaltimer after every level (FDE_TRACE_LEVELS)
  double* Kr;                    // k_run split units: node store [C | Sc^{-1} | G] (k x k each) per node, or null
  long long krlev[LMAX], krinst; // per-instance offset of level m's node store, instance stride
  int kp, lds, ldk, lda, rch_max;  // smem geometry (host computed)
  int off_B, off_C, off_M, off_M2, off_S, off_T, off_Z, off_U;
};

__device__ __forceinline__ unsigned tr_ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void tr_grid_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (tr_ld_acquire(bar) < target) __nanosleep(20);
    __threadfence();
  }
  __syncthreads();
}

#define TR_SUB 16                // Q_mu rows per streamed sub-chunk
#define TR_STG 4                 // sub-chunk pipeline stages (3 sub-chunks in flight)
#define TR_MW (TR_SUB / 8)       // m-tiles per sub-chunk
#define TR_NS (8 / TR_MW)        // warps per m-tile (n-tile stride)
#define TR_NT (24 / TR_NS)       // n-tiles per warp in the Q update (24 n-tiles = 192 columns)

// O[q][c] = Cin[q][c] + sgn * sum_p A[q][p] B[p][c]  (q < M, c < N; Cin may be null = 0).
// Row-major shared-memory operands.  A warp item = 4 rows x 32 consecutive columns (lane =
// column: conflict-free B / Cin / O accesses, broadcast A loads), four independent FMA chains.
__device__ __forceinline__ void tr_mm(double* O, int ldo, const double* Cin, int ldci, const double* A,
                                      int lda, const double* B, int ldb, int M, int N, int K, double sgn,
                                      double diag_add = 0.0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int MQ = (M + 3) >> 2, NG = (N + 31) >> 5;
  for (int it = warp; it < MQ * NG; it += TR_WARPS) {
    const int q0 = (it / NG) * 4, c = (it % NG) * 32 + lane;
    const bool cok = c < N;
    double v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      v[i] = ((Cin && cok && q0 + i < M) ? Cin[(q0 + i) * ldci + c] : 0.0) + (q0 + i == c ? diag_add : 0.0);
#pragma unroll 2
    for (int p = 0; p < K; ++p) {
      const double bv = cok ? B[p * ldb + c] : 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i) v[i] = fma(sgn * A[min(q0 + i, M - 1) * lda + p], bv, v[i]);
    }
    if (cok)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (q0 + i < M) O[(q0 + i) * ldo + c] = v[i];
  }
}


// O[q][c] = Cin[q][c] (+ diag_add on q == c) + sgn * sum_p A[q][p] B[p][c] on the FP64 tensor
// cores (DMMA m8n8k4): row-major shared-memory operands, out-of-range rows / columns / K
// entries read as zero (bounds-checked fragments).  Warp item = one m-tile x up to 4 n-tiles
// (A fragment reused); items over all warps of the CTA.  No barrier inside.
__device__ __forceinline__ void tr_dmma(double* O, int ldo, const double* Cin, int ldci, const double* A,
                                        int lda, const double* B, int ldb, int M, int N, int K, double sgn,
                                        double diag_add = 0.0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
  const int MT = (M + 7) >> 3, NT = (N + 7) >> 3, NG = (NT + 3) >> 2;
  for (int it = warp; it < MT * NG; it += TR_WARPS) {
    const int mt = it % MT, ng = it / MT;
    const int q = 8 * mt + gid;
    double d[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = 8 * (4 * ng + u) + 2 * tig;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const bool in = q < M && c + h < N;
        d[u][h] = in ? ((Cin ? Cin[q * ldci + c + h] : 0.0) + (q == c + h ? diag_add : 0.0)) : 0.0;
      }
    }
    for (int k0 = 0; k0 < K; k0 += 4) {
      const int p = k0 + tig;
      const double av = (q < M && p < K) ? sgn * A[q * lda + p] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int n = 8 * (4 * ng + u) + gid;
        const double bv = (p < K && n < N) ? B[p * ldb + n] : 0.0;
        dmma884(d[u][0], d[u][1], av, bv);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = 8 * (4 * ng + u) + 2 * tig;
      if (q < M) {
        if (c < N) O[q * ldo + c] = d[u][0];
        if (c + 1 < N) O[q * ldo + c + 1] = d[u][1];
      }
    }
  }
}

__device__ __forceinline__ double tr_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}


// Sc^{-1} for k <= KG by ONE warp, no CTA barrier: unpivoted Gauss-Jordan (reading R17) with
// lane r owning row r of the KG x KG matrix (identity padding beyond k), the pivot row
// broadcast by shuffles, and the columns rotated left by one per pivot so that the pivot
// column is always register 0 (compile-time register indices; after KG pivots the rotation
// is the identity).  In: M (k x k, ld ldm); out: Mi (k x k, ld ldm).
template <int KG>
__device__ __noinline__ void tr_warp_gj(const double* M, double* Mi, int ldm, int k, DevStatus* st, int where) {
  const int r = threadIdx.x & 31;
  double row[KG];
#pragma unroll
  for (int c = 0; c < KG; ++c) row[c] = (r < k && c < k) ? M[r * ldm + c] : (r == c ? 1.0 : 0.0);
  bool bad = false;
#pragma unroll 1
  for (int p = 0; p < KG; ++p) {
    double pr[KG];
#pragma unroll
    for (int c = 0; c < KG; ++c) pr[c] = __shfl_sync(0xffffffffu, row[c], p);
    const double piv = pr[0];
    bad |= !(isfinite(piv) && piv != 0.0);
    const double rp = tr_rcp(piv);
    const bool me = r == p;
    const double f = row[0] * rp;
#pragma unroll
    for (int c = 1; c < KG; ++c) row[c - 1] = me ? pr[c] * rp : fma(-f, pr[c], row[c]);
    row[KG - 1] = me ? rp : -f;
  }
  if (bad && r == 0) latch_status(st, FDE_ESINGULAR, where);
  if (r < k)
#pragma unroll
    for (int c = 0; c < KG; ++c)
      if (c < k) Mi[r * ldm + c] = row[c];
}

// One warp's share of a TR_SUB-row sub-chunk of the node update (tr_unit step 5): m-tile
// warp % TR_MW, n-tiles warp / TR_MW + TR_NS i (i < NTI, all with columns < xm):
//   Q_mu[r][c] = U1[r][c] + U2[r][c] - sum_q [U1 m-cols | U2 m-cols][r][q] S[q][c].
template <int NTI>
__device__ __forceinline__ void tr_upd_tiles(const double* U1, const double* U2, const double* Ss, double* Qo,
                                             int rs, int nr, int ncol1, int xm, int k, int K4, int lds) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
  const int mt = warp % TR_MW, nt0 = warp / TR_MW;
  const int r = 8 * mt + gid;
  const bool rok = r < nr;
  if (8 * mt >= nr) return;
  double d[NTI][2];
#pragma unroll
  for (int i = 0; i < NTI; ++i) {
    const int c = 8 * (nt0 + TR_NS * i) + 2 * tig;
    d[i][0] = (rok && c < xm) ? U1[r * ncol1 + c] + U2[r * ncol1 + c] : 0.0;
    d[i][1] = (rok && c + 1 < xm) ? U1[r * ncol1 + c + 1] + U2[r * ncol1 + c + 1] : 0.0;
  }
  const double* bp = Ss + tig * lds + 8 * nt0 + gid;
  const double* u1 = U1 + r * ncol1 + xm;
  const double* u2 = U2 + r * ncol1 + xm - k;
#pragma unroll 4
  for (int k0 = 0; k0 < K4; k0 += 4) {
    const int q = k0 + tig;                          // A = -[U1 m-cols | U2 m-cols] (zero padded)
    const double av = (rok && q < 2 * k) ? -(q < k ? u1[q] : u2[q]) : 0.0;
#pragma unroll
    for (int i = 0; i < NTI; ++i) dmma884(d[i][0], d[i][1], av, bp[k0 * lds + 8 * TR_NS * i]);
  }
  if (rok) {
    double* qr = Qo + (long long)(rs + r) * xm;
#pragma unroll
    for (int i = 0; i < NTI; ++i) {
      const int c = 8 * (nt0 + TR_NS * i) + 2 * tig;
      if (c < xm) qr[c] = d[i][0];
      if (c + 1 < xm) qr[c + 1] = d[i][1];
    }
  }
}

// One (node, row chunk) unit of level m.  All global reads are asynchronous copies into
// shared memory (cp.async), so the latency of L2/HBM is paid once per stage, not per load.
__device__ void tr_unit(const TrArgs& a, double* sm, int inst, int m, int j, int chunk) {
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31, gid = lane >> 2, tig = lane & 3;
  const int xm = a.xc[m], k = a.xc[m + 1] - xm, ncol1 = a.xc[m + 1];   // child Q: (ncol1-1) x ncol1
  const int lds = a.lds, ldk = a.ldk;
  double* Ms = sm + a.off_M;      // Sc, then Sc^{-1} (Gauss-Jordan ping-pong with M2)
  double* M2 = sm + a.off_M2;
  double* Ss = sm + a.off_S;      // rows 0..k-1: S_top; rows k..2k-1: T, then S_bot (ld lds)
  double* Ts = sm + a.off_T;      // k x xm scratch (S_bot before it moves into Ss)
  // level-m rows of Q_c1 / Q_c2 (k x ncol1 each; contiguous runs staged by 16-byte copies, each
  // placed at its base + the source parity)
  const long long qs1_ = (long long)(ncol1 - 1) * ncol1;
  const double* Q1s = a.Q + (long long)inst * a.qinst + a.qlev[m + 1] + (long long)(2 * j) * qs1_ + (long long)(xm - 1) * ncol1;
  double* Z1 = cp_contig_dst(sm + a.off_Z, Q1s);
  double* Z2 = cp_contig_dst(sm + a.off_Z + round_up(k * ncol1 + 2, 2), Q1s + qs1_);
  double* Ub = sm + a.off_U;      // TR_STG buffers x [Q_c1 rows | Q_c2 rows] (TR_SUB x ncol1 each);
                                  // aliases Ts and Z: streamed only after the S phase
  const long long qs1 = (long long)(ncol1 - 1) * ncol1;
  const double* Q1 = a.Q + (long long)inst * a.qinst + a.qlev[m + 1] + (long long)(2 * j) * qs1;
  const double* Q2 = Q1 + qs1;
  const int r0 = xm - 1;          // first level-m row of the child Q
  // row chunk of Q_mu handled by this unit
  const int nrow = xm - 1;
  const int rch = m > 0 ? round_up((nrow + a.rc[m] - 1) / a.rc[m], 8) : 0;
  const int ra = chunk * rch, rb = m > 0 ? min(nrow, ra + rch) : 0;
  const int nsub = rb > ra ? (rb - ra + TR_SUB - 1) / TR_SUB : 0;
  FDE_ASSERT(k >= 1 && k <= a.kmaxc && rb <= max(nrow, 0) && ra >= 0 && ncol1 <= a.NC);
  // sub-chunk buffers: [U1 | U2] x TR_STG, each TR_SUB x ncol1 (+2 spare doubles: 16-byte copies)
  const int usz = TR_SUB * ncol1 + 2;
  auto ubuf = [&](int sc, int which) -> double* {
    const int rs = ra + sc * TR_SUB;
    return cp_contig_dst(Ub + (sc % TR_STG) * 2 * usz + which * usz, (which ? Q2 : Q1) + (long long)rs * ncol1);
  };
  auto issue_sub = [&](int sc) {
    const int rs = ra + sc * TR_SUB, nr = min(TR_SUB, rb - rs);
    cp_contig(Ub + (sc % TR_STG) * 2 * usz, Q1 + (long long)rs * ncol1, nr * ncol1, t, TR_THREADS);
    cp_contig(Ub + (sc % TR_STG) * 2 * usz + usz, Q2 + (long long)rs * ncol1, nr * ncol1, t, TR_THREADS);
    cp_async_commit();
  };
  const bool tdbg = a.trace && t == 0;
  long long tcl = clock64();
  const int tsl = 1100 + (m == a.L - 1 ? 0 : 8);   // phase clocks: bottom level / the others
#define TPH(i) do { if (tdbg) { const long long t_ = clock64(); atomicAdd(a.trace + tsl + (i), (unsigned long long)(t_ - tcl)); tcl = t_; } } while (0)
  if (tdbg) atomicAdd(a.trace + tsl + 7, 1ULL);
  // 1. stage the level-m rows of both children (+ the first Q sub-chunk, in flight meanwhile)
  cp_contig(sm + a.off_Z, Q1 + (long long)r0 * ncol1, k * ncol1, t, TR_THREADS);
  cp_contig(sm + a.off_Z + round_up(k * ncol1 + 2, 2), Q2 + (long long)r0 * ncol1, k * ncol1, t, TR_THREADS);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  TPH(0);
  // 2. Sc = I - C B ; T = R_bot - C R_top   (B = Z2[:, m-cols], C = Z1[:, m-cols], read in place)
  const double* Bz = Z2 + xm;
  const double* Cz = Z1 + xm;
  tr_dmma(Ms, ldk, nullptr, 0, Cz, ncol1, Bz, ncol1, k, k, k, -1.0, 1.0);
  tr_dmma(Ts, lds, Z1, ncol1, Cz, ncol1, Z2, ncol1, k, xm, k, -1.0);
  __shared__ double rcp_buf[2];
  if (t == 0) rcp_buf[0] = 0.0;
  __syncthreads();
  if (t == 0) {
    const double p0 = Ms[0];
    if (!(isfinite(p0) && fabs(p0) > 0.0)) latch_status(a.st, FDE_ESINGULAR, inst * 65536 + 32768 + node_index(m, j));
    rcp_buf[0] = tr_rcp(p0);
  }
  __syncthreads();
  TPH(1);
  // 3. Sc^{-1}: warp-level Gauss-Jordan in registers (tr_warp_gj) for k <= 32, else the
  //    CTA-wide ping-pong version with one barrier per pivot
  const double* Mi;
  double* Gs;
  if (k <= 32) {
    if (warp == 0) {
      const int where = inst * 65536 + 32768 + node_index(m, j);
      if (k <= 16) tr_warp_gj<16>(Ms, M2, ldk, k, a.st, where);
      else if (k <= 24) tr_warp_gj<24>(Ms, M2, ldk, k, a.st, where);
      else tr_warp_gj<32>(Ms, M2, ldk, k, a.st, where);
    }
    __syncthreads();
    Mi = M2;
    Gs = Ms;
  } else {
    const int kk = k * k;
    for (int p = 0; p < k; ++p) {
      const double* src = (p & 1) ? M2 : Ms;
      double* dst = (p & 1) ? Ms : M2;
      const double rp = rcp_buf[p & 1];
      const int op = p * ldk;
      for (int e = t; e < kk; e += TR_THREADS) {
        const int q = e / k, cc = e - q * k;
        const double mqp = src[q * ldk + p], mpc = src[op + cc], mqc = src[q * ldk + cc];
        const double fq = -mqp * rp;
        const double v = (q == p) ? ((cc == p) ? rp : mpc * rp) : ((cc == p) ? fq : fma(fq, mpc, mqc));
        dst[q * ldk + cc] = v;
        if (q == p + 1 && cc == p + 1) {
          if (!(isfinite(v) && fabs(v) > 0.0)) latch_status(a.st, FDE_ESINGULAR, inst * 65536 + 32768 + node_index(m, j));
          rcp_buf[(p + 1) & 1] = tr_rcp(v);
        }
      }
      __syncthreads();
    }
    Mi = (k & 1) ? M2 : Ms;
    Gs = (k & 1) ? Ms : M2;
  }
  TPH(2);
  tr_dmma(Gs, ldk, nullptr, 0, Bz, ncol1, Mi, ldk, k, k, k, 1.0);          // G = B Sc^{-1}
  __syncthreads();
  if (a.Kr && chunk == 0) {               // U unit of the split run: what the R unit needs
    double* Kn = a.Kr + (long long)inst * a.krinst + a.krlev[m] + (long long)j * 3 * k * k;
    for (int e = t; e < k * k; e += TR_THREADS) {
      const int q = e / k, p = e - q * k;
      Kn[e] = Cz[q * ncol1 + p];
      Kn[k * k + e] = Mi[q * ldk + p];
      Kn[2 * k * k + e] = Gs[q * ldk + p];
    }
  }
  // 4. S_bot = Sc^{-1} T -> Ss rows k..2k-1 ; S_top = R_top - G T -> Ss rows 0..k-1
  tr_dmma(Ss + k * lds, lds, nullptr, 0, Mi, ldk, Ts, lds, k, xm, k, 1.0);
  tr_dmma(Ss, lds, Z2, ncol1, Gs, ldk, Ts, lds, k, xm, k, -1.0);
  // zero the K padding rows 2k .. round4(2k) and the column padding of S
  const int K4 = round_up(2 * k, 4), xmp = round_up(xm, 16);
  if (xmp > xm)
    for (int e = t; e < K4 * (xmp - xm); e += TR_THREADS) Ss[(e / (xmp - xm)) * lds + xm + e % (xmp - xm)] = 0.0;
  for (int e = t; e < (K4 - 2 * k) * xmp; e += TR_THREADS) Ss[(2 * k + e / xmp) * lds + e % xmp] = 0.0;
  __syncthreads();
  if (chunk == 0) {                       // keep S for the per-leaf v recursion
    double* So = a.Sst + (long long)inst * a.sinst + a.slev[m] + (long long)j * 2 * k * xm;
    for (int q = warp; q < 2 * k; q += TR_WARPS)
      for (int c = lane; c < xm; c += 32) So[q * xm + c] = Ss[q * lds + c];
  }
  TPH(3);
  if (nsub == 0) { __syncthreads(); return; }
  // 5. Q_mu rows [ra, rb) = Q1 + Q2 - [Q1 m-cols | Q2 m-cols] [S_top; S_bot], streamed in
  //    sub-chunks of TR_SUB rows.  Warp -> m-tile (warp % TR_MW) x n-tiles (warp / TR_MW) +
  //    TR_NS i: A fragment reused TR_NT times.
  double* Qo = a.Q + (long long)inst * a.qinst + a.qlev[m] + (long long)j * (long long)nrow * xm;
  // valid n-tiles of this warp (cols < xm): a warp-uniform trip count, so the DMMA loop has no
  // per-instruction predicate (a predicated mma.sync costs a WARPSYNC each)
  const int nti = max(0, min(TR_NT, ((xm + 7) / 8 - warp / TR_MW + TR_NS - 1) / TR_NS));
  auto update = [&](const double* U1, const double* U2, int rs, int nr) {
    switch (nti) {
      case 6: tr_upd_tiles<6>(U1, U2, Ss, Qo, rs, nr, ncol1, xm, k, K4, lds); break;
      case 5: tr_upd_tiles<5>(U1, U2, Ss, Qo, rs, nr, ncol1, xm, k, K4, lds); break;
      case 4: tr_upd_tiles<4>(U1, U2, Ss, Qo, rs, nr, ncol1, xm, k, K4, lds); break;
      case 3: tr_upd_tiles<3>(U1, U2, Ss, Qo, rs, nr, ncol1, xm, k, K4, lds); break;
      case 2: tr_upd_tiles<2>(U1, U2, Ss, Qo, rs, nr, ncol1, xm, k, K4, lds); break;
      case 1: tr_upd_tiles<1>(U1, U2, Ss, Qo, rs, nr, ncol1, xm, k, K4, lds); break;
      default: break;
    }
  };
  // TMA-engine path: each sub-chunk's Q1 / Q2 rows are one contiguous run (rounded up to an
  // even count of doubles: the extra one stays inside the child Q) -> two bulk copies into a
  // ring slot with an mbarrier; the last warp done with a slot refills it (no CTA barrier).
  __shared__ unsigned long long qbar[TR_STG];
  __shared__ int qcnt[TR_STG];
  const bool qbulk = ((reinterpret_cast<unsigned long long>(Q1) | reinterpret_cast<unsigned long long>(Q2) |
                       reinterpret_cast<unsigned long long>(Ub)) & 15) == 0 && (ra & 1) == 0 && TR_SUB % 2 == 0;
  if (qbulk) {
    auto issue_b = [&](int sc) {                      // (one thread)
      const int rs = ra + sc * TR_SUB, nr = min(TR_SUB, rb - rs);
      const unsigned bytes = (unsigned)round_up(nr * ncol1, 2) * 8u;
      FDE_ASSERT(nr >= 1 && rs + nr <= rb && (int)(bytes / 8) <= usz);
      double* dst = Ub + (sc % TR_STG) * 2 * usz;
      mbar_expect_tx(qbar + sc % TR_STG, 2 * bytes);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(dst)), "l"(Q1 + (long long)rs * ncol1), "r"(bytes), "r"(smem_u32(qbar + sc % TR_STG)) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(dst + usz)), "l"(Q2 + (long long)rs * ncol1), "r"(bytes), "r"(smem_u32(qbar + sc % TR_STG)) : "memory");
    };
    if (t == 0) {
      for (int i = 0; i < TR_STG; ++i) mbar_init(qbar + i, 1u);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      // (generic accesses of the aliased staging buffers, and Q written by other CTAs, before
      //  the async-proxy copies)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("fence.proxy.async.global;" ::: "memory");
      for (int sc = 0; sc < TR_STG && sc < nsub; ++sc) issue_b(sc);
    } else if (t >= 32 && t < 32 + TR_STG) {
      qcnt[t - 32] = 0;
    }
    __syncthreads();
    for (int sc = 0; sc < nsub; ++sc) {
      mbar_wait(qbar + sc % TR_STG, (sc / TR_STG) & 1);
      TPH(6);                                            // (wait)
      const int rs = ra + sc * TR_SUB;
      const double* U1 = Ub + (sc % TR_STG) * 2 * usz;
      update(U1, U1 + usz, rs, min(TR_SUB, rb - rs));
      TPH(5);                                            // (update)
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        if (atomicAdd(&qcnt[sc % TR_STG], 1) == TR_WARPS - 1 && sc + TR_STG < nsub) {
          qcnt[sc % TR_STG] = 0;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue_b(sc + TR_STG);
        }
      }
    }
    __syncthreads();
    if (t == 0)
      for (int i = 0; i < TR_STG; ++i) mbar_inval(qbar + i);
  } else {
    // cp.async pipeline (TR_STG - 1 sub-chunks' copies in flight during one's DMMA)
    for (int sc = 0; sc < TR_STG - 1 && sc < nsub; ++sc) issue_sub(sc);
    for (int sc = 0; sc < nsub; ++sc) {
      if (sc + TR_STG - 1 < nsub) issue_sub(sc + TR_STG - 1);
      TPH(5);                                            // (issue)
      const int ahead = min(TR_STG - 1, nsub - 1 - sc);   // groups allowed to stay in flight
      if (ahead >= 3) asm volatile("cp.async.wait_group 3;" ::: "memory");
      else if (ahead == 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
      else if (ahead == 1) cp_async_wait_group1();
      else cp_async_wait_all();
      __syncthreads();
      TPH(6);                                            // (wait)
      const int rs = ra + sc * TR_SUB;
      update(ubuf(sc, 0), ubuf(sc, 1), rs, min(TR_SUB, rb - rs));
      __syncthreads();
    }
  }
  TPH(4);
#undef TPH
}

// R unit of node (m, j) in the split pipelined run (k_run.cuh): the right-hand-side column alone.
// The node's U unit (tr_unit over all columns, column 0 left as don't-care) stored C, Sc^{-1} and
// G = B Sc^{-1}; with R_top0 = Q_c2[lvl m, 0], R_bot0 = Q_c1[lvl m, 0]:
//   t = R_bot0 - C R_top0,  S_bot[:, 0] = Sc^{-1} t,  S_top[:, 0] = R_top0 - G t,
//   Q_node[r, 0] = Q_c1[r, 0] + Q_c2[r, 0] - Q_c1[r, m-cols] S_top[:, 0] - Q_c2[r, m-cols] S_bot[:, 0]
// (the same algebra as tr_unit, restricted to column 0).
__device__ void tr_unit_R(const TrArgs& a, double* sm, int inst, int m, int j) {
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int xm = a.xc[m], k = a.xc[m + 1] - xm, ncol1 = a.xc[m + 1];
  const long long qs1 = (long long)(ncol1 - 1) * ncol1;
  const double* Q1 = a.Q + (long long)inst * a.qinst + a.qlev[m + 1] + (long long)(2 * j) * qs1;
  const double* Q2 = Q1 + qs1;
  const double* Kn = a.Kr + (long long)inst * a.krinst + a.krlev[m] + (long long)j * 3 * k * k;
  const int nr = ncol1 - 1;                          // rows of the child Q (incl. the level-m rows)
  const int kp1 = k + 1;                             // staged row: [column 0 | m-cols]
  double* Ks = sm;                                   // [C | Sc^-1 | G]
  double* R1 = Ks + 3 * k * k;                       // [nr][k+1] of Q_c1
  double* R2 = R1 + nr * kp1;                        // [nr][k+1] of Q_c2
  double* tv = R2 + nr * kp1;                        // t [k], s_top [k], s_bot [k]
  FDE_ASSERT(xm >= 1 && k >= 1 && ncol1 <= a.NC);
  for (int e = t; e < 3 * k * k; e += TR_THREADS) cp_async8(Ks + e, Kn + e);
  for (int e = t; e < nr * kp1; e += TR_THREADS) {
    const int r = e / kp1, c = e - r * kp1;
    const int col = c == 0 ? 0 : xm + c - 1;
    cp_async8(R1 + e, Q1 + (long long)r * ncol1 + col);
    cp_async8(R2 + e, Q2 + (long long)r * ncol1 + col);
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  const double* C = Ks;
  const double* Mi = Ks + k * k;
  const double* G = Ks + 2 * k * k;
  if (warp == 0) {
    for (int q = lane; q < k; q += 32) {           // t = R_bot0 - C R_top0
      double acc = R1[(xm - 1 + q) * kp1];
      for (int p = 0; p < k; ++p) acc = fma(-C[q * k + p], R2[(xm - 1 + p) * kp1], acc);
      tv[q] = acc;
    }
    __syncwarp();
    for (int q = lane; q < k; q += 32) {           // S_bot0 = Sc^-1 t ; S_top0 = R_top0 - G t
      double sb = 0.0, st = R2[(xm - 1 + q) * kp1];
      for (int p = 0; p < k; ++p) { sb = fma(Mi[q * k + p], tv[p], sb); st = fma(-G[q * k + p], tv[p], st); }
      tv[k + q] = st; tv[2 * k + q] = sb;
    }
  }
  __syncthreads();
  double* So = a.Sst + (long long)inst * a.sinst + a.slev[m] + (long long)j * 2 * k * xm;
  for (int q = t; q < 2 * k; q += TR_THREADS) So[(long long)q * xm] = tv[k + q];   // [S_top; S_bot][:, 0]
  if (m > 0) {
    double* Qo = a.Q + (long long)inst * a.qinst + a.qlev[m] + (long long)j * (long long)(xm - 1) * xm;
    for (int r = t; r < xm - 1; r += TR_THREADS) {
      const double* r1 = R1 + r * kp1;
      const double* r2 = R2 + r * kp1;
      double acc = r1[0] + r2[0];
      for (int q = 0; q < k; ++q) acc = fma(-r1[1 + q], tv[k + q], fma(-r2[1 + q], tv[2 * k + q], acc));
      Qo[(long long)r * xm] = acc;
    }
  }
  __syncthreads();
}

#define TR_NL 4                  // leaves per final-pass group (one warp each in the v phase)

// Final pass for the leaves lu0 .. lu0+nl-1 (global index inst * nleaf + leaf): per-leaf v
// recursion (one warp per leaf, S blocks double-buffered through shared memory), then
// u = X v with each leaf's panel block copied to shared memory.
__device__ void tr_final(const TrArgs& a, double* sm, int lu0, int nl) {
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int vstride = round_up(a.NC, 8), sbuf = a.kmaxc * a.NC;
  double* vs = sm;                                   // [TR_NL][vstride]
  double* Sb = sm + TR_NL * vstride;                 // v phase: [TR_NL warps][2][kmax x NC]
  double* Xs = sm + TR_NL * vstride;                 // u phase: [NC cols][128 rows] (aliases Sb)
  double* part = Xs + (long long)a.NC * 128;         // [2][128]
  if (warp < nl) {
    const int lu = lu0 + warp, inst = lu / a.nleaf, leaf = lu % a.nleaf;
    double* v = vs + warp * vstride;
    double* buf = Sb + warp * 2 * sbuf;
    auto S_of = [&](int m) {
      const int xm = a.xc[m], k = a.xc[m + 1] - xm;
      const int jn = leaf >> (a.L - m), side = (leaf >> (a.L - m - 1)) & 1;
      return a.Sst + (long long)inst * a.sinst + a.slev[m] + (long long)jn * 2 * k * xm + (long long)side * k * xm;
    };
    auto issue = [&](int m) {
      const int xm = a.xc[m], k = a.xc[m + 1] - xm;
      const double* g = S_of(m);
      double* d = buf + (m & 1) * sbuf;
      for (int e = lane; e < k * xm; e += 32) cp_async8(d + e, g + e);
      cp_async_commit();
    };
    for (int c = lane; c < a.NC; c += 32) v[c] = (c == 0) ? 1.0 : 0.0;
    issue(0);
    for (int m = 0; m < a.L; ++m) {
      if (m + 1 < a.L) { issue(m + 1); cp_async_wait_group1(); } else cp_async_wait_all();
      __syncwarp();
      const int xm = a.xc[m], k = a.xc[m + 1] - xm;
      const double* S = buf + (m & 1) * sbuf;
      if (lane < k) {                            // lane = row q of S_side, 4 FMA chains
        const double* sr = S + lane * xm;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int c = 0;
        for (; c + 3 < xm; c += 4) {
          a0 = fma(sr[c], v[c], a0); a1 = fma(sr[c + 1], v[c + 1], a1);
          a2 = fma(sr[c + 2], v[c + 2], a2); a3 = fma(sr[c + 3], v[c + 3], a3);
        }
        for (; c < xm; ++c) a0 = fma(sr[c], v[c], a0);
        v[xm + lane] = -((a0 + a1) + (a2 + a3));
      }
      for (int q = 32 + lane; q < k; q += 32) {  // (k > 32: remaining rows, one per lane)
        double acc = 0.0;
        for (int c = 0; c < xm; ++c) acc = fma(S[q * xm + c], v[c], acc);
        v[xm + q] = -acc;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int w = 0; w < nl; ++w) {
    const int lu = lu0 + w, inst = lu / a.nleaf, leaf = lu % a.nleaf;
    const int r0 = a.leaf_r0[leaf], s = a.leaf_n[leaf];
    const double* Xi = a.X + (long long)inst * a.xstride + r0;
    for (int e = t; e < a.NC * 128; e += TR_THREADS) {
      const int c = e >> 7, i = e & 127;
      if (i < s) cp_async8(Xs + e, Xi + (long long)c * a.n + i);
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    const double* v = vs + w * vstride;
    {
      const int i = t & 127, h = t >> 7;           // two column halves, fixed-order sums
      double acc = 0.0;
      if (i < s)
        for (int c = h; c < a.NC; c += 2) acc = fma(Xs[c * 128 + i], v[c], acc);
      part[h * 128 + i] = acc;
    }
    __syncthreads();
    for (int i = t; i < s; i += TR_THREADS) a.u[(long long)inst * a.n + r0 + i] = part[i] + part[128 + i];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(TR_THREADS, 1)
k_tree(const TrArgs a) {
  extern __shared__ double sm[];
  const int G = gridDim.x, b = blockIdx.x;
  unsigned nbar = 0;
  auto stamp = [&](int i) {
    if (a.trace && b == 0 && threadIdx.x == 0) {
      unsigned long long tm;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm));
      a.trace[1024 + i] = tm;
    }
  };
  stamp(0);
  for (int m = a.L - 1; m >= 0; --m) {
    const int per_inst = (1 << m) * a.rc[m];
    for (int u = b; u < a.batch * per_inst; u += G) {
      const int inst = u / per_inst, w = u % per_inst;
      tr_unit(a, sm, inst, m, w / a.rc[m], w % a.rc[m]);
    }
    stamp(2 * (a.L - m) - 1);
    tr_grid_barrier(a.bar, (++nbar) * G);
    stamp(2 * (a.L - m));
  }
  const int total = a.batch * a.nleaf;
  for (int base = b * TR_NL; base < total; base += TR_NL * G) tr_final(a, sm, base, min(TR_NL, total - base));
  stamp(2 * a.L + 1);
}
