// k_leaf.cuh -- S3 + S4: fused leaf assembly, block LU and block triangular solves.
//
// One CTA per (leaf, instance).  The leaf block of
//   A_m = shift I + c (D+ T + D- T^T),  T[i,j] = -g_{i-j+1}            (Eq. 2.5-2.6)
// is generated from g and d+- straight into shared memory (the identity shift and the
// diagonal scaling touch only the leaves and the factors) and factorised
// without pivoting (A_m and every principal sub-block are strictly diagonally dominant,
// P:231).  The factorisation is a block LU with 32 x 32 blocks kept in "inverse-diagonal"
// form, so that both the factorisation and the two block triangular sweeps are GEMMs on the
// FP64 tensor cores (DMMA):
//   for each block column k:  D_k <- (A_kk)^{-1}            (unpivoted Gauss-Jordan, 32 pivots)
//                             Lt_ik = A_ik D_k   (i > k),   Ut_jk = A_jk D_k   (j < k)
//                             A_ij -= Lt_ik A_kj            (i, j > k)
//   forward  y_i -= Lt_ik y_k                 (k = 0 .. nb-2)
//   backward x_j -= Ut_jk y_k, x_k = D_k y_k  (k = nb-1 .. 0)
// The leaf is padded to a multiple of 32 with an identity block.
//   factor mode: X = [b | U_0 | ... | U_{L-1}] rows of this leaf, b = u_prev + dt f (fused solve,
//     optional), U_l = the column factor of the level-l off-diagonal block containing the leaf:
//       first child  rows: U12 = [-c D-  J L_l[:n1],  -c d+[r0+n1-1] e_{n1-1}]
//       second child rows: U21 = [-c D+  L_l[:n2],    -c d-[r0+n1]   e_0      ]
//     X <- A_leaf^{-1} X is written to HBM for the level kernel (k_levels.cuh);
//   solve mode: y <- A_leaf^{-1} (b + dt f) with the factor kept in HBM.
#pragma once
#include "fde_common.cuh"
#include "fde_dmma.cuh"

#define LEAF_THREADS 256             // 8 warps: 2 per SM sub-partition (DMMA issue is per SMSP)
#define LEAF_WARPS (LEAF_THREADS / 32)
#define LDA_LEAF 132                 // column-major leading dims (= 4 mod 16: conflict-free DMMA frags)
#define LDP_LEAF 132
#define YLD 132                      // warp stripe buffer (128 x 8) leading dim (= 4 mod 16)
#define LEAF_SLOT (LEAF_MAX * LEAF_MAX)   // doubles per kept leaf factor
#define LEAF_RSLOT (LEAF_MAX * LDA_LEAF)  // doubles per stored run LU (the shared-memory layout)
#define NCOL_MAX 384                 // panel columns (1 + sum of k_l) held as descriptors in smem
#define LEAF_FRONT (32 * 33 + 3 * LEAF_MAX + 2 * NCOL_MAX)        // doubles before the LU region
#define LEAF_BIG (LEAF_MAX * LDA_LEAF + LEAF_WARPS * 8 * YLD)       // LU + stripe buffers (reused by Q)
#define LEAF_SMEM ((LEAF_FRONT + LEAF_BIG) * 8)
#define GJ_WARPS 4                   // warps of the 32 x 32 diagonal-block Gauss-Jordan
#define LEAF_OVW 8                   // register tiles per warp of an overwrite GEMM
#define LEAF_LDV 132                 // row pitch of the TMA boxes of the projection (= LDA_LEAF)
struct alignas(64) CUtensorMapLike { unsigned long long opaque[16]; };   // (= CUtensorMap, 128 bytes)

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
  double* LU; long long lustride; int keep;  // kept factors, LEAF_SLOT doubles per leaf
  int nf;                                    // fused RHS columns (0/1), factor mode
  const double* u_prev; const double* f;     // [batch*n], factor mode with nf = 1
  const double* b; double* y; int nrhs; int ld;   // solve mode
  double* Q; long long qstride, qinst;       // factor mode: Q_leaf = V_all^T X_leaf (or null)
  int store_lu;                              // factor mode: write the LU (inverse-diagonal form, pitch
                                             // LDA_LEAF, LEAF_RSLOT doubles per leaf) -- k_run
  unsigned long long* prof;                  // optional: phase cycle sums (k_run FDE_TRACE_RUN)
  DevStatus* st;
  unsigned long long* trace;                 // optional phase clocks (FDE_TRACE_LEVELS)
  const void* lmap;                          // TMA maps of L_l: [inst * L + l] (CUtensorMap), or null
  const void* xmap;                          // TMA map of this X buffer (n x NC x batch), or null
};

// ---- DMMA GEMMs on column-major shared-memory operands ---------------------------------
// C[M x N] -= A[M x K] B[K x N]; tiles round-robin over warps [w0, w0 + nw); M, N % 8 == 0,
// K % 4 == 0.  Optionally skips the tile block (skip_m0.., skip_n0..) of size 32 x 32.
// Warp roles of the overlapped Gauss-Jordan.  Warp w runs on SM sub-partition w % 4, whose
// FP64 pipe is shared by DFMA and DMMA (tools/gj_bench.cu: 233 cycles per pivot alone, 928
// with DMMA warps on the same SMSPs, 306 with them on the other two).  SPLIT puts the GJ on
// warps 0,1,4,5 (SMSPs 0,1) and the other work on SMSPs 2,3: used while the leaf is built
// (FMA work), not in the LU, where the DMMA trailing update needs all four pipes
// (measured: build+gj0 10.6 -> 9.6 us, but lu+store 27.1 -> 29.1 us per leaf with SPLIT).
template <bool SPLIT>
__device__ __forceinline__ bool gj_role(int warp) { return SPLIT ? (warp & 2) == 0 : warp < GJ_WARPS; }
template <bool SPLIT>
__device__ __forceinline__ int role_idx(int warp) { return SPLIT ? (warp & 1) | ((warp >> 2) << 1) : warp & 3; }

// A predicated mma.sync costs the warp a WARPSYNC + branch per instruction, so the DMMA loops
// below run a warp-uniform, compile-time number of tiles; only loads / stores are guarded.
// The skip block (skip_m0 = skip_n0 = 0: the leading 32 x 32 tiles, already updated by the
// lookahead) is left out of the tile enumeration.
template <bool ADD = false, int U = 4>
__device__ __forceinline__ void cm_gemm_sub(double* C, int ldc, const double* A, int lda,
                                            const double* B, int ldb, int M, int N, int K, int w0,
                                            int nw, int skip_m0 = -1, int skip_n0 = -1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gid = lane >> 2, tig = lane & 3;
  const int w = warp - w0;
  if (w < 0 || w >= nw) return;
  FDE_ASSERT(skip_m0 < 0 || (skip_m0 == 0 && skip_n0 == 0 && M >= 32 && N >= 32));
  const int MB = M >> 3, NB8 = N >> 3;
  const bool skip = skip_m0 >= 0;
  const int ns = skip ? 4 * (MB - 4) : 0;            // tiles of the first 4 n-tiles (below the skip)
  const int NT = MB * NB8 - (skip ? 16 : 0);
  auto tile = [&](int t, int& mo, int& no) {
    if (t < ns) { no = (t / (MB - 4)) * 8; mo = (4 + t % (MB - 4)) * 8; }
    else { const int t2 = t - ns; no = ((skip ? 4 : 0) + t2 / MB) * 8; mo = (t2 % MB) * 8; }
  };
  for (int t0 = w; t0 < NT; t0 += U * nw) {
    double d[U][2];
    const double* ap[U];
    const double* bp[U];
    bool ok[U];
    int mo[U], no[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = t0 + u * nw;
      ok[u] = t < NT;
      tile(ok[u] ? t : t0, mo[u], no[u]);             // (a valid tile for the unused slots)
      d[u][0] = ok[u] ? C[mo[u] + gid + (no[u] + 2 * tig) * ldc] : 0.0;
      d[u][1] = ok[u] ? C[mo[u] + gid + (no[u] + 2 * tig + 1) * ldc] : 0.0;
      ap[u] = A + mo[u] + gid + tig * lda;
      bp[u] = B + tig + (no[u] + gid) * ldb;
    }
    for (int k0 = 0; k0 < K; k0 += 4) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        dmma884(d[u][0], d[u][1], ADD ? ap[u][k0 * lda] : -ap[u][k0 * lda], bp[u][k0]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (ok[u]) {
        C[mo[u] + gid + (no[u] + 2 * tig) * ldc] = d[u][0];
        C[mo[u] + gid + (no[u] + 2 * tig + 1) * ldc] = d[u][1];
      }
  }
}

// Register tiles of an overwrite product O = A B (O may alias A or B): compute() keeps up to
// LEAF_OVW 8x8 tiles per warp in registers; the caller synchronises before store().
struct OvwTiles {
  double d[LEAF_OVW][2];
  int mo[LEAF_OVW], no[LEAF_OVW];
  int cnt;
};

template <int CNT>
__device__ __forceinline__ void ovw_mma(OvwTiles& T, const double* A, int lda, const double* B, int ldb, int K) {
  const int lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
  for (int k0 = 0; k0 < K; k0 += 4) {
#pragma unroll
    for (int u = 0; u < CNT; ++u)
      dmma884(T.d[u][0], T.d[u][1], A[T.mo[u] + gid + (k0 + tig) * lda], B[k0 + tig + (T.no[u] + gid) * ldb]);
  }
}

// tiles over the rows [r_lo, r_hi) and [r2_lo, r2_hi) (two row ranges) x N columns
__device__ __forceinline__ void ovw_compute(OvwTiles& T, const double* A, int lda, const double* B,
                                            int ldb, int r_lo, int r_hi, int r2_lo, int r2_hi, int N,
                                            int K) {
  const int warp = threadIdx.x >> 5;
  const int M1 = (r_hi - r_lo) >> 3, M2 = (r2_hi - r2_lo) >> 3, MB = M1 + M2;
  const int NT = MB * (N >> 3);
  T.cnt = 0;
#pragma unroll
  for (int u = 0; u < LEAF_OVW; ++u) {
    const int t = warp + u * LEAF_WARPS;
    const int mbi = t % MB;
    T.mo[u] = mbi < M1 ? r_lo + mbi * 8 : r2_lo + (mbi - M1) * 8;
    T.no[u] = (t / MB) * 8;
    T.d[u][0] = 0.0; T.d[u][1] = 0.0;
    if (t < NT) T.cnt = u + 1;
  }
  switch (T.cnt) {                                   // (warp-uniform)
    case 8: ovw_mma<8>(T, A, lda, B, ldb, K); break;
    case 7: ovw_mma<7>(T, A, lda, B, ldb, K); break;
    case 6: ovw_mma<6>(T, A, lda, B, ldb, K); break;
    case 5: ovw_mma<5>(T, A, lda, B, ldb, K); break;
    case 4: ovw_mma<4>(T, A, lda, B, ldb, K); break;
    case 3: ovw_mma<3>(T, A, lda, B, ldb, K); break;
    case 2: ovw_mma<2>(T, A, lda, B, ldb, K); break;
    case 1: ovw_mma<1>(T, A, lda, B, ldb, K); break;
    default: break;
  }
}

__device__ __forceinline__ void ovw_store(const OvwTiles& T, double* O, int ldo, double sgn = 1.0) {
  const int lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
#pragma unroll
  for (int u = 0; u < LEAF_OVW; ++u)
    if (u < T.cnt) {
      O[T.mo[u] + gid + (T.no[u] + 2 * tig) * ldo] = sgn * T.d[u][0];
      O[T.mo[u] + gid + (T.no[u] + 2 * tig + 1) * ldo] = sgn * T.d[u][1];
    }
}

// In-place inverse of a 32 x 32 column-major block with all threads: unpivoted Gauss-Jordan,
// one barrier per pivot, ping-pong between D and the scratch S (ld 33).
__device__ void blk_gj_inv32(double* D, int ld, double* S, DevStatus* st, int where) {
  const int t = threadIdx.x;
  for (int kk = 0; kk < 32; ++kk) {
    const double* src = (kk & 1) ? S : D;
    double* dst = (kk & 1) ? D : S;
    const int ls = (kk & 1) ? 33 : ld, lt = (kk & 1) ? ld : 33;
    const double piv = src[kk + kk * ls];
    if (t == 0 && !(isfinite(piv) && piv != 0.0)) latch_status(st, FDE_ESINGULAR, where);
    const double rp = 1.0 / piv;
    for (int e = t; e < 1024; e += LEAF_THREADS) {
      const int i = e & 31, c = e >> 5;
      const double aic = src[i + c * ls], aik = src[i + kk * ls], akc = src[kk + c * ls];
      double v;
      if (i == kk) v = (c == kk) ? rp : akc * rp;
      else v = (c == kk) ? -aik * rp : fma(-aik * rp, akc, aic);
      dst[i + c * lt] = v;
    }
    __syncthreads();
  }
}

// Reciprocal to full double precision without the IEEE division routine: hardware
// approximation + two Newton steps (error well below 1 ulp of the pivots' conditioning).
__device__ __forceinline__ double fast_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

// In-place inverse of a 32 x 32 column-major block by the gj_role warps (named barrier 1): unpivoted
// Gauss-Jordan in registers, lane r of role warp w owns A[r, 8w .. 8w+7].  Per pivot the pivot
// row and column are published through a double-buffered shared scratch (buf, 128 doubles)
// and one 128-thread barrier.  The blocks are diagonal blocks of Schur complements of a
// strictly diagonally dominant matrix: no pivoting; a zero / non-finite pivot
// latches FDE_ESINGULAR.
template <bool SPLIT>
__device__ __noinline__ void quad_gj_inv32(double* D, int ld, double* buf, DevStatus* st, int where) {
  const int w = role_idx<SPLIT>(threadIdx.x >> 5), r = threadIdx.x & 31;
  double col[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) col[c] = D[r + (8 * w + c) * ld];
  bool bad = false;
#pragma unroll 1
  for (int kb8 = 0; kb8 < 4; ++kb8) {
#pragma unroll
    for (int k8 = 0; k8 < 8; ++k8) {
      const int kk = 8 * kb8 + k8;
      double* pr = buf + (k8 & 1) * 64;              // [0, 32): pivot row ; [32, 64): pivot column
      if (w == kb8) pr[32 + r] = col[k8];
      if (r == kk) {
        double2* pv = reinterpret_cast<double2*>(pr + 8 * w);
#pragma unroll
        for (int c = 0; c < 4; ++c) pv[c] = make_double2(col[2 * c], col[2 * c + 1]);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(GJ_WARPS * 32) : "memory");
      const double piv = pr[kk];
      bad |= !(isfinite(piv) && piv != 0.0);
      const double rp = fast_rcp(piv);
      const double f = pr[32 + r] * rp;              // A[r, kk] / pivot
      const bool me = r == kk;
      const double2* pv = reinterpret_cast<const double2*>(pr + 8 * w);
#pragma unroll
      for (int c2 = 0; c2 < 4; ++c2) {
        const double2 q = pv[c2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = 2 * c2 + h;
          const double p = h ? q.y : q.x;
          if (w == kb8 && c == k8) col[c] = me ? rp : -f;
          else col[c] = me ? p * rp : fma(-f, p, col[c]);
        }
      }
    }
  }
  if (bad && threadIdx.x == 0) latch_status(st, FDE_ESINGULAR, where);
#pragma unroll
  for (int c = 0; c < 8; ++c) D[r + (8 * w + c) * ld] = col[c];
}

// Block LU in inverse-diagonal form of A (sp x sp, sp % 32 == 0) in shared memory; the
// off-diagonal blocks are stored negated (-Lt, -Ut) for the accumulate-only stripe solve:
//   for kb:  D_k = (A_kk)^{-1} ;  -Lt_ik = -A_ik D_k (i > k) ;  -Ut_jk = -A_jk D_k (j < k)
//            A_ij += (-Lt_ik) A_kj   (i, j > k)
// With lookahead: the next diagonal block is updated first and inverted by warps 0..3
// while the other four finish the trailing update (three CTA barriers per block column).
__device__ void leaf_block_lu(double* A, int sp, double* prow, DevStatus* st, int where,
                              unsigned long long* trace = nullptr, bool gj0_done = false) {
  const int nb = sp >> 5, warp = threadIdx.x >> 5;
  const bool tr = trace && threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0;
  long long tl = clock64();
#define LUT(i) do { if (tr) { const long long t_ = clock64(); trace[960 + (i)] += t_ - tl; tl = t_; } } while (0)
  if (!gj0_done) {
    if (warp < GJ_WARPS) quad_gj_inv32<false>(A, LDA_LEAF, prow, st, where);
    __syncthreads();
  }
  LUT(0);
  for (int kb = 0; kb < nb; ++kb) {
    const int k0 = kb * 32;
    if (nb > 1) {
      OvwTiles T;
      ovw_compute(T, A + k0 * LDA_LEAF, LDA_LEAF, A + k0 + k0 * LDA_LEAF, LDA_LEAF, 0, k0,
                  k0 + 32, sp, 32, 32);
      __syncthreads();
      ovw_store(T, A + k0 * LDA_LEAF, LDA_LEAF, -1.0);
      __syncthreads();
    }
    LUT(1);
    if (kb + 1 < nb) {
      const int k1 = k0 + 32;
      double* Akk = A + k1 + k1 * LDA_LEAF;
      const double* Lk = A + k1 + k0 * LDA_LEAF;
      const double* Uk = A + k0 + k1 * LDA_LEAF;
      cm_gemm_sub<true, 2>(Akk, LDA_LEAF, Lk, LDA_LEAF, Uk, LDA_LEAF, 32, 32, 32, 0, LEAF_WARPS);
      __syncthreads();
      LUT(2);
#ifdef FDE_LU_SERIAL
      if (warp < GJ_WARPS) quad_gj_inv32<false>(Akk, LDA_LEAF, prow, st, where);
      __syncthreads();
      if (sp - k1 > 32)
        cm_gemm_sub<true>(Akk, LDA_LEAF, Lk, LDA_LEAF, Uk, LDA_LEAF, sp - k1, sp - k1, 32, 0,
                          LEAF_WARPS, 0, 0);
      __syncthreads();
#else
      if (warp < GJ_WARPS) quad_gj_inv32<false>(Akk, LDA_LEAF, prow, st, where);
      else if (sp - k1 > 32)
        cm_gemm_sub<true>(Akk, LDA_LEAF, Lk, LDA_LEAF, Uk, LDA_LEAF, sp - k1, sp - k1, 32, GJ_WARPS,
                          LEAF_WARPS - GJ_WARPS, 0, 0);
      __syncthreads();
#endif
      LUT(3);
    }
  }
#undef LUT
}

// ---- warp-stripe block triangular solve -------------------------------------------------
// One warp solves A_leaf x = p for an 8-column stripe with no CTA barrier: the stripe lives in
// the warp's registers as DMMA accumulator fragments (tile t = rows 8t..8t+7:
// acc[t][j] = x[8t + gid][2 tig + j]); finished 32-row blocks z_kb are published through a
// warp-private 32 x 8 shared buffer (Ys) to serve as the B operand of the block updates.
// The factor is in inverse-diagonal form with the off-diagonal blocks stored NEGATED
// (leaf_block_lu): -Lt_ik (i > k), -Ut_jk (j < k), D_k = (U_kk)^{-1}:
//   forward   z_i += (-Lt_ik) z_k                       (k = 0 .. nb-2, i > k)
//   backward  x_k  = D_k z_k,  z_j += (-Ut_jk) z_k       (k = nb-1 .. 0, j < k)

__device__ __forceinline__ void ys_publish(double* Ys, const double (&acc)[16][2], int kb) {
  const int lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    Ys[8 * i + gid + (2 * tig) * YLD] = acc[4 * kb + i][0];
    Ys[8 * i + gid + (2 * tig + 1) * YLD] = acc[4 * kb + i][1];
  }
}

__device__ __forceinline__ void stripe_solve(double (&acc)[16][2], const double* __restrict__ A, int nb,
                                             double* Ys) {
  const int lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
#pragma unroll
  for (int kb = 0; kb < 3; ++kb) {                 // forward
    if (kb + 1 < nb) {
      ys_publish(Ys, acc, kb);
      __syncwarp();
#pragma unroll
      for (int k4 = 0; k4 < 8; ++k4) {
        const double b = Ys[4 * k4 + tig + gid * YLD];
        const double* Ak = A + (kb * 32 + 4 * k4 + tig) * LDA_LEAF + gid;
#pragma unroll
        for (int t = 4 * (kb + 1); t < 16; ++t)      // (tiles >= 4 nb: unused accumulators)
          dmma884(acc[t][0], acc[t][1], Ak[8 * t], b);
      }
      __syncwarp();
    }
  }
#pragma unroll
  for (int kb = 3; kb >= 0; --kb) {                // backward
    if (kb < nb) {
      ys_publish(Ys, acc, kb);
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 4; ++i) { acc[4 * kb + i][0] = 0.0; acc[4 * kb + i][1] = 0.0; }
#pragma unroll
      for (int k4 = 0; k4 < 8; ++k4) {
        const double b = Ys[4 * k4 + tig + gid * YLD];
        const double* Ak = A + (kb * 32 + 4 * k4 + tig) * LDA_LEAF + gid;
#pragma unroll
        for (int t = 0; t < 4 * (kb + 1); ++t) dmma884(acc[t][0], acc[t][1], Ak[8 * t], b);
      }
      __syncwarp();
    }
  }
}

// Panel column descriptor (factor mode): X column cg of this leaf's rows.
//   kind 0: zero (padding) ; 1: fused rhs b = u_prev + dt f ; 2: scaled low-rank column
//   -c ds[i] L_l[li0 + lstep i, q] ; 3: exact column -c de[i] at the row with li == 0.
struct PanelCol {        // 16 bytes (NCOL_MAX of them live in shared memory)
  const double* Lq;      // kind 2: &L_l[0, q]; otherwise any valid address (read, unused)
  int li0;
  signed char kind, lstep;
  signed char sel;       // scaling: 0 -> d+ rows, 1 -> d- rows
  signed char pad;
};
static_assert(sizeof(PanelCol) == 16, "PanelCol layout");

__device__ __forceinline__ PanelCol panel_col(const LeafArgs& a, int inst, int leaf, int r0, int cg,
                                              int c_end) {
  PanelCol pc{a.Lf, 0, 0, 0, 0, 0};
  if (cg >= c_end) return pc;
  if (cg == 0) { pc.kind = 1; return pc; }
  const TreeDev& tr = a.tree;
  const int L = tr.L;
  int l = 0;
  while (l + 1 < L && a.xcol[l + 1] <= cg) ++l;
  const int q = cg - a.xcol[l], r = a.rank[inst * L + l], kq = a.kl[l];
  const int jn = leaf >> (L - l), child = (leaf >> (L - l - 1)) & 1;
  const int nd = node_index(l, jn);
  const int r0n = tr.node_r0[nd], n1 = tr.node_n1[nd];
  // row index into L_l: child 0 -> n1-1-(R-r0n) (decreasing), child 1 -> R-r0n-n1
  const int li0 = child == 0 ? n1 - 1 - (r0 - r0n) : r0 - r0n - n1;
  const int lstep = child == 0 ? -1 : 1;
  if (q == kq - 1) { pc.kind = 3; pc.sel = child == 0 ? 0 : 1; pc.li0 = li0; pc.lstep = lstep; }
  else if (q < r) {
    pc.kind = 2; pc.sel = child == 0 ? 1 : 0; pc.li0 = li0; pc.lstep = lstep;
    pc.Lq = a.Lf + (long long)inst * a.lf_stride + tr.lev_lofs[l] + (long long)q * tr.lev_m[l];
  }
  return pc;
}

// One panel stripe (8 columns) solved by a group of 4 warps (named barrier 2 + group): warp w of
// the group owns row block w (4 DMMA m-tiles).  Same block sweeps as stripe_solve -- forward
// z_i += (-Lt_ik) z_k, backward x_k = D_k z_k, z_j += (-Ut_jk) z_k -- with each finished block
// published through a double-buffered 32 x 8 shared buffer; identical arithmetic per element
// (same DMMA chains in the same order), so results equal the single-warp stripe bitwise.
//   buf: 3 warp-private stripe buffers of the group (8 x YLD each): [stripe | pub0 | pub1]
__device__ __noinline__ void leaf_coop_stripe(const double* __restrict__ A, int nb, int s, double c,
                                              const LeafArgs& a, const PanelCol* pcd, int c_begin,
                                              int c_end, int st, const double* dps, const double* dms,
                                              const double* bs, double* buf, double* Xi, int n) {
  const int lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
  const int w = (threadIdx.x >> 5) & 3, bar = 2 + (threadIdx.x >> 7);
  double* Sb = buf;                                   // stripe columns (rows 0..127, pitch YLD)
  double* Pb[2] = {buf + 8 * YLD, buf + 16 * YLD};    // published blocks (32 rows, pitch YLD)
  const int cs = c_begin + 8 * st;
  auto gsync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(128) : "memory"); };
  // generate: warp w scales columns 2w, 2w+1
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int cc = 2 * w + h;
    const PanelCol pc = cs + cc < c_end ? pcd[cs + cc - c_begin] : PanelCol{a.Lf, 0, 0, 0, 0, 0};
    const double* sc = pc.sel ? dms : dps;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = lane + 32 * q;
      const int ic = i < s ? i : s - 1;
      const double x = __ldg(pc.Lq + pc.li0 + pc.lstep * ic);
      double v = 0.0;
      if (i < s) {
        if (pc.kind == 2) v = x * (-c * sc[i]);
        else if (pc.kind == 3) v = (pc.li0 + pc.lstep * i == 0) ? -c * sc[i] : 0.0;
        else if (pc.kind == 1) v = bs[i];
      }
      Sb[i + cc * YLD] = v;
    }
  }
  gsync();
  double acc[4][2];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int i = 32 * w + 8 * u + gid;
    acc[u][0] = w < nb ? Sb[i + 2 * tig * YLD] : 0.0;
    acc[u][1] = w < nb ? Sb[i + (2 * tig + 1) * YLD] : 0.0;
  }
  auto publish = [&](double* P) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      P[8 * u + gid + (2 * tig) * YLD] = acc[u][0];
      P[8 * u + gid + (2 * tig + 1) * YLD] = acc[u][1];
    }
  };
  int pb = 0;
  for (int kb = 0; kb + 1 < nb; ++kb) {               // forward
    if (w == kb) publish(Pb[pb]);
    gsync();
    if (w > kb && w < nb) {
#pragma unroll
      for (int k4 = 0; k4 < 8; ++k4) {
        const double b = Pb[pb][4 * k4 + tig + gid * YLD];
        const double* Ak = A + (kb * 32 + 4 * k4 + tig) * LDA_LEAF + gid;
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma884(acc[u][0], acc[u][1], Ak[8 * (4 * w + u)], b);
      }
    }
    pb ^= 1;
  }
  for (int kb = nb - 1; kb >= 0; --kb) {              // backward
    if (w == kb) publish(Pb[pb]);
    gsync();
    if (w <= kb) {
      if (w == kb) {
#pragma unroll
        for (int u = 0; u < 4; ++u) { acc[u][0] = 0.0; acc[u][1] = 0.0; }
      }
#pragma unroll
      for (int k4 = 0; k4 < 8; ++k4) {
        const double b = Pb[pb][4 * k4 + tig + gid * YLD];
        const double* Ak = A + (kb * 32 + 4 * k4 + tig) * LDA_LEAF + gid;
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma884(acc[u][0], acc[u][1], Ak[8 * (4 * w + u)], b);
      }
    }
    pb ^= 1;
  }
  // each warp's rows -> stripe buffer -> X (columns contiguous over rows)
  if (w < nb) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = 32 * w + 8 * u + gid;
      Sb[i + 2 * tig * YLD] = acc[u][0];
      Sb[i + (2 * tig + 1) * YLD] = acc[u][1];
    }
  }
  __syncwarp();
  if (w < nb)
    for (int cc = 0; cc < 8 && cs + cc < c_end; ++cc) {
      const int i = 32 * w + lane;
      if (i < s) Xi[(long long)(cs + cc) * n + i] = Sb[i + cc * YLD];
    }
}

// ---- S5 input: projection of the leaf panel on every ancestor's V factor -----------------
// Q_leaf = V_all[leaf rows]^T X_leaf  ((NC-1) x NC, row-major, ld NC), where V-column j is
// the V factor column of X column j+1 (level l, q): child 0 rows of a level-l node carry
// V21 = [J L_l, e_{n1-1}], child 1 rows V12 = [L_l, e_0] (k_levels.cuh / k_tree.cuh).  Runs
// after all stripes: the LU + stripe buffers are reused for V (NV x 128 col-major) and
// chunks of X re-read from L2.  DMMA tiles: warp unit = (m-tile, 2 n-tiles), A reused.
__device__ void leaf_project(const LeafArgs& a, double* big, const PanelCol* pcd, int c_begin,
                             int NC, int s, int sp, const double* Xi, double* Qo, int c_lo = 0,
                             unsigned long long* prof = nullptr) {
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31, gid = lane >> 2, tig = lane & 3;
  long long ph_t = clock64();
  auto ph = [&](int i) {                              // (debug: B phase cycle sums, prof[i])
    if (prof && t == 0) { const long long t_ = clock64(); atomicAdd(prof + i, (unsigned long long)(t_ - ph_t)); ph_t = t_; }
  };
  const int n = a.tree.n, NV = NC - 1, NVP = round_up(NV, 8), MT = NVP >> 3;
  FDE_ASSERT((long long)NV * NC <= a.qstride && NVP * LDA_LEAF + 16 * LDA_LEAF <= LEAF_BIG && s <= LEAF_MAX);
  double* Vs = big;                                   // [NVP cols][LDA_LEAF]
  double* Xs = big + NVP * LDA_LEAF;
  const int XCH = min(((LEAF_BIG - NVP * LDA_LEAF) / LDA_LEAF) & ~15, round_up(NC - c_lo, 16));
  // row pairs of X are 16-byte aligned when the leaf start, n and the instance stride are even
  const bool xvec = (reinterpret_cast<unsigned long long>(Xi) & 15) == 0 && (n & 1) == 0;
  __syncthreads();                                    // every warp is done with the LU
  for (int j = warp; j < NVP; j += LEAF_WARPS) {
    const PanelCol pc = j < NV ? pcd[j + 1 - c_begin] : PanelCol{a.Lf, 0, 0, 0, 0, 0};
    for (int q = 0; q < LEAF_MAX / 32; ++q) {
      const int i = lane + 32 * q;
      if (pc.kind == 2 && i < s) cp_async8(&Vs[i + j * LDA_LEAF], pc.Lq + pc.li0 + pc.lstep * i);
      else Vs[i + j * LDA_LEAF] = (pc.kind == 3 && i < s && pc.li0 + pc.lstep * i == 0) ? 1.0 : 0.0;
    }
  }
  cp_async_commit();
  // balanced column chunks of whole n-tile pairs (16 columns), at most XCH wide
  const int NPT = round_up(NC - c_lo, 16) >> 4, maxp = XCH >> 4;
  const int nchunk = (NPT + maxp - 1) / maxp;
  const int MP = (MT + 1) >> 1;                       // m-tile pairs
  int c0 = c_lo;                                      // (c_lo = 1: the rhs column is projected later)
  for (int ch = 0; ch < nchunk; ++ch) {
    const int npc = (NPT * (ch + 1)) / nchunk - (NPT * ch) / nchunk;   // n-pairs in this chunk
    const int ncp = 16 * npc;
    if (xvec) {                                        // 16-byte copies of row pairs
      for (int cc = warp; cc < ncp; cc += LEAF_WARPS)
#pragma unroll
        for (int q = 0; q < LEAF_MAX / 64; ++q) {
          const int i = 2 * lane + 64 * q;
          double* d = &Xs[i + cc * LDA_LEAF];
          if (c0 + cc < NC && i + 1 < s) cp_async16(d, Xi + (long long)(c0 + cc) * n + i);
          else {
            d[0] = (c0 + cc < NC && i < s) ? __ldcg(Xi + (long long)(c0 + cc) * n + i) : 0.0;
            d[1] = 0.0;
          }
        }
    } else {
      for (int cc = warp; cc < ncp; cc += LEAF_WARPS)
        for (int q = 0; q < LEAF_MAX / 32; ++q) {
          const int i = lane + 32 * q;
          if (c0 + cc < NC && i < s) cp_async8(&Xs[i + cc * LDA_LEAF], Xi + (long long)(c0 + cc) * n + i);
          else Xs[i + cc * LDA_LEAF] = 0.0;
        }
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    ph(1);
    // warp unit = (m-tile pair) x (n-tile pair): 2 A + 2 B fragments feed 4 DMMAs per k-step
    for (int u = warp; u < MP * npc; u += LEAF_WARPS) {
      const int mp = u % MP, n0 = (u / MP) * 16;
      const bool m2 = 2 * mp + 1 < MT;
      double d[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};
      const double* ap0 = Vs + (16 * mp + gid) * LDA_LEAF + tig;
      const double* ap1 = ap0 + 8 * LDA_LEAF;
      const double* bp0 = Xs + (n0 + gid) * LDA_LEAF + tig;
      const double* bp1 = bp0 + 8 * LDA_LEAF;
#pragma unroll 4
      for (int k0 = 0; k0 < sp; k0 += 4) {
        const double a0 = ap0[k0], a1 = m2 ? ap1[k0] : 0.0, b0 = bp0[k0], b1 = bp1[k0];
        dmma884(d[0][0][0], d[0][0][1], a0, b0);
        dmma884(d[0][1][0], d[0][1][1], a0, b1);
        dmma884(d[1][0][0], d[1][0][1], a1, b0);
        dmma884(d[1][1][0], d[1][1][1], a1, b1);
      }
#pragma unroll
      for (int hm = 0; hm < 2; ++hm) {
        const int j = 16 * mp + 8 * hm + gid;
        if (j < NV) {
          double* qr = Qo + (long long)j * NC;
#pragma unroll
          for (int hn = 0; hn < 2; ++hn) {
            const int c = c0 + n0 + 8 * hn + 2 * tig;
            if (c < NC) qr[c] = d[hm][hn][0];
            if (c + 1 < NC) qr[c + 1] = d[hm][hn][1];
          }
        }
      }
    }
    __syncthreads();
    ph(2);
    c0 += ncp;
  }
  if (prof && t == 0) atomicAdd(prof + 3, 1ULL);
}

// The same projection for whole leaves (s % 32 == 0) with every operand moved by the TMA
// engine (cp.async.bulk.tensor, host-encoded maps, LeafArgs::lmap / xmap) and no CTA barrier
// in the product loop:
//   * V: one 132 x r_l box of L_l per level (rows li0 .. li0+131, or li0-s+1 .. for a child-0
//     leaf, whose run is then reversed in place); each level's k_l columns form a 128-byte
//     aligned block at pitch LEAF_LDV (colofs[j] = shared offset of V column j); the exact /
//     padding columns are written by the threads;
//   * X: 132 x 16 boxes (16 panel columns) through a ring of NB slots, each with a "full"
//     mbarrier (bytes in flight) and a shared counter of the warps done with it: the last warp
//     to finish a chunk refills its slot with chunk c + NB at once (no producer warp);
//   * work unit = (m-tile pair) x (16-column chunk); unit u of the global order (chunk-major)
//     belongs to warp (u + 1) % 8, balanced across chunks (warp 0, which issues the first
//     copies, gets the smaller share).
// Output rows >= NV / columns >= NC of a tile are dropped (a product column depends only on its
// own B column; out-of-range box columns are zero-filled by the TMA).  Same per-element
// arithmetic as leaf_project: Q[j][c] = sum over k0 ascending of the 4-term DMMA k-steps.
#define PB_NB_MAX 4
__device__ __forceinline__ void tma_load_2d(void* dst, const void* map, int c0, int c1, unsigned long long* bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const void* map, int c0, int c1, int c2,
                                            unsigned long long* bar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
               ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)) : "memory");
}

// 2 x 2 DMMA tiles of the projection over K = S (S = 0: runtime K = s)
template <int S>
__device__ __forceinline__ void proj_tile2x2(double (&d)[2][2][2], const double* ap0, const double* ap1,
                                             const double* bp0, const double* bp1, int s) {
  const int K = S ? S : s;
#pragma unroll 8
  for (int k0 = 0; k0 < K; k0 += 4) {
    const double a0 = ap0[k0], a1 = ap1[k0], b0 = bp0[k0], b1 = bp1[k0];
    dmma884(d[0][0][0], d[0][0][1], a0, b0);
    dmma884(d[0][1][0], d[0][1][1], a0, b1);
    dmma884(d[1][0][0], d[1][0][1], a1, b0);
    dmma884(d[1][1][0], d[1][1][1], a1, b1);
  }
}

__device__ __forceinline__ bool leaf_project_tma(const LeafArgs& a, double* smem, const PanelCol* pcd,
                                                 int c_begin, int NC, int s, int inst, int r0, double* Qo,
                                                 int c_lo, unsigned long long* prof = nullptr,
                                                 const double* x0s = nullptr) {
  __shared__ unsigned long long bars[1 + PB_NB_MAX];   // [0] V, [1..NB] chunk slots "full"
  __shared__ int cnt[PB_NB_MAX];                        // warps done with a chunk slot
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31, gid = lane >> 2, tig = lane & 3;
  const TreeDev& tr = a.tree;
  const int L = tr.L, NV = NC - 1, MP = (NV + 15) >> 4;
  constexpr int LDV = LEAF_LDV, CW = 16;
  const int NCOL = NC - c_lo, NCH = (NCOL + CW - 1) / CW;
  if (!a.lmap || !a.xmap || (s & 31) || s > LEAF_MAX || NCOL < 1 || L < 1) return false;
  long long ph_t = clock64();
  const bool pw = prof && t == 32;                    // (debug: warp 1's phase clocks)
  auto ph = [&](int i) {
    if (pw) { const long long t_ = clock64(); atomicAdd(prof + i, (unsigned long long)(t_ - ph_t)); ph_t = t_; }
  };
  // shared layout: colofs (ints) in the front scratch; V level blocks after the descriptors
  int* colofs = reinterpret_cast<int*>(smem);
  // (offsets from the dynamic shared array itself, so that the loads below stay LDS)
  int voff = (int)(reinterpret_cast<const double*>(pcd + (NC - c_begin)) - smem);
  voff += (int)(((128u - ((smem_u32(smem) + 8u * (unsigned)voff) & 127u)) & 127u) >> 3);
  double* Vs = smem + voff;
  auto lev_block = [&](int l) { return round_up(a.kl[l] * LDV, 16); };
  int vtot = 0;
  for (int l = 0; l < L; ++l) vtot += lev_block(l);
  double* Xb = Vs + vtot;
  const int NB = min(PB_NB_MAX, (int)((smem + LEAF_FRONT + LEAF_BIG - Xb) / (CW * LDV)));
  if (NB < 2) return false;
  FDE_ASSERT(NV <= NCOL_MAX && (smem_u32(Vs) & 127) == 0 && (smem_u32(Xb) & 127) == 0 &&
             Xb + NB * CW * LDV <= smem + LEAF_FRONT + LEAF_BIG && s <= LDV);
  for (int j = t; j < NV; j += LEAF_THREADS) {        // V column j = X column j + 1
    int l = 0, o = 0;
    while (l + 1 < L && a.xcol[l + 1] - 1 <= j) { o += lev_block(l); ++l; }
    colofs[j] = o + (j - (a.xcol[l] - 1)) * LDV;
  }
  const unsigned xbytes = CW * LDV * 8;
  auto issue_chunk = [&](int c) {                     // (lane 0 of the issuing warp)
    unsigned long long* fb = bars + 1 + (c % NB);
    mbar_expect_tx(fb, xbytes);
    tma_load_3d(Xb + (c % NB) * CW * LDV, a.xmap, r0, c_lo + c * CW, inst, fb);
  };
  if (warp == 0) {
    // the previous task's generic accesses of this shared memory, and X (written by other CTAs,
    // acquired by the scheduler), ordered before the TMA (async proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
    const int rl = lane < L ? a.rank[inst * L + lane] : 0;
    int vbytes = rl * LDV * 8;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) vbytes += __shfl_xor_sync(0xffffffffu, vbytes, o);
    if (lane == 0) {
      for (int i = 0; i < 1 + PB_NB_MAX; ++i) mbar_init(bars + i, 1u);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(bars, (unsigned)vbytes);
    }
    __syncwarp();
    if (rl > 0) {                                     // lane l: the kind-2 columns of level l
      int o = 0;
      for (int l = 0; l < lane; ++l) o += lev_block(l);
      const PanelCol pc = pcd[a.xcol[lane] - c_begin];
      FDE_ASSERT(pc.kind == 2 && rl < a.kl[lane] && o + rl * LDV <= vtot);
      const int row0 = pc.lstep < 0 ? pc.li0 - (s - 1) : pc.li0;
      tma_load_2d(Vs + o, static_cast<const CUtensorMapLike*>(a.lmap) + (inst * L + lane), row0, 0, bars);
    }
    if (lane == 0)
      for (int c = 0; c < min(NB, NCH); ++c) issue_chunk(c);
  } else if (t >= 32 && t < 32 + PB_NB_MAX) {
    cnt[t - 32] = 0;
  }
  __syncthreads();                                    // (colofs complete)
  // exact / padding V columns: warp per column, lanes over rows (columns the TMA does not touch)
  for (int j = warp; j < NV; j += LEAF_WARPS) {
    const PanelCol pc = pcd[j + 1 - c_begin];
    if (pc.kind != 2)
      for (int i = lane; i < s; i += 32) Vs[colofs[j] + i] = (pc.kind == 3 && pc.li0 + pc.lstep * i == 0) ? 1.0 : 0.0;
  }
  ph(4);
  mbar_wait(bars, 0);
  ph(5);
  // child-0 runs arrived forward: reverse them in place (warp per column, lanes over pairs)
  for (int j = warp; j < NV; j += LEAF_WARPS) {
    const PanelCol pc = pcd[j + 1 - c_begin];
    if (pc.kind == 2 && pc.lstep < 0) {
      double* col = Vs + colofs[j];
      for (int i = lane; i < (s >> 1); i += 32) {
        const double x = col[i], y = col[s - 1 - i];
        col[i] = y; col[s - 1 - i] = x;
      }
    }
  }
  __syncthreads();
  for (int c = 0; c < NCH; ++c) {
    ph(6);
    mbar_wait(bars + 1 + c % NB, (c / NB) & 1);
    ph(7);
    const double* Xs = Xb + (c % NB) * CW * LDV;
    const int col0 = c_lo + c * CW;
    for (int mp = (warp - 1 - (c * MP) % LEAF_WARPS + 2 * LEAF_WARPS) % LEAF_WARPS; mp < MP; mp += LEAF_WARPS) {
      const int j0 = 16 * mp + gid, j1 = j0 + 8;
      const double* ap0 = Vs + colofs[j0 < NV ? j0 : 0] + tig;
      const double* ap1 = Vs + colofs[j1 < NV ? j1 : 0] + tig;
      const double* bp0 = Xs + gid * LDV + tig;
      const double* bp1 = bp0 + 8 * LDV;
      double d[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};
      if (s == LEAF_MAX) proj_tile2x2<LEAF_MAX>(d, ap0, ap1, bp0, bp1, s);   // (compile-time trip count)
      else proj_tile2x2<0>(d, ap0, ap1, bp0, bp1, s);
#pragma unroll
      for (int hm = 0; hm < 2; ++hm) {
        const int j = 16 * mp + 8 * hm + gid;
        if (j < NV) {
          double* qr = Qo + (long long)j * NC;
#pragma unroll
          for (int hn = 0; hn < 2; ++hn) {
            const int cc = col0 + 8 * hn + 2 * tig;
            if (cc < NC) qr[cc] = d[hm][hn][0];
            if (cc + 1 < NC) qr[cc + 1] = d[hm][hn][1];
          }
        }
      }
    }
    // the last warp done with this slot refills it with chunk c + NB
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&cnt[c % NB], 1) == LEAF_WARPS - 1 && c + NB < NCH) {
        cnt[c % NB] = 0;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_chunk(c + NB);
      }
    }
  }
  if (x0s) {
    // Q[:, 0] = V_all^T x0 with the staged V (fused BB' task): one m-tile per warp item, the
    // right-hand side in B-fragment column 0 (the other 7 columns zero)
    __syncthreads();                                  // (V reversal visible; x0s written before entry)
    const int MT = (NV + 7) >> 3;
    for (int mt = warp; mt < MT; mt += LEAF_WARPS) {
      const int j = 8 * mt + gid;
      const double* ap = Vs + colofs[j < NV ? j : 0] + tig;
      double d0 = 0.0, d1 = 0.0;
#pragma unroll 8
      for (int k0 = 0; k0 < s; k0 += 4) dmma884(d0, d1, ap[k0], gid == 0 ? x0s[k0 + tig] : 0.0);
      if (tig == 0 && j < NV) Qo[(long long)j * NC] = d0;
    }
  }
  ph(6);
  __syncthreads();                                    // (smem and barriers free for the next task)
  ph(8);
  if (pw) atomicAdd(prof + 3, 1ULL);
  if (t == 0)
    for (int i = 0; i < 1 + PB_NB_MAX; ++i) mbar_inval(bars + i);
  return true;
}

// COOP: solve a last round of 1-2 stripes with 4-warp groups (k_run; the extra call raises the
// register pressure of the fused k_step kernel into spills, so it stays off there)
template <bool COOP = false>
__device__ __forceinline__ void leaf_task(const LeafArgs& a, double* smem, int leaf, int inst,
                                          bool do_proj = true) {
  double* S = smem;                               // 32 x 33 scratch (g staging, Gauss-Jordan)
  double* dps = S + 32 * 33;                      // d+ / d- of the leaf rows
  double* dms = dps + LEAF_MAX;
  double* bs = dms + LEAF_MAX;                    // fused rhs b = u + dt f of the leaf
  PanelCol* pcd = reinterpret_cast<PanelCol*>(bs + LEAF_MAX);   // panel column descriptors
  double* A = smem + LEAF_FRONT;                  // [LEAF_MAX cols][LDA_LEAF]
  const TreeDev& tr = a.tree;
  const int t = threadIdx.x, warp = t >> 5;
  const int lane = t & 31, gid = lane >> 2, tig = lane & 3;
  double* Ys = A + LEAF_MAX * LDA_LEAF + warp * 8 * YLD;   // warp-private 128 x 8 stripe buffer
  const int n = tr.n;
  const int r0 = tr.leaf_r0[leaf], s = tr.leaf_n[leaf];
  const int sp = round_up(s, 32), nb = sp >> 5;
  const int where = inst * 65536 + leaf;
  FDE_ASSERT(s >= 1 && s <= LEAF_MAX && r0 >= 0 && r0 + s <= tr.n && a.xcol[tr.L] <= NCOL_MAX);
  double* LUg = a.LU + (long long)inst * a.lustride + (long long)leaf * LEAF_SLOT;
  double acc[16][2];
  // debug (FDE_TRACE_LEVELS): per-CTA globaltimer stamps at the phase boundaries
  const bool trc = a.trace && t == 0 && leaf < 1024 && inst == 0;
  auto stamp = [&](int ph) {
    if (a.trace) {
      __syncthreads();
      if (trc) {
        unsigned long long tm;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm));
        a.trace[2048 + leaf * 8 + ph] = tm;
      }
    }
  };
  stamp(0);
  long long lph_t = clock64();
  auto lph = [&](int i) {                         // (a.prof: CTA-synchronised phase clocks)
    if (a.prof) {
      __syncthreads();
      if (t == 0) { const long long t_ = clock64(); atomicAdd(a.prof + i, (unsigned long long)(t_ - lph_t)); lph_t = t_; }
    }
  };

  const long long bclk = clock64();
  if (a.mode == 0) {
    // ---- S3: generate the leaf block from g and d+- (column-major), identity padding
    const double c = a.cfac[inst];
    const double* gi = a.g + (long long)inst * a.gstride;
    const double* dpi = a.dp + (long long)inst * n + r0;
    const double* dmi = a.dm + (long long)inst * n + r0;
    // Toeplitz entries by offset: tt[d + sp] = T[i, j] for d = i - j (-g_{d+1} for d >= -1,
    // else 0), d in [-sp, sp] (S is free scratch; 2 sp + 1 <= 257 doubles)
    double* tt = S;
    for (int e = t; e <= 2 * sp; e += LEAF_THREADS) {
      const int d = e - sp;
      tt[e] = (d >= -1 && d + 1 <= n + 1) ? -gi[d + 1] : 0.0;
    }
    for (int i = t; i < s; i += LEAF_THREADS) {
      dps[i] = dpi[i]; dms[i] = dmi[i];
      if (a.nf) bs[i] = a.u_prev[(long long)inst * n + r0 + i] + a.dt * a.f[(long long)inst * n + r0 + i];
    }
    {                                                // panel column descriptors (one per column)
      const int cb = 1 - a.nf, ce = a.xcol[tr.L];
      for (int cc = t; cc < ce - cb; cc += LEAF_THREADS) pcd[cc] = panel_col(a, inst, leaf, r0, cb + cc, ce);
    }
    __syncthreads();
    const bool btr = a.trace && leaf == 0 && inst == 0 && (t == 0 || t == 128);
    long long bt0 = clock64();
    if (btr) a.trace[980 + (t >> 7) * 4] = bt0 - bclk;
    {
      // lane owns rows lane + 32u (their d+- in registers); 4 independent elements per column
      double dpr[LEAF_MAX / 32], dmr[LEAF_MAX / 32];
#pragma unroll
      for (int u = 0; u < LEAF_MAX / 32; ++u) {
        const int i = lane + 32 * u;
        dpr[u] = i < s ? dps[i] : 0.0;
        dmr[u] = i < s ? dms[i] : 0.0;
      }
      // the gj_role warps build block column 0 first and invert its diagonal block (quad GJ)
      // while the others build the remaining columns (the first pivot chain overlaps the build)
      const bool gjw = gj_role<true>(warp);
      const int rw = role_idx<true>(warp);
      const int jlo = gjw ? 8 * rw : 32 + rw;
      const int jhi = gjw ? min(8 * rw + 8, sp) : sp;
      const int jst = gjw ? 1 : LEAF_WARPS - GJ_WARPS;
      for (int j = jlo; j < jhi; j += jst) {
#pragma unroll
        for (int u = 0; u < LEAF_MAX / 32; ++u) {
          const int i = lane + 32 * u;
          if (i < sp) {
            const double tij = tt[i - j + sp], tji = tt[j - i + sp];   // T[i,j], T^T[i,j] = T[j,i]
            const double v = (i < s && j < s) ? fma(c, fma(dpr[u], tij, dmr[u] * tji), i == j ? a.shift : 0.0)
                                              : (i == j ? 1.0 : 0.0);
            A[i + j * LDA_LEAF] = v;
          }
        }
      }
      if (btr) { const long long t_ = clock64(); a.trace[981 + (t >> 7) * 4] = t_ - bt0; bt0 = t_; }
      if (gjw) {
        asm volatile("bar.sync 1, %0;" ::"n"(GJ_WARPS * 32) : "memory");
        quad_gj_inv32<true>(A, LDA_LEAF, S + 272, a.st, where);    // (S + 272: clear of the staged tt)
        if (btr) { const long long t_ = clock64(); a.trace[982] = t_ - bt0; }
      }
    }
    __syncthreads();
    stamp(1);
    lph(0);
    // ---- S4: block LU (inverse-diagonal form, off-diagonal blocks negated); block 0 done
    leaf_block_lu(A, sp, S + 272, a.st, where, a.trace, true);
    // for the deferred rhs column (leaf_rhs_final): the LU in its shared-memory layout as one
    // bulk store of the TMA engine, overlapped with the panel (which only reads it); completed
    // before the task ends (lu_bulk_wait)
    double* LUr = a.store_lu ? a.LU + (long long)inst * a.lustride + (long long)leaf * LEAF_RSLOT : nullptr;
    const bool lu_bulk = a.store_lu && (reinterpret_cast<unsigned long long>(LUr) & 15) == 0;
    if (lu_bulk) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // (this thread's LU writes)
      __syncthreads();
      if (t == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(LUr), "r"(smem_u32(A)), "r"((unsigned)(sp * LDA_LEAF * 8)) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else if (a.store_lu) {
      for (int j = warp; j < sp; j += LEAF_WARPS)
        for (int i = lane; i < sp; i += 32) LUr[i + j * LDA_LEAF] = A[i + j * LDA_LEAF];
    }
    lph(1);
    stamp(2);
    // ---- panel X = A_leaf^{-1} [b | U_0 .. U_{L-1}] by warp stripes of 8 columns
    const int c_begin = 1 - a.nf, c_end = a.xcol[tr.L];
    const int nstripe = (c_end - c_begin + 7) >> 3;
    double* Xi = a.X + (long long)inst * a.xstride + r0;
    const bool ptr = a.trace && t == 0 && leaf == 0 && inst == 0;
    long long pt0 = clock64(), pt1 = clock64();
#define PTR(i) do { if (ptr) { const long long t_ = clock64(); a.trace[970 + (i)] += t_ - pt0; pt0 = t_; } \
                       if (a.prof && t == 0) { const long long t_ = clock64(); atomicAdd(a.prof + 5 + (i), (unsigned long long)(t_ - pt1)); pt1 = t_; } } while (0)
    // software pipeline: the raw L_l gathers of the warp's next stripe are in flight (in
    // registers) while the current stripe is solved
    double pv[8][4];
    auto load_raw = [&](int st) {
      const int cs = c_begin + 8 * st;
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        const PanelCol pc = cs + cc < c_end ? pcd[cs + cc - c_begin] : PanelCol{a.Lf, 0, 0, 0, 0, 0};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int i = lane + 32 * q;
          // branch-free: every descriptor carries a valid pointer (kind != 2: step 0 at a.Lf)
          const int ic = i < s ? i : s - 1;
          // (no use of the value here: the load stays in flight over the current stripe's solve;
          //  the kind / row masks are applied where the value is scaled)
          pv[cc][q] = __ldg(pc.Lq + pc.li0 + pc.lstep * ic);
        }
      }
    };
    // The last round of stripes (nstripe % 8 of them) would keep only that many warps busy: when
    // it holds at most 2 stripes, each is solved by a group of 4 warps that split its row blocks
    // (leaf_coop_stripe), and the per-warp loop stops at the last full round.
    const int ntail = nstripe % LEAF_WARPS;
#ifdef FDE_ALL_COOP
    const int nsolo = (COOP && nb > 1) ? 0 : nstripe;
#else
    const int nsolo = (COOP && ntail >= 1 && ntail <= 2 && nb > 1) ? nstripe - ntail : nstripe;
#endif
    if (warp < nsolo) load_raw(warp);
    for (int st = warp; st < nsolo; st += LEAF_WARPS) {
      // scale the 8 panel columns into the warp's stripe buffer, then into registers
      const int cs = c_begin + 8 * st;
      // (branch-free: every load is unconditional and in range, the kind picks by selects, so
      //  the 32 shared loads of a lane are in flight together)
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        const PanelCol pc = cs + cc < c_end ? pcd[cs + cc - c_begin] : PanelCol{a.Lf, 0, 0, 0, 0, 0};
        const double* sc = pc.sel ? dms : dps;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int i = lane + 32 * q, ic = i < s ? i : s - 1;
          const double scv = sc[ic], bv = bs[ic];
          const double v2 = pv[cc][q] * (-c * scv);
          const double v3 = (pc.li0 + pc.lstep * i == 0) ? -c * scv : 0.0;
          double v = pc.kind == 2 ? v2 : pc.kind == 3 ? v3 : pc.kind == 1 ? bv : 0.0;
          Ys[i + cc * YLD] = i < s ? v : 0.0;
        }
      }
      __syncwarp();
      if (a.prof && t == 0 && st == warp) { const long long t_ = clock64(); atomicAdd(a.prof + 9, (unsigned long long)(t_ - pt1)); }
      PTR(0);
#pragma unroll
      for (int tt = 0; tt < 16; ++tt) {
        const int i = 8 * tt + gid;
        acc[tt][0] = tt < 4 * nb ? Ys[i + 2 * tig * YLD] : 0.0;
        acc[tt][1] = tt < 4 * nb ? Ys[i + (2 * tig + 1) * YLD] : 0.0;
      }
      __syncwarp();
      PTR(1);
      if (st + LEAF_WARPS < nsolo) load_raw(st + LEAF_WARPS);
      stripe_solve(acc, A, nb, Ys);
      PTR(2);
#pragma unroll
      for (int tt = 0; tt < 16; ++tt) {
        if (tt < 4 * nb) {
          const int i = 8 * tt + gid;
          Ys[i + 2 * tig * YLD] = acc[tt][0];
          Ys[i + (2 * tig + 1) * YLD] = acc[tt][1];
        }
      }
      __syncwarp();
      for (int cc = 0; cc < 8 && cs + cc < c_end; ++cc)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int i = lane + 32 * q;
          if (i < s) Xi[(long long)(cs + cc) * n + i] = Ys[i + cc * YLD];
        }
      __syncwarp();
      PTR(3);
    }
#undef PTR
    if (COOP && nsolo < nstripe) {
      __syncthreads();                               // (every warp-private stripe buffer free)
      const int g = warp >> 2;                       // group g solves stripes nsolo + g, + 2, ..
      for (int st2 = nsolo + g; st2 < nstripe; st2 += 2) {
        if (st2 > nsolo + g) asm volatile("bar.sync %0, %1;" ::"r"(2 + g), "n"(128) : "memory");
        leaf_coop_stripe(A, nb, s, c, a, pcd, c_begin, c_end, st2, dps, dms, bs,
                         A + LEAF_MAX * LDA_LEAF + (4 * g) * 8 * YLD, Xi, n);
      }
      __syncthreads();
    }
    lph(4);
    if (a.keep) {
      // kept factor = the explicit leaf inverse (stripe solves of the identity): a later solve
      // is one streaming pass over it (k_solve.cuh), not a sequential block sweep
      for (int st = warp; st < sp / 8; st += LEAF_WARPS) {
#pragma unroll
        for (int tt = 0; tt < 16; ++tt) {
          const int i = 8 * tt + gid;
          acc[tt][0] = (i == 8 * st + 2 * tig) ? 1.0 : 0.0;
          acc[tt][1] = (i == 8 * st + 2 * tig + 1) ? 1.0 : 0.0;
        }
        stripe_solve(acc, A, nb, Ys);
#pragma unroll
        for (int tt = 0; tt < 16; ++tt)
          if (tt < 4 * nb) {
            const int i = 8 * tt + gid;
            LUg[i + (8 * st + 2 * tig) * sp] = acc[tt][0];
            LUg[i + (8 * st + 2 * tig + 1) * sp] = acc[tt][1];
          }
      }
    }
    if (lu_bulk && t == 0) {                         // (the store has read the LU region and landed)
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    stamp(3);
    if (a.Q && do_proj)
      leaf_project(a, A, pcd, c_begin, c_end, s, sp, Xi, a.Q + (long long)inst * a.qinst + (long long)leaf * a.qstride,
                   c_begin);
    stamp(4);
  } else {
    // ---- solve mode: factor from HBM, right-hand sides b (+ dt f) -> y (y may alias b)
    for (int j = warp; j < sp; j += LEAF_WARPS)
      for (int i = lane; i < sp; i += 32) A[i + j * LDA_LEAF] = LUg[i + j * sp];
    __syncthreads();
    const long long ib = (long long)inst * a.ld * a.nrhs + r0;
    const int nstripe = (a.nrhs + 7) >> 3;
    for (int st = warp; st < nstripe; st += LEAF_WARPS) {
      const int cA = 8 * st + 2 * tig;
#pragma unroll
      for (int tt = 0; tt < 16; ++tt) {
        const int i = 8 * tt + gid;
        const bool in = tt < 4 * nb && i < s;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          double v = 0.0;
          if (in && cA + j < a.nrhs) {
            const long long o = ib + (long long)(cA + j) * a.ld + i;
            v = a.b[o];
            if (a.f) v += a.dt * a.f[o];               // b = u + dt f (S7)
          }
          acc[tt][j] = v;
        }
      }
      stripe_solve(acc, A, nb, Ys);
#pragma unroll
      for (int tt = 0; tt < 16; ++tt) {
        const int i = 8 * tt + gid;
        if (tt < 4 * nb && i < s) {
          if (cA < a.nrhs) a.y[ib + (long long)cA * a.ld + i] = acc[tt][0];
          if (cA + 1 < a.nrhs) a.y[ib + (long long)(cA + 1) * a.ld + i] = acc[tt][1];
        }
      }
    }
  }
}

__global__ void __launch_bounds__(LEAF_THREADS, 1)
k_leaf(const LeafArgs a) {
  extern __shared__ double smem[];
  leaf_task(a, smem, blockIdx.x, blockIdx.y);
}

// The projection Q_leaf = V_all^T X_leaf as a task of its own (k_step.cuh): X is read back from
// global memory, so it can run on any SM once the leaf's panel is written.
// q0 (k_run fused BB' task): x0 = X[:, 0] of the leaf sits in smem[0, s) (leaf_rhs_final) and the
// projection also forms Q[:, 0] = V_all^T x0.
__device__ __forceinline__ void leaf_proj_task(const LeafArgs& a, double* smem, int leaf, int inst,
                                               bool q0 = false) {
  double* bs = smem + 32 * 33 + 2 * LEAF_MAX;
  PanelCol* pcd = reinterpret_cast<PanelCol*>(bs + LEAF_MAX);
  const TreeDev& tr = a.tree;
  const int r0 = tr.leaf_r0[leaf], s = tr.leaf_n[leaf], sp = round_up(s, 32);
  const int c_begin = 1 - a.nf, c_end = a.xcol[tr.L];
  for (int cc = threadIdx.x; cc < c_end - c_begin; cc += LEAF_THREADS)
    pcd[cc] = panel_col(a, inst, leaf, r0, c_begin + cc, c_end);
  const double* Xi = a.X + (long long)inst * a.xstride + r0;
  double* Qo = a.Q + (long long)inst * a.qinst + (long long)leaf * a.qstride;
  double* x0s = smem + 512;                           // (clear of the projection's colofs)
  if (q0)
    for (int i = threadIdx.x; i < s; i += LEAF_THREADS) x0s[i] = smem[i];
  __syncthreads();                                    // (descriptors visible)
  if (leaf_project_tma(a, smem, pcd, c_begin, c_end, s, inst, r0, Qo, c_begin, a.prof ? a.prof + 8 : nullptr,
                       q0 ? x0s : nullptr))
    return;
  // (cp.async path: column 0 is projected with the others, read back from X)
  leaf_project(a, smem + LEAF_FRONT, pcd, c_begin, c_end, s, sp, Xi, Qo, q0 ? 0 : c_begin,
               a.prof ? a.prof + 8 : nullptr);
}
