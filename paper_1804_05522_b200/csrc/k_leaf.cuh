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

#define LEAF_THREADS 256
#define LEAF_WARPS (LEAF_THREADS / 32)
#define LDA_LEAF 132                 // column-major leading dims (= 4 mod 16: conflict-free DMMA frags)
#define LDP_LEAF 132
#define NCHUNK 64                    // right-hand-side columns per panel chunk
#define LEAF_SLOT (LEAF_MAX * LEAF_MAX)   // doubles per kept leaf factor
#define LEAF_SMEM ((LEAF_MAX * LDA_LEAF + NCHUNK * LDP_LEAF + 32 * 33 + 2 * LEAF_MAX) * 8)
#define LEAF_OVW 8                   // register tiles per warp of an overwrite GEMM

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
  DevStatus* st;
  unsigned long long* trace;                 // optional phase clocks (FDE_TRACE_LEVELS)
};

// ---- DMMA GEMMs on column-major shared-memory operands ---------------------------------
// C[M x N] -= A[M x K] B[K x N]; tiles round-robin over warps [w0, w0 + nw); M, N % 8 == 0,
// K % 4 == 0.  Optionally skips the tile block (skip_m0.., skip_n0..) of size 32 x 32.
__device__ __forceinline__ void cm_gemm_sub(double* C, int ldc, const double* A, int lda,
                                            const double* B, int ldb, int M, int N, int K, int w0,
                                            int nw, int skip_m0 = -1, int skip_n0 = -1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gid = lane >> 2, tig = lane & 3;
  const int w = warp - w0;
  if (w < 0 || w >= nw) return;
  const int MB = M >> 3, NT = MB * (N >> 3);
  for (int t0 = w; t0 < NT; t0 += 4 * nw) {
    double d[4][2];
    int mo[4], no[4];
    bool ok[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = t0 + u * nw;
      mo[u] = (t % MB) * 8; no[u] = (t / MB) * 8;
      ok[u] = t < NT && !(skip_m0 >= 0 && mo[u] >= skip_m0 && mo[u] < skip_m0 + 32 &&
                          no[u] >= skip_n0 && no[u] < skip_n0 + 32);
      if (ok[u]) {
        d[u][0] = C[mo[u] + gid + (no[u] + 2 * tig) * ldc];
        d[u][1] = C[mo[u] + gid + (no[u] + 2 * tig + 1) * ldc];
      }
    }
    for (int k0 = 0; k0 < K; k0 += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (ok[u])
          dmma884(d[u][0], d[u][1], -A[mo[u] + gid + (k0 + tig) * lda],
                  B[k0 + tig + (no[u] + gid) * ldb]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
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

// tiles over the rows [r_lo, r_hi) and [r2_lo, r2_hi) (two row ranges) x N columns
__device__ __forceinline__ void ovw_compute(OvwTiles& T, const double* A, int lda, const double* B,
                                            int ldb, int r_lo, int r_hi, int r2_lo, int r2_hi, int N,
                                            int K) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gid = lane >> 2, tig = lane & 3;
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
  for (int k0 = 0; k0 < K; k0 += 4) {
#pragma unroll
    for (int u = 0; u < LEAF_OVW; ++u)
      if (u < T.cnt)
        dmma884(T.d[u][0], T.d[u][1], A[T.mo[u] + gid + (k0 + tig) * lda],
                B[k0 + tig + (T.no[u] + gid) * ldb]);
  }
}

__device__ __forceinline__ void ovw_store(const OvwTiles& T, double* O, int ldo) {
  const int lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
#pragma unroll
  for (int u = 0; u < LEAF_OVW; ++u)
    if (u < T.cnt) {
      O[T.mo[u] + gid + (T.no[u] + 2 * tig) * ldo] = T.d[u][0];
      O[T.mo[u] + gid + (T.no[u] + 2 * tig + 1) * ldo] = T.d[u][1];
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
#pragma unroll
    for (int j = 0; j < 1024 / LEAF_THREADS; ++j) {
      const int e = t + j * LEAF_THREADS, i = e & 31, c = e >> 5;
      const double aic = src[i + c * ls], aik = src[i + kk * ls], akc = src[kk + c * ls];
      double v;
      if (i == kk) v = (c == kk) ? rp : akc * rp;
      else v = (c == kk) ? -aik * rp : fma(-aik * rp, akc, aic);
      dst[i + c * lt] = v;
    }
    __syncthreads();
  }
}

// Block LU in inverse-diagonal form of A (sp x sp, sp % 32 == 0) in shared memory.
// On entry the first diagonal block must already be inverted.
__device__ void leaf_block_lu(double* A, int sp, double* S, DevStatus* st, int where) {
  const int nb = sp >> 5;
  for (int kb = 0; kb < nb; ++kb) {
    const int k0 = kb * 32;
    // Lt / Ut = A(rows != kb, kb) D_k   (overwrite the block column)
    if (nb > 1) {
      OvwTiles T;
      ovw_compute(T, A + k0 * LDA_LEAF, LDA_LEAF, A + k0 + k0 * LDA_LEAF, LDA_LEAF, 0, k0,
                  k0 + 32, sp, 32, 32);
      __syncthreads();
      ovw_store(T, A + k0 * LDA_LEAF, LDA_LEAF);
      __syncthreads();
    }
    if (kb + 1 < nb) {
      const int k1 = k0 + 32;
      // trailing update, then the next diagonal block is inverted
      cm_gemm_sub(A + k1 + k1 * LDA_LEAF, LDA_LEAF, A + k1 + k0 * LDA_LEAF, LDA_LEAF,
                  A + k0 + k1 * LDA_LEAF, LDA_LEAF, sp - k1, sp - k1, 32, 0, LEAF_WARPS);
      __syncthreads();
      blk_gj_inv32(A + k1 + k1 * LDA_LEAF, LDA_LEAF, S, st, where);
    }
  }
}

// P (sp x ncp) <- A^{-1} P with the block factor in A.
__device__ void leaf_block_solve(const double* A, int sp, double* P, int ncp) {
  const int nb = sp >> 5;
  for (int kb = 0; kb + 1 < nb; ++kb) {             // forward: y_i -= Lt_ik y_k
    const int k0 = kb * 32;
    cm_gemm_sub(P + k0 + 32, LDP_LEAF, A + k0 + 32 + k0 * LDA_LEAF, LDA_LEAF, P + k0, LDP_LEAF,
                sp - k0 - 32, ncp, 32, 0, LEAF_WARPS);
    __syncthreads();
  }
  for (int kb = nb - 1; kb >= 0; --kb) {            // backward: x_j -= Ut_jk y_k ; x_k = D_k y_k
    const int k0 = kb * 32;
    OvwTiles T;
    ovw_compute(T, A + k0 + k0 * LDA_LEAF, LDA_LEAF, P + k0, LDP_LEAF, 0, 32, 0, 0, ncp, 32);
    if (k0 > 0)
      cm_gemm_sub(P, LDP_LEAF, A + k0 * LDA_LEAF, LDA_LEAF, P + k0, LDP_LEAF, k0, ncp, 32, 0,
                  LEAF_WARPS);
    __syncthreads();
    {
      // ovw tiles index rows from 0: shift to block row k0
      const int lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
#pragma unroll
      for (int u = 0; u < LEAF_OVW; ++u)
        if (u < T.cnt) {
          P[k0 + T.mo[u] + gid + (T.no[u] + 2 * tig) * LDP_LEAF] = T.d[u][0];
          P[k0 + T.mo[u] + gid + (T.no[u] + 2 * tig + 1) * LDP_LEAF] = T.d[u][1];
        }
    }
    __syncthreads();
  }
}

// Panel chunk generation (factor mode): X columns [c_first, c_first + nc) of this leaf's rows
// into P (sp x ncp, zero padded).  Warp per column (level, node and rank are warp-uniform),
// lanes over rows; d+- of the leaf rows are staged in shared memory (dps, dms).
//   column 0 (fused rhs): b = u_prev + dt f
//   level l column q:  q < r: scaled low-rank column; r <= q < k-1: zero padding;
//                      q = k-1: exact column (the single entry -g_0 of the other triangle)
__device__ void gen_chunk(const LeafArgs& a, int inst, int leaf, int r0, int s, int sp, int c_first,
                          int nc, int ncp, double* P, const double* dps, const double* dms, double c) {
  const TreeDev& tr = a.tree;
  const int n = tr.n, L = tr.L, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int cc = warp; cc < ncp; cc += LEAF_WARPS) {
    double* pc = P + cc * LDP_LEAF;
    const int cg = c_first + cc;
    if (cc >= nc) {
      for (int i = lane; i < sp; i += 32) pc[i] = 0.0;
      continue;
    }
    if (cg == 0) {
      const double* u = a.u_prev + (long long)inst * n + r0;
      const double* f = a.f + (long long)inst * n + r0;
      for (int i = lane; i < sp; i += 32) pc[i] = (i < s) ? u[i] + a.dt * f[i] : 0.0;
      continue;
    }
    int l = 0;
    while (l + 1 < L && a.xcol[l + 1] <= cg) ++l;
    const int q = cg - a.xcol[l], r = a.rank[inst * L + l], kq = a.kl[l];
    const int jn = leaf >> (L - l), child = (leaf >> (L - l - 1)) & 1;
    const int nd = node_index(l, jn);
    const int r0n = tr.node_r0[nd], n1 = tr.node_n1[nd];
    const int m = tr.lev_m[l];
    const double* Lq = a.Lf + (long long)inst * a.lf_stride + tr.lev_lofs[l] + (long long)q * m;
    // row index into L_l: child 0 -> n1-1-(R-r0n) (decreasing), child 1 -> R-r0n-n1
    const int li0 = child == 0 ? n1 - 1 - (r0 - r0n) : r0 - r0n - n1, lstep = child == 0 ? -1 : 1;
    const double* ds = child == 0 ? dms : dps;      // scaling of the low-rank columns
    const double* de = child == 0 ? dps : dms;      // scaling of the exact column
#pragma unroll
    for (int u = 0; u < LEAF_MAX / 32; ++u) {
      const int i = lane + 32 * u;
      if (i >= sp) break;
      double v = 0.0;
      if (i < s) {
        const int li = li0 + lstep * i;
        if (q == kq - 1) v = (li == 0) ? -c * de[i] : 0.0;
        else if (q < r) v = -c * ds[i] * Lq[li];
      }
      pc[i] = v;
    }
  }
}

__global__ void __launch_bounds__(LEAF_THREADS)
k_leaf(const LeafArgs a) {
  extern __shared__ double smem[];
  double* A = smem;                               // [LEAF_MAX cols][LDA_LEAF]
  double* P = smem + LEAF_MAX * LDA_LEAF;         // [NCHUNK cols][LDP_LEAF]
  double* S = P + NCHUNK * LDP_LEAF;              // 32 x 33 Gauss-Jordan scratch
  double* dps = S + 32 * 33;                      // d+ / d- of the leaf rows
  double* dms = dps + LEAF_MAX;
  const TreeDev& tr = a.tree;
  const int leaf = blockIdx.x, inst = blockIdx.y, t = threadIdx.x, warp = t >> 5;
  const int n = tr.n;
  const int r0 = tr.leaf_r0[leaf], s = tr.leaf_n[leaf];
  const int sp = round_up(s, 32);
  const int where = inst * 65536 + leaf;
  double* LUg = a.LU + (long long)inst * a.lustride + (long long)leaf * LEAF_SLOT;

  if (a.mode == 0) {
    // ---- S3: generate the leaf block from g and d+- (column-major), identity padding
    const double c = a.cfac[inst];
    const double* gi = a.g + (long long)inst * a.gstride;
    const double* dpi = a.dp + (long long)inst * n + r0;
    const double* dmi = a.dm + (long long)inst * n + r0;
    for (int j = warp; j < sp; j += LEAF_WARPS)
      for (int i = t & 31; i < sp; i += 32) {
        double v;
        if (i < s && j < s) {
          const int k1 = i - j + 1, k2 = j - i + 1;     // T[i,j] = -g_{i-j+1}, T^T[i,j] = T[j,i]
          const double tij = (k1 >= 0) ? -gi[k1] : 0.0;
          const double tji = (k2 >= 0) ? -gi[k2] : 0.0;
          v = (i == j ? a.shift : 0.0) + c * (dpi[i] * tij + dmi[i] * tji);
        } else {
          v = (i == j) ? 1.0 : 0.0;
        }
        A[i + j * LDA_LEAF] = v;
      }
    for (int i = t; i < s; i += LEAF_THREADS) { dps[i] = dpi[i]; dms[i] = dmi[i]; }
    __syncthreads();
    const bool ldbg = a.trace && blockIdx.x == 0 && blockIdx.y == 0 && t == 0;
    long long llast = clock64();
#define LT(i) do { if (ldbg) { const long long t_ = clock64(); a.trace[900 + (i)] += t_ - llast; llast = t_; } } while (0)
    LT(0);
    const int c_begin = 1 - a.nf, c_end = a.xcol[tr.L];
    blk_gj_inv32(A, LDA_LEAF, S, a.st, where);
    LT(1);
    leaf_block_lu(A, sp, S, a.st, where);
    if (a.keep)
      for (int j = warp; j < sp; j += LEAF_WARPS)
        for (int i = t & 31; i < sp; i += 32) LUg[i + j * sp] = A[i + j * LDA_LEAF];
    LT(2);
    double* Xi = a.X + (long long)inst * a.xstride;
    for (int c0 = c_begin; c0 < c_end; c0 += NCHUNK) {
      const int nc = min(NCHUNK, c_end - c0), ncp = round_up(nc, 8);
      gen_chunk(a, inst, leaf, r0, s, sp, c0, nc, ncp, P, dps, dms, c);
      __syncthreads();
      LT(3);
      leaf_block_solve(A, sp, P, ncp);
      LT(4);
      for (int cc = warp; cc < nc; cc += LEAF_WARPS)
        for (int i = t & 31; i < s; i += 32) Xi[(long long)(c0 + cc) * n + r0 + i] = P[i + cc * LDP_LEAF];
      __syncthreads();
      LT(5);
    }
  } else {
    // ---- solve mode: factor from HBM, right-hand sides b (+ dt f) -> y (y may alias b)
    for (int j = warp; j < sp; j += LEAF_WARPS)
      for (int i = t & 31; i < sp; i += 32) A[i + j * LDA_LEAF] = LUg[i + j * sp];
    const long long ib = (long long)inst * a.ld * a.nrhs;
    for (int c0 = 0; c0 < a.nrhs; c0 += NCHUNK) {
      const int nc = min(NCHUNK, a.nrhs - c0), ncp = round_up(nc, 8);
      for (int e = t; e < sp * ncp; e += LEAF_THREADS) {
        const int i = e % sp, cc = e / sp;
        double v = 0.0;
        if (i < s && cc < nc) {
          const long long o = ib + (long long)(c0 + cc) * a.ld + r0 + i;
          v = a.b[o];
          if (a.f) v += a.dt * a.f[o];                  // b = u + dt f (S7)
        }
        P[i + cc * LDP_LEAF] = v;
      }
      __syncthreads();
      leaf_block_solve(A, sp, P, ncp);
      for (int cc = warp; cc < nc; cc += LEAF_WARPS)
        for (int i = t & 31; i < s; i += 32)
          a.y[ib + (long long)(c0 + cc) * a.ld + r0 + i] = P[i + cc * LDP_LEAF];
      __syncthreads();
    }
  }
}
