// k_levels.cuh -- S5 (Sherman-Morrison-Woodbury level factorisation) and S6 (tree solve)
// as ONE persistent kernel over all levels.
//
// Algebra (node of level l, rows [r0, r0+n1+n2)):
//   A = blkdiag(A11, A22)(I + blkdiag(W1, W2) Z^T),  W1 = A11^{-1} U12,  W2 = A22^{-1} U21,
//   Z^T = [[0, V12^T], [V21^T, 0]],  V12 = [L_l[:n2], e_0],  V21 = [J L_l[:n1], e_{n1-1}],
//   A^{-1} = (I - W K^{-1} Z^T) blkdiag(A11, A22)^{-1},  K = [[I, B], [C, I]],
//   B = V12^T W2,  C = V21^T W1,  Sc = I - C B,
//   K^{-1} [a; b] = [a - B y; y],  y = Sc^{-1} (b - C a).
// Processing the levels from the leaves to the root applies these factors to the ancestor
// columns of X (factor mode; the fused right-hand side is X column 0) or to the right-hand
// sides Y (solve mode, with the kept B, C, Sc^{-1}).
//
// Work decomposition: P = 2^p CTAs per instance; CTA c owns the rows of node c of level p.
//  * local phase (levels L-1 .. p): the CTA walks its subtree in post-order; every node is
//    solved by this CTA alone (no grid synchronisation).
//  * global phase (levels p-1 .. 0): one counter barrier per level; the per-CTA partial
//    products are summed in a fixed order (directly by every CTA of the node when it has
//    <= 8 pieces per child, else split over the node's CTAs + one more barrier); every CTA
//    of a node solves the small K system redundantly (bitwise identical).
//  * every pass over rows is fused: X_targets -= W S_half for level l and, on the updated
//    rows still in shared memory, the partial products V^T X for level l-1 (the targets of
//    level l are exactly the columns level l-1 reduces).  Both contractions run on the FP64
//    tensor cores (DMMA m8n8k4, fde_dmma.cuh).
#pragma once
#include "fde_common.cuh"
#include "fde_dmma.cuh"

#define LV_THREADS 256
#define LV_WARPS (LV_THREADS / 32)
#define MT_RED 16                      // reduce accumulator tiles per warp (8x8 each)
#define LV_SMEM_MAX (226 * 1024)       // dynamic smem cap (static smem of the node solve on top)

struct LvArgs {
  TreeDev tree;
  int mode;                            // 0 factor, 1 solve
  int L, p, P;
  int nf;                              // factor: fused rhs columns (X column 0)
  int CR, lgCR;                        // rows per chunk (power of two >= 8) and its log2
  int ldx, lds, ldk, ldm;              // smem leading dimensions
  int off_Xc, off_Wn, off_Vc, off_Pt, off_Pb, off_T, off_B, off_C, off_Si, off_M;  // doubles
  int xbuf, wbuf, vbuf;                // size of one pipeline buffer of Xc / Wn / Vc (doubles)
  int kl[LMAX];                        // k_l = R_l + 1 (R_l = max rank over the batch)
  int xcol[LMAX + 1];                  // first X column of level l's W block; xcol[L] = end
  long long kofs[LMAX];                // per-instance offset of level l's node store
  long long kstride_inst;
  const double* Lf; long long lf_stride;
  const int* rank;                     // actual per-instance ranks [batch * L]
  double* X; long long xstride;
  double* Y; int ld, nrhs; long long ystride;
  double* Kst;                         // node store: B, C, Sc^{-1} (k x k row-major each)
  double* sums; long long sum_half;    // [inst][node][2][sum_half]; entry (q, col) at q*sum_nc+col
  int sum_nc;
  double* part;                        // [2][inst][P][sum_half]
  unsigned* bar;
  const int* post; int npost;          // post-order template of a level-p subtree (d, jrel)
  DevStatus* st;
  unsigned long long* trace;           // optional phase timestamps (FDE_TRACE_LEVELS), or null
};

struct LvSmem {
  double *Xc, *Wn, *Vc, *Pt, *Pb, *T, *B, *C, *Si, *M;
  int xbuf, wbuf, vbuf;                // second pipeline buffer offsets (doubles)
};

__device__ __forceinline__ unsigned lv_ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void lv_grid_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (lv_ld_acquire(bar) < target) __nanosleep(16);
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ int lv_ncols(const LvArgs& a, int lvl) {   // reduce columns of level lvl
  return a.mode == 1 ? a.nrhs : a.xcol[lvl + 1] - (1 - a.nf);
}
__device__ __forceinline__ int lv_ntgt(const LvArgs& a, int lvl) {    // target columns of level lvl
  return a.mode == 1 ? a.nrhs : a.xcol[lvl] - (1 - a.nf);
}

// ---------------------------------------------------------------------------------------
// One fused pass over up to two contiguous row ranges.
//   update (upd >= 0): T[rows, 0:NT) -= W_upd[rows] S_s, S_s = S half of the sub-range
//   reduce (red >= 0): out[q, c] = sum_rows V_red[row, q] T[row, c]  (node red_node, child red_child)
// T = X[:, tb:] (factor) or Y (solve).  out is k_red x NC row-major with leading dim out_ld.
// Rows are streamed in chunks of CR through a double-buffered cp.async pipeline: the loads of
// chunk i+1 are in flight while the DMMA update/reduce of chunk i runs.
template <int MT>
__device__ void lv_pass(const LvArgs& a, const LvSmem& sm, int inst, int nsub, int ra0, int rb0,
                        const double* S0, int ra1, int rb1, const double* S1, int upd, int red,
                        int red_node, int red_child, double* out, int out_ld) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int n = a.tree.n, CR = a.CR, ldx = a.ldx, lds = a.lds;
  const bool solve = a.mode == 1;
  const int tb = 1 - a.nf;
  const int NC = solve ? a.nrhs : (upd >= 0 ? a.xcol[upd] : a.xcol[red + 1]) - tb;
  const int NCP = round_up(NC, 8);
  if (NC <= 0 && red < 0) return;                 // root without fused right-hand side
  FDE_ASSERT(NCP <= a.lds && rb0 <= n && (nsub < 2 || rb1 <= n) && ra0 >= 0);
  double* T;
  long long cst;
  if (solve) { T = a.Y + (long long)inst * a.ystride; cst = a.ld; }
  else { T = a.X + (long long)inst * a.xstride + (long long)tb * n; cst = n; }
  const double* Xi = a.X + (long long)inst * a.xstride;
  int ku = 0, kp4u = 0, xw = 0;
  if (upd >= 0) { ku = a.kl[upd]; kp4u = round_up(ku, 4); xw = a.xcol[upd]; }
  int kr = 0, kp8r = 0, QB = 1, ntile = 0, rr = 0, m = 1, r0n = 0, n1 = 0;
  const double* Ll = nullptr;
  if (red >= 0) {
    kr = a.kl[red]; kp8r = round_up(kr, 8); QB = kp8r / 8; ntile = QB * (NCP / 8);
    rr = a.rank[inst * a.L + red];
    const int nd = node_index(red, red_node);
    r0n = a.tree.node_r0[nd]; n1 = a.tree.node_n1[nd]; m = a.tree.lev_m[red];
    Ll = a.Lf + (long long)inst * a.lf_stride + a.tree.lev_lofs[red];
  }
  // debug phase clocks (FDE_TRACE_LEVELS): thread 0 of CTA 0 accumulates cycles per phase
  const bool dbg = a.trace && blockIdx.x == 0 && tid == 0;
  long long pacc[5] = {0, 0, 0, 0, 0}, plast = clock64();
#define PT(i) do { if (dbg) { const long long t_ = clock64(); pacc[i] += t_ - plast; plast = t_; } } while (0)
  double acc[MT][2];
  int aoff[MT], boff[MT];                 // smem offsets of this warp's reduce tiles
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    acc[i][0] = 0.0; acc[i][1] = 0.0;
    const int t = warp + i * LV_WARPS;
    const int qb = (t < ntile ? t : 0) % QB, cb = (t < ntile ? t : 0) / QB;
    aoff[i] = (qb * 8 + gid) * ldx + tig;
    boff[i] = (cb * 8 + gid) * ldx + tig;
  }
  // chunk enumeration over the sub-ranges
  const int n0 = (rb0 - ra0 + CR - 1) / CR;
  const int nch = n0 + (nsub > 1 ? (rb1 - ra1 + CR - 1) / CR : 0);
  auto chunk_rows = [&](int ci, int& r0, int& nr, const double*& S) {
    if (ci < n0) { r0 = ra0 + ci * CR; nr = min(CR, rb0 - r0); S = S0; }
    else { r0 = ra1 + (ci - n0) * CR; nr = min(CR, rb1 - r0); S = S1; }
  };
  // thread -> (row r, first column c0); columns advance by cstep (CR is a power of two)
  const int lg = a.lgCR, rr_t = tid & (CR - 1), c0_t = tid >> lg, cstep = LV_THREADS >> lg;
  auto issue = [&](int ci) {
    int r0, nr; const double* S;
    chunk_rows(ci, r0, nr, S);
    const int b = ci & 1;
    double* Xc = sm.Xc + b * sm.xbuf + rr_t;
    double* Wn = sm.Wn + b * sm.wbuf + rr_t;
    double* Vc = sm.Vc + b * sm.vbuf + rr_t;
    const bool rok = rr_t < nr;
    const int R = r0 + rr_t;
    {
      const double* src = T + (long long)c0_t * cst + R;
      const long long sstep = (long long)cstep * cst;
      for (int c = c0_t; c < NCP; c += cstep, src += sstep) {
        if (rok && c < NC) cp_async8(&Xc[c * ldx], src);
        else Xc[c * ldx] = 0.0;
      }
    }
    if (upd >= 0) {
      const double* src = Xi + (long long)(xw + c0_t) * n + R;
      const long long sstep = (long long)cstep * n;
      for (int kk = c0_t; kk < kp4u; kk += cstep, src += sstep) {
        if (rok && kk < ku) cp_async8(&Wn[kk * ldx], src);
        else Wn[kk * ldx] = 0.0;
      }
    }
    if (red >= 0) {
      // V rows: child 1 -> L_l[i2, q] with e_0 as the exact column; child 0 -> L_l[n1-1-j1, q]
      const int li = red_child == 1 ? R - r0n - n1 : n1 - 1 - (R - r0n);
      const double ex = (li == 0) ? 1.0 : 0.0;    // li == 0 <=> i2 == 0 resp. j1 == n1-1
      const double* src = Ll + li + (long long)c0_t * m;
      const long long sstep = (long long)cstep * m;
      for (int q = c0_t; q < kp8r; q += cstep, src += sstep) {
        if (rok && q < rr) cp_async8(&Vc[q * ldx], src);
        else Vc[q * ldx] = (rok && q == kr - 1) ? ex : 0.0;
      }
    }
    cp_async_commit();
  };

  issue(0);
  for (int ci = 0; ci < nch; ++ci) {
    if (ci + 1 < nch) { issue(ci + 1); cp_async_wait_group1(); }
    else cp_async_wait_all();
    __syncthreads();
    PT(1);
    int r0, nr; const double* S;
    chunk_rows(ci, r0, nr, S);
    const int b = ci & 1;
    double* Xc = sm.Xc + b * sm.xbuf;
    const double* Wn = sm.Wn + b * sm.wbuf;
    const double* Vc = sm.Vc + b * sm.vbuf;
    if (upd >= 0) {
      // X_chunk -= W S.  Warp -> fixed row block mb (A fragment reused), column blocks
      // nb0, nb0 + nbs, ...; 4 independent accumulator tiles in flight.
      const int MB = CR >> 3, NB = NCP >> 3, nbs = LV_WARPS / MB;
      const int mb = warp & (MB - 1), nb0 = warp / MB;
      const double* ap = Wn + tig * ldx + mb * 8 + gid;
      double* cb = Xc + 2 * tig * ldx + mb * 8 + gid;
      const double* bb = S + tig * lds + gid;
      for (int nb = nb0; nb < NB; nb += 4 * nbs) {
        const int cnt = min(4, (NB - nb + nbs - 1) / nbs);
        double d[4][2];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (u < cnt) {
            d[u][0] = cb[(nb + u * nbs) * 8 * ldx];
            d[u][1] = cb[(nb + u * nbs) * 8 * ldx + ldx];
          }
        for (int k0 = 0; k0 < kp4u; k0 += 4) {
          const double av = -ap[k0 * ldx];
          const double* bk = bb + k0 * lds + nb * 8;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (u < cnt) dmma884(d[u][0], d[u][1], av, bk[u * nbs * 8]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (u < cnt) {
            cb[(nb + u * nbs) * 8 * ldx] = d[u][0];
            cb[(nb + u * nbs) * 8 * ldx + ldx] = d[u][1];
          }
      }
      __syncthreads();
    }
    PT(2);
    if (red >= 0) {
      // acc += V^T X_chunk: all of this warp's tiles advance together along the rows
      for (int k0 = 0; k0 < CR; k0 += 4) {
#pragma unroll
        for (int i = 0; i < MT; ++i)
          if (warp + i * LV_WARPS < ntile)
            dmma884(acc[i][0], acc[i][1], Vc[aoff[i] + k0], Xc[boff[i] + k0]);
      }
    }
    PT(3);
    if (upd >= 0 && rr_t < nr) {
      double* dst = T + (long long)c0_t * cst + r0 + rr_t;
      const long long sstep = (long long)cstep * cst;
      for (int c = c0_t; c < NC; c += cstep, dst += sstep) *dst = Xc[c * ldx + rr_t];
    }
    __syncthreads();                              // buffer b is refilled by issue(ci + 2)
    PT(4);
  }
  if (dbg) for (int i = 0; i < 5; ++i) a.trace[1100 + i] += pacc[i];
  if (red >= 0) {
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int t = warp + i * LV_WARPS;
      if (t < ntile) {
        const int qb = t % QB, cb = t / QB;
        const int q = qb * 8 + gid, c = cb * 8 + 2 * tig;
        if (q < kr) {
          if (c < NC) out[(long long)q * out_ld + c] = acc[i][0];
          if (c + 1 < NC) out[(long long)q * out_ld + c + 1] = acc[i][1];
        }
      }
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------------------
// D = (Cin ? Cin : 0) + sgn * A B, row-major shared-memory operands; m, n multiples of 8,
// K a multiple of 4 (operands zero padded).  DMMA tiles, 4 independent tiles per warp.
__device__ void blk_dmma(double* D, int ldd, const double* Cin, int ldc, const double* A, int lda,
                         const double* B, int ldb, int m, int n, int K, double sgn) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gid = lane >> 2, tig = lane & 3;
  const int MB = m / 8, NT = MB * (n / 8);
  for (int t0 = warp; t0 < NT; t0 += 4 * LV_WARPS) {
    double d[4][2];
    int mb[4], nb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = t0 + u * LV_WARPS, tt = t < NT ? t : 0;
      mb[u] = tt % MB; nb[u] = tt / MB;
      if (Cin) {
        d[u][0] = Cin[(mb[u] * 8 + gid) * ldc + nb[u] * 8 + 2 * tig];
        d[u][1] = Cin[(mb[u] * 8 + gid) * ldc + nb[u] * 8 + 2 * tig + 1];
      } else {
        d[u][0] = 0.0; d[u][1] = 0.0;
      }
    }
    for (int k0 = 0; k0 < K; k0 += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (t0 + u * LV_WARPS < NT)
          dmma884(d[u][0], d[u][1], sgn * A[(mb[u] * 8 + gid) * lda + k0 + tig],
                  B[(k0 + tig) * ldb + nb[u] * 8 + gid]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (t0 + u * LV_WARPS < NT) {
        D[(mb[u] * 8 + gid) * ldd + nb[u] * 8 + 2 * tig] = d[u][0];
        D[(mb[u] * 8 + gid) * ldd + nb[u] * 8 + 2 * tig + 1] = d[u][1];
      }
  }
}

// Node solve.  In: sm.Pt = V12^T X2, sm.Pb = V21^T X1 (k x ncols, zero padded to the
// smem extents).  Out: S_top in sm.Pt, S_bot in sm.Pb (round8(k) x round8(ntgt); rows >= k
// are exactly zero, as the K padding of the DMMA update requires).
__device__ void lv_node_solve(const LvArgs& a, const LvSmem& sm, int inst, int lvl, int j,
                              bool store) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = a.kl[lvl], kp4 = round_up(k, 4), kp8 = round_up(k, 8);
  const bool solve = a.mode == 1;
  const int ntgt = lv_ntgt(a, lvl), ntp = round_up(ntgt, 8);
  const int lds = a.lds, ldk = a.ldk, ldm = a.ldm;
  double* Kn = a.Kst + (long long)inst * a.kstride_inst + a.kofs[lvl] + (long long)j * 3 * k * k;
  const bool ndbg = a.trace && blockIdx.x == 0 && tid == 0;
  long long nlast = clock64();
#define NT(i) do { if (ndbg) { const long long t_ = clock64(); a.trace[1110 + (i)] += t_ - nlast; nlast = t_; } } while (0)
  if (!solve) {
    // B = V12^T W2, C = V21^T W1 live in the W columns of the sums; copy them out
    for (int e = tid; e < kp8 * kp8; e += LV_THREADS) {
      const int i = e / kp8, jj = e % kp8;
      const bool in = i < k && jj < k;
      sm.B[i * ldk + jj] = in ? sm.Pt[i * lds + ntgt + jj] : 0.0;
      sm.C[i * ldk + jj] = in ? sm.Pb[i * lds + ntgt + jj] : 0.0;
    }
    __syncthreads();
    blk_dmma(sm.M, ldm, nullptr, 0, sm.C, ldk, sm.B, ldk, kp8, kp8, kp4, -1.0);   // -C B
    __syncthreads();
    for (int e = tid; e < k * 2 * k; e += LV_THREADS) {           // [Sc | I], Sc = I - C B
      const int i = e / (2 * k), jj = e % (2 * k);
      if (jj < k) { if (i == jj) sm.M[i * ldm + jj] += 1.0; }
      else sm.M[i * ldm + jj] = (jj - k == i) ? 1.0 : 0.0;
    }
    __syncthreads();
    NT(0);
    // Gauss-Jordan on [Sc | I] by one warp, no pivoting (reading R17: Sc = I - C B
    // with rho(C B) < 1 for the M-matrix A_m; measured element growth 1.0).  Lane owns
    // columns lane, lane+32, lane+64; a pivot smaller than PIV_MIN x its row latches
    // FDE_ESINGULAR instead of silently amplifying rounding.
    {
      // rows i = warp, warp + LV_WARPS, ...; lanes own columns lane, lane+32, lane+64.
      // Rows are never normalised during the sweep (one barrier per pivot); the inverse is
      // the right half divided by the final diagonal.
      const int k2 = 2 * k;
      const int c0 = lane, c1 = lane + 32, c2 = lane + 64;
      if (warp == 0) {                              // scale for the pivot test: max |Sc|
        double rm = 0.0;
        for (int e = lane; e < k * k; e += 32) rm = fmax(rm, fabs(sm.M[(e / k) * ldm + e % k]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) rm = fmax(rm, __shfl_xor_sync(0xffffffffu, rm, o));
        if (lane == 0) sm.Si[0] = rm;               // Si is rewritten below
      }
      __syncthreads();
      const double rm = sm.Si[0];
      for (int jc = 0; jc < k; ++jc) {
        const double* mp = sm.M + jc * ldm;
        const double piv = mp[jc];
        if (tid == 0 && (!(fabs(piv) > 1e-10 * rm) || !isfinite(piv)))
          latch_status(a.st, FDE_ESINGULAR, inst * 65536 + 32768 + node_index(lvl, j));
        const double rp = 1.0 / piv;
        const bool u0 = c0 > jc && c0 < k2, u1 = c1 > jc && c1 < k2, u2 = c2 > jc && c2 < k2;
        const double p0 = u0 ? mp[c0] : 0.0, p1 = u1 ? mp[c1] : 0.0, p2 = u2 ? mp[c2] : 0.0;
        for (int i = warp; i < k; i += LV_WARPS) {
          if (i == jc) continue;
          double* mi = sm.M + i * ldm;
          const double f = mi[jc] * rp;             // column jc is not written in this step
          const double x0 = u0 ? mi[c0] : 0.0, x1 = u1 ? mi[c1] : 0.0, x2 = u2 ? mi[c2] : 0.0;
          if (u0) mi[c0] = x0 - f * p0;
          if (u1) mi[c1] = x1 - f * p1;
          if (u2) mi[c2] = x2 - f * p2;
        }
        __syncthreads();
      }
    }
    NT(1);
    for (int e = tid; e < kp8 * kp8; e += LV_THREADS) {
      const int i = e / kp8, jj = e % kp8;
      sm.Si[i * ldk + jj] = (i < k && jj < k) ? sm.M[i * ldm + k + jj] / sm.M[i * ldm + i] : 0.0;
    }
    __syncthreads();
    NT(2);
    if (store)
      for (int e = tid; e < k * k; e += LV_THREADS) {
        const int i = e / k, jj = e % k;
        Kn[e] = sm.B[i * ldk + jj];
        Kn[k * k + e] = sm.C[i * ldk + jj];
        Kn[2 * k * k + e] = sm.Si[i * ldk + jj];
      }
  } else {
    for (int e = tid; e < kp8 * kp8; e += LV_THREADS) {
      const int i = e / kp8, jj = e % kp8;
      const bool in = i < k && jj < k;
      sm.B[i * ldk + jj] = in ? Kn[i * k + jj] : 0.0;
      sm.C[i * ldk + jj] = in ? Kn[k * k + i * k + jj] : 0.0;
      sm.Si[i * ldk + jj] = in ? Kn[2 * k * k + i * k + jj] : 0.0;
    }
    __syncthreads();
  }
  NT(3);
  // T = Pb - C Pt ;  S_bot = Sc^{-1} T -> Pb ;  S_top = Pt - B S_bot -> Pt   (targets)
  blk_dmma(sm.T, lds, sm.Pb, lds, sm.C, ldk, sm.Pt, lds, kp8, ntp, kp4, -1.0);
  __syncthreads();
  blk_dmma(sm.Pb, lds, nullptr, 0, sm.Si, ldk, sm.T, lds, kp8, ntp, kp4, 1.0);
  __syncthreads();
  blk_dmma(sm.Pt, lds, sm.Pt, lds, sm.B, ldk, sm.Pb, lds, kp8, ntp, kp4, -1.0);
  __syncthreads();
  NT(4);
}

// load the k x ncols node sums into Pt / Pb, zero filling the rest of the smem extents
__device__ void lv_load_sums(const LvArgs& a, const LvSmem& sm, const double* top,
                             const double* bot, int k, int ncols) {
  const int kp8 = round_up(k, 8), lds = a.lds;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q = warp; q < kp8; q += LV_WARPS)
    for (int c = lane; c < lds; c += 32) {
      const bool in = q < k && c < ncols;
      sm.Pt[q * lds + c] = in ? __ldcg(top + (long long)q * a.sum_nc + c) : 0.0;
      sm.Pb[q * lds + c] = in ? __ldcg(bot + (long long)q * a.sum_nc + c) : 0.0;
    }
  __syncthreads();
}

// ---------------------------------------------------------------------------------------
template <int MT>
__global__ void __launch_bounds__(LV_THREADS, 1)
k_levels(const LvArgs a) {
  extern __shared__ double smem[];
  LvSmem sm;
  sm.Xc = smem + a.off_Xc; sm.Wn = smem + a.off_Wn; sm.Vc = smem + a.off_Vc;
  sm.Pt = smem + a.off_Pt; sm.Pb = smem + a.off_Pb; sm.T = smem + a.off_T;
  sm.B = smem + a.off_B; sm.C = smem + a.off_C; sm.Si = smem + a.off_Si; sm.M = smem + a.off_M;
  sm.xbuf = a.xbuf; sm.wbuf = a.wbuf; sm.vbuf = a.vbuf;
  const TreeDev& tr = a.tree;
  const int P = a.P, p = a.p, L = a.L;
  const int inst = blockIdx.x / P, c = blockIdx.x % P;
  const bool solve = a.mode == 1;
  const long long nnodes = (1LL << L) - 1;
  const long long sh = a.sum_half;
  double* sums_i = a.sums + (long long)inst * nnodes * 2 * sh;
  unsigned nbar = 0;
  int tix = 0;
  const bool tracer = a.trace && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1);
  auto TR = [&](int tag) {
    if (tracer && tix < 255) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      unsigned long long* b = a.trace + (blockIdx.x == 0 ? 0 : 512);
      b[2 * tix] = tag; b[2 * tix + 1] = t; ++tix;
    }
  };
  TR(0);
  int r_lo, r_hi;
  if (p < L) {
    const int nd = node_index(p, c);
    r_lo = tr.node_r0[nd]; r_hi = r_lo + tr.node_n1[nd] + tr.node_n2[nd];
  } else {
    r_lo = tr.leaf_r0[c]; r_hi = r_lo + tr.leaf_n[c];
  }
  auto part_slot = [&](int lvl, int cta) -> double* {
    return a.part + (((long long)(lvl & 1) * (gridDim.x / P) + inst) * P + cta) * sh;
  };

  // ---------------- local phase: post-order over the subtree of node (p, c)
  if (p == L) {
    if (L > 0)
      lv_pass<MT>(a, sm, inst, 1, r_lo, r_hi, nullptr, 0, 0, nullptr, -1, L - 1, c >> 1, c & 1,
              part_slot(L - 1, c), a.sum_nc);
  } else {
    for (int it = 0; it < a.npost; ++it) {
      const int d = a.post[2 * it], jrel = a.post[2 * it + 1];
      const int lvl = p + d, j = (c << d) + jrel;
      const int nd = node_index(lvl, j);
      const int r0 = tr.node_r0[nd], n1 = tr.node_n1[nd], n2 = tr.node_n2[nd];
      double* top = sums_i + (long long)nd * 2 * sh;
      double* bot = top + sh;
      if (lvl == L - 1) {                         // leaves below: reduce-only passes
        lv_pass<MT>(a, sm, inst, 1, r0, r0 + n1, nullptr, 0, 0, nullptr, -1, lvl, j, 0, bot, a.sum_nc);
        lv_pass<MT>(a, sm, inst, 1, r0 + n1, r0 + n1 + n2, nullptr, 0, 0, nullptr, -1, lvl, j, 1, top,
                a.sum_nc);
      }
      TR(100 + lvl);
      lv_load_sums(a, sm, top, bot, a.kl[lvl], lv_ncols(a, lvl));
      lv_node_solve(a, sm, inst, lvl, j, !solve);
      TR(200 + lvl);
      int red = -1, rn = 0, rc = 0;
      double* out = nullptr;
      if (lvl > p) {
        red = lvl - 1; rn = j >> 1; rc = j & 1;
        double* pt = sums_i + (long long)node_index(red, rn) * 2 * sh;
        out = rc ? pt : pt + sh;
      } else if (lvl > 0) {
        red = lvl - 1; rn = c >> 1; rc = c & 1;
        out = part_slot(red, c);
      }
      lv_pass<MT>(a, sm, inst, 2, r0, r0 + n1, sm.Pt, r0 + n1, r0 + n1 + n2, sm.Pb, lvl, red, rn, rc,
              out, a.sum_nc);
      TR(300 + lvl);
    }
  }

  // ---------------- global phase: levels p-1 .. 0
  for (int lvl = p - 1; lvl >= 0; --lvl) {
    const int G = 1 << (p - lvl);
    const int j = c >> (p - lvl), ch = (c >> (p - lvl - 1)) & 1, c0 = j * G;
    const int k = a.kl[lvl], ncols = lv_ncols(a, lvl);
    lv_grid_barrier(a.bar, (++nbar) * gridDim.x);
    TR(400 + lvl);
    if (G / 2 <= 8) {
      const int kp8 = round_up(k, 8);
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G2 = G / 2;
      const double* p0 = part_slot(lvl, c0);
      for (int q = warp; q < kp8; q += LV_WARPS)
        for (int cc = lane; cc < a.lds; cc += 32) {
          double st = 0.0, sb = 0.0;
          if (q < k && cc < ncols) {
            const double* pp = p0 + (long long)q * a.sum_nc + cc;
            double vb[8], vt[8];                      // all loads in flight, fixed-order sums
#pragma unroll
            for (int g = 0; g < 8; ++g)
              if (g < G2) { vb[g] = __ldcg(pp + g * sh); vt[g] = __ldcg(pp + (g + G2) * sh); }
#pragma unroll
            for (int g = 0; g < 8; ++g)
              if (g < G2) { sb += vb[g]; st += vt[g]; }
          }
          sm.Pt[q * a.lds + cc] = st;
          sm.Pb[q * a.lds + cc] = sb;
        }
      __syncthreads();
    } else {
      const int nd = node_index(lvl, j);
      double* top = sums_i + (long long)nd * 2 * sh;
      const int E = k * ncols, chunk = (2 * E + G - 1) / G, g = c - c0;
      for (int e = g * chunk + threadIdx.x; e < min(2 * E, (g + 1) * chunk); e += LV_THREADS) {
        const int half = e / E, inner = e % E;       // half 0: top (child 1), 1: bot (child 0)
        const int q = inner / ncols, cc = inner % ncols;
        const long long o = (long long)q * a.sum_nc + cc;
        double s = 0.0;
        const int g0 = half == 0 ? G / 2 : 0;
        for (int gg = g0; gg < g0 + G / 2; ++gg) s += __ldcg(part_slot(lvl, c0 + gg) + o);
        top[half * sh + o] = s;
      }
      lv_grid_barrier(a.bar, (++nbar) * gridDim.x);
      lv_load_sums(a, sm, top, top + sh, k, ncols);
    }
    TR(500 + lvl);
    lv_node_solve(a, sm, inst, lvl, j, !solve && c == c0);
    TR(600 + lvl);
    int red = -1, rn = 0, rc = 0;
    double* out = nullptr;
    if (lvl > 0) {
      red = lvl - 1; rn = c >> (p - lvl + 1); rc = (c >> (p - lvl)) & 1;
      out = part_slot(red, c);
    }
    lv_pass<MT>(a, sm, inst, 1, r_lo, r_hi, ch ? sm.Pb : sm.Pt, 0, 0, nullptr, lvl, red, rn, rc, out,
            a.sum_nc);
    TR(700 + lvl);
  }
  TR(999);
}
