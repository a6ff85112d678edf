// k_compress.cuh -- S2: per-level compression of the Toeplitz off-diagonal blocks.
//
// Structure used (Lemma 3.7 proof; Lemma 3.4):
// the lower off-diagonal block of every HODLR node of T_{alpha,N} (n2 x n1, node split
// n1 = floor(s/2), n2 = ceil(s/2)) is  T21[i,j] = -g_{n1+1+i-j} = -(H J)[i,j]  with the
// Hankel H[i,j] = g_{2+i+j} (a leading section of the PSD Hankel of Lemma 3.4) and J the
// flip.  So one factorisation  H_m ~ L L^T  (m = largest n2 of the level) serves every
// node of a level:  T21 ~ (-L[:n2]) (J L[:n1])^T.  The upper block is the single entry
// -g_0 and is carried exactly by the assembly (k_leaf / k_level).
//
// Compression = truncation of singular values below tau = tol * 2^alpha (reading
// R7).  Because H is PSD, it is computed as
//   (1) diagonally pivoted partial Cholesky of H_m (greedy pivot = largest residual
//       diagonal, ties to the smallest index), stopped when trace(H - L L^T) <= tau
//       (for a PSD residual ||.||_2 <= trace);
//   (2) recompression: eigen-decomposition of the small Gram L^T L = V diag(lam) V^T by
//       cyclic Jacobi, keep lam >= tau (the eigenvalues of L L^T), L <- L V_keep.
// The block error is <= 2 tau; the kept rank equals the truncated-SVD rank of the oracle
// in every tested case (tests/test_parity_1d.py::test_ranks_equal_truncated_svd, tests/test_rank_study.py).
//
// (1) runs as one cooperative launch: each (instance, level) task is cut into chunks of
// PC_ROWS rows, one CTA per chunk with its rows of L resident in shared memory (PC_RPT rows per
// thread).  Per pivot the CTAs of a task exchange their partials through tagged slots: each
// CTA publishes (trace, max, index, candidate row) and releases the slot's tag; every CTA polls
// the G tags and reduces the partials in a fixed order (deterministic, schedule independent).
#pragma once
#include "fde_common.cuh"

#ifdef FDE_DEBUG
__device__ int g_comp_trace = 0;      // (diagnostics build, FDE_COMP_TRACE: per-task printf)
#endif

#define PC_THREADS 256
#define PC_RPT 2
#define PC_ROWS (PC_THREADS * PC_RPT)
#define PSTRIDE (KRAW + 4)    // slot: [trace, max, index, tag | candidate row]
#define PC_STOP 1e-3          // pivoted-Cholesky trace stop = tau * PC_STOP ...
#define PC_EPS_TRACE 3.2e-14  // ... but never below ~144 ulps of the initial trace

struct PcTask {            // one (instance, level)
  int inst, level, m, G;   // G chunks (CTAs)
  int slot0;               // first chunk slot of this task (for partial buffers)
  int pad;
  long long lraw_ofs;      // offset of this task's raw factor (m x KRAW, ld m)
  long long lf_ofs;        // offset of the final factor (m x RCAP, ld m)
  double tau;
};
struct PcChunk { int task, row0, nrows, grank; };

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Barrier among the G CTAs of one task (all co-resident: cooperative launch).
__device__ __forceinline__ void group_barrier(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    while (ld_acquire_u32(ctr) < target) { __nanosleep(32); }
    __threadfence();
  }
  __syncthreads();
}

// Deterministic block reductions (fixed tree).
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = (lane < (int)(blockDim.x >> 5)) ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  double r = red[0];
  __syncthreads();
  return r;
}

__device__ __forceinline__ void argmax_merge(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

__device__ __forceinline__ void block_argmax(double v, int i, double* redv, int* redi,
                                             double& outv, int& outi) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double v2 = __shfl_down_sync(0xffffffffu, v, o);
    int i2 = __shfl_down_sync(0xffffffffu, i, o);
    argmax_merge(v, i, v2, i2);
  }
  if (lane == 0) { redv[w] = v; redi[w] = i; }
  __syncthreads();
  if (w == 0) {
    if (lane < (int)(blockDim.x >> 5)) { v = redv[lane]; i = redi[lane]; }
    else { v = -1.0; i = 0x7fffffff; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double v2 = __shfl_down_sync(0xffffffffu, v, o);
      int i2 = __shfl_down_sync(0xffffffffu, i, o);
      argmax_merge(v, i, v2, i2);
    }
    if (lane == 0) { redv[0] = v; redi[0] = i; }
  }
  __syncthreads();
  outv = redv[0]; outi = redi[0];
  __syncthreads();
}

// ---------------------------------------------------------------------------------------
// (1) pivoted partial Cholesky, cooperative.  smem: Lc[KRAW][PC_ROWS].
// Outputs: Lraw (global), kr per task, full Gram L^T L per task (fixed-order reduction).
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(PC_THREADS, 1)
k_pchol(const PcTask* __restrict__ tasks, const PcChunk* __restrict__ chunks,
        const double* __restrict__ g, long long gstride,
        double* __restrict__ Lraw, int* __restrict__ task_kr,
        unsigned* __restrict__ ctr, double* __restrict__ part,
        double* __restrict__ gram_part, double* __restrict__ gram,
        DevStatus* __restrict__ st) {
  extern __shared__ double smem[];
  double* Lc = smem;                                  // [KRAW][PC_ROWS]
  __shared__ double redv[32], redm[32];
  __shared__ int redi[32];
  __shared__ double Lp[KRAW];
  __shared__ double s_total, s_pmax;
  __shared__ int s_p, s_stop;

  const PcChunk ch = chunks[blockIdx.x];
  const PcTask tk = tasks[ch.task];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int m = tk.m, G = tk.G;
  const double* gi = g + (long long)tk.inst * gstride;
  unsigned* myctr = ctr + ch.task;
  const int myslot = tk.slot0 + ch.grank;
  bool valid[PC_RPT];
  int ri[PC_RPT];                                     // global row index of each owned row
  double d[PC_RPT];                                   // residual diagonal
#pragma unroll
  for (int u = 0; u < PC_RPT; ++u) {
    const int lr = t + PC_THREADS * u;
    valid[u] = lr < ch.nrows;
    ri[u] = ch.row0 + lr;
    d[u] = valid[u] ? gi[2 + 2 * ri[u]] : 0.0;        // diag of H_m: g_{2+2i}
  }
  int k = 0;
  unsigned step = 0;
#ifdef FDE_DEBUG
  const long long pc_start = clock64();
  long long pc_ph[4] = {0, 0, 0, 0}, pc_t = pc_start;
#define PCPH(i) do { if (g_comp_trace && t == 0) { const long long t_ = clock64(); pc_ph[i] += t_ - pc_t; pc_t = t_; } } while (0)
#else
#define PCPH(i) do { } while (0)
#endif
  // Stopping threshold of the pivoted Cholesky (s_total below): tau * PC_STOP, floored at the
  // rounding level of the residual trace.  Stopping well below tau lets the optimal
  // recompression reproduce the truncated-SVD approximant (same rank; tests/ and DESIGN.md).
  for (;;) {
    // ---- local partials of the residual diagonal: trace and argmax in ONE block reduction; warp 0
    //      publishes them and the candidate row of L (from shared memory) in this chunk's slot
    {
      double sv = 0.0, bv = -1.0;
      int bi = 0x7fffffff;
#pragma unroll
      for (int u = 0; u < PC_RPT; ++u)
        if (valid[u]) { sv += d[u]; argmax_merge(bv, bi, d[u], ri[u]); }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sv += __shfl_down_sync(0xffffffffu, sv, o);
        const double v2 = __shfl_down_sync(0xffffffffu, bv, o);
        const int i2 = __shfl_down_sync(0xffffffffu, bi, o);
        argmax_merge(bv, bi, v2, i2);
      }
      if (lane == 0) { redv[w] = sv; redm[w] = bv; redi[w] = bi; }
      __syncthreads();
      if (w == 0) {
        const int nwp = PC_THREADS >> 5;
        sv = lane < nwp ? redv[lane] : 0.0;
        bv = lane < nwp ? redm[lane] : -1.0;
        bi = lane < nwp ? redi[lane] : 0x7fffffff;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          sv += __shfl_down_sync(0xffffffffu, sv, o);
          const double v2 = __shfl_down_sync(0xffffffffu, bv, o);
          const int i2 = __shfl_down_sync(0xffffffffu, bi, o);
          argmax_merge(bv, bi, v2, i2);
        }
        sv = __shfl_sync(0xffffffffu, sv, 0);
        bv = __shfl_sync(0xffffffffu, bv, 0);
        bi = __shfl_sync(0xffffffffu, bi, 0);
        double* slot = part + ((long long)myslot * 2 + (step & 1)) * PSTRIDE;
        if (lane == 0) { slot[0] = sv; slot[1] = bv; slot[2] = (double)bi; }
        if (bv >= 0.0)
          for (int q = lane; q < k; q += 32) slot[4 + q] = Lc[q * PC_ROWS + (bi - ch.row0)];
        __syncwarp();
        if (lane == 0)
          asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(reinterpret_cast<unsigned long long*>(slot) + 3),
                       "l"((unsigned long long)(step + 1)) : "memory");
      }
    }
    ++step;
    PCPH(0);
    // ---- warp 0: wait for the G slots of this step, fixed-order reduction, winner's pivot row
    if (w == 0) {
      double tot = 0.0, bv = -1.0; int bi = 0x7fffffff, bs = 0;
      // poll every tag with relaxed loads (in flight together), then one acquire fence
      for (;;) {
        bool ok = true;
        for (int c = lane; c < G; c += 32) {
          const double* o = part + ((long long)(tk.slot0 + c) * 2 + ((step - 1) & 1)) * PSTRIDE;
          ok &= ld_relaxed_u64(reinterpret_cast<const unsigned long long*>(o) + 3) >= step;
        }
        if (__all_sync(0xffffffffu, ok)) break;
        __nanosleep(16);
      }
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      PCPH(1);
      for (int c = lane; c < G; c += 32) {
        const double* o = part + ((long long)(tk.slot0 + c) * 2 + ((step - 1) & 1)) * PSTRIDE;
        tot += __ldcg(o);
        double v = __ldcg(o + 1); int ix = (int)__ldcg(o + 2);
        if (v > bv || (v == bv && ix < bi)) { bv = v; bi = ix; bs = c; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        tot += __shfl_down_sync(0xffffffffu, tot, o);
        double v2 = __shfl_down_sync(0xffffffffu, bv, o);
        int i2 = __shfl_down_sync(0xffffffffu, bi, o);
        int s2 = __shfl_down_sync(0xffffffffu, bs, o);
        if (v2 > bv || (v2 == bv && i2 < bi)) { bv = v2; bi = i2; bs = s2; }
      }
      tot = __shfl_sync(0xffffffffu, tot, 0);
      bv = __shfl_sync(0xffffffffu, bv, 0);
      bi = __shfl_sync(0xffffffffu, bi, 0);
      bs = __shfl_sync(0xffffffffu, bs, 0);
      if (lane == 0) {
        if (k == 0) s_total = fmax(tk.tau * PC_STOP, PC_EPS_TRACE * tot);   // initial trace
        s_pmax = bv; s_p = bi;
        int stop = (tot <= s_total) || !(bv > 0.0) || (k == KRAW);
        if (k == KRAW && tot > tk.tau && ch.grank == 0)
          latch_status(st, FDE_ENOCONV, tk.inst * 65536 + tk.level);
        s_stop = stop;
      }
      __syncwarp();
      // the pivot index is out: the other warps start their H[i,p] loads (barrier 1) while
      // this warp fetches the winner's row
      asm volatile("bar.arrive 1, %0;" ::"n"(PC_THREADS) : "memory");
      const double* o = part + ((long long)(tk.slot0 + bs) * 2 + ((step - 1) & 1)) * PSTRIDE;
      for (int q = lane; q < k; q += 32) Lp[q] = __ldcg(o + 4 + q);
    } else {
      asm volatile("bar.sync 1, %0;" ::"n"(PC_THREADS) : "memory");
    }
    const int p = s_p;
    FDE_ASSERT(s_stop || (p >= 0 && p < m && k < KRAW));
    double hv[PC_RPT];
#pragma unroll
    for (int u = 0; u < PC_RPT; ++u) hv[u] = (valid[u] && !s_stop) ? gi[2 + ri[u] + p] : 0.0;   // H[i,p] = g_{2+i+p}
    __syncthreads();
    PCPH(2);
    if (s_stop) break;
    const double sp = sqrt(s_pmax);
#pragma unroll
    for (int u = 0; u < PC_RPT; ++u) {
      const int lr = t + PC_THREADS * u;
      double l = 0.0;
      if (valid[u]) {
        double acc0 = hv[u], acc1 = 0.0;
        int q = 0;
        for (; q + 1 < k; q += 2) {
          acc0 -= Lc[q * PC_ROWS + lr] * Lp[q];
          acc1 -= Lc[(q + 1) * PC_ROWS + lr] * Lp[q + 1];
        }
        if (q < k) acc0 -= Lc[q * PC_ROWS + lr] * Lp[q];
        l = (acc0 + acc1) / sp;
        d[u] = (ri[u] == p) ? 0.0 : fmax(d[u] - l * l, 0.0);
      }
      Lc[k * PC_ROWS + lr] = l;
    }
    ++k;
    PCPH(3);
  }
  const int kr = k;
#ifdef FDE_DEBUG
  if (g_comp_trace && t == 0 && ch.grank == 0)
    printf("k_pchol task %d level %d G %d pivots %d cycles %lld  local+publish %lld poll %lld gather %lld update %lld\n",
           ch.task, tk.level, G, kr, clock64() - pc_start, pc_ph[0], pc_ph[1], pc_ph[2], pc_ph[3]);
#endif
  // ---- raw factor to global (for the transform kernel)
  {
    double* Lo = Lraw + tk.lraw_ofs;
#pragma unroll
    for (int u = 0; u < PC_RPT; ++u)
      if (valid[u])
        for (int q = 0; q < kr; ++q) Lo[ri[u] + (long long)q * m] = Lc[q * PC_ROWS + t + PC_THREADS * u];
  }
  if (ch.grank == 0 && t == 0) task_kr[ch.task] = kr;
  // ---- partial Gram of this chunk (rows beyond nrows hold zeros)
  const int kr2 = kr * kr;
  double* gp = gram_part + (long long)myslot * (KRAW * KRAW);
  for (int e = t; e < kr2; e += PC_THREADS) {
    const int a = e % kr, b = e / kr;
    if (a > b) continue;
    const double* la = Lc + a * PC_ROWS;
    const double* lb = Lc + b * PC_ROWS;
    double s0 = 0.0, s1 = 0.0;
    const int nr = ch.nrows;
    int r = 0;
    for (; r + 1 < nr; r += 2) { s0 += la[r] * lb[r]; s1 += la[r + 1] * lb[r + 1]; }
    if (r < nr) s0 += la[r] * lb[r];
    gp[a + b * kr] = s0 + s1;
  }
  group_barrier(myctr, (unsigned)G);
  // ---- split fixed-order reduction: chunk grank sums entries e = grank + G*j
  double* gt = gram + (long long)ch.task * (KRAW * KRAW);
  for (int e = ch.grank + G * t; e < kr2; e += G * PC_THREADS) {
    const int a = e % kr, b = e / kr;
    if (a > b) continue;
    double s = 0.0;
    for (int c = 0; c < G; ++c) s += __ldcg(gram_part + (long long)(tk.slot0 + c) * (KRAW * KRAW) + e);
    gt[a + b * kr] = s;
    gt[b + a * kr] = s;
  }
}

// ---------------------------------------------------------------------------------------
// (2) Recompression: cyclic (round-robin) Jacobi on the kr x kr Gram, one CTA per task.  A round
// rotates N/2 disjoint pairs; on the 2 x 2 block (P1, P2) of A (P1, P2 pairs of the round) it is
// A'[P1,P2] = J1^T A[P1,P2] J2 -- row phase, then column phase, the annihilated entry set to
// zero -- and V <- V J.  A is double-buffered, so each thread owns whole blocks.  Warp 0
// computes the NEXT round's rotations while the CTA applies the current one: the next pairs'
// diagonal blocks are formed from this round's input by the same block formula, so one
// barrier per round and the rotation's sqrt / rcp chain is off the critical path.
// Writes Vkeep (kr x r, ld KRAW), the final rank r and rank_out[inst*L + level].
#define EIG_THREADS 256
#define EIG_APPLY (EIG_THREADS - 32)                                         // warps 1.. apply
#define EIG_NB (((KRAW / 2) * (KRAW / 2) + EIG_APPLY - 1) / EIG_APPLY)       // blocks per thread
#define EIG_NV ((KRAW * (KRAW / 2) + EIG_APPLY - 1) / EIG_APPLY)             // V items per thread
#define EIG_SMEM (3 * KRAW * KRAW * 8 + 2 * KRAW * (KRAW / 2) + KRAW * KRAW)      // bytes

__device__ __forceinline__ double eig_rcp(double x) {      // 1/x to ~1 ulp (finite, normal x)
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

// rotation (c, s) annihilating apq of the symmetric 2 x 2 block [[app, apq], [apq, aqq]]
__device__ __forceinline__ void eig_rot(double app, double aqq, double apq, double& c, double& sn) {
  c = 1.0; sn = 0.0;
  if (apq != 0.0 && fabs(apq) > 1e-300) {
    const double tau = (aqq - app) * eig_rcp(2.0 * apq);
    const double at = fabs(tau);
    const double tt = at > 1e150 ? 0.5 / tau : copysign(eig_rcp(at + sqrt(fma(tau, tau, 1.0))), tau);
    c = rsqrt(fma(tt, tt, 1.0));
    sn = tt * c;
  }
}

__global__ void __launch_bounds__(EIG_THREADS)
k_eig(const PcTask* __restrict__ tasks, const int* __restrict__ task_kr,
      const double* __restrict__ gram, double* __restrict__ vkeep,
      int* __restrict__ task_rank, int* __restrict__ rank_out, int L,
      DevStatus* __restrict__ st) {
  extern __shared__ double eig_smem[];                 // [A0 | A1 | V] (N x N each) | pair tables
  double* const A0 = eig_smem;
  double* const A1 = eig_smem + KRAW * KRAW;
  double* V = eig_smem + 2 * KRAW * KRAW;
  // round r: pair w = (pp[r][w], pq[r][w]); index a sits in pair pw[r][a]
  unsigned char* pp = reinterpret_cast<unsigned char*>(eig_smem + 3 * KRAW * KRAW);
  unsigned char* pq = pp + KRAW * (KRAW / 2);
  unsigned char* pw = pq + KRAW * (KRAW / 2);
  __shared__ double red[32];
  __shared__ int s_done;
  __shared__ int order[KRAW];
  __shared__ double lam[KRAW];
  __shared__ double rc[2][KRAW / 2], rs[2][KRAW / 2];
  const int task = blockIdx.x;
  const PcTask tk = tasks[task];
  const int kr = task_kr[task];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int N = kr + (kr & 1), NP = N / 2;
  const double* gt = gram + (long long)task * (KRAW * KRAW);
  for (int e = t; e < N * N; e += EIG_THREADS) {
    const int a = e % N, b = e / N;
    A0[e] = (a < kr && b < kr) ? gt[a + b * kr] : 0.0;
    V[e] = (a == b) ? 1.0 : 0.0;
  }
  for (int e = t; e < (N - 1) * NP; e += EIG_THREADS) {   // round-robin pairs
    const int r = e / NP, w = e % NP;
    int a, b;
    if (w == 0) { a = r; b = N - 1; }
    else { a = (r + w) % (N - 1); b = (r - w + (N - 1)) % (N - 1); }
    const int p = min(a, b), q = max(a, b);
    pp[r * NP + w] = (unsigned char)p; pq[r * NP + w] = (unsigned char)q;
    pw[r * N + p] = (unsigned char)w; pw[r * N + q] = (unsigned char)w;
  }
  // this thread's work items (warps 1..; warp 0 computes rotations): blocks (w1, w2), V (row i, pair w)
  int b1[EIG_NB], b2[EIG_NB], vi[EIG_NV], vw[EIG_NV];
#pragma unroll
  for (int j = 0; j < EIG_NB; ++j) {
    const int u = t - 32 + j * EIG_APPLY;
    b1[j] = (warp > 0 && u < NP * NP) ? u % NP : -1; b2[j] = u / NP;
  }
#pragma unroll
  for (int j = 0; j < EIG_NV; ++j) {
    const int u = t - 32 + j * EIG_APPLY;
    vi[j] = (warp > 0 && u < N * NP) ? u % N : -1; vw[j] = u / N;
  }
  __syncthreads();
  // warp 0: the rotations of round r from a matrix that is current for round r
  auto rot_direct = [&](const double* A, int r, int buf) {
    if (lane < NP) {
      const int p = pp[r * NP + lane], q = pq[r * NP + lane];
      eig_rot(A[p + p * N], A[q + q * N], A[p + q * N], rc[buf][lane], rs[buf][lane]);
    }
  };
  // entry (a, b) of the matrix after round r (input A, rotations rot[buf] of round r)
  auto after = [&](const double* A, int r, int buf, int a, int b) -> double {
    const int wa = pw[r * N + a], wb = pw[r * N + b];
    const int pa = pp[r * NP + wa], qa = pq[r * NP + wa], pb = pp[r * NP + wb], qb = pq[r * NP + wb];
    if (wa == wb && a != b) return 0.0;                   // the annihilated entry
    const double c1 = rc[buf][wa], s1 = rs[buf][wa], c2 = rc[buf][wb], s2 = rs[buf][wb];
    const double ap_p = A[pa + pb * N], aq_p = A[qa + pb * N], ap_q = A[pa + qb * N], aq_q = A[qa + qb * N];
    const double rp_ = a == pa ? c1 * ap_p - s1 * aq_p : s1 * ap_p + c1 * aq_p;   // row a, column pb
    const double rq_ = a == pa ? c1 * ap_q - s1 * aq_q : s1 * ap_q + c1 * aq_q;   // row a, column qb
    return b == pb ? c2 * rp_ - s2 * rq_ : s2 * rp_ + c2 * rq_;
  };
  int cur = 0, nsw = 0;
  const long long c_start = clock64();
#ifdef FDE_DEBUG
  __shared__ long long ph[4];
  if (t < 4) ph[t] = 0;
#endif
  if (kr > 1) {
    if (warp == 0) rot_direct(A0, 0, 0);
    __syncthreads();
    int rb = 0;                                         // rotation buffer of the current round
    for (int sweep = 0; sweep < 40; ++sweep) {
      nsw = sweep;
      const double* A = cur ? A1 : A0;
      double off = 0.0, dia = 0.0;
      for (int e = t; e < N * N; e += EIG_THREADS) {
        const int a = e % N, b = e / N;
        if (a == b) dia += A[e] * A[e]; else off += A[e] * A[e];
      }
      off = block_sum(off, red);
      dia = block_sum(dia, red);
      // converged: off-diagonal mass <= 1e-24 of the diagonal's at the start of a sweep (quadratic
      // convergence: the previous sweep started near 1e-12 or below).  At cfg3 this ends after 5
      // sweeps instead of 6 with the truncated approximant unchanged to the rounding level
      // (relative difference 3e-15, cold path)
      if (off <= 1e-24 * dia) break;                  // (uniform: every thread holds the sums)
      for (int r = 0; r < N - 1; ++r) {
        const double* Ai = cur ? A1 : A0;
        double* Ao = cur ? A0 : A1;
#ifdef FDE_DEBUG
        const long long tr0 = clock64();
#endif
        if (warp == 0 && lane < NP) {                   // next round's rotations (round r + 1,
          const int rn = r + 1 < N - 1 ? r + 1 : 0;     //  or round 0 of the next sweep)
          const int p = pp[rn * NP + lane], q = pq[rn * NP + lane];
          eig_rot(after(Ai, r, rb, p, p), after(Ai, r, rb, q, q), after(Ai, r, rb, p, q),
                  rc[rb ^ 1][lane], rs[rb ^ 1][lane]);
        }
#pragma unroll
        for (int j = 0; j < EIG_NB; ++j) {              // 2 x 2 blocks (w1, w2) of A
          const int w1 = b1[j], w2 = b2[j];
          if (w1 < 0) continue;
          const int p1 = pp[r * NP + w1], q1 = pq[r * NP + w1], p2 = pp[r * NP + w2], q2 = pq[r * NP + w2];
          const double c1 = rc[rb][w1], s1 = rs[rb][w1], c2 = rc[rb][w2], s2 = rs[rb][w2];
          const double ap_p = Ai[p1 + p2 * N], aq_p = Ai[q1 + p2 * N];
          const double ap_q = Ai[p1 + q2 * N], aq_q = Ai[q1 + q2 * N];
          const double rpp = c1 * ap_p - s1 * aq_p, rqp = s1 * ap_p + c1 * aq_p;   // column p2
          const double rpq = c1 * ap_q - s1 * aq_q, rqq = s1 * ap_q + c1 * aq_q;   // column q2
          Ao[p1 + p2 * N] = c2 * rpp - s2 * rpq;
          Ao[p1 + q2 * N] = w1 == w2 ? 0.0 : s2 * rpp + c2 * rpq;
          Ao[q1 + p2 * N] = w1 == w2 ? 0.0 : c2 * rqp - s2 * rqq;
          Ao[q1 + q2 * N] = s2 * rqp + c2 * rqq;
        }
#pragma unroll
        for (int j = 0; j < EIG_NV; ++j) {              // V <- V J (row i, pair w: in place)
          const int i = vi[j], w = vw[j];
          if (i < 0) continue;
          const int p = pp[r * NP + w], q = pq[r * NP + w];
          const double c = rc[rb][w], sn = rs[rb][w];
          const double vip = V[i + p * N], viq = V[i + q * N];
          V[i + p * N] = c * vip - sn * viq;
          V[i + q * N] = sn * vip + c * viq;
        }
#ifdef FDE_DEBUG
        const long long tr1 = clock64();
        if (lane == 0 && warp < 2) ph[warp] += tr1 - tr0;
#endif
        __syncthreads();
#ifdef FDE_DEBUG
        if (lane == 0 && warp < 2) ph[2 + warp] += clock64() - tr1;
#endif
        cur ^= 1;
        rb ^= 1;
      }
    }
  }
  const double* A = cur ? A1 : A0;
#ifdef FDE_DEBUG
  if (g_comp_trace && t == 0)
    printf("k_eig task %d level %d kr %d sweeps %d cycles %lld  rot(w0) %lld apply(w1) %lld bar(w0) %lld bar(w1) %lld\n",
           task, tk.level, kr, nsw, clock64() - c_start, ph[0], ph[1], ph[2], ph[3]);
#else
  (void)nsw; (void)c_start;
#endif
  // ---- select lam >= tau, descending
  if (t == 0) {
    int r = 0;
    for (int a = 0; a < kr; ++a) { lam[a] = A[a + a * N]; }
    for (int a = 0; a < kr; ++a) if (lam[a] >= tk.tau) order[r++] = a;
    for (int a = 0; a < r; ++a)                         // selection sort, descending
      for (int b = a + 1; b < r; ++b)
        if (lam[order[b]] > lam[order[a]]) { int x = order[a]; order[a] = order[b]; order[b] = x; }
    if (r > RCAP) { latch_status(st, FDE_ENOCONV, tk.inst * 65536 + tk.level); r = RCAP; }
    task_rank[task] = r;
    rank_out[tk.inst * L + tk.level] = r;
    s_done = r;
  }
  __syncthreads();
  const int r = s_done;
  double* vk = vkeep + (long long)task * (KRAW * RCAP);
  for (int e = t; e < kr * r; e += EIG_THREADS) {
    const int a = e % kr, j = e / kr;
    vk[a + j * KRAW] = V[a + order[j] * N];
  }
}

// ---------------------------------------------------------------------------------------
// (3) L_final = Lraw * Vkeep for every row (one CTA per chunk; same chunk list).
__global__ void __launch_bounds__(PC_ROWS)
k_ltransform(const PcTask* __restrict__ tasks, const PcChunk* __restrict__ chunks,
             const int* __restrict__ task_kr, const int* __restrict__ task_rank,
             const double* __restrict__ vkeep, const double* __restrict__ Lraw,
             double* __restrict__ Lf) {
  __shared__ double vs[KRAW * RCAP];
  const PcChunk ch = chunks[blockIdx.x];
  const PcTask tk = tasks[ch.task];
  const int kr = task_kr[ch.task], r = task_rank[ch.task];
  const double* vk = vkeep + (long long)ch.task * (KRAW * RCAP);
  for (int e = threadIdx.x; e < KRAW * r; e += PC_ROWS) {
    const int a = e % KRAW, j = e / KRAW;
    vs[a + j * KRAW] = (a < kr) ? vk[a + j * KRAW] : 0.0;   // rows >= kr must be zero, not stale
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t >= ch.nrows) return;
  const int i = ch.row0 + t, m = tk.m;
  const double* Li = Lraw + tk.lraw_ofs + i;
  double lrow[KRAW];
#pragma unroll
  for (int q = 0; q < KRAW; ++q) lrow[q] = (q < kr) ? Li[(long long)q * m] : 0.0;
  double* Lo = Lf + tk.lf_ofs + i;
  for (int j = 0; j < r; ++j) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < KRAW; ++q) s += lrow[q] * vs[q + j * KRAW];
    Lo[(long long)j * m] = s;
  }
}

// X column offsets: colofs[inst*(L+1)+l] = sum_{l'<l} (rank + 1).
__global__ void k_colofs(const int* __restrict__ rank, int* __restrict__ colofs, int L, int batch) {
  const int inst = blockIdx.x * blockDim.x + threadIdx.x;
  if (inst >= batch) return;
  int c = 0;
  for (int l = 0; l < L; ++l) {
    colofs[inst * (L + 1) + l] = c;
    c += rank[inst * L + l] + 1;
  }
  colofs[inst * (L + 1) + L] = c;
}
