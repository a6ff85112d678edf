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
// PC_ROWS rows, one CTA per chunk with its rows of L resident in shared memory; the CTAs
// of a task synchronise through a counter barrier once per pivot and reduce the trace /
// argmax partials in a fixed order (deterministic, schedule independent).
#pragma once
#include "fde_common.cuh"

#define PC_ROWS 256
#define PSTRIDE (KRAW + 4)
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
__global__ void __launch_bounds__(PC_ROWS)
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
  const int t = threadIdx.x;
  const int m = tk.m, G = tk.G;
  const bool valid = t < ch.nrows;
  const int i = ch.row0 + t;
  const double* gi = g + (long long)tk.inst * gstride;
  unsigned* myctr = ctr + ch.task;
  const int myslot = tk.slot0 + ch.grank;

  double d = valid ? gi[2 + 2 * i] : 0.0;            // diag of H_m: g_{2+2i}
  int k = 0;
  unsigned step = 0;
  // Stopping threshold of the pivoted Cholesky (s_total below): tau * PC_STOP, floored at the
  // rounding level of the residual trace.  Stopping well below tau lets the optimal
  // recompression reproduce the truncated-SVD approximant (same rank; tests/ and DESIGN.md).
  for (;;) {
    // ---- local partials of the residual diagonal: trace and argmax in ONE block reduction; warp 0
    //      writes them and the candidate row of L (from shared memory) into this chunk's slot
    {
      double sv = valid ? d : 0.0, bv = valid ? d : -1.0;
      int bi = valid ? i : 0x7fffffff;
      const int lane = t & 31, w = t >> 5;
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
        const int nwp = PC_ROWS >> 5;
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
      }
    }
    ++step;
    group_barrier(myctr, step * (unsigned)G);
    // ---- fixed-order reduction over the G chunks of this task; warp 0 then fetches the
    //      winning chunk's pivot row of L
    if (t < 32) {
      double tot = 0.0, bv = -1.0; int bi = 0x7fffffff, bs = 0;
      for (int c = t; c < G; c += 32) {
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
      if (t == 0) {
        if (k == 0) s_total = fmax(tk.tau * PC_STOP, PC_EPS_TRACE * tot);   // initial trace
        s_pmax = bv; s_p = bi;
        int stop = (tot <= s_total) || !(bv > 0.0) || (k == KRAW);
        if (k == KRAW && tot > tk.tau && ch.grank == 0)
          latch_status(st, FDE_ENOCONV, tk.inst * 65536 + tk.level);
        s_stop = stop;
      }
      const double* o = part + ((long long)(tk.slot0 + bs) * 2 + ((step - 1) & 1)) * PSTRIDE;
      for (int q = t; q < k; q += 32) Lp[q] = __ldcg(o + 4 + q);
    }
    __syncthreads();
    if (s_stop) break;
    const int p = s_p;
    const double sp = sqrt(s_pmax);
    double l = 0.0;
    if (valid) {
      double acc0 = gi[2 + i + p], acc1 = 0.0;       // H[i,p] = g_{2+i+p}
      int q = 0;
      for (; q + 1 < k; q += 2) {
        acc0 -= Lc[q * PC_ROWS + t] * Lp[q];
        acc1 -= Lc[(q + 1) * PC_ROWS + t] * Lp[q + 1];
      }
      if (q < k) acc0 -= Lc[q * PC_ROWS + t] * Lp[q];
      l = (acc0 + acc1) / sp;
      d = (i == p) ? 0.0 : fmax(d - l * l, 0.0);
    }
    Lc[k * PC_ROWS + t] = l;
    ++k;
  }
  const int kr = k;
  // ---- raw factor to global (for the transform kernel)
  if (valid) {
    double* Lo = Lraw + tk.lraw_ofs;
    for (int q = 0; q < kr; ++q) Lo[i + (long long)q * m] = Lc[q * PC_ROWS + t];
  }
  if (ch.grank == 0 && t == 0) task_kr[ch.task] = kr;
  // ---- partial Gram of this chunk (rows beyond nrows hold zeros)
  const int kr2 = kr * kr;
  double* gp = gram_part + (long long)myslot * (KRAW * KRAW);
  for (int e = t; e < kr2; e += PC_ROWS) {
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
  ++step;
  group_barrier(myctr, step * (unsigned)G);
  // ---- split fixed-order reduction: chunk grank sums entries e = grank + G*j
  double* gt = gram + (long long)ch.task * (KRAW * KRAW);
  for (int e = ch.grank + G * t; e < kr2; e += G * PC_ROWS) {
    const int a = e % kr, b = e / kr;
    if (a > b) continue;
    double s = 0.0;
    for (int c = 0; c < G; ++c) s += __ldcg(gram_part + (long long)(tk.slot0 + c) * (KRAW * KRAW) + e);
    gt[a + b * kr] = s;
    gt[b + a * kr] = s;
  }
}

// ---------------------------------------------------------------------------------------
// (2) Recompression: cyclic (round-robin) Jacobi on the kr x kr Gram, one CTA per task; one warp
// per rotation pair of a round (kr/2 disjoint pairs), applied as a row phase (A <- J^T A) and a
// column phase (A <- A J, V <- V J) separated by barriers -- two barriers per round.
// Writes Vkeep (kr x r, ld KRAW), the final rank r and rank_out[inst*L + level].
#define EIG_THREADS 768                                  // >= KRAW/2 warps
__global__ void __launch_bounds__(EIG_THREADS)
k_eig(const PcTask* __restrict__ tasks, const int* __restrict__ task_kr,
      const double* __restrict__ gram, double* __restrict__ vkeep,
      int* __restrict__ task_rank, int* __restrict__ rank_out, int L,
      DevStatus* __restrict__ st) {
  extern __shared__ double eig_smem[];                 // [A | V] (N x N each)
  double* A = eig_smem;
  double* V = A + KRAW * KRAW;
  __shared__ double red[32];
  __shared__ int s_done;
  __shared__ int order[KRAW];
  __shared__ double lam[KRAW];
  __shared__ double rc[KRAW / 2], rs[KRAW / 2];
  const int task = blockIdx.x;
  const PcTask tk = tasks[task];
  const int kr = task_kr[task];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int N = kr + (kr & 1);
  const double* gt = gram + (long long)task * (KRAW * KRAW);
  for (int e = t; e < N * N; e += EIG_THREADS) {
    const int a = e % N, b = e / N;
    A[e] = (a < kr && b < kr) ? gt[a + b * kr] : 0.0;
    V[e] = (a == b) ? 1.0 : 0.0;
  }
  __syncthreads();
  if (kr > 1) {
    for (int sweep = 0; sweep < 40; ++sweep) {
      double off = 0.0, dia = 0.0;
      for (int e = t; e < N * N; e += EIG_THREADS) {
        const int a = e % N, b = e / N;
        if (a == b) dia += A[e] * A[e]; else off += A[e] * A[e];
      }
      off = block_sum(off, red);
      dia = block_sum(dia, red);
      if (t == 0) s_done = (off <= 1e-34 * dia);
      __syncthreads();
      if (s_done) break;
      for (int r = 0; r < N - 1; ++r) {
        int p = 0, q = 0;
        if (warp < N / 2) {
          int a, b;
          if (warp == 0) { a = r; b = N - 1; }
          else { a = (r + warp) % (N - 1); b = (r - warp + (N - 1)) % (N - 1); }
          p = min(a, b); q = max(a, b);
          const double app = A[p + p * N], aqq = A[q + q * N], apq = A[p + q * N];
          double c = 1.0, sn = 0.0;
          if (apq != 0.0 && fabs(apq) > 1e-300) {
            const double tau = (aqq - app) / (2.0 * apq);
            const double tt = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + tt * tt);
            sn = tt * c;
          }
          if (lane == 0) { rc[warp] = c; rs[warp] = sn; }
          __syncwarp();
          for (int j = lane; j < N; j += 32) {             // rows p, q:  A <- J^T A
            const double apj = A[p + j * N], aqj = A[q + j * N];
            A[p + j * N] = c * apj - sn * aqj;
            A[q + j * N] = sn * apj + c * aqj;
          }
        }
        __syncthreads();
        if (warp < N / 2) {
          const double c = rc[warp], sn = rs[warp];
          for (int i = lane; i < N; i += 32) {             // columns p, q:  A <- A J,  V <- V J
            const double aip = A[i + p * N], aiq = A[i + q * N];
            A[i + p * N] = c * aip - sn * aiq;
            A[i + q * N] = sn * aip + c * aiq;
            const double vip = V[i + p * N], viq = V[i + q * N];
            V[i + p * N] = c * vip - sn * viq;
            V[i + q * N] = sn * vip + c * viq;
          }
          __syncwarp();
          if (lane == 0) { A[p + q * N] = 0.0; A[q + p * N] = 0.0; }   // annihilated pair entry
        }
        __syncthreads();
      }
    }
  }
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
