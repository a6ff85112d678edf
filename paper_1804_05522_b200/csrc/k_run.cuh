// k_run.cuh -- K implicit-Euler steps (S3-S7) in ONE persistent dataflow launch, pipelined
// across time steps.  Only the right-hand-side column of the leaf panel depends on the previous
// step's solution; everything else of step m (leaf LU, the U columns of the panel and their
// projection) depends only on d+-(t_m).  So each step is split into
//   A  (leaf): build + LU + U-column stripes, LU stored          (k_leaf.cuh leaf_task, nf = 0)
//   B  (leaf): projection Q[:, 1:] = V^T X[:, 1:]                 (leaf_proj_task)
//   A' (leaf): x0 = A_leaf^{-1}(u^(m-1) + dt f), Q[:, 0] = V^T x0 (leaf_rhs_task)
//   tree units of every level, then u^(m) = X v per leaf group    (k_tree.cuh)
// and the task queue of step m+1 follows that of step m: the A and B tasks of step m+1 run on
// the SMs the latency-bound tree levels of step m leave idle.  Dependencies are per-task
// counters (release/acquire at gpu scope); a task only waits for tasks with smaller indices
// (claimed earlier by co-resident CTAs), so progress is guaranteed.  Step parity selects one
// of two buffer sets (X, LU, Q, S); a step-m task never overwrites data a step m-2 task still
// reads (A(m) waits for the final(m-2) group of its leaf).  Same arithmetic as k_step.
#pragma once
#include "k_step.cuh"

struct RunArgs {
  LeafArgs la;                   // template (tree, g, L_l, ...); per-step fields set per task
  TrArgs ta;
  int K;
  const double* dp; const double* dm; long long coef_stride;   // step m: dp + m * coef_stride
  const double* f; long long f_stride;
  const double* u0; double* uout;                              // uout + m * batch * n
  double* X[2]; double* LU[2]; double* Q[2]; double* S[2];
  unsigned* ctr;
  int* done; long long per_step;                               // step m counters: done + m * per_step
  long long o_A, o_pair, o_fin, o_lvl[LMAX];
};

__global__ void __launch_bounds__(TR_THREADS, 1)
k_run(const RunArgs ra) {
  extern __shared__ double smem[];
  __shared__ int task;
  const TrArgs& a0 = ra.ta;
  const int B = a0.batch, L = a0.L, nleaf = a0.nleaf, n = a0.n;
  const long long n_leaf = (long long)B * nleaf;
  long long n_lvl[LMAX];
  long long T = 3 * n_leaf;
  for (int m = L - 1; m >= 0; --m) { n_lvl[m] = (long long)B * (1LL << m) * a0.rc[m]; T += n_lvl[m]; }
  const long long n_fin = (n_leaf + TR_NL - 1) / TR_NL;
  T += n_fin;
  const long long total = T * ra.K;
  while (true) {
    __syncthreads();
    if (threadIdx.x == 0) task = (int)atomicAdd(ra.ctr, 1u);
    __syncthreads();
    long long tk = task;
    if (tk >= total) break;
    const int step = (int)(tk / T), p = step & 1;
    tk -= (long long)step * T;
    int* dn = ra.done + (long long)step * ra.per_step;
    int* dprev = ra.done + (long long)(step - 1) * ra.per_step;     // (valid for step >= 1)
    int* dprev2 = ra.done + (long long)(step - 2) * ra.per_step;    // (valid for step >= 2)
    // per-step views
    LeafArgs la = ra.la;
    la.dp = ra.dp + (long long)step * ra.coef_stride;
    la.dm = ra.dm + (long long)step * ra.coef_stride;
    la.f = ra.f + (long long)step * ra.f_stride;
    la.u_prev = step == 0 ? ra.u0 : ra.uout + (long long)(step - 1) * B * n;
    la.X = ra.X[p]; la.LU = ra.LU[p];
    la.Q = ra.Q[p] + a0.qlev[L];
    if (tk < n_leaf) {                                  // ---- A: build, LU (stored), U columns
      const int inst = (int)(tk / nleaf), leaf = (int)(tk % nleaf);
      if (step >= 2) st_wait(dprev2 + ra.o_fin + tk / TR_NL, 1);
      la.nf = 0; la.store_lu = 1;
      leaf_task(la, smem, leaf, inst, false);
      st_signal(dn + ra.o_A + tk);
      continue;
    }
    tk -= n_leaf;
    if (tk < n_leaf) {                                  // ---- B: projection of the U columns
      const int inst = (int)(tk / nleaf), leaf = (int)(tk % nleaf);
      st_wait(dn + ra.o_A + tk, 1);
      la.nf = 0;
      leaf_proj_task(la, smem, leaf, inst);
      st_signal(dn + ra.o_pair + (long long)inst * (1 << (L - 1)) + (leaf >> 1));
      continue;
    }
    tk -= n_leaf;
    if (tk < n_leaf) {                                  // ---- A': the rhs column
      const int inst = (int)(tk / nleaf), leaf = (int)(tk % nleaf);
      st_wait(dn + ra.o_A + tk, 1);
      if (step >= 1) st_wait(dprev + ra.o_fin + tk / TR_NL, 1);
      leaf_rhs_task(la, smem, leaf, inst);
      st_signal(dn + ra.o_pair + (long long)inst * (1 << (L - 1)) + (leaf >> 1));
      continue;
    }
    tk -= n_leaf;
    TrArgs a = a0;
    a.Q = ra.Q[p]; a.Qleaf = ra.Q[p] + a0.qlev[L]; a.Sst = ra.S[p]; a.X = ra.X[p];
    a.u = ra.uout + (long long)step * B * n;
    int m = L - 1;
    while (m >= 0 && tk >= n_lvl[m]) { tk -= n_lvl[m]; --m; }
    if (m >= 0) {                                       // ---- SMW unit of level m
      const long long per_inst = (1LL << m) * a.rc[m];
      const int inst = (int)(tk / per_inst), w = (int)(tk % per_inst);
      const int j = w / a.rc[m], chunk = w % a.rc[m];
      if (m == L - 1) {
        st_wait(dn + ra.o_pair + (long long)inst * (1 << (L - 1)) + j, 4);
      } else {
        const int* c = dn + ra.o_lvl[m + 1] + (long long)inst * (1 << (m + 1)) + 2 * j;
        st_wait(c, a.rc[m + 1]);
        st_wait(c + 1, a.rc[m + 1]);
      }
      tr_unit(a, smem, inst, m, j, chunk);
      st_signal(dn + ra.o_lvl[m] + (long long)inst * (1 << m) + j);
      continue;
    }
    // ---- final group: u^(step) = X v for TR_NL leaves
    const long long lu0 = tk * TR_NL;
    const int nl = (int)min((long long)TR_NL, n_leaf - lu0);
    const int i0 = (int)(lu0 / nleaf), i1 = (int)((lu0 + nl - 1) / nleaf);
    for (int inst = i0; inst <= i1; ++inst) st_wait(dn + ra.o_lvl[0] + inst, a.rc[0]);
    tr_final(a, smem, (int)lu0, nl);
    st_signal(dn + ra.o_fin + tk);
  }
}
