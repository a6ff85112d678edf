// k_step.cuh -- the whole fused factor + solve step (S3-S6, tree path) as ONE persistent
// dataflow kernel: leaf tasks (k_leaf.cuh leaf_task), then the SMW tree units of every level
// (k_tree.cuh tr_unit), then the final u = X v groups (tr_final), claimed in that
// topological order from a single atomic counter.  A unit waits only for its own inputs
// (completion counters of its two children, release/acquire at gpu scope) instead of a grid
// barrier per level, so the tree's bottom levels fill the SMs left idle by the last wave of
// leaves, and no level waits for unrelated nodes.  Every claimed task only depends on tasks
// with smaller indices, all claimed by co-resident CTAs (cooperative launch): progress is
// guaranteed.  The arithmetic is exactly that of k_leaf + k_tree (same functions).
#pragma once
#include "k_leaf.cuh"
#include "k_tree.cuh"
#include "k_final.cuh"

struct StepArgs {
  LeafArgs la;
  TrArgs ta;
  unsigned* ctr;                 // task counter (zeroed before the launch)
  int* done;                     // completion counters (zeroed before the launch)
  long long dofs[LMAX + 1];      // per level m (0..L-1): offset of [inst][node] counters;
                                 // dofs[L]: [inst][level L-1 node] count of projected leaves
  long long lofs;                // [inst][leaf] panel-done flags
  unsigned long long* trace;     // optional: [task][start, end, kind, sm] (FDE_TRACE_STEP)
  // part of the step (the top-level split of one problem over ranks; batch 1):
  //   leaf tasks and finals for leaves [lf0, lf1); tree levels m in [mlo, mhi); restrict = 1:
  //   only the nodes of level m above [lf0, lf1); level mhi - 1's children (level mhi) were
  //   completed by an earlier launch when mhi < L (no wait).  Whole step: lf0 = 0, lf1 = nleaf,
  //   mlo = 0, mhi = L, restrict = 0, do_leaf = do_final = 1.
  int lf0, lf1, mlo, mhi, restrict_nodes, do_leaf, do_final;
};

__device__ __forceinline__ int st_ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_wait(const int* p, int target) {
  if (threadIdx.x == 0)
    while (st_ld_acquire(p) < target) __nanosleep(64);
  __syncthreads();
}

__device__ __forceinline__ void st_signal(int* p) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(p, 1);
  }
}

__global__ void __launch_bounds__(TR_THREADS, 1)
k_step(const StepArgs sa) {
  extern __shared__ double smem[];
  __shared__ int task;
  const TrArgs& a = sa.ta;
  const int B = a.batch, L = a.L, nleaf = a.nleaf;
  // leaves of the part (per instance) and the nodes of each processed level
  const int lcnt = sa.lf1 - sa.lf0;
  const long long n_leaf = sa.do_leaf ? (long long)B * lcnt : 0;
  __shared__ long long n_lvl[LMAX];                // (shared: indexed by the task's level)
  __shared__ int j0[LMAX], jn[LMAX];
  long long total = 2 * n_leaf;                    // panel tasks, then projection tasks
  for (int m = L - 1; m >= 0; --m) {
    const bool on = m >= sa.mlo && m < sa.mhi;
    const int j0m = sa.restrict_nodes ? (sa.lf0 >> (L - m)) : 0;
    const int jnm = !on ? 0 : (sa.restrict_nodes ? (lcnt >> (L - m)) : (1 << m));
    const long long nl = (long long)B * jnm * a.rc[m];
    if (threadIdx.x == 0) { j0[m] = j0m; jn[m] = jnm; n_lvl[m] = nl; }
    total += nl;
  }
  __syncthreads();
  const long long n_fin_leaves = sa.do_final ? (long long)B * lcnt : 0;
  const long long n_fin = (n_fin_leaves + TR_NL - 1) / TR_NL;
  total += n_fin;
  while (true) {
    __syncthreads();                               // (task of the previous iteration consumed)
    if (threadIdx.x == 0) task = (int)atomicAdd(sa.ctr, 1u);
    __syncthreads();
    long long tk = task;
    if (tk >= total) break;
    const long long tk0 = tk;
    unsigned long long t_start = 0;
    if (sa.trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    auto rec = [&](int kind) {
      if (sa.trace && threadIdx.x == 0 && tk0 < 4000) {
        unsigned long long te, smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(te));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(*(unsigned*)&smid));
        sa.trace[4 * tk0] = t_start; sa.trace[4 * tk0 + 1] = te; sa.trace[4 * tk0 + 2] = kind;
        sa.trace[4 * tk0 + 3] = smid & 0xffffffffu;
      }
    };
    if (tk < n_leaf) {                             // ---- leaf: build, LU, panel X
      const int inst = (int)(tk / lcnt), leaf = sa.lf0 + (int)(tk % lcnt);
      const long long gl = (long long)inst * nleaf + leaf;
      leaf_task(sa.la, smem, leaf, inst, false);
      st_signal(sa.done + sa.lofs + gl);
      rec(100);
      continue;
    }
    tk -= n_leaf;
    if (tk < n_leaf) {                             // ---- leaf: projection Q = V^T X
      const int inst = (int)(tk / lcnt), leaf = sa.lf0 + (int)(tk % lcnt);
      const long long gl = (long long)inst * nleaf + leaf;
      st_wait(sa.done + sa.lofs + gl, 1);
      leaf_proj_task(sa.la, smem, leaf, inst);
      st_signal(sa.done + sa.dofs[L] + (long long)inst * (1 << (L - 1)) + (leaf >> 1));
      rec(101);
      continue;
    }
    tk -= n_leaf;
    int m = L - 1;
    while (m >= 0 && tk >= n_lvl[m]) { tk -= n_lvl[m]; --m; }
    if (m >= 0) {                                  // ---- SMW unit of level m
      const long long per_inst = (long long)jn[m] * a.rc[m];
      const int inst = (int)(tk / per_inst), w = (int)(tk % per_inst);
      const int j = j0[m] + w / a.rc[m], chunk = w % a.rc[m];
      if (m == L - 1) {
        st_wait(sa.done + sa.dofs[L] + (long long)inst * (1 << (L - 1)) + j, 2);
      } else if (m + 1 < sa.mhi) {
        const int* c = sa.done + sa.dofs[m + 1] + (long long)inst * (1 << (m + 1)) + 2 * j;
        st_wait(c, a.rc[m + 1]);
        st_wait(c + 1, a.rc[m + 1]);
      }                                            // (else: children from an earlier launch)
      tr_unit(a, smem, inst, m, j, chunk);
      st_signal(sa.done + sa.dofs[m] + (long long)inst * (1 << m) + j);
      rec(m);
      continue;
    }
    // ---- final group: u = X v for TR_NL leaves of the part (needs every ancestor's S: the
    //      root's done -- in this launch if it holds level 0, else from an earlier launch)
    const long long lu0 = tk * TR_NL;
    const int nl = (int)min((long long)TR_NL, n_fin_leaves - lu0);
    const int i0 = (int)(lu0 / lcnt), i1 = (int)((lu0 + nl - 1) / lcnt);
    if (sa.mlo == 0 && sa.mhi > 0)
      for (int inst = i0; inst <= i1; ++inst) st_wait(sa.done + sa.dofs[0] + inst, a.rc[0]);
    for (int q = 0; q < nl; ) {                    // (contiguous runs of one instance)
      const long long g = lu0 + q;
      const int inst = (int)(g / lcnt), l = (int)(g % lcnt);
      const int run = min(nl - q, lcnt - l);
      tr_final(a, smem, inst * nleaf + sa.lf0 + l, run);
      q += run;
    }
    rec(200);
  }
}
