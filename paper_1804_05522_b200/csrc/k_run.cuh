// k_run.cuh -- K implicit-Euler steps (S3-S7) in ONE persistent dataflow launch, pipelined
// across time steps.  Of step m, only the right-hand-side column depends on u^(m-1); the leaf
// LUs, the U columns of the panel (X[:, 1:] = A_leaf^{-1} U) and their projections depend on
// d+-(t_m) alone.  Per leaf and step the work is therefore split into
//   A  : build + LU (stored, inverse-diagonal form) + U-column stripes   (k_leaf.cuh leaf_task, nf = 0)
//   B  : projection Q[:, 1:] = V_all^T X[:, 1:]                           (leaf_proj_task)
//   B' : u^(m-1) on the leaf's rows = X^(m-1) v^(m-1) (the "final" of step m-1, see k_tree.cuh),
//        x0 = A_leaf^{-1}(u^(m-1) + dt f^(m)) with the stored LU, X[:, 0] = x0,
//        Q[:, 0] = V_all^T x0                                             (leaf_rhs_final, k_final.cuh)
// and the SMW tree units of every level follow (k_tree.cuh tr_unit).  With whole tree units
// (fuse = 1, the default unless units are split) B runs inside B' as one task BB': after x0 the
// projection stages V once (TMA) and forms Q[:, 1:] and Q[:, 0] from it (tickets per step: A, BB').
// A virtual step K holds
// the last finals (u^(K-1)).  Only B' and the tree lie on the step-to-step chain; A and B of
// step m+1 fill the SMs while the tree of step m climbs its latency-bound upper levels.
//
// Scheduling.  Leaf work comes from one ticket queue (atomicAdd): A(m), B(m), B'(m) for
// m = 0..K-1, then the finals of step K.  Tree units never wait: a unit is released by the task
// whose completion makes it ready -- the CTA completing the last input of a node runs the
// node's first row chunk itself next (continuation: the step's critical chain runs without any
// queue round trip) and publishes the other chunks in a ready queue.  A CTA takes ready-queue
// work first (a ticket drawn when the queue is non-empty; a ticket drawn by a race past the
// tail is kept and served by a later release), then continuation, then its leaf ticket, whose
// inputs it polls.
// Every dependency points to an earlier task of the order A(0) B(0) B'(0) tree(0) A(1) ..., so
// the earliest incomplete task can always run: no deadlock for any number of co-resident CTAs.
// Buffers alternate by step parity (X, stored LU, Q, S); the waits below protect every reuse:
//   A(m)_i   waits B'(m-1)_i   (X^(m-2) of the leaf was last read by the final in B'(m-1)_i)
//   B(m)_i   waits A(m)_i
//   B'(m)_i  waits A(m)_i and root(m-1) of its instance (S^(m-1) complete)
//   tree(m) level L-1 unit j waits B and B' of leaves 2j, 2j+1; level m units their children.
// Same arithmetic as k_step except the rhs column: its leaf solve is a plain FMA block sweep
// (not the DMMA stripe) and u^(m-1) is formed per leaf.
//
// Time-invariant coefficients (inv = 1: coef_stride 0, A_m the same matrix every step; "the LU
// can be computed only once at the beginning"): the factor is formed once.  Step 0 runs A, B, B' and split tree
// units (U + R); steps 1..K-1 run only B' and the R units against the step-0 factor (one buffer set,
// no parity): tickets A(0) B(0) B'(0) B'(1) .. B'(K-1), finals(K).  Reuse safety on the single set:
//   X[:, 0] / Q_leaf[:, 0] of leaf i: read (final, bottom R unit) before B'(m+1)_i writes them --
//     B'(m+1)_i reads X^(m)[:, 0] itself, and waits root(m), so every R unit of step m is done;
//   S[:, 0] / Q_node[:, 0] of node p: R(m+1)_p runs after B'(m+1) of every leaf below p, the only
//     readers of S^(m)_p; the U-unit data ([C | Sc^-1 | G], S[:, 1:], Q[:, 1:]) is read-only after
//     step 0.  An R unit of a step >= 1 has no U input: it is released by its 2 children alone.
#pragma once
#include "k_step.cuh"   // (k_final.cuh: leaf_rhs_final, rn_copy)


// Steps per k_run launch: the step index is the 16-bit field of the tree task ids (rn_tid, kept
// non-negative); fde1d_run splits longer runs into launches of at most RUN_KMAX steps.
#define RUN_KMAX 8192

struct RunArgs {
  // per-step argument blocks in device memory (host-filled): step m's d+-, f, u^(m-1), u^(m)
  // and the parity-(m & 1) buffer set (X, stored leaf LU, Q, S).  Read by reference from
  // global memory, never copied into per-thread local memory.
  const LeafArgs* las;           // [K]
  const TrArgs* tas;             // [K]
  int K;
  int smem_doubles;              // dynamic shared memory of the launch
  unsigned* heads;               // [0] tree units done, [1] leaf tickets, [2] rq tail, [3] rq head
  unsigned long long* rq;        // ready queue: task id + 1 per slot (zeroed), K * units per step
  long long rq_cap;              // slots
  int use_rq;                    // some level splits its nodes into row chunks
  int* done; long long per_step; // step m counters: done + m * per_step (m = 0..K-1)
  long long o_A, o_R, o_lvl[LMAX];   // A done, B' done [leaf]; R unit done [node of level m]
  long long o_ku[LMAX], o_kr[LMAX];  // release counters of level-m nodes: U (2 inputs), R (3 inputs)
  int split;                         // 1: U / R tree units (one of each per node)
  int fuse;                          // 1 (whole units only): B runs inside B' (tickets A, BB' per step)
  int inv;                           // 1: factor once (step 0), B' + R units only after it (split units)
  unsigned long long* trace;     // optional (FDE_TRACE_RUN): [0] count, then [start,end,code,sm]
  unsigned long long* prof;      // optional: B' phase cycle sums [16]
  long long trace_cap;
};

__device__ __forceinline__ bool rn_ready(const int* p, int target) { return st_ld_acquire(p) >= target; }

// Leaf-queue ticket l: per step A of every leaf, B of every leaf, B' of every leaf (fused: A,
// BB'; inv: A, B, B' at step 0, then B' only); step K: finals.  -> (step, kind, leaf index tk)
__device__ __forceinline__ int rn_decode(const RunArgs& ra, long long n_leaf, long long l, long long& tk,
                                         int& step) {
  if (ra.inv) {
    if (l < 3 * n_leaf) { step = 0; tk = l % n_leaf; return (int)(l / n_leaf); }
    const long long l2 = l - 3 * n_leaf;
    step = 1 + (int)(l2 / n_leaf);
    tk = l2 - (long long)(step - 1) * n_leaf;
    return step == ra.K ? 3 : 2;
  }
  const int per = ra.fuse ? 2 : 3;
  step = (int)(l / (per * n_leaf));
  tk = l - (long long)step * per * n_leaf;
  int kind = step == ra.K ? 3 : (int)(tk / n_leaf);
  const int slot = kind == 3 ? 0 : kind;
  if (ra.fuse && kind == 1) kind = 2;
  tk -= slot * n_leaf;
  return kind;
}

// Are the inputs of leaf ticket l complete?
__device__ __forceinline__ bool rn_leaf_ready(const RunArgs& ra, long long n_leaf, long long l) {
  const TrArgs& a = ra.tas[0];
  long long tk;
  int step;
  const int kind = rn_decode(ra, n_leaf, l, tk, step);
  const int* dn = ra.done + (long long)step * ra.per_step;
  const int inst = (int)(tk / a.nleaf);
  if (kind == 0) return step < 2 || rn_ready(dn - ra.per_step + ra.o_R + tk, 1);
  if (kind == 1) return rn_ready(dn + ra.o_A + tk, 1);
  if (kind == 2 && !rn_ready((ra.inv ? ra.done : dn) + ra.o_A + tk, 1)) return false;   // (inv: A of step 0)
  return step < 1 || rn_ready(dn - ra.per_step + ra.o_lvl[0] + inst, a.rc[0]);
}

// Tree task ids: step (16 bits) | level m (8) | chunk (8) | node jj = inst 2^m + j (32).
__device__ __forceinline__ long long rn_tid(int step, int m, int chunk, long long jj) {
  // step < RUN_KMAX < 2^15, m < 2^8, chunk < 2^8, jj < 2^32: the id stays non-negative
  return ((long long)step << 48) | ((long long)m << 40) | ((long long)chunk << 32) | jj;
}

// Node jj of level m (step `step`) just became ready: its chunk 0 is this CTA's continuation,
// chunks 1.. go to the ready queue.  (thread 0)
__device__ __forceinline__ void rn_push(const RunArgs& ra, long long tid) {
  const unsigned slot = atomicAdd(ra.heads + 2, 1u);
  FDE_ASSERT((long long)slot < ra.rq_cap);
  const unsigned long long v = (unsigned long long)tid + 1ULL;
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(ra.rq + slot), "l"(v) : "memory");
}
__device__ __forceinline__ long long rn_release(const RunArgs& ra, int step, int m, long long jj) {
  const int rc = ra.tas[0].rc[m];
  for (int c = 1; c < rc; ++c) rn_push(ra, rn_tid(step, m, c, jj));
  return rn_tid(step, m, 0, jj);
}
// split run: a unit (part 0 = U, 1 = R) became ready -- the continuation if the CTA has none yet,
// else the ready queue  (thread 0)
__device__ __forceinline__ void rn_ready_unit(const RunArgs& ra, int step, int m, int part, long long jj,
                                              long long& cont) {
  const long long tid = rn_tid(step, m, part, jj);
  if (cont < 0) cont = tid; else rn_push(ra, tid);
}

__global__ void __launch_bounds__(TR_THREADS, 1)
k_run(const RunArgs ra) {
  extern __shared__ double smem[];
  __shared__ long long task;
  __shared__ int queue;
  // the task's argument blocks, copied from global memory once per task: the kernels read
  // their geometry (xcol, ranks, offsets, ...) from shared memory, not through the L1
  __shared__ LeafArgs s_la;
  __shared__ TrArgs s_ta, s_tp;
  __shared__ int s_la_step, s_ta_step, s_tp_step;   // which step's block each copy holds
  if (threadIdx.x == 0) { s_la_step = -1; s_ta_step = -1; s_tp_step = -1; }
  FDE_ASSERT((long long)ra.smem_doubles * 8 >= LEAF_SMEM);
  const TrArgs& a0 = ra.tas[0];
  const int L = a0.L, nleaf = a0.nleaf;
  const long long n_leaf = (long long)a0.batch * nleaf;
  long long Tt = 0;
  for (int m = 0; m < L; ++m) Tt += (long long)a0.batch * (1LL << m) * (ra.split ? 2 : a0.rc[m]);
  // (inv: U + R units at step 0, R units only after it; A, B, B' tickets at step 0, B' only after it)
  const unsigned tot_t = (unsigned)(ra.inv ? Tt + (Tt / 2) * (ra.K - 1) : Tt * ra.K);
  const unsigned tot_l = (unsigned)(ra.inv ? (ra.K + 3) * n_leaf : (ra.fuse ? 2 : 3) * n_leaf * ra.K + n_leaf);
  volatile unsigned* vh = ra.heads;     // [0] tree units completed, [1] leaf tickets, [2] rq tail, [3] rq head
  long long held = -1;                  // thread 0: leaf ticket not yet runnable
  long long iou = -1;                   // thread 0: ready-queue ticket not yet served
  long long cont = -1;                  // thread 0: continuation tree task
  bool leaf_out = false;                // thread 0: leaf queue exhausted
  while (true) {
    __syncthreads();                                  // (previous task consumed)
    if (threadIdx.x == 0) {
      int q = -1;
      long long idx = 0;
      while (true) {
        if (cont >= 0) {                              // (released by our relaxed RMW on the
          asm volatile("fence.acq_rel.gpu;" ::: "memory");   // children's counters: acquire here)
          q = 0; idx = cont; cont = -1; break;
        }
        if (!ra.use_rq) {                             // (one unit per node: nothing is ever queued)
        } else if (iou >= 0) {                        // then ready-queue work
          unsigned long long v;
          asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ra.rq + iou) : "memory");
          if (v) { q = 0; idx = (long long)(v - 1); iou = -1; break; }
        } else if (vh[2] > vh[3]) {
          iou = atomicAdd(ra.heads + 3, 1u);
          if (iou >= ra.rq_cap) iou = -1;             // (a race past the last slot: never filled)
          else continue;
        }
        if (held < 0 && !leaf_out) {
          const unsigned l = atomicAdd(ra.heads + 1, 1u);
          if (l < tot_l) held = l; else leaf_out = true;
        }
        if (held >= 0 && rn_leaf_ready(ra, n_leaf, held)) { q = 1; idx = held; held = -1; break; }
        if (leaf_out && held < 0 && vh[0] >= tot_t) break;
        __nanosleep(32);
      }
      queue = q; task = idx;
    }
    __syncthreads();
    if (queue < 0) break;
    unsigned long long t_start = 0;
    if (ra.trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    int code;
    if (queue == 1) {                                 // ---- leaf ticket
      long long tk;
      int step;
      const int kind = rn_decode(ra, n_leaf, task, tk, step);
      const int inst = (int)(tk / nleaf), leaf = (int)(tk % nleaf);
      FDE_ASSERT(step >= 0 && step <= ra.K && kind >= 0 && kind <= 3 && (kind == 3) == (step == ra.K));
      FDE_ASSERT(inst >= 0 && inst < a0.batch && leaf >= 0 && leaf < nleaf);
      int* dn = ra.done + (long long)step * ra.per_step;
      if (kind == 0) {                                // A: build, LU (stored), U columns
        if (s_la_step != step) { rn_copy(&s_la, &ra.las[step]); if (threadIdx.x == 0) s_la_step = step; }
        leaf_task<true>(s_la, smem, leaf, inst, false);
      } else if (kind == 1) {                         // B: projection of the U columns
        if (s_la_step != step) { rn_copy(&s_la, &ra.las[step]); if (threadIdx.x == 0) s_la_step = step; }
        leaf_proj_task(s_la, smem, leaf, inst);
      } else {                                        // B': final of step-1 + rhs column
        if (kind == 2 && s_la_step != step) { rn_copy(&s_la, &ra.las[step]); if (threadIdx.x == 0) s_la_step = step; }
        const int tps = step > 0 ? step - 1 : 0;
        if (s_tp_step != tps) { rn_copy(&s_tp, &ra.tas[tps]); if (threadIdx.x == 0) s_tp_step = tps; }
        leaf_rhs_final(s_tp, step > 0 ? &s_tp : nullptr, kind == 2 ? &s_la : nullptr,
                       smem, ra.smem_doubles, inst, leaf, ra.prof, !(ra.fuse && kind == 2));
        if (ra.prof && threadIdx.x == 0) atomicAdd(ra.prof + (kind == 2 ? 7 : 15), 1ULL);
        if (ra.fuse && kind == 2) {                   // BB': the projection with Q[:, 0] (x0 in smem[0, s))
          __syncthreads();
          leaf_proj_task(s_la, smem, leaf, inst, true);
        }
      }
      __syncthreads();
      if (threadIdx.x == 0 && kind < 3) {
        __threadfence();
        if (kind == 0) atomicAdd(dn + ra.o_A + tk, 1);
        if (kind == 2) atomicAdd(dn + ra.o_R + tk, 1);
        if (kind >= 1) {
          const long long jj = (long long)inst * (1 << (L - 1)) + (leaf >> 1);
          if (ra.split) {                           // B -> U of the bottom node; B' -> its R
            if (kind == 1) { if (atomicAdd(dn + ra.o_ku[L - 1] + jj, 1) == 1) rn_ready_unit(ra, step, L - 1, 0, jj, cont); }
            else if (atomicAdd(dn + ra.o_kr[L - 1] + jj, 1) == (ra.inv && step > 0 ? 1 : 2))
              rn_ready_unit(ra, step, L - 1, 1, jj, cont);
          } else if (atomicAdd(dn + ra.o_ku[L - 1] + jj, 1) == (ra.fuse ? 1 : 3)) {
            cont = rn_release(ra, step, L - 1, jj);
          }
        }
      }
      code = 100 + kind + 1000 * step;
    } else {                                          // ---- tree unit
      const int step = (int)(task >> 48), m = (int)((task >> 40) & 0xff), chunk = (int)((task >> 32) & 0xff);
      const long long jj = task & 0xffffffffLL;
      const int inst = (int)(jj >> m), j = (int)(jj & ((1LL << m) - 1));
      FDE_ASSERT(step >= 0 && step < ra.K && m >= 0 && m < L && chunk >= 0 && chunk < (ra.split ? 2 : a0.rc[m]));
      FDE_ASSERT(inst >= 0 && inst < a0.batch && j >= 0 && j < (1 << m));
      int* dn = ra.done + (long long)step * ra.per_step;
      if (s_ta_step != step) { rn_copy(&s_ta, &ra.tas[step]); if (threadIdx.x == 0) s_ta_step = step; }
      const TrArgs& a = s_ta;
      const bool runit = ra.split && chunk == 1;
      if (runit) tr_unit_R(a, smem, inst, m, j);
      else tr_unit(a, smem, inst, m, j, ra.split ? 0 : chunk);
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        const long long pj = m > 0 ? (long long)inst * (1 << (m - 1)) + (j >> 1) : 0;
        if (!ra.split) {
          if (atomicAdd(dn + ra.o_lvl[m] + jj, 1) == a.rc[m] - 1 && m > 0) {   // node complete
            if (atomicAdd(dn + ra.o_ku[m - 1] + pj, 1) == 1) cont = rn_release(ra, step, m - 1, pj);
          }
        } else if (!runit) {                        // U: parent's U (2 children), own R (+1)
          if (m > 0 && atomicAdd(dn + ra.o_ku[m - 1] + pj, 1) == 1) rn_ready_unit(ra, step, m - 1, 0, pj, cont);
          if (atomicAdd(dn + ra.o_kr[m] + jj, 1) == 2) rn_ready_unit(ra, step, m, 1, jj, cont);
        } else {                                    // R: node done, parent's R (+1)
          atomicAdd(dn + ra.o_lvl[m] + jj, 1);
          if (m > 0 && atomicAdd(dn + ra.o_kr[m - 1] + pj, 1) == (ra.inv && step > 0 ? 1 : 2))
            rn_ready_unit(ra, step, m - 1, 1, pj, cont);
        }
        atomicAdd(ra.heads, 1u);
      }
      code = (runit ? 50 : 0) + m + 1000 * step;
    }
    if (ra.trace && threadIdx.x == 0) {
      const unsigned long long e = atomicAdd(ra.trace, 1ULL);
      if ((long long)e < ra.trace_cap) {
        unsigned long long te; unsigned smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(te));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        unsigned long long* r = ra.trace + 4 + 4 * e;
        r[0] = t_start; r[1] = te; r[2] = (unsigned long long)code; r[3] = smid;
      }
    }
  }
}
