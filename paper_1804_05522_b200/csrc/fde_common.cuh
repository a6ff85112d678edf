// fde_common.cuh -- shared definitions of the sm_100a HODLR library (no torch types).
// Citations: P:<n> = PAPER.md line n.  See include/fdehodlr.h and DESIGN.md.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fdehodlr.h"

// ---- diagnostics switches ----------------------------------------------------------------
// Trace / experiment switches (FDE_TRACE_RUN, FDE_TRACE_STEP, FDE_TRACE_LEVELS, FDE_DEBUG2D,
// FDE_LEVEL_PASSES, FDE_SPLIT_KERNELS) exist only in the diagnostics build
// (libfdehodlr_dbg.so, compiled with -DFDE_DEBUG by build.py); the product library never reads
// the environment, so its behaviour is fixed by the C-ABI arguments alone.
#ifdef FDE_DEBUG
#include <cstdlib>
#include <cstdio>
static inline const char* fde_dbg_env(const char* name) { return getenv(name); }
#else
static inline const char* fde_dbg_env(const char*) { return nullptr; }
#endif

// Device bounds / invariant checks of the diagnostics build (compute-sanitizer is not available
// on the GPU pool, profiles/r02_sanitizer.md): a failed check prints its location and traps, so
// the launch fails with an error instead of touching memory it does not own.  Compiled out of
// the product library.
#ifdef FDE_DEBUG
#define FDE_ASSERT(c)                                                               \
  do {                                                                              \
    if (!(c)) {                                                                     \
      printf("FDE_ASSERT failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
             (int)blockIdx.x, (int)threadIdx.x);                                    \
      __trap();                                                                     \
    }                                                                               \
  } while (0)
#else
#define FDE_ASSERT(c) do { } while (0)
#endif

// ---- capacities ---------------------------------------------------------------------
#define LEAF_MAX   FDE_LEAF_MAX          // leaf held in shared memory (128 x 129 doubles)
#define RCAP       FDE_RANK_MAX          // max compressed rank per level (T-block)
#define KCAP       (RCAP + 1)            // X columns per level: r low-rank + 1 exact column
#define KRAW       48                    // max pivots of the partial pivoted Cholesky
#define NRHS_MAX   64                    // max right-hand sides of one hodlr_solve call
#define LMAX       24                    // max tree depth
#define SEG        128                   // rows per segment of the level passes
#define PB         32                    // diagonal block of the blocked leaf LU

static_assert(KRAW >= RCAP, "raw pivot cap must cover the final rank cap");

// ---- device status word (latched first failure) ----------------------------------------
struct DevStatus {
  int code;    // FDE_OK / FDE_ESINGULAR / FDE_ENOCONV
  int where;   // instance * 65536 + index
};

__device__ __forceinline__ void latch_status(DevStatus* st, int code, int where) {
  if (atomicCAS(&st->code, 0, code) == 0) atomicExch(&st->where, where);
}

// ---- tree description (host computed, copied once) -------------------------------------
// Nodes of level l are indexed (1<<l)-1+j, j < 2^l; leaves j < 2^L.
// Segments: per level, the children of every node are cut into pieces of <= SEG rows.
struct TreeDev {
  int n, L, nleaf;
  const int* node_r0;     // [2^L - 1]
  const int* node_n1;
  const int* node_n2;
  const int* node_seg;    // [2^L - 1][3]: first segment of child 0, of child 1, end (level-local)
  const int* leaf_r0;     // [2^L]
  const int* leaf_n;
  const int* seg_ofs;     // [L+1] start of each level's segment list
  const int* seg_node;    // level-local node index j
  const int* seg_child;   // 0 (first child, rows [r0, r0+n1)) or 1
  const int* seg_row0;    // global first row
  const int* seg_len;     // rows
  const int* lev_m;       // [L] Hankel section size of level l (max n2 over its nodes)
  const long long* lev_lofs;  // [L] offset of level l's factor inside an instance's block
};

// ---- per-instance, per-level rank bookkeeping written by the compression ----------------
// rank[inst*L + l] = r_l ; colofs[inst*(L+1) + l] = sum_{l'<l} (r_l'+1)   (X column offsets)

__host__ __device__ __forceinline__ int node_index(int l, int j) { return (1 << l) - 1 + j; }
