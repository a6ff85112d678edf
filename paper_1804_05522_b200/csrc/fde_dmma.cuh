// fde_dmma.cuh -- FP64 tensor-core MMA (mma.sync.m8n8k4.f64, SASS DMMA.8x8x4) helpers.
// tcgen05.mma has no f64 kind; on sm_100a the FP64 tensor path is the warp-level DMMA.
// Fragment layout (verified on B200 by tools/dmma_layout.cu):
//   gid = lane >> 2, tig = lane & 3
//   A (8x4, row-major): a = A[gid][tig]
//   B (4x8):            b = B[tig][gid]
//   C/D (8x8):          c0 = C[gid][2*tig], c1 = C[gid][2*tig + 1]
#pragma once

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__host__ __device__ __forceinline__ int round_up(int x, int m) { return (x + m - 1) / m * m; }

// Asynchronous global -> shared copies (SASS LDGSTS): a whole tile is put in flight before
// the single wait, instead of one load round trip per loop iteration.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {   // both 16-byte aligned
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_group1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
