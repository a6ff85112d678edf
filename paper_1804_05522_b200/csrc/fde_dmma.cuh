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

// ---- mbarriers for the TMA-engine copies (k_leaf.cuh leaf_project_tma) -------------------
// A copy signals its bytes on an mbarrier (complete_tx), so one wait covers every copy of a phase.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_inval(unsigned long long* b) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {   // = arrive + tx
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned parity) {
  unsigned ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
               : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  while (!mbar_try(b, parity)) { }
}

// Contiguous run of `count` doubles -> shared memory with 16-byte cp.async for the aligned body
// (8-byte copies for an odd head / tail).  dst_base: 16-byte aligned with one spare double; the
// run lands at dst_base + (src parity), which is returned (the same for every thread).
__device__ __forceinline__ double* cp_contig_dst(double* dst_base, const double* src) {
  return dst_base + (int)((reinterpret_cast<unsigned long long>(src) >> 3) & 1);
}
__device__ __forceinline__ void cp_contig(double* dst_base, const double* src, int count, int t, int nt) {
  double* dst = cp_contig_dst(dst_base, src);
  const int h = (int)(dst - dst_base);               // 1: odd head element
  if (h && t == 0 && count > 0) cp_async8(dst, src);
  const int body = (count - h) >> 1;
  for (int e = t; e < body; e += nt) cp_async16(dst + h + 2 * e, src + h + 2 * e);
  const int done = h + 2 * body;
  if (done < count && t == nt - 1) cp_async8(dst + done, src + done);
}
