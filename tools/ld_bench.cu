// Per-SM streaming read bandwidth by load method (one CTA of 256 threads per SM, each CTA reads
// its own 148 KB "leaf panel" = 145 columns x 1 KB strided by n, as the B' final does).
// usage: ld_bench <nctas>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __launch_bounds__(256, 1) k_ld(const double* __restrict__ X, long long n, int NC, double* out,
                                              unsigned long long* cyc) {
  extern __shared__ double sm[];
  __shared__ unsigned long long bar;
  const int t = threadIdx.x;
  const double* Xi = X + (long long)blockIdx.x * 128;
  double acc = 0.0;
  __syncthreads();
  const long long t0 = clock64();
  if (MODE == 0) {                        // plain double2 loads, all columns of a quarter in flight
    const int i2 = 2 * (t & 63), h = t >> 6;
    for (int c = h; c < NC; c += 4 * 24) {
      double2 x[24];
#pragma unroll
      for (int u = 0; u < 24; ++u) x[u] = c + 4 * u < NC ? *reinterpret_cast<const double2*>(Xi + (long long)(c + 4 * u) * n + i2) : make_double2(0, 0);
#pragma unroll
      for (int u = 0; u < 24; ++u) acc += x[u].x + x[u].y;
    }
  } else if (MODE == 1) {                 // cp.async 16 B into smem, one wait
    for (int e = t; e < NC * 64; e += 256) {
      const int c = e >> 6, i2 = 2 * (e & 63);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(sm + c * 128 + i2)), "l"(Xi + (long long)c * n + i2) : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    acc = sm[t];
  } else if (MODE == 3) {                 // cp.async 8 B into smem, one wait
    for (int e = t; e < NC * 128; e += 256) {
      const int c = e >> 7, i = e & 127;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(su32(sm + c * 128 + i)), "l"(Xi + (long long)c * n + i) : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    acc = sm[t];
  } else if (MODE == 4) {                 // plain 8-byte loads, 32 in flight per thread
    const int i = t & 127, h = t >> 7;
    for (int c = h; c < NC; c += 2 * 32) {
      double x[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) x[u] = c + 2 * u < NC ? Xi[(long long)(c + 2 * u) * n + i] : 0.0;
#pragma unroll
      for (int u = 0; u < 32; ++u) acc += x[u];
    }
  } else {                                // TMA 1D bulk copies (1 KB per column), one mbarrier
    if (t == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (t == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(NC * 1024) : "memory");
      for (int c = 0; c < NC; ++c)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 1024, [%2];"
                     ::"r"(su32(sm + c * 128)), "l"(Xi + (long long)c * n), "r"(su32(&bar)) : "memory");
    }
    unsigned ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(su32(&bar)) : "memory");
    acc = sm[t];
  }
  __syncthreads();
  const long long t1 = clock64();
  if (t == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 12345.0) out[t] = acc;
}

int main(int argc, char** argv) {
  const long long n = 65536; const int NC = 145;
  double* X; double* out; unsigned long long* cyc;
  cudaMalloc(&X, n * NC * 8 * 4); cudaMemset(X, 0, n * NC * 8 * 4);
  cudaMalloc(&out, 4096); cudaMalloc(&cyc, 4096 * 8);
  void* flush; cudaMalloc(&flush, 512 << 20);
  for (int mode = 0; mode < 5; ++mode)
    for (int nct : {1, 16, 148}) {
      auto f = mode == 0 ? k_ld<0> : mode == 1 ? k_ld<1> : mode == 2 ? k_ld<2> : mode == 3 ? k_ld<3> : k_ld<4>;
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      unsigned long long h[148];
      double best = 1e30, avg = 0;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(flush, rep, 512 << 20);       // cold: X in HBM
        f<<<nct, 256, 160 * 1024>>>(X, n, NC, out, cyc);
        cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, nct * 8, cudaMemcpyDeviceToHost);
        double a = 0; for (int i = 0; i < nct; ++i) a += h[i]; a /= nct;
        avg = a;
      }
      printf("mode %d (%s) ctas %3d: %.2f us per CTA for %d KB -> %.1f GB/s per SM  [%s]\n", mode,
             mode == 0 ? "ld.v2 x24" : mode == 1 ? "cp.async16" : mode == 2 ? "TMA 1D" : mode == 3 ? "cp.async8" : "ld.f64 x32", nct, avg / 1965.0, NC, NC * 1024 / (avg / 1965.0) / 1e3,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
