// Dependent-chain latencies (SM cycles) of the primitives the latency-bound kernels are built
// from: FP64 FMA / sqrt / div / rcp.approx / rsqrt, shared-memory load, __syncthreads at 8 and 16
// warps, L2 round trip, gpu-scope fences, release-store + relaxed-load poll of the same CTA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_fp64 tools/lat_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

#define N 256

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__device__ __forceinline__ double rcp_approx(double x) {
  double y;
  asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

__global__ void k_lat(double* out, long long* cyc, double seed, volatile double* gbuf,
                      unsigned long long* flag) {
  __shared__ double sm[1024];
  const int t = threadIdx.x;
  for (int i = t; i < 1024; i += blockDim.x) sm[i] = 1.0 + 1e-9 * i;
  __syncthreads();
  double x = seed + t * 1e-12;
  long long c0, c1;
  int k = 0;
#define TIME(expr)                                                     \
  c0 = clock64();                                                      \
  for (int i = 0; i < N; ++i) { expr; }                                \
  c1 = clock64();                                                      \
  if (t == 0) cyc[k] = (c1 - c0);                                      \
  ++k;
  TIME(x = fma(x, 1.0000001, 1e-9))                    // 0 dfma
  TIME(x = sqrt(x + 1.0))                              // 1 sqrt
  TIME(x = 1.0 / (x + 0.5))                            // 2 div
  TIME(x = rcp_approx(x + 0.5))                        // 3 rcp.approx
  TIME(x = rsqrt(x + 0.5))                             // 4 rsqrt
  {
    int idx = (int)(x * 0.0) + t;
    c0 = clock64();
    for (int i = 0; i < N; ++i) idx = (int)sm[idx & 1023] + (idx & 511);   // 5 lds chain (+cvt)
    c1 = clock64();
    if (t == 0) cyc[k] = c1 - c0;
    ++k;
    x += idx;
  }
  TIME(__syncthreads())                                 // 6 bar (blockDim warps)
  {
    double v = x;
    c0 = clock64();
    for (int i = 0; i < 32; ++i) v = gbuf[((long long)(v * 0.0) + i * 4099) & 0xfffff] + v;   // 7 L2 (32 dependent)
    c1 = clock64();
    if (t == 0) cyc[k] = (c1 - c0) * N / 32;
    ++k;
    x += v;
  }
  c0 = clock64();
  for (int i = 0; i < 32; ++i) { __threadfence(); if (t == 0) gbuf[i] = x; }
  c1 = clock64();
  if (t == 0) cyc[k] = (c1 - c0) * N / 32;              // 8 threadfence + store
  ++k;
  c0 = clock64();
  for (int i = 0; i < 32; ++i) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  c1 = clock64();
  if (t == 0) cyc[k] = (c1 - c0) * N / 32;              // 9 fence.acq_rel.gpu
  ++k;
  if (t == 0) {                                         // 10 release store + relaxed poll (own)
    unsigned long long* f = flag + blockIdx.x * 32;
    c0 = clock64();
    for (int i = 0; i < 32; ++i) {
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(f), "l"((unsigned long long)(i + 1)) : "memory");
      unsigned long long v;
      do { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory"); } while (v < (unsigned long long)(i + 1));
    }
    c1 = clock64();
    cyc[k] = (c1 - c0) * N / 32;
  }
  ++k;
  if (t == 0) {                                         // 11 atomicAdd round trip
    c0 = clock64();
    unsigned long long v = 0;
    for (int i = 0; i < 32; ++i) v += atomicAdd(flag + 4096 + blockIdx.x, 1ULL + (v & 0));
    c1 = clock64();
    cyc[k] = (c1 - c0) * N / 32;
    x += (double)v;
  }
  ++k;
  if (t == 0) {                                         // 12 nanosleep(16)
    c0 = clock64();
    for (int i = 0; i < 32; ++i) __nanosleep(16);
    c1 = clock64();
    cyc[k] = (c1 - c0) * N / 32;
  }
  ++k;
  {                                                     // 13 DMMA dependent chain
    double c0 = x, c1 = 0.0;
    c0 = clock64();
    c0 = x;
    long long s0 = clock64();
    for (int i = 0; i < N; ++i) dmma884(c0, c1, 1.0000001, 0.5);
    long long s1 = clock64();
    if (t == 0) cyc[k] = s1 - s0;
    ++k;
    x += c0 + c1;
  }
  {                                                     // 14 DMMA 4 independent chains (per DMMA)
    double c[4][2] = {{x, 0}, {x, 1}, {x, 2}, {x, 3}};
    long long s0 = clock64();
    for (int i = 0; i < N / 4; ++i) {
#pragma unroll
      for (int u = 0; u < 4; ++u) dmma884(c[u][0], c[u][1], 1.0000001, 0.5);
    }
    long long s1 = clock64();
    if (t == 0) cyc[k] = s1 - s0;
    ++k;
    x += c[0][0] + c[1][0] + c[2][0] + c[3][0];
  }
  {                                                     // 15 DMMA 8 independent chains (per DMMA)
    double c[8][2];
#pragma unroll
    for (int u = 0; u < 8; ++u) { c[u][0] = x + u; c[u][1] = 0.0; }
    long long s0 = clock64();
    for (int i = 0; i < N / 8; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u) dmma884(c[u][0], c[u][1], 1.0000001, 0.5);
    }
    long long s1 = clock64();
    if (t == 0) cyc[k] = s1 - s0;
    ++k;
#pragma unroll
    for (int u = 0; u < 8; ++u) x += c[u][0];
  }
  {                                                     // 16 shfl (double) chain
    double v = x;
    long long s0 = clock64();
    for (int i = 0; i < N; ++i) v = __shfl_sync(0xffffffffu, v, (t + 1) & 31) + 1e-9;
    long long s1 = clock64();
    if (t == 0) cyc[k] = s1 - s0;
    ++k;
    x += v;
  }
  out[t] = x;
}

int main() {
  double *out, *gbuf;
  long long* cyc;
  unsigned long long* flag;
  cudaMalloc(&out, 1024 * 8);
  cudaMalloc(&cyc, 64 * 8);
  cudaMalloc(&gbuf, (1 << 20) * 8);
  cudaMemset(gbuf, 0, (1 << 20) * 8);
  cudaMalloc(&flag, 8192 * 8);
  cudaMemset(flag, 0, 8192 * 8);
  const char* names[] = {"dfma", "sqrt(f64)", "div(f64)", "rcp.approx.f64", "rsqrt(f64)", "lds+cvt chain",
                         "__syncthreads", "L2 load (dep)", "threadfence+st", "fence.acq_rel.gpu",
                         "st.release+ld.relaxed poll", "atomicAdd (rt)", "nanosleep(16)",
                         "dmma dep chain", "dmma 4 chains (per op)", "dmma 8 chains (per op)", "shfl f64 + dadd chain"};
  for (int warps : {8, 16}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(flag, 0, 8192 * 8);
      k_lat<<<1, 32 * warps>>>(out, cyc, 1.5, gbuf, flag);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    }
    long long h[64];
    cudaMemcpy(h, cyc, 17 * 8, cudaMemcpyDeviceToHost);
    printf("warps=%d\n", warps);
    for (int i = 0; i < 17; ++i) printf("  %-28s %7.1f cycles\n", names[i], (double)h[i] / N);
  }
  return 0;
}
