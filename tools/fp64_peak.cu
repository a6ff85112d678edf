// fp64_peak.cu -- measure the B200 FP64 throughput ceilings used as roofline denominators:
//   (a) DFMA (CUDA-core FP64) and (b) DMMA (mma.sync m8n8k4 f64 tensor path).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
         a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-9 + 1.0, b = 0.5;
  double d[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) { d[k][0] = 0; d[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[k][0]), "+d"(d[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = nsm * 4, threads = 512;
  for (int rep = 0; rep < 2; ++rep) {
    const int it = 20000;
    dfma_loop<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, it);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)it * blocks * threads;
    printf("{\"kind\": \"dfma\", \"tflops\": %.3f, \"ms\": %.3f}\n", flops / ms * 1e-9, ms);
    const int it2 = 20000;
    dmma_loop<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    dmma_loop<<<blocks, threads>>>(out, it2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double f2 = 2.0 * 8 * 8 * 4 * 8 * (double)it2 * blocks * (threads / 32);
    printf("{\"kind\": \"dmma_m8n8k4\", \"tflops\": %.3f, \"ms\": %.3f}\n", f2 / ms * 1e-9, ms);
  }
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", nsm, clk);
  return 0;
}
