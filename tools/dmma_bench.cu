// dmma_bench.cu -- latency / throughput of the FP64 tensor-core MMA shapes on sm_100a, as a
// function of warps per SM and independent accumulators per warp (guides the tiling of
// k_leaf / k_tree).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_bench dmma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC>
__global__ void k884(double* out, int iters, long long* cyc) {
  double a = threadIdx.x * 1e-9 + 1.0, b = 0.5;
  double d[ACC][2];
#pragma unroll
  for (int k = 0; k < ACC; ++k) { d[k][0] = 0; d[k][1] = 0; }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ACC; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[k][0]), "+d"(d[k][1]) : "d"(a), "d"(b));
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < ACC; ++k) s += d[k][0] + d[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int ACC>
__global__ void k1684(double* out, int iters, long long* cyc) {
  double a0 = threadIdx.x * 1e-9 + 1.0, a1 = 0.25, b = 0.5;
  double d[ACC][4];
#pragma unroll
  for (int k = 0; k < ACC; ++k) { d[k][0] = 0; d[k][1] = 0; d[k][2] = 0; d[k][3] = 0; }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ACC; ++k)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(d[k][0]), "+d"(d[k][1]), "+d"(d[k][2]), "+d"(d[k][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < ACC; ++k) s += d[k][0] + d[k][1] + d[k][2] + d[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int ACC>
__global__ void k1688(double* out, int iters, long long* cyc) {
  double a0 = threadIdx.x * 1e-9 + 1.0, a1 = 0.25, a2 = 0.125, a3 = 0.0625, b0 = 0.5, b1 = 0.75;
  double d[ACC][4];
#pragma unroll
  for (int k = 0; k < ACC; ++k) { d[k][0] = 0; d[k][1] = 0; d[k][2] = 0; d[k][3] = 0; }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ACC; ++k)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(d[k][0]), "+d"(d[k][1]), "+d"(d[k][2]), "+d"(d[k][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < ACC; ++k) s += d[k][0] + d[k][1] + d[k][2] + d[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int ACC>
__global__ void k16816(double* out, int iters, long long* cyc) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + 0.125 * i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 0.5 + 0.25 * i;
  double d[ACC][4];
#pragma unroll
  for (int k = 0; k < ACC; ++k) { d[k][0] = 0; d[k][1] = 0; d[k][2] = 0; d[k][3] = 0; }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ACC; ++k)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(d[k][0]), "+d"(d[k][1]), "+d"(d[k][2]), "+d"(d[k][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < ACC; ++k) s += d[k][0] + d[k][1] + d[k][2] + d[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void kshfl(double* out, int iters, long long* cyc) {
  double v = threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __shfl_sync(0xffffffffu, v, (threadIdx.x + 1) & 31) + 1.0;
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void klds(double* out, int iters, long long* cyc) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = (int)s[p];
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = p;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void kbar(double* out, int iters, long long* cyc) {
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename K>
static double run(K kern, int warps, int iters, double* out, long long* cyc, int nsm) {
  kern<<<nsm, warps * 32>>>(out, 10, cyc);
  kern<<<nsm, warps * 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  return (double)h / iters;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 1 << 16);
  const int it = 2000;
  printf("# cycles per loop iteration (per warp); flops/clk/SM = shape_flops*ACC*warps / cycles\n");
  int ws[] = {1, 2, 4, 8, 10, 16};
  for (int w : ws) {
    double c1 = run(k884<1>, w, it, out, cyc, nsm), c4 = run(k884<4>, w, it, out, cyc, nsm),
           c8 = run(k884<8>, w, it, out, cyc, nsm), c16 = run(k884<16>, w, it, out, cyc, nsm);
    printf("m8n8k4  warps %2d: acc1 %.1f (lat) acc4 %.1f acc8 %.1f acc16 %.1f | flop/clk/SM acc8 %.1f acc16 %.1f\n",
           w, c1, c4, c8, c16, 512.0 * 8 * w / c8, 512.0 * 16 * w / c16);
  }
  for (int w : ws) {
    double c1 = run(k1684<1>, w, it, out, cyc, nsm), c4 = run(k1684<4>, w, it, out, cyc, nsm),
           c8 = run(k1684<8>, w, it, out, cyc, nsm);
    printf("m16n8k4 warps %2d: acc1 %.1f (lat) acc4 %.1f acc8 %.1f | flop/clk/SM acc4 %.1f acc8 %.1f\n",
           w, c1, c4, c8, 1024.0 * 4 * w / c4, 1024.0 * 8 * w / c8);
  }
  for (int w : ws) {
    double c1 = run(k1688<1>, w, it, out, cyc, nsm), c4 = run(k1688<4>, w, it, out, cyc, nsm),
           c8 = run(k1688<8>, w, it, out, cyc, nsm);
    printf("m16n8k8 warps %2d: acc1 %.1f (lat) acc4 %.1f acc8 %.1f | flop/clk/SM acc4 %.1f acc8 %.1f\n",
           w, c1, c4, c8, 2048.0 * 4 * w / c4, 2048.0 * 8 * w / c8);
  }
  for (int w : ws) {
    double c1 = run(k16816<1>, w, it, out, cyc, nsm), c2 = run(k16816<2>, w, it, out, cyc, nsm),
           c4 = run(k16816<4>, w, it, out, cyc, nsm);
    printf("m16n8k16 warps %2d: acc1 %.1f (lat) acc2 %.1f acc4 %.1f | flop/clk/SM acc1 %.1f acc2 %.1f acc4 %.1f\n",
           w, c1, c2, c4, 4096.0 * w / c1, 4096.0 * 2 * w / c2, 4096.0 * 4 * w / c4);
  }
  printf("shfl f64 dependent latency: %.1f cycles\n", run(kshfl, 1, it, out, cyc, nsm));
  printf("lds f64 dependent latency: %.1f cycles\n", run(klds, 1, it, out, cyc, nsm));
  for (int w : ws) printf("__syncthreads %2d warps: %.1f cycles\n", w, run(kbar, w, it, out, cyc, nsm));
  return 0;
}
