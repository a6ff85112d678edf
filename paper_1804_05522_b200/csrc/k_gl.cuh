// k_gl.cuh -- S1: Grünwald–Letnikov weights on the device.
//   g_0 = 1, g_1 = -alpha, g_{k+1} = g_k (k - alpha)/(k + 1)
// computed as a multiplicative scan g_k = prod_{j=1..k} (j-1-alpha)/j: each thread forms
// the product of a contiguous chunk of factors, a block-wide exclusive product scan joins
// the chunks, and each thread re-expands its chunk from its prefix.  Rounding grows like
// (chunk + log2 threads) ulps instead of k ulps for the sequential recursion.
#pragma once
#include "fde_common.cuh"

#define GL_THREADS 1024

// One CTA per instance.  g[inst*gstride + k] for k = 0..nk-1 (nk = n + 2).
__global__ void __launch_bounds__(GL_THREADS)
k_gl_weights(const double* __restrict__ alpha, int nk, double* __restrict__ g, long long gstride) {
  const int inst = blockIdx.x;
  const double a = alpha[inst];
  double* gi = g + (long long)inst * gstride;
  const int nf = nk - 1;                                  // factors j = 1..nk-1
  const int chunk = (nf + GL_THREADS - 1) / GL_THREADS;
  const int t = threadIdx.x;
  const int j0 = 1 + t * chunk;
  const int j1 = min(nf + 1, j0 + chunk);
  double p = 1.0;
  for (int j = j0; j < j1; ++j) p *= ((double)(j - 1) - a) / (double)j;

  // block-wide inclusive product scan (fixed order => deterministic)
  __shared__ double warp_tot[GL_THREADS / 32];
  const int lane = t & 31, w = t >> 5;
  double incl = p;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl = v * incl;
  }
  if (lane == 31) warp_tot[w] = incl;
  __syncthreads();
  if (w == 0) {
    double v = (lane < GL_THREADS / 32) ? warp_tot[lane] : 1.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      double u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v = u * v;
    }
    warp_tot[lane] = v;                                    // inclusive over warps
  }
  __syncthreads();
  double excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = 1.0;
  if (w > 0) excl = warp_tot[w - 1] * excl;
  if (t == 0) gi[0] = 1.0;
  double v = excl;
  for (int j = j0; j < j1; ++j) {
    v *= ((double)(j - 1) - a) / (double)j;
    gi[j] = v;                                             // g_j
  }
}
