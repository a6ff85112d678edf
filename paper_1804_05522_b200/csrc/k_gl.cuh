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

// Multi-CTA variant for long weight vectors (the handle's S1): the factors j = 1..nk-1 are cut
// into segments of GLS_SEG, one CTA each.  k_gl_seg writes every segment's product; k_gl_expand
// joins the products of the preceding segments (fixed order), runs the block-wide exclusive
// product scan of the per-thread chunks and re-expands.  Rounding grows like
// (GLS_CH + log2 GLS_THREADS + log2 segments) ulps.
#define GLS_THREADS 256
#define GLS_CH 4
#define GLS_SEG (GLS_THREADS * GLS_CH)

__device__ __forceinline__ double gl_chunk_prod(double a, int j0, int j1) {
  double p = 1.0;
  for (int j = j0; j < j1; ++j) p *= ((double)(j - 1) - a) / (double)j;
  return p;
}

// grid (segments, batch): seg[inst * nseg + b] = product of the factors of segment b
__global__ void __launch_bounds__(GLS_THREADS)
k_gl_seg(const double* __restrict__ alpha, int nk, double* __restrict__ seg) {
  const int b = blockIdx.x, inst = blockIdx.y, t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int nf = nk - 1;
  const int j0 = 1 + b * GLS_SEG + t * GLS_CH, j1 = min(nf + 1, j0 + GLS_CH);
  double p = gl_chunk_prod(alpha[inst], j0, j1);
  __shared__ double wp[GLS_THREADS / 32];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {                     // fixed-order tree
    const double v = __shfl_down_sync(0xffffffffu, p, o);
    if ((lane & (2 * o - 1)) == 0) p *= v;
  }
  if (lane == 0) wp[w] = p;
  __syncthreads();
  if (t == 0) {
    double q = 1.0;
    for (int i = 0; i < GLS_THREADS / 32; ++i) q *= wp[i];
    seg[(long long)inst * gridDim.x + b] = q;
  }
}

// grid (segments, batch): g[inst*gstride + k], k = 0..nk-1
__global__ void __launch_bounds__(GLS_THREADS)
k_gl_expand(const double* __restrict__ alpha, int nk, const double* __restrict__ seg,
            double* __restrict__ g, long long gstride) {
  const int b = blockIdx.x, inst = blockIdx.y, t = threadIdx.x, lane = t & 31, w = t >> 5;
  const double a = alpha[inst];
  double* gi = g + (long long)inst * gstride;
  const int nf = nk - 1;
  const int j0 = 1 + b * GLS_SEG + t * GLS_CH, j1 = min(nf + 1, j0 + GLS_CH);
  __shared__ double warp_tot[GLS_THREADS / 32];
  __shared__ double s_pre;
  if (w == 0) {                                           // product of segments 0..b-1
    const double* sg = seg + (long long)inst * gridDim.x;
    double q = 1.0;
    for (int i = lane; i < b; i += 32) q *= sg[i];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double v = __shfl_down_sync(0xffffffffu, q, o);
      if ((lane & (2 * o - 1)) == 0) q *= v;
    }
    if (lane == 0) s_pre = q;
  }
  const double p = gl_chunk_prod(a, j0, j1);
  double incl = p;                                        // block-wide inclusive product scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl = v * incl;
  }
  if (lane == 31) warp_tot[w] = incl;
  __syncthreads();
  if (w == 0) {
    double v = (lane < GLS_THREADS / 32) ? warp_tot[lane] : 1.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v = u * v;
    }
    if (lane < GLS_THREADS / 32) warp_tot[lane] = v;
  }
  __syncthreads();
  double excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = 1.0;
  if (w > 0) excl = warp_tot[w - 1] * excl;
  if (b == 0 && t == 0) gi[0] = 1.0;
  double v = s_pre * excl;
  for (int j = j0; j < j1; ++j) {
    v *= ((double)(j - 1) - a) / (double)j;
    gi[j] = v;                                             // g_j
  }
}
