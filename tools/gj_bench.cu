// Latency of the 4-warp Gauss-Jordan inverse of a 32x32 block (k_leaf.cuh quad_gj_inv32), alone
// and next to DMMA-heavy warps (the LU's concurrent trailing update).  usage: gj_bench
#include <cstdio>
#include <cuda_runtime.h>
#define LEAF_MAX 128
#define LDA_LEAF 132
#define GJ_WARPS 4
struct DevStatus { int code; int where; };
__device__ __forceinline__ void latch_status(DevStatus* st, int code, int where) { if (st) atomicCAS(&st->code, 0, code); }
#define FDE_ESINGULAR 3
__device__ __forceinline__ double fast_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__device__ __noinline__ void quad_gj_inv32(double* D, int ld, double* buf, DevStatus* st, int where) {
  const int w = threadIdx.x >> 5, r = threadIdx.x & 31;
  double col[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) col[c] = D[r + (8 * w + c) * ld];
  bool bad = false;
#pragma unroll 1
  for (int kb8 = 0; kb8 < 4; ++kb8) {
#pragma unroll
    for (int k8 = 0; k8 < 8; ++k8) {
      const int kk = 8 * kb8 + k8;
      double* pr = buf + (k8 & 1) * 64;
      if (w == kb8) pr[32 + r] = col[k8];
      if (r == kk) {
        double2* pv = reinterpret_cast<double2*>(pr + 8 * w);
#pragma unroll
        for (int c = 0; c < 4; ++c) pv[c] = make_double2(col[2 * c], col[2 * c + 1]);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(GJ_WARPS * 32) : "memory");
      const double piv = pr[kk];
      bad |= !(isfinite(piv) && piv != 0.0);
      const double rp = fast_rcp(piv);
      const double f = pr[32 + r] * rp;
      const bool me = r == kk;
      const double2* pv = reinterpret_cast<const double2*>(pr + 8 * w);
#pragma unroll
      for (int c2 = 0; c2 < 4; ++c2) {
        const double2 q = pv[c2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = 2 * c2 + h;
          const double p = h ? q.y : q.x;
          if (w == kb8 && c == k8) col[c] = me ? rp : -f;
          else col[c] = me ? p * rp : fma(-f, p, col[c]);
        }
      }
    }
  }
  if (bad && threadIdx.x == 0) latch_status(st, FDE_ESINGULAR, where);
#pragma unroll
  for (int c = 0; c < 8; ++c) D[r + (8 * w + c) * ld] = col[c];
}

// 2-warp variant: lane r of warp w (0..1) owns A[r, 16w .. 16w+15]; named barrier 1 over 64 threads
__device__ __noinline__ void duo_gj_inv32(double* D, int ld, double* buf) {
  const int w = threadIdx.x >> 5, r = threadIdx.x & 31;
  double col[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) col[c] = D[r + (16 * w + c) * ld];
#pragma unroll 1
  for (int kb = 0; kb < 2; ++kb) {
#pragma unroll
    for (int k16 = 0; k16 < 16; ++k16) {
      const int kk = 16 * kb + k16;
      double* pr = buf + (k16 & 1) * 64;
      if (w == kb) pr[32 + r] = col[k16];
      if (r == kk) {
        double2* pv = reinterpret_cast<double2*>(pr + 16 * w);
#pragma unroll
        for (int c = 0; c < 8; ++c) pv[c] = make_double2(col[2 * c], col[2 * c + 1]);
      }
      asm volatile("bar.sync 1, 64;" ::: "memory");
      const double piv = pr[kk];
      const double rp = fast_rcp(piv);
      const double f = pr[32 + r] * rp;
      const bool me = r == kk;
      const double2* pv = reinterpret_cast<const double2*>(pr + 16 * w);
#pragma unroll
      for (int c2 = 0; c2 < 8; ++c2) {
        const double2 q = pv[c2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = 2 * c2 + h;
          const double p = h ? q.y : q.x;
          if (w == kb && c == k16) col[c] = me ? rp : -f;
          else col[c] = me ? p * rp : fma(-f, p, col[c]);
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < 16; ++c) D[r + (16 * w + c) * ld] = col[c];
}

template <int MODE>   // 0: GJ alone (warps 4-7 idle), 1: warps 4-7 run DMMA chains meanwhile
__global__ void __launch_bounds__(256, 1) k_gj(int reps, unsigned long long* cyc, double* out) {
  __shared__ double A[32 * 33 + 8], buf[256], B[64 * 33];
  __shared__ volatile int stop;
  const int t = threadIdx.x, warp = t >> 5;
  for (int e = t; e < 32 * 32; e += 256) { const int i = e % 32, j = e / 32; A[i + j * 33] = (i == j) ? 40.0 : 1.0 / (1 + i + 2 * j); }
  for (int e = t; e < 64 * 33; e += 256) B[e] = 0.001 * e;
  if (t == 0) stop = 0;
  __syncthreads();
  const bool gj = MODE <= 1 ? warp < GJ_WARPS : warp < 2;                 // modes 2/3: 2-warp GJ
  const bool dm = MODE == 1 ? warp >= GJ_WARPS : MODE == 3 ? (warp & 3) >= 2 : false;   // DMMA warps
  if (gj) {
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) { if (MODE <= 1) quad_gj_inv32(A, 33, buf, nullptr, 0); else duo_gj_inv32(A, 33, buf); }
    const long long t1 = clock64();
    if (t == 0) { cyc[blockIdx.x] = t1 - t0; stop = 1; }
  } else if (dm) {
    const int lane = t & 31, gid = lane >> 2, tig = lane & 3;
    double acc[12][2] = {};
    while (!stop) {
#pragma unroll
      for (int k4 = 0; k4 < 8; ++k4) {
        const double b = B[4 * k4 + tig + gid * 33];
#pragma unroll
        for (int u = 0; u < 12; ++u) dmma884(acc[u][0], acc[u][1], B[(u * 8 + gid) % 64 + (4 * k4 + tig) * 33 % 2000], b);
      }
    }
    double s = 0; for (int u = 0; u < 12; ++u) s += acc[u][0] + acc[u][1];
    if (s == 12345.0) out[0] = s;
  }
  __syncthreads();
  if (t < 32) out[1 + t] = A[t];
}

int main() {
  unsigned long long* cyc; double* out;
  cudaMalloc(&cyc, 148 * 8); cudaMalloc(&out, 64 * 8);
  const int reps = 64;
  for (int mode = 0; mode < 4; ++mode) {
    for (int it = 0; it < 2; ++it) {
      if (mode == 0) k_gj<0><<<148, 256>>>(reps, cyc, out);
      else if (mode == 1) k_gj<1><<<148, 256>>>(reps, cyc, out);
      else if (mode == 2) k_gj<2><<<148, 256>>>(reps, cyc, out);
      else k_gj<3><<<148, 256>>>(reps, cyc, out);
      cudaDeviceSynchronize();
    }
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double a = 0; for (int i = 0; i < 148; ++i) a += h[i]; a /= 148;
    printf("mode %d (%s): %.0f cycles per 32x32 GJ = %.1f cycles per pivot [%s]\n", mode,
           mode == 0 ? "quad alone" : mode == 1 ? "quad + 4 DMMA warps (same SMSPs)" : mode == 2 ? "duo alone" : "duo + 4 DMMA warps on SMSPs 2,3", a / reps, a / reps / 32, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
