// Verify the mma.sync m8n8k4 f64 fragment layout assumed by csrc/fde_dmma.cuh:
//   gid = lane >> 2, tig = lane & 3
//   A (8x4, row-major): a = A[gid][tig]
//   B (4x8):            b = B[tig][gid]
//   C/D (8x8):          c0 = C[gid][2*tig], c1 = C[gid][2*tig+1]
#include <cstdio>
#include <cmath>
__global__ void k(const double* A, const double* B, double* C) {
  int lane = threadIdx.x, gid = lane >> 2, tig = lane & 3;
  double a = A[gid * 4 + tig], b = B[tig * 8 + gid];
  double c0 = 0, c1 = 0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  C[gid * 8 + 2 * tig] = c0;
  C[gid * 8 + 2 * tig + 1] = c1;
}
int main() {
  double hA[32], hB[32], hC[64], ref[64];
  for (int i = 0; i < 32; ++i) { hA[i] = 1 + i * 0.37; hB[i] = 2 - i * 0.11; }
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      double s = 0;
      for (int q = 0; q < 4; ++q) s += hA[i * 4 + q] * hB[q * 8 + j];
      ref[i * 8 + j] = s;
    }
  double *A, *B, *C;
  cudaMalloc(&A, 256); cudaMalloc(&B, 256); cudaMalloc(&C, 512);
  cudaMemcpy(A, hA, 256, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, 256, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(A, B, C);
  cudaMemcpy(hC, C, 512, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < 64; ++i) err = fmax(err, fabs(hC[i] - ref[i]));
  printf("{\"dmma_layout_max_err\": %g, \"ok\": %s}\n", err, err < 1e-12 ? "true" : "false");
  return err < 1e-12 ? 0 : 1;
}
