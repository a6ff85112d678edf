// k_pgmres.cuh -- SURVEY §8(f) NEXT-3: the paper's 1D comparison method:
// GMRES, left-preconditioned by the tridiagonal structure-preserving preconditioners P1 / P2 of
// [DMS] -- A_m with T_{alpha,N} replaced by the first- (alpha = 1) or second-order (alpha = 2)
// Grunwald-Letnikov matrix, i.e.
//   P1 = I + c (D+ T_1 + D- T_1^T),  T_1 = I - (superdiagonal)          (bidiagonal, g^(1) = [1, -1])
//   P2 = I + c (D+ + D-) tridiag(-1, 2, -1)                              (T_2 symmetric)
// -- on the exact operator applied matrix-free: A_m u = u + c (D+ T u + D- T^T u), T u and T^T u by
// circulant embedding of size M = 2^ceil(log2 2n) and FFTs.
//   * FFT: four-step, M = M1 M2 (both <= 1024): k_fft_cols (M1 interleaved FFTs of size M2, times
//     the twiddles w_M^{j1 k2}) then k_fft_rows (M2 FFTs of size M1); radix-2 in shared memory.
//   * tridiagonal solves: partitioned Thomas (SPIKE): blocks of TD_M rows solved independently
//     with their two coupling spikes, a reduced 2x2-block tridiagonal system for the block ends
//     (one thread, block Thomas), reconstruction; no pivoting (P1, P2 strictly diagonally dominant).
//   * GMRES: full (no restart), classical Gram-Schmidt twice, Givens rotations on the device.
#pragma once
#include "fde_common.cuh"

// ---- FFT ----------------------------------------------------------------------------------
#define FFT_T 256

// In-place radix-2 FFT (decimation in time) of `cnt` interleaved sequences of length P held in
// shared memory as s[q * P + i] (double2), sign = -1 forward / +1 inverse (unscaled).  tw: the P/2
// twiddles exp(sign 2 pi i k / P) in shared memory (built by the caller).
__device__ void smem_fft(double2* s, const double2* tw, int P, int lgP, int cnt) {
  const int t = threadIdx.x;
  for (int e = t; e < cnt * P; e += FFT_T) {          // bit reversal
    const int q = e / P, i = e - q * P;
    const int r = __brev(i) >> (32 - lgP);
    if (i < r) { double2* a = s + q * P; const double2 x = a[i]; a[i] = a[r]; a[r] = x; }
  }
  __syncthreads();
  for (int len = 2, lgl = 1; len <= P; len <<= 1, ++lgl) {
    const int half = len >> 1;
    for (int e = t; e < cnt * (P >> 1); e += FFT_T) {
      const int q = e / (P >> 1), b = e - q * (P >> 1);
      const int grp = b >> (lgl - 1), k = b & (half - 1);
      const int i0 = grp * len + k, i1 = i0 + half;
      const double2 w0 = tw[k << (lgP - lgl)];
      double2* a = s + q * P;
      const double2 u = a[i0], v = a[i1];
      const double2 w = make_double2(w0.x * v.x - w0.y * v.y, w0.x * v.y + w0.y * v.x);
      a[i0] = make_double2(u.x + w.x, u.y + w.y);
      a[i1] = make_double2(u.x - w.x, u.y - w.y);
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void build_twiddles(double2* tw, int P, double sign) {
  for (int k = threadIdx.x; k < P / 2; k += FFT_T) {
    double sn, cs;
    sincospi(sign * 2.0 * k / P, &sn, &cs);
    tw[k] = make_double2(cs, sn);
  }
}

#define FFT_G 8                   // sequences per CTA (coalesced 128-byte rows of double2)
// Step 1: Y[k2 * M1 + j1] = w_M^{j1 k2} sum_{j2} x[j1 + M1 j2] w_M2^{j2 k2}   (j1 in this CTA's group)
__global__ void __launch_bounds__(FFT_T)
k_fft_cols(const double2* __restrict__ x, double2* __restrict__ Y, int M1, int M2, int lgM2, double sign) {
  extern __shared__ double2 fs[];
  double2* tw = fs + FFT_G * M2;
  const int j10 = blockIdx.x * FFT_G;
  build_twiddles(tw, M2, sign);
  for (int e = threadIdx.x; e < FFT_G * M2; e += FFT_T) {
    const int g = e % FFT_G, j2 = e / FFT_G;
    fs[g * M2 + j2] = x[(long long)j2 * M1 + j10 + g];
  }
  __syncthreads();
  smem_fft(fs, tw, M2, lgM2, FFT_G);
  const long long M = (long long)M1 * M2;
  for (int e = threadIdx.x; e < FFT_G * M2; e += FFT_T) {
    const int g = e % FFT_G, k2 = e / FFT_G, j1 = j10 + g;
    double sn, cs;
    sincospi(sign * 2.0 * (double)(((long long)j1 * k2) % M) / (double)M, &sn, &cs);
    const double2 v = fs[g * M2 + k2];
    Y[(long long)k2 * M1 + j1] = make_double2(cs * v.x - sn * v.y, cs * v.y + sn * v.x);
  }
}

// Step 2: X[k2 + M2 k1] = scale * sum_{j1} Y[k2 * M1 + j1] w_M1^{j1 k1}   (k2 in this CTA's group)
__global__ void __launch_bounds__(FFT_T)
k_fft_rows(const double2* __restrict__ Y, double2* __restrict__ X, int M1, int lgM1, int M2, double sign,
           double scale) {
  extern __shared__ double2 fs[];
  double2* tw = fs + FFT_G * M1;
  const int k20 = blockIdx.x * FFT_G;
  build_twiddles(tw, M1, sign);
  for (int e = threadIdx.x; e < FFT_G * M1; e += FFT_T) {
    const int g = e / M1, j1 = e - g * M1;
    fs[g * M1 + j1] = Y[(long long)(k20 + g) * M1 + j1];
  }
  __syncthreads();
  smem_fft(fs, tw, M1, lgM1, FFT_G);
  for (int e = threadIdx.x; e < FFT_G * M1; e += FFT_T) {
    const int g = e % FFT_G, k1 = e / FFT_G;
    const double2 v = fs[g * M1 + k1];
    X[(long long)k1 * M2 + k20 + g] = make_double2(scale * v.x, scale * v.y);
  }
}

// circulant embedding columns of T and T^T (size M, real -> complex):  c_T = [t_0..t_{n-1}, 0.., r_{n-1}..r_1]
// with t_i = T[i, 0] = -g_{i+1}, r_j = T[0, j] = -g_{1-j} (r_0 = -g_1, r_1 = -g_0, r_j = 0 for j >= 2)
__global__ void k_embed_T(const double* __restrict__ g, int n, long long M, double2* __restrict__ cT,
                          double2* __restrict__ cTt) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  double a = 0.0, b = 0.0;                            // a: column of T, b: column of T^T
  if (i < n) { a = -g[i + 1]; b = i == 0 ? -g[1] : (i == 1 ? -g[0] : 0.0); }
  else if (i > M - n) {                               // j = M - i in 1..n-1: first-row tail
    const long long j = M - i;
    a = j == 1 ? -g[0] : 0.0;
    b = -g[j + 1];
  }
  cT[i] = make_double2(a, 0.0);
  cTt[i] = make_double2(b, 0.0);
}

__global__ void k_pad_complex(const double* __restrict__ x, int n, long long M, double2* __restrict__ z) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < M) z[i] = make_double2(i < n ? x[i] : 0.0, 0.0);
}

// z1 = s1 * z, z2 = s2 * z (complex products)
__global__ void k_spec_mul(const double2* __restrict__ z, const double2* __restrict__ s1, const double2* __restrict__ s2,
                           long long M, double2* __restrict__ z1, double2* __restrict__ z2) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  const double2 a = z[i], p = s1[i], q = s2[i];
  z1[i] = make_double2(a.x * p.x - a.y * p.y, a.x * p.y + a.y * p.x);
  z2[i] = make_double2(a.x * q.x - a.y * q.y, a.x * q.y + a.y * q.x);
}

// y = x + c (d+ Re(y1) + d- Re(y2))   (A_m u, Eq. 2.5)
__global__ void k_apply_combine(int n, const double* __restrict__ x, const double2* __restrict__ y1,
                                const double2* __restrict__ y2, const double* __restrict__ dp,
                                const double* __restrict__ dm, double c, double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[i] + c * (dp[i] * y1[i].x + dm[i] * y2[i].x);
}

// ---- tridiagonal preconditioner (partitioned Thomas / SPIKE) ------------------------------
#define TD_M 256                  // rows per block
// P row i: lo_i x_{i-1} + di_i x_i + up_i x_{i+1}
__global__ void k_prec_coeffs(int n, int kind, double c, const double* __restrict__ dp, const double* __restrict__ dm,
                              double* __restrict__ lo, double* __restrict__ di, double* __restrict__ up) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (kind == 1) {                // T_1 = I - superdiag: D+ T_1 + D- T_1^T -> lo -d-, di d+ + d-, up -d+
    lo[i] = i > 0 ? -c * dm[i] : 0.0;
    di[i] = 1.0 + c * (dp[i] + dm[i]);
    up[i] = i + 1 < n ? -c * dp[i] : 0.0;
  } else {                        // T_2 = tridiag(-1, 2, -1)
    const double s = c * (dp[i] + dm[i]);
    lo[i] = i > 0 ? -s : 0.0;
    di[i] = 1.0 + 2.0 * s;
    up[i] = i + 1 < n ? -s : 0.0;
  }
}

// Factor each block (Thomas, no pivoting) and its spikes: v = T_k^{-1} (lo_s e_first), w = T_k^{-1}
// (up_{e-1} e_last).  cp[i] = modified superdiagonal, dd[i] = 1 / modified diagonal.
__global__ void k_td_block_setup(int n, const double* __restrict__ lo, const double* __restrict__ di,
                                 const double* __restrict__ up, double* __restrict__ cp, double* __restrict__ dd,
                                 double* __restrict__ v, double* __restrict__ w) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = k * TD_M, e = min(n, s + TD_M);
  if (s >= n) return;
  // forward elimination (LU of the block: L unit lower with multipliers lo_i dd_{i-1})
  double prev_c = 0.0;
  for (int i = s; i < e; ++i) {
    const double l = i > s ? lo[i] : 0.0;
    const double d = di[i] - l * prev_c;
    dd[i] = 1.0 / d;
    cp[i] = (i + 1 < e ? up[i] : 0.0) * dd[i];
    prev_c = cp[i];
  }
  // spikes: solve T_k v = lo_s e_1 and T_k w = up_{e-1} e_m
  double fv = 0.0, fw = 0.0;
  for (int i = s; i < e; ++i) {
    const double l = i > s ? lo[i] : 0.0;
    const double rv = (i == s ? lo[s] : 0.0) - l * fv;
    const double rw = (i == e - 1 ? up[e - 1] : 0.0) - l * fw;
    fv = rv * dd[i]; fw = rw * dd[i];
    v[i] = fv; w[i] = fw;
  }
  for (int i = e - 2; i >= s; --i) { v[i] -= cp[i] * v[i + 1]; w[i] -= cp[i] * w[i + 1]; }
}

// y = T_k^{-1} r per block (same factors)
__global__ void k_td_block_solve(int n, const double* __restrict__ lo, const double* __restrict__ cp,
                                 const double* __restrict__ dd, const double* __restrict__ r, double* __restrict__ y) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = k * TD_M, e = min(n, s + TD_M);
  if (s >= n) return;
  double f = 0.0;
  for (int i = s; i < e; ++i) { const double l = i > s ? lo[i] : 0.0; f = (r[i] - l * f) * dd[i]; y[i] = f; }
  for (int i = e - 2; i >= s; --i) y[i] -= cp[i] * y[i + 1];
}

// Reduced system for the block-end unknowns (one thread): with a_k = x_{s_k} (first), b_k = x_{e_k-1}
// (last):  a_k + v_{s} b_{k-1} + w_{s} a_{k+1} = y_{s},   b_k + v_{e-1} b_{k-1} + w_{e-1} a_{k+1} = y_{e-1}.
// Unknown pairs z_k = (b_{k-1}?)...  solved in the ordering u_k = (a_k, b_k) as a block-tridiagonal
// system  E_k u_{k-1} + I u_k + F_k u_{k+1} = (y_s, y_{e-1})  with E_k = [[0, v_s], [0, v_{e-1}]],
// F_k = [[w_s, 0], [w_{e-1}, 0]] -- block Thomas with 2x2 blocks (SDD: no pivoting).
__global__ void k_td_reduced(int n, int nb, const double* __restrict__ v, const double* __restrict__ w,
                             const double* __restrict__ y, double* __restrict__ ab, double* __restrict__ work) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  // work: per block: G (2x2 inverse of the modified diagonal block) and modified rhs / F
  double* Fm = work;                  // [nb][4] modified F_k (= D_k^{-1} F_k)
  double* rm = work + 4 * nb;         // [nb][2] modified rhs
  double Fp[4] = {0, 0, 0, 0};        // previous modified F
  double rp[2] = {0, 0};
  for (int k = 0; k < nb; ++k) {
    const int s = k * TD_M, e = min(n, s + TD_M);
    const double E01 = k > 0 ? v[s] : 0.0, E11 = k > 0 ? v[e - 1] : 0.0;   // E = [[0, E01], [0, E11]]
    // D = I - E Fp,  r = y - E rp
    const double D00 = 1.0 - E01 * Fp[2], D01 = -E01 * Fp[3];
    const double D10 = -E11 * Fp[2], D11 = 1.0 - E11 * Fp[3];
    const double r0 = y[s] - E01 * rp[1], r1 = y[e - 1] - E11 * rp[1];
    const double det = D00 * D11 - D01 * D10, id = 1.0 / det;
    const double I00 = D11 * id, I01 = -D01 * id, I10 = -D10 * id, I11 = D00 * id;
    const double F00 = k + 1 < nb ? w[s] : 0.0, F10 = k + 1 < nb ? w[e - 1] : 0.0;   // F = [[F00, 0], [F10, 0]]
    Fp[0] = I00 * F00 + I01 * F10; Fp[1] = 0.0; Fp[2] = I10 * F00 + I11 * F10; Fp[3] = 0.0;
    rp[0] = I00 * r0 + I01 * r1; rp[1] = I10 * r0 + I11 * r1;
    for (int q = 0; q < 4; ++q) Fm[4 * k + q] = Fp[q];
    rm[2 * k] = rp[0]; rm[2 * k + 1] = rp[1];
  }
  double un[2] = {0, 0};
  for (int k = nb - 1; k >= 0; --k) {
    const double u0 = rm[2 * k] - Fm[4 * k] * un[0], u1 = rm[2 * k + 1] - Fm[4 * k + 2] * un[0];
    ab[2 * k] = u0; ab[2 * k + 1] = u1;
    un[0] = u0; un[1] = u1;
  }
}

// x_i = y_i - v_i b_{k-1} - w_i a_{k+1}
__global__ void k_td_reconstruct(int n, int nb, const double* __restrict__ y, const double* __restrict__ v,
                                 const double* __restrict__ w, const double* __restrict__ ab, double* __restrict__ x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int k = i / TD_M;
  const double bprev = k > 0 ? ab[2 * (k - 1) + 1] : 0.0, anext = k + 1 < nb ? ab[2 * (k + 1)] : 0.0;
  x[i] = y[i] - v[i] * bprev - w[i] * anext;
}

// ---- GMRES helpers ------------------------------------------------------------------------
#define GM_T 256
// h[j] = V[:, j]^T w for j < k (partials per CTA: P[blockIdx.x][j]); fixed order
__global__ void __launch_bounds__(GM_T)
k_gm_dots(int n, int k, const double* __restrict__ V, const double* __restrict__ w, double* __restrict__ P) {
  __shared__ double red[GM_T / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int chunk = (n + gridDim.x - 1) / gridDim.x, i0 = blockIdx.x * chunk, i1 = min(n, i0 + chunk);
  for (int j = 0; j < k; ++j) {
    double a = 0.0;
    for (int i = i0 + t; i < i1; i += GM_T) a = fma(V[(long long)j * n + i], w[i], a);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) red[warp] = a;
    __syncthreads();
    if (t == 0) { double s = 0.0; for (int q = 0; q < GM_T / 32; ++q) s += red[q]; P[(long long)blockIdx.x * 128 + j] = s; }
    __syncthreads();
  }
}
__global__ void k_gm_sum(int k, int nparts, const double* __restrict__ P, double* __restrict__ h) {
  const int j = threadIdx.x;
  if (j >= k) return;
  double s = 0.0;
  for (int q = 0; q < nparts; ++q) s += P[(long long)q * 128 + j];
  h[j] = s;
}
// w -= V[:, 0:k] h
__global__ void k_gm_axpy(int n, int k, const double* __restrict__ V, const double* __restrict__ h, double* __restrict__ w) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double a = w[i];
  for (int j = 0; j < k; ++j) a = fma(-V[(long long)j * n + i], h[j], a);
  w[i] = a;
}
__global__ void k_gm_scale(int n, const double* __restrict__ w, const double* __restrict__ nrm, double* __restrict__ v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = w[i] / nrm[0];
}
// Hessenberg column j (H[0..j+1], ld 128) -> apply previous Givens, new rotation, residual g;
// out[0] = |g_{j+1}|.  cs/sn/g stored in gs (3 x 128).  (one thread)
__global__ void k_gm_givens(int j, double* __restrict__ Hcol, double* __restrict__ gs, double* __restrict__ out) {
  double* cs = gs; double* sn = gs + 128; double* g = gs + 256;
  for (int i = 0; i < j; ++i) {
    const double a = Hcol[i], b = Hcol[i + 1];
    Hcol[i] = cs[i] * a + sn[i] * b;
    Hcol[i + 1] = -sn[i] * a + cs[i] * b;
  }
  const double a = Hcol[j], b = Hcol[j + 1];
  const double r = hypot(a, b);
  cs[j] = r > 0.0 ? a / r : 1.0; sn[j] = r > 0.0 ? b / r : 0.0;
  Hcol[j] = r; Hcol[j + 1] = 0.0;
  g[j + 1] = -sn[j] * g[j];
  g[j] = cs[j] * g[j];
  out[0] = fabs(g[j + 1]);
}
// y = R^{-1} g (k x k upper triangular R = H[0:k, 0:k], ld 128) (one thread)
__global__ void k_gm_backsolve(int k, const double* __restrict__ H, const double* __restrict__ gs, double* __restrict__ y) {
  const double* g = gs + 256;
  for (int i = k - 1; i >= 0; --i) {
    double a = g[i];
    for (int j = i + 1; j < k; ++j) a -= H[(long long)j * 128 + i] * y[j];
    y[i] = a / H[(long long)i * 128 + i];
  }
}
__global__ void k_gm_setg(double* __restrict__ gs, const double* __restrict__ beta) {
  for (int i = 0; i < 128; ++i) gs[256 + i] = 0.0;
  gs[256] = beta[0];
}

__global__ void k_sqrt1(double* v) { v[0] = sqrt(v[0]); }
// H[j] += h[j] (j < k)
__global__ void k_add_vec(int k, const double* __restrict__ h, double* __restrict__ H) {
  const int j = threadIdx.x;
  if (j < k) H[j] += h[j];
}
// x += V[:, 0:k] y
__global__ void k_gm_axpy_neg(int n, int k, const double* __restrict__ V, const double* __restrict__ y, double* __restrict__ x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double a = x[i];
  for (int j = 0; j < k; ++j) a = fma(V[(long long)j * n + i], y[j], a);
  x[i] = a;
}
