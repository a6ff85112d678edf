// fdehodlr.cu -- host side of the C-ABI (include/fdehodlr.h): argument checking, tree
// bookkeeping, workspace management and kernel orchestration on the caller's stream.
// All arithmetic of the method runs in the kernels of k_*.cuh.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "fde_common.cuh"
#include "k_gl.cuh"
#include "k_compress.cuh"
#include "k_leaf.cuh"
#include "k_level.cuh"
#include "k_levels.cuh"
#include "k_matvec.cuh"
#include "k_tree.cuh"
#include "k_solve.cuh"
#include "k_step.cuh"
#include "k_run.cuh"

// ---------------------------------------------------------------------------------------
// errors, launch accounting
static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

static int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define CU(call)                                                                     \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
      return set_err(e_ == cudaErrorMemoryAllocation ? FDE_ENOMEM : FDE_ECUDA,       \
                     "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__,      \
                     __LINE__);                                                      \
  } while (0)

#define LAUNCHED()                                                                   \
  do {                                                                               \
    g_launches.fetch_add(1, std::memory_order_relaxed);                              \
    cudaError_t e_ = cudaGetLastError();                                             \
    if (e_ != cudaSuccess)                                                           \
      return set_err(FDE_ECUDA, "kernel launch: %s (%s:%d)", cudaGetErrorString(e_), \
                     __FILE__, __LINE__);                                            \
  } while (0)

// ---------------------------------------------------------------------------------------
// tracing: optional CUDA-event pair around every kernel launch (fde_profile_enable)
struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
};
static bool g_prof = false;
static std::vector<ProfRec> g_prof_recs;
static std::vector<cudaEvent_t> g_ev_free;

static cudaEvent_t prof_event() {
  if (!g_ev_free.empty()) {
    cudaEvent_t e = g_ev_free.back();
    g_ev_free.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct ProfScope {
  const char* name;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  ProfScope(const char* nm, cudaStream_t st) : name(nm), s(st) {
    if (g_prof) { a = prof_event(); cudaEventRecord(a, s); }
  }
  ~ProfScope() {
    if (g_prof) {
      cudaEvent_t b = prof_event();
      cudaEventRecord(b, s);
      g_prof_recs.push_back({name, a, b});
    }
  }
};
#define PROF(nm) ProfScope prof_scope_(nm, s)

struct fde_hodlr {
  int batch = 0, n = 0, leaf = 0, L = 0, nleaf = 0, nnodes = 0;
  double h = 0, dt = 0, shift = 1, tol = 0;
  std::vector<double> alpha;
  // tree (host)
  std::vector<int> node_r0, node_n1, node_n2, node_seg, leaf_r0, leaf_n;
  std::vector<int> seg_ofs, seg_node, seg_child, seg_row0, seg_len, lev_m;
  std::vector<long long> lev_lofs, lev_lraw;
  long long lf_stride = 0, lraw_stride = 0;
  int max_seg = 0, max_nodes_lvl = 0;
  TreeDev tree{};
  // compression plan
  std::vector<PcTask> tasks;
  std::vector<PcChunk> chunks;
  std::vector<int> launch_chunk0;   // chunk ranges of the cooperative launches
  // device memory
  std::vector<void*> allocs;
  int* d_tree_int = nullptr;
  long long* d_lev_lofs = nullptr;
  double *d_alpha = nullptr, *d_cfac = nullptr, *d_g = nullptr;
  double *d_Lf = nullptr, *d_Lraw = nullptr;
  int *d_rank = nullptr, *d_colofs = nullptr;
  double *d_dp = nullptr, *d_dm = nullptr;
  double *d_X = nullptr, *d_LU = nullptr, *d_P = nullptr;
  long long gstride = 0, xstride = 0, lustride = 0, pstride_seg = 0, pstride_inst = 0;
  long long lurstride = 0;          // stored run LUs (k_run): LEAF_RSLOT doubles per leaf
  int ncap = 0;
  // level layout (host-known after the compression): k_l = max rank over the batch + 1
  bool layout_done = false;
  std::vector<int> kl, xcol;
  std::vector<long long> kofs;
  long long kstride_inst = 0, sum_half = 0;
  int sum_nc = 0, kmax = 0, p = 0, P = 1, coop_capacity = 1;
  double *d_Kst = nullptr, *d_sums = nullptr, *d_lvpart = nullptr;
  unsigned* d_bar = nullptr;
  int* d_post = nullptr;
  // projected-tree path (k_leaf Q phase + k_tree) for the fused factor + solve step
  bool tree_ok = false;
  double *d_Q = nullptr, *d_S = nullptr;
  long long qlev[LMAX + 1] = {}, slev[LMAX] = {}, qinst = 0, sinst = 0;
  int trc[LMAX] = {};
  int tr_grid = 0;
  TrArgs tr_geo{};
  size_t tr_smem = 0;
  int* d_done = nullptr;            // k_step task counter + completion counters
  long long dofs[LMAX + 1] = {}, ndone = 0, lofs = 0;
  bool compress_only = false;       // built with FDE_COMPRESS_ONLY (hodlr_ranks only)
  int step_grid = 0;
  size_t step_smem = 0;
  // pipelined multi-step run (k_run.cuh): second buffer set and stored leaf LUs
  double *d_X2 = nullptr, *d_Q2 = nullptr, *d_S2 = nullptr, *d_LUr[2] = {nullptr, nullptr};
  int* d_runctr = nullptr;
  long long runctr_cap = 0;
  unsigned long long* d_runrq = nullptr;
  long long runrq_cap = 0;
  std::vector<LeafArgs> run_las;
  std::vector<TrArgs> run_tas;
  void* d_run_args = nullptr;
  size_t run_args_cap = 0;
  int npost = 0;
  // compression scratch
  PcTask* d_tasks = nullptr;
  PcChunk* d_chunks = nullptr;
  unsigned* d_ctr = nullptr;
  double* d_glseg = nullptr;            // S1 segment products (k_gl_seg)
  double* d_Kr[2] = {nullptr, nullptr}; // k_run split units: node stores [C | Sc^-1 | G] (2 parities)
  long long krlev[LMAX] = {}, krinst = 0;
  double *d_part = nullptr, *d_gram_part = nullptr, *d_gram = nullptr, *d_vkeep = nullptr;
  int *d_task_kr = nullptr, *d_task_rank = nullptr;
  DevStatus* d_status = nullptr;
  int* d_flag = nullptr;            // FDE_CHECK result word (own allocation, never aliased)
  // staging for FDE_HOST_PTRS
  double *d_in = nullptr;   // 4 * batch * n
  double* d_rhs = nullptr;  // batch * n (solve-only rhs)
  bool factored = false;
  const double *src_dp = nullptr, *src_dm = nullptr;   // fde2d_step: coefficient arrays factorised
  double* d_split = nullptr;        // fde1d_step_split: send staging (n doubles)
  double* d_solve_split = nullptr;  // kept-factor solve of large nodes: partials + K-solve results
  double* d_hstage = nullptr;       // fde1d_run with FDE_HOST_PTRS: device staging
  size_t hstage_cap = 0;
  size_t solve_split_cap = 0;
  // TMA tensor maps of the projection (k_leaf.cuh leaf_project_tma): per (instance, level) a
  // 2D map of L_l (rows x rank, box 132 x rank), then the 3D maps of X and X2 (n x NC x batch,
  // box 132 x 16 x 1); null when some operand is not 16-byte aligned (the projection then
  // stages through cp.async)
  CUtensorMap* d_tmaps = nullptr;
  bool tma_ok = false;
  cudaStream_t last_stream = nullptr;
};

static int tmaps_build(fde_hodlr* H, const std::vector<int>& rk);
static int tmaps_add_x2(fde_hodlr* H);

template <typename T>
static int dalloc(fde_hodlr* H, T** p, size_t count) {
  void* q = nullptr;
  size_t bytes = count * sizeof(T);
  if (bytes == 0) bytes = 8;
  cudaError_t e = cudaMalloc(&q, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_err(FDE_ENOMEM, "cudaMalloc(%zu bytes) failed: %s", bytes, cudaGetErrorString(e));
  }
  H->allocs.push_back(q);
  *p = (T*)q;
  return FDE_OK;
}

#define TRY(x)               \
  do {                       \
    int rc_ = (x);           \
    if (rc_ != FDE_OK) return rc_; \
  } while (0)

static void free_handle(fde_hodlr* H) {
  if (!H) return;
  for (void* p : H->allocs) cudaFree(p);
  delete H;
}

// ---------------------------------------------------------------------------------------
// tree (reading R10: uniform depth, N1 = floor, N2 = ceil)
static void build_tree(fde_hodlr* H) {
  const int n = H->n, leaf = H->leaf;
  std::vector<std::pair<int, int>> nodes{{0, n}};
  int L = 0;
  H->node_r0.clear(); H->node_n1.clear(); H->node_n2.clear();
  while (true) {
    int mx = 0;
    for (auto& nd : nodes) mx = std::max(mx, nd.second);
    if (mx <= leaf) break;
    std::vector<std::pair<int, int>> nxt;
    for (auto& nd : nodes) {
      const int n1 = nd.second / 2, n2 = nd.second - n1;
      H->node_r0.push_back(nd.first);
      H->node_n1.push_back(n1);
      H->node_n2.push_back(n2);
      nxt.push_back({nd.first, n1});
      nxt.push_back({nd.first + n1, n2});
    }
    nodes.swap(nxt);
    ++L;
  }
  H->L = L;
  H->nleaf = (int)nodes.size();
  H->nnodes = (1 << L) - 1;
  H->leaf_r0.clear(); H->leaf_n.clear();
  for (auto& nd : nodes) { H->leaf_r0.push_back(nd.first); H->leaf_n.push_back(nd.second); }
  // segments and per-level sizes
  H->seg_ofs.assign(L + 1, 0);
  H->seg_node.clear(); H->seg_child.clear(); H->seg_row0.clear(); H->seg_len.clear();
  H->node_seg.assign(3 * std::max(1, H->nnodes), 0);
  H->lev_m.assign(std::max(1, L), 0);
  H->lev_lofs.assign(std::max(1, L), 0);
  H->lev_lraw.assign(std::max(1, L), 0);
  H->max_seg = 0;
  long long lofs = 0, lraw = 0;
  for (int l = 0; l < L; ++l) {
    H->seg_ofs[l] = (int)H->seg_node.size();
    int local = 0, m = 0;
    for (int j = 0; j < (1 << l); ++j) {
      const int nd = (1 << l) - 1 + j;
      const int r0 = H->node_r0[nd], n1 = H->node_n1[nd], n2 = H->node_n2[nd];
      m = std::max(m, n2);
      H->node_seg[3 * nd + 0] = local;
      for (int c = 0; c < 2; ++c) {
        if (c == 1) H->node_seg[3 * nd + 1] = local;
        const int rs = c == 0 ? r0 : r0 + n1, len = c == 0 ? n1 : n2;
        for (int o = 0; o < len; o += SEG) {
          H->seg_node.push_back(j);
          H->seg_child.push_back(c);
          H->seg_row0.push_back(rs + o);
          H->seg_len.push_back(std::min(SEG, len - o));
          ++local;
        }
      }
      H->node_seg[3 * nd + 2] = local;
    }
    H->max_seg = std::max(H->max_seg, local);
    H->lev_m[l] = m;
    H->lev_lofs[l] = lofs;
    H->lev_lraw[l] = lraw;
    lofs += (long long)m * RCAP;
    lraw += (long long)m * KRAW;
  }
  H->seg_ofs[L] = (int)H->seg_node.size();
  H->lf_stride = std::max(1LL, lofs);
  H->lraw_stride = std::max(1LL, lraw);
  H->max_nodes_lvl = L > 0 ? (1 << (L - 1)) : 1;
}

static int upload_tree(fde_hodlr* H) {
  // pack all int tables in one buffer
  std::vector<int> buf;
  auto put = [&](const std::vector<int>& v) { size_t o = buf.size(); buf.insert(buf.end(), v.begin(), v.end()); if (v.empty()) buf.push_back(0); return o; };
  size_t o_r0 = put(H->node_r0), o_n1 = put(H->node_n1), o_n2 = put(H->node_n2), o_ns = put(H->node_seg);
  size_t o_lr = put(H->leaf_r0), o_ln = put(H->leaf_n), o_so = put(H->seg_ofs), o_sn = put(H->seg_node);
  size_t o_sc = put(H->seg_child), o_s0 = put(H->seg_row0), o_sl = put(H->seg_len), o_m = put(H->lev_m);
  TRY(dalloc(H, &H->d_tree_int, buf.size()));
  CU(cudaMemcpy(H->d_tree_int, buf.data(), buf.size() * sizeof(int), cudaMemcpyHostToDevice));
  TRY(dalloc(H, &H->d_lev_lofs, H->lev_lofs.size()));
  CU(cudaMemcpy(H->d_lev_lofs, H->lev_lofs.data(), H->lev_lofs.size() * sizeof(long long), cudaMemcpyHostToDevice));
  int* b = H->d_tree_int;
  TreeDev& t = H->tree;
  t.n = H->n; t.L = H->L; t.nleaf = H->nleaf;
  t.node_r0 = b + o_r0; t.node_n1 = b + o_n1; t.node_n2 = b + o_n2; t.node_seg = b + o_ns;
  t.leaf_r0 = b + o_lr; t.leaf_n = b + o_ln; t.seg_ofs = b + o_so; t.seg_node = b + o_sn;
  t.seg_child = b + o_sc; t.seg_row0 = b + o_s0; t.seg_len = b + o_sl; t.lev_m = b + o_m;
  t.lev_lofs = H->d_lev_lofs;
  return FDE_OK;
}

// ---------------------------------------------------------------------------------------
// compression plan: tasks (instance, level) cut into PC_ROWS chunks, packed into
// cooperative launches that fit on the device at once.
static int plan_compression(fde_hodlr* H, int capacity) {
  H->tasks.clear(); H->chunks.clear(); H->launch_chunk0.clear();
  int slot = 0, in_launch = 0;
  H->launch_chunk0.push_back(0);
  for (int b = 0; b < H->batch; ++b) {
    for (int l = 0; l < H->L; ++l) {
      const int m = H->lev_m[l];
      const int G = (m + PC_ROWS - 1) / PC_ROWS;
      if (G > capacity)
        return set_err(FDE_EDIM, "n=%d too large: level %d needs %d co-resident CTAs (device holds %d)",
                       H->n, l, G, capacity);
      if (in_launch + G > capacity) { H->launch_chunk0.push_back((int)H->chunks.size()); in_launch = 0; }
      PcTask tk{};
      tk.inst = b; tk.level = l; tk.m = m; tk.G = G; tk.slot0 = slot;
      tk.lraw_ofs = (long long)b * H->lraw_stride + H->lev_lraw[l];
      tk.lf_ofs = (long long)b * H->lf_stride + H->lev_lofs[l];
      tk.tau = H->tol * std::exp2(H->alpha[b]);         // reading R7: ||T||_2 <= 2^alpha
      const int tid = (int)H->tasks.size();
      H->tasks.push_back(tk);
      for (int c = 0; c < G; ++c) {
        PcChunk ch{tid, c * PC_ROWS, std::min(PC_ROWS, m - c * PC_ROWS), c};
        H->chunks.push_back(ch);
      }
      slot += G;
      in_launch += G;
    }
  }
  H->launch_chunk0.push_back((int)H->chunks.size());
  return FDE_OK;
}

// S1: GL weights g_0..g_{n+1} of every instance (two multi-CTA passes, k_gl.cuh)
static int launch_gl(fde_hodlr* H, cudaStream_t s) {
  const int nk = H->n + 2, nseg = (nk - 1 + GLS_SEG - 1) / GLS_SEG;
  { PROF("k_gl_seg"); k_gl_seg<<<dim3(nseg, H->batch), GLS_THREADS, 0, s>>>(H->d_alpha, nk, H->d_glseg); }
  LAUNCHED();
  { PROF("k_gl_expand"); k_gl_expand<<<dim3(nseg, H->batch), GLS_THREADS, 0, s>>>(H->d_alpha, nk, H->d_glseg, H->d_g, H->gstride); }
  LAUNCHED();
  return FDE_OK;
}

static int run_compression(fde_hodlr* H, cudaStream_t s) {
  if (H->L == 0) return FDE_OK;
  const int ntask = (int)H->tasks.size();
#ifdef FDE_DEBUG
  if (fde_dbg_env("FDE_COMP_TRACE")) { const int one = 1; CU(cudaMemcpyToSymbol(g_comp_trace, &one, sizeof(int))); }
#endif
  CU(cudaMemsetAsync(H->d_ctr, 0, sizeof(unsigned) * ntask, s));
  CU(cudaMemsetAsync(H->d_part, 0, sizeof(double) * std::max<size_t>(1, H->chunks.size()) * 2 * PSTRIDE, s));   // slot tags
  const size_t smem = (size_t)KRAW * PC_ROWS * sizeof(double);
  for (size_t li = 0; li + 1 < H->launch_chunk0.size(); ++li) {
    const int c0 = H->launch_chunk0[li], c1 = H->launch_chunk0[li + 1];
    if (c1 <= c0) continue;
    const PcTask* tasks = H->d_tasks;
    const PcChunk* chunks = H->d_chunks + c0;
    const double* g = H->d_g;
    long long gs = H->gstride;
    double* Lraw = H->d_Lraw;
    int* tkr = H->d_task_kr;
    unsigned* ctr = H->d_ctr;
    double* part = H->d_part;
    double* gp = H->d_gram_part;
    double* gram = H->d_gram;
    DevStatus* st = H->d_status;
    void* args[] = {&tasks, &chunks, &g, &gs, &Lraw, &tkr, &ctr, &part, &gp, &gram, &st};
    { PROF("k_pchol"); CU(cudaLaunchCooperativeKernel((void*)k_pchol, dim3(c1 - c0), dim3(PC_THREADS), args, smem, s)); }
    LAUNCHED();
  }
  { PROF("k_eig"); k_eig<<<ntask, EIG_THREADS, EIG_SMEM, s>>>(
      H->d_tasks, H->d_task_kr, H->d_gram, H->d_vkeep, H->d_task_rank, H->d_rank, H->L, H->d_status); }
  LAUNCHED();
  { PROF("k_ltransform"); k_ltransform<<<(int)H->chunks.size(), PC_ROWS, 0, s>>>(
      H->d_tasks, H->d_chunks, H->d_task_kr, H->d_task_rank, H->d_vkeep, H->d_Lraw, H->d_Lf); }
  LAUNCHED();
  { PROF("k_colofs"); k_colofs<<<(H->batch + 127) / 128, 128, 0, s>>>(H->d_rank, H->d_colofs, H->L, H->batch); }
  LAUNCHED();
  return FDE_OK;
}

__global__ void k_cfac(const double* __restrict__ alpha, double dt, double h, double* __restrict__ c,
                       int batch) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < batch) c[i] = dt / pow(h, alpha[i]);        // c = dt / h^alpha (Eq. 2.5)
}

static int set_dt(fde_hodlr* H, double dt, cudaStream_t s) {
  H->dt = dt;
  { PROF("k_cfac"); k_cfac<<<(H->batch + 127) / 128, 128, 0, s>>>(H->d_alpha, dt, H->h, H->d_cfac, H->batch); }
  LAUNCHED();
  return FDE_OK;
}

// cudaFuncSetAttribute applies to the current device: one bit per device that has them
static std::atomic<unsigned long long> g_attr_mask{0};
static int set_attrs() {
  int dev = 0;
  CU(cudaGetDevice(&dev));
  const unsigned long long bit = 1ULL << (dev & 63);
  if (g_attr_mask.load() & bit) return FDE_OK;
  CU(cudaFuncSetAttribute(k_pchol, cudaFuncAttributeMaxDynamicSharedMemorySize, KRAW * PC_ROWS * 8));
  CU(cudaFuncSetAttribute(k_eig, cudaFuncAttributeMaxDynamicSharedMemorySize, EIG_SMEM));
  CU(cudaFuncSetAttribute(k_solve_level, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * KCAP * KCAP * 8));
  CU(cudaFuncSetAttribute(k_leaf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          LEAF_SMEM));
  CU(cudaFuncSetAttribute(k_lvl_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_REDUCE));
  CU(cudaFuncSetAttribute(k_mv_leaf, cudaFuncAttributeMaxDynamicSharedMemorySize, MV_LEAF_SMEM));
  CU(cudaFuncSetAttribute(k_mv_update, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MV_UPDATE));
  CU(cudaFuncSetAttribute(k_levels<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, LV_SMEM_MAX));
  CU(cudaFuncSetAttribute(k_levels<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, LV_SMEM_MAX));
  CU(cudaFuncSetAttribute(k_levels<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, LV_SMEM_MAX));
  g_attr_mask.fetch_or(bit);
  return FDE_OK;
}

static int check_common(int batch, int n, const double* alpha, double h, double dt, double tol,
                        int leaf) {
  if (batch < 1) return set_err(FDE_EDOMAIN, "batch=%d must be >= 1", batch);
  if (n < 1) return set_err(FDE_EDOMAIN, "n=%d must be >= 1", n);
  if (!alpha) return set_err(FDE_EDOMAIN, "alpha is NULL");
  for (int b = 0; b < batch; ++b)
    if (!(alpha[b] > 1.0 && alpha[b] <= 2.0))
      return set_err(FDE_EDOMAIN, "alpha[%d]=%g outside (1, 2]", b, alpha[b]);
  if (!(h > 0.0) || !std::isfinite(h)) return set_err(FDE_EDOMAIN, "h=%g must be > 0", h);
  if (!(dt >= 0.0) || !std::isfinite(dt)) return set_err(FDE_EDOMAIN, "dt=%g must be >= 0", dt);
  if (!(tol > 0.0 && tol < 1.0)) return set_err(FDE_EDOMAIN, "tol=%g outside (0, 1)", tol);
  if (leaf < 2 || leaf > LEAF_MAX) return set_err(FDE_EDOMAIN, "leaf=%d outside [2, %d]", leaf, LEAF_MAX);
  return FDE_OK;
}

// d >= 0 check (FDE_CHECK)
__global__ void k_check_nonneg(const double* __restrict__ a, long long cnt, int* __restrict__ bad) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt && !(a[i] >= 0.0)) atomicExch(bad, 1);
}

static int check_nonneg(fde_hodlr* H, const double* dp, const double* dm, cudaStream_t s) {
  int* bad = H->d_flag;
  CU(cudaMemsetAsync(bad, 0, sizeof(int), s));
  const long long cnt = (long long)H->batch * H->n;
  { PROF("k_check_nonneg"); k_check_nonneg<<<(unsigned)((cnt + 255) / 256), 256, 0, s>>>(dp, cnt, bad); }
  LAUNCHED();
  { PROF("k_check_nonneg"); k_check_nonneg<<<(unsigned)((cnt + 255) / 256), 256, 0, s>>>(dm, cnt, bad); }
  LAUNCHED();
  int hb = 0;
  CU(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (hb) return set_err(FDE_EDOMAIN, "d_plus / d_minus has a negative or non-finite entry (P:56)");
  return FDE_OK;
}

// Read the latched device status after a synchronisation.  A failure is reported once: the
// word is cleared when it is returned, so a later call on the same handle starts clean.
static int read_status(fde_hodlr* H, DevStatus* out) {
  DevStatus st{};
  CU(cudaMemcpy(&st, H->d_status, sizeof(st), cudaMemcpyDeviceToHost));
  if (st.code != FDE_OK) CU(cudaMemset(H->d_status, 0, sizeof(DevStatus)));
  *out = st;
  return FDE_OK;
}

static int sync_and_status(fde_hodlr* H, cudaStream_t s) {
  CU(cudaStreamSynchronize(s));
  DevStatus st{};
  TRY(read_status(H, &st));
  if (st.code != FDE_OK)
    return set_err(st.code, "device status %d at instance %d index %d", st.code, st.where / 65536,
                   st.where % 65536);
  return FDE_OK;
}

// ---------------------------------------------------------------------------------------
// Level layout and the persistent level kernel's configuration
static unsigned long long* g_trace = nullptr;

struct LvCfg {
  int CR, ldx, lds, ldk, ldm, offs[10], xbuf, wbuf, vbuf;
  size_t bytes;
};

static int lv_config(const fde_hodlr* H, int mode, int nrhs, LvCfg* cfg) {
  const int L = H->L;
  const int NCPX = round_up(mode == 0 ? H->xcol[L] : nrhs, 8);
  const int KP8 = round_up(H->kmax, 8), KP4 = round_up(H->kmax, 4);
  if ((KP8 / 8) * (NCPX / 8) > MT_RED * LV_WARPS)
    return set_err(FDE_EDIM, "level width %d x %d exceeds the reduce tile budget", KP8, NCPX);
  const int lds = NCPX + ((NCPX % 16 == 0) ? 20 : 28);   // >= NCPX + 16 (padded views), = 4 mod 16
  const int ldk = KP8 + 1, ldm = 2 * KP8 + 1;
  for (int CR = 64; CR >= 8; CR /= 2) {
    const int ldx = CR + 4;
    long long o = 0;
    int offs[10];
    const int xb = NCPX * ldx, wb = KP4 * ldx, vb = KP8 * ldx;   // one pipeline buffer each
    offs[0] = (int)o; o += 2LL * xb;                         // Xc x 2
    offs[1] = (int)o; o += 2LL * wb;                         // Wn x 2
    offs[2] = (int)o; o += 2LL * vb;                         // Vc x 2
    offs[3] = (int)o; o += (long long)KP8 * lds;             // Pt
    offs[4] = (int)o; o += (long long)KP8 * lds;             // Pb
    if ((long long)KP8 * lds <= 2LL * xb) offs[5] = offs[0];   // T aliases Xc
    else { offs[5] = (int)o; o += (long long)KP8 * lds; }
    offs[6] = (int)o; o += (long long)KP8 * ldk;             // B
    offs[7] = (int)o; o += (long long)KP8 * ldk;             // C
    offs[8] = (int)o; o += (long long)KP8 * ldk;             // Sci
    offs[9] = (int)o; o += (long long)KP8 * ldm;             // GJ workspace
    const size_t bytes = (size_t)o * sizeof(double);
    if (bytes <= LV_SMEM_MAX) {
      cfg->CR = CR; cfg->ldx = ldx; cfg->lds = lds; cfg->ldk = ldk; cfg->ldm = ldm; cfg->bytes = bytes;
      cfg->xbuf = xb; cfg->wbuf = wb; cfg->vbuf = vb;
      for (int i = 0; i < 10; ++i) cfg->offs[i] = offs[i];
      return FDE_OK;
    }
  }
  return set_err(FDE_EDIM, "level kernel workspace does not fit in shared memory (k=%d, cols=%d)",
                 H->kmax, NCPX);
}

static void print_leaf_trace(unsigned long long* d_trace) {
  std::vector<unsigned long long> lt(4096), h(1024);
  cudaDeviceSynchronize();
  cudaMemcpy(lt.data(), d_trace + 2048, 4096 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaMemcpy(h.data(), d_trace, 1024 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double ph[4] = {0, 0, 0, 0};
  unsigned long long t0 = ~0ULL, t1 = 0;
  int cnt = 0;
  for (int l = 0; l < 512 && lt[l * 8 + 4]; ++l, ++cnt) {
    for (int q = 0; q < 4; ++q) ph[q] += (double)(lt[l * 8 + q + 1] - lt[l * 8 + q]);
    t0 = std::min(t0, lt[l * 8]);
    t1 = std::max(t1, lt[l * 8 + 4]);
  }
  fprintf(stderr, "k_leaf build cycles leaf0: warp0 staging %llu build %llu gj0 %llu | warp4 staging %llu build %llu\n",
          h[980], h[981], h[982], h[984], h[985]);
  fprintf(stderr, "k_leaf LU cycles CTA0: gj0 %llu ovw %llu diagupd %llu gj||trail %llu\n", h[960], h[961], h[962], h[963]);
  fprintf(stderr, "k_leaf panel cycles CTA0 warp0: gen %llu ld %llu solve %llu store %llu\n", h[970], h[971], h[972], h[973]);
  if (cnt)
    fprintf(stderr, "k_leaf per-CTA avg us: build %.2f lu %.2f panel %.2f proj %.2f (%d CTAs, span %.1f us)\n",
            ph[0] / cnt * 1e-3, ph[1] / cnt * 1e-3, ph[2] / cnt * 1e-3, ph[3] / cnt * 1e-3, cnt, (t1 - t0) * 1e-3);
}

// Layout of the projected-tree path (k_tree.cuh): Q stores of levels 1..L (leaves: L), S
// stores of levels 0..L-1, work split and shared-memory geometry.  Leaves tree_ok = false
// (the level-pass path is used) when the panel is too wide for the leaf Q phase.
static int tree_layout(fde_hodlr* H) {
  const int L = H->L, B = H->batch, NC = H->xcol[L];
  H->tree_ok = false;
  if (L < 1 || NC - 1 > 176) return FDE_OK;
  long long q = 0, sofs = 0;
  for (int m = 1; m <= L; ++m) {
    H->qlev[m] = q;
    q += (1LL << m) * (long long)(H->xcol[m] - 1) * H->xcol[m];
  }
  for (int m = 0; m < L; ++m) {
    H->slev[m] = sofs;
    sofs += (1LL << m) * 2LL * H->kl[m] * H->xcol[m];
  }
  H->qinst = q; H->sinst = sofs;
  int dev = 0, nsm = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  TrArgs& g = H->tr_geo;
  const int kp = round_up(H->kmax, 8), K4 = round_up(2 * H->kmax, 4);
  g.kp = kp; g.ldk = kp + 1;
  g.lds = round_up(NC, 16) + 4;                       // = 4 mod 16: conflict-free B fragments
  g.lda = K4 + ((4 - K4 % 16) + 16) % 16;
  int rch_max = 8;
  for (int m = 0; m < L; ++m) {
    const int nodes = B << m, rows = H->xcol[m] - 1;
    int rc = std::max(1, nsm / std::max(1, nodes));
    rc = std::min(rc, std::max(1, (rows + 15) / 16));
    H->trc[m] = rc;
    rch_max = std::max(rch_max, round_up((std::max(rows, 1) + rc - 1) / rc, 8));
  }
  g.rch_max = rch_max;
  long long o = 0;
  g.off_B = (int)o; o += (long long)kp * g.ldk;
  g.off_C = (int)o; o += (long long)kp * g.ldk;
  g.off_M = (int)o; o += (long long)kp * g.ldk;
  g.off_M2 = (int)o; o += (long long)kp * g.ldk;
  o = round_up((int)o, 2);
  g.off_S = (int)o; o += (long long)K4 * g.lds;
  g.off_T = (int)o;                                   // union { T + Z (S phase), U (Q update) }
  g.off_Z = round_up((int)(o + (long long)kp * g.lds), 2);   // (16-byte aligned: contiguous staging)
  g.off_U = (int)o;
  o += std::max((long long)(g.off_Z - o) + 2LL * H->kmax * NC + 6, 2LL * TR_STG * (TR_SUB * NC + 2));
  // final pass: 4 v vectors + max(4 warps x 2 S buffers, X block + partials)
  const long long fin = 4LL * round_up(NC, 8) + std::max(8LL * H->kmax * NC, (long long)NC * 128 + 256);
  const size_t bytes = (size_t)std::max(o, fin) * sizeof(double);
  if (bytes > 227 * 1024) return FDE_OK;
  CU(cudaFuncSetAttribute(k_tree, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  int per_sm = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tree, TR_THREADS, bytes));
  if (per_sm < 1) return FDE_OK;
  H->tr_grid = nsm * per_sm;
  H->tr_smem = bytes;
  TRY(dalloc(H, &H->d_Q, (size_t)B * H->qinst));
  TRY(dalloc(H, &H->d_S, (size_t)B * H->sinst));
  // persistent dataflow kernel (k_step.cuh): counters and launch geometry
  long long dn = 1;                                   // [0] = task counter
  for (int m = 0; m < L; ++m) { H->dofs[m] = dn; dn += (long long)B << m; }
  H->dofs[L] = dn; dn += (long long)B << (L - 1);
  H->lofs = dn; dn += (long long)B * H->nleaf;
  H->ndone = dn;
  TRY(dalloc(H, &H->d_done, (size_t)dn));
  H->step_smem = std::max((size_t)LEAF_SMEM, bytes);
  CU(cudaFuncSetAttribute(k_step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)H->step_smem));
  int per_sm2 = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, k_step, TR_THREADS, H->step_smem));
  H->step_grid = nsm * std::max(1, per_sm2);
  H->tree_ok = true;
  return FDE_OK;
}

static int launch_tree(fde_hodlr* H, double* u_next, cudaStream_t s) {
  TrArgs a = H->tr_geo;
  const int L = H->L;
  a.L = L; a.NC = H->xcol[L]; a.nleaf = H->nleaf; a.batch = H->batch; a.kmaxc = H->kmax;
  for (int l = 0; l <= L; ++l) a.xc[l] = H->xcol[l];
  for (int m = 0; m < L; ++m) { a.rc[m] = H->trc[m]; a.slev[m] = H->slev[m]; }
  for (int m = 1; m <= L; ++m) a.qlev[m] = H->qlev[m];
  a.qinst = H->qinst; a.sinst = H->sinst;
  a.Qleaf = H->d_Q + H->qlev[L]; a.Q = H->d_Q; a.Sst = H->d_S;
  a.X = H->d_X; a.xstride = H->xstride; a.n = H->n;
  a.leaf_r0 = H->tree.leaf_r0; a.leaf_n = H->tree.leaf_n;
  a.u = u_next; a.bar = H->d_bar; a.st = H->d_status;
  a.trace = g_trace;                                   // (reset by factor_impl)
  CU(cudaMemsetAsync(H->d_bar, 0, sizeof(unsigned), s));
  void* args[] = {&a};
  { PROF("k_tree"); CU(cudaLaunchCooperativeKernel((void*)k_tree, dim3(H->tr_grid), dim3(TR_THREADS), args, H->tr_smem, s)); }
  LAUNCHED();
  if (g_trace) {
    print_leaf_trace(g_trace);
    std::vector<unsigned long long> h(64);
    CU(cudaStreamSynchronize(s));
    CU(cudaMemcpy(h.data(), g_trace + 1024, 64 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    fprintf(stderr, "k_tree CTA0 (us): ");
    for (int m = 0; m < H->L; ++m)
      fprintf(stderr, "L%d work %.1f bar %.1f | ", H->L - 1 - m, (h[2 * m + 1] - h[2 * m]) * 1e-3,
              (h[2 * m + 2] - h[2 * m + 1]) * 1e-3);
    fprintf(stderr, "final %.1f ; rc:", (h[2 * H->L + 1] - h[2 * H->L]) * 1e-3);
    for (int m = 0; m < H->L; ++m) fprintf(stderr, " %d", H->trc[m]);
    fprintf(stderr, " grid %d smem %zu\n", H->tr_grid, H->tr_smem);
    std::vector<unsigned long long> c(16);
    CU(cudaMemcpy(c.data(), g_trace + 1100, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    fprintf(stderr, "k_tree CTA0 unit cycles: stage %llu sc+T %llu gj %llu S %llu Qupd %llu | final: vrec %llu xwait %llu gemv %llu\n",
            c[0], c[1], c[2], c[3], c[4], c[10], c[11], c[12]);
  }
  return FDE_OK;
}

static void post_order(int d, int j, int D, std::vector<int>& out) {
  if (d + 1 < D) { post_order(d + 1, 2 * j, D, out); post_order(d + 1, 2 * j + 1, D, out); }
  out.push_back(d);
  out.push_back(j);
}

static int finalize_layout(fde_hodlr* H, cudaStream_t s) {
  const int L = H->L, B = H->batch, n = H->n;
  std::vector<int> rk((size_t)B * std::max(1, L), 0);
  if (L > 0) {
    CU(cudaStreamSynchronize(s));
    CU(cudaMemcpy(rk.data(), H->d_rank, rk.size() * sizeof(int), cudaMemcpyDeviceToHost));
    DevStatus st{};
    CU(cudaMemcpy(&st, H->d_status, sizeof(st), cudaMemcpyDeviceToHost));
    if (st.code != FDE_OK)
      return set_err(st.code, "compression failed (status %d) at instance %d level %d", st.code,
                     st.where / 65536, st.where % 65536);
  }
  H->kl.assign(std::max(1, L), 1);
  H->xcol.assign(L + 1, 1);
  H->kofs.assign(std::max(1, L), 0);
  H->kmax = 1;
  long long ko = 0;
  for (int l = 0; l < L; ++l) {
    int R = 0;
    for (int b = 0; b < B; ++b) R = std::max(R, rk[(size_t)b * L + l]);
    H->kl[l] = R + 1;
    H->kmax = std::max(H->kmax, R + 1);
    H->xcol[l + 1] = H->xcol[l] + R + 1;
    H->kofs[l] = ko;
    ko += (1LL << l) * 3LL * (R + 1) * (R + 1);
  }
  if (H->xcol[L] > NCOL_MAX)
    return set_err(FDE_EDIM, "panel width %d exceeds %d columns (ranks too large for this build)",
                   H->xcol[L], NCOL_MAX);
  H->kstride_inst = std::max(1LL, ko);
  H->xstride = (long long)n * H->xcol[L];
  H->sum_nc = std::max(H->xcol[L], NRHS_MAX);
  H->sum_half = (long long)round_up(H->kmax, 8) * H->sum_nc;
  // CTAs per instance for the persistent level kernel: P = 2^p co-resident with the batch
  LvCfg cfg;
  TRY(lv_config(H, 0, 1, &cfg));
  int dev = 0, nsm = 0, per_sm = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_levels<16>, LV_THREADS, cfg.bytes));
  H->coop_capacity = std::max(1, nsm * per_sm);
  int p = 0;
  while (p < L && ((long long)B << (p + 1)) <= H->coop_capacity) ++p;
  H->p = p;
  H->P = 1 << p;
  std::vector<int> post;
  if (p < L) post_order(0, 0, L - p, post);
  H->npost = (int)post.size() / 2;
  const size_t nn = std::max(1, H->nnodes);
  TRY(dalloc(H, &H->d_X, (size_t)B * H->xstride));
  TRY(dalloc(H, &H->d_Kst, (size_t)B * H->kstride_inst));
  TRY(dalloc(H, &H->d_sums, (size_t)B * nn * 2 * H->sum_half));
  TRY(dalloc(H, &H->d_lvpart, (size_t)2 * B * H->P * H->sum_half));
  TRY(dalloc(H, &H->d_bar, 1));
  TRY(dalloc(H, &H->d_post, std::max<size_t>(2, post.size())));
  if (!post.empty())
    CU(cudaMemcpy(H->d_post, post.data(), post.size() * sizeof(int), cudaMemcpyHostToDevice));
  TRY(tree_layout(H));
  TRY(tmaps_build(H, rk));
  H->layout_done = true;
  return FDE_OK;
}

static int launch_levels(fde_hodlr* H, int mode, int nf, double* Y, int ld, int nrhs, cudaStream_t s) {
  const int L = H->L;
  if (L == 0) return FDE_OK;
  LvCfg cfg;
  TRY(lv_config(H, mode, nrhs, &cfg));
  LvArgs a{};
  a.tree = H->tree; a.mode = mode; a.L = L; a.p = H->p; a.P = H->P; a.nf = nf; a.CR = cfg.CR;
  a.lgCR = 0;
  while ((1 << a.lgCR) < cfg.CR) ++a.lgCR;
  a.ldx = cfg.ldx; a.lds = cfg.lds; a.ldk = cfg.ldk; a.ldm = cfg.ldm;
  a.off_Xc = cfg.offs[0]; a.off_Wn = cfg.offs[1]; a.off_Vc = cfg.offs[2]; a.off_Pt = cfg.offs[3];
  a.off_Pb = cfg.offs[4]; a.off_T = cfg.offs[5]; a.off_B = cfg.offs[6]; a.off_C = cfg.offs[7];
  a.off_Si = cfg.offs[8]; a.off_M = cfg.offs[9];
  a.xbuf = cfg.xbuf; a.wbuf = cfg.wbuf; a.vbuf = cfg.vbuf;
  for (int l = 0; l < L; ++l) { a.kl[l] = H->kl[l]; a.xcol[l] = H->xcol[l]; a.kofs[l] = H->kofs[l]; }
  a.xcol[L] = H->xcol[L];
  a.kstride_inst = H->kstride_inst;
  a.Lf = H->d_Lf; a.lf_stride = H->lf_stride; a.rank = H->d_rank;
  a.X = H->d_X; a.xstride = H->xstride;
  a.Y = Y; a.ld = ld; a.nrhs = nrhs; a.ystride = (long long)ld * nrhs;
  a.Kst = H->d_Kst; a.sums = H->d_sums; a.sum_half = H->sum_half; a.sum_nc = H->sum_nc;
  a.part = H->d_lvpart; a.bar = H->d_bar; a.post = H->d_post; a.npost = H->npost; a.st = H->d_status;
  const bool trace = g_trace != nullptr;                 // debug: FDE_TRACE_LEVELS=1
  unsigned long long* d_trace = g_trace;
  if (trace) a.trace = d_trace;
  const int grid = H->P * H->batch;
  // reduce tiles per warp: (round8(k)/8) x (cols/8) tiles over LV_WARPS warps
  const int ntile = (round_up(H->kmax, 8) / 8) * (round_up(mode == 0 ? H->xcol[L] : nrhs, 8) / 8);
  const int mt = ntile <= 4 * LV_WARPS ? 4 : (ntile <= 8 * LV_WARPS ? 8 : 16);
  void* fn = mt == 4 ? (void*)k_levels<4> : (mt == 8 ? (void*)k_levels<8> : (void*)k_levels<16>);
  void* args[] = {&a};
  if (H->P > 1) {
    CU(cudaMemsetAsync(H->d_bar, 0, sizeof(unsigned), s));
    { PROF("k_levels"); CU(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(LV_THREADS), args, cfg.bytes, s)); }
  } else {
    { PROF("k_levels"); CU(cudaLaunchKernel(fn, dim3(grid), dim3(LV_THREADS), args, cfg.bytes, s)); }
  }
  LAUNCHED();
  if (trace) {
    static unsigned long long h[2048];
    CU(cudaStreamSynchronize(s));
    CU(cudaMemcpy(h, d_trace, sizeof(h), cudaMemcpyDeviceToHost));
    for (int b = 0; b < 2; ++b) {
      fprintf(stderr, "k_levels trace CTA %s:", b ? "last" : "0");
      for (int i = 0; i < 255 && h[b * 512 + 2 * i + 1]; ++i)
        fprintf(stderr, " %llu:%.2f", h[b * 512 + 2 * i],
                (h[b * 512 + 2 * i + 1] - h[b * 512 + 1]) * 1e-3);
      fprintf(stderr, "\n");
    }
    fprintf(stderr, "k_levels pass cycles CTA 0: sync %llu load %llu update %llu reduce %llu store %llu\n",
            h[1100], h[1101], h[1102], h[1103], h[1104]);
    fprintf(stderr, "k_levels node cycles CTA 0: prep %llu GJ %llu Si %llu store %llu solves %llu\n",
            h[1110], h[1111], h[1112], h[1113], h[1114]);
    print_leaf_trace(d_trace);
  }
  return FDE_OK;
}

// debug tracing buffer (FDE_TRACE_LEVELS): cleared before every leaf launch
static int trace_reset(cudaStream_t s) {
  if (!fde_dbg_env("FDE_TRACE_LEVELS")) { g_trace = nullptr; return FDE_OK; }
  if (!g_trace) CU(cudaMalloc(&g_trace, 8192 * sizeof(unsigned long long)));
  CU(cudaMemsetAsync(g_trace, 0, 8192 * sizeof(unsigned long long), s));
  return FDE_OK;
}

// ---------------------------------------------------------------------------------------
static int build_impl(int batch, int n, const double* alpha, double h, double dt, const double* dp,
                      const double* dm, double shift, double tol, int leaf, unsigned flags,
                      cudaStream_t s, fde_hodlr** out) {
  TRY(check_common(batch, n, alpha, h, dt, tol, leaf));
  if (!(shift > 0.0) || !std::isfinite(shift)) return set_err(FDE_EDOMAIN, "shift=%g must be > 0", shift);
  if (!out) return set_err(FDE_EDOMAIN, "out is NULL");
  TRY(set_attrs());
  fde_hodlr* H = new fde_hodlr();
  auto fail = [&](int rc) { free_handle(H); return rc; };
  H->batch = batch; H->n = n; H->leaf = leaf; H->h = h; H->dt = dt; H->shift = shift; H->tol = tol;
  H->alpha.assign(alpha, alpha + batch);
  build_tree(H);
  if (H->L > LMAX) return fail(set_err(FDE_EDIM, "tree depth %d exceeds %d", H->L, LMAX));
  int rc;
  if ((rc = upload_tree(H)) != FDE_OK) return fail(rc);
  // capacity for the cooperative compression
  int dev = 0, nsm = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pchol, PC_THREADS, KRAW * PC_ROWS * 8) != cudaSuccess)
    return fail(set_err(FDE_ECUDA, "device query failed: %s", cudaGetErrorString(cudaGetLastError())));
  if ((rc = plan_compression(H, std::max(1, nsm * per_sm))) != FDE_OK) return fail(rc);
  const int L = H->L;
  H->gstride = n + 2;
  H->ncap = NRHS_MAX;                                   // matvec partials (k_lvl_reduce)
  H->lustride = (long long)H->nleaf * LEAF_SLOT;          // one padded block factor per leaf
  H->pstride_seg = (long long)KCAP * H->ncap;
  H->pstride_inst = (long long)std::max(1, H->max_seg) * H->pstride_seg;
  const size_t B = batch;
  const size_t ntask = H->tasks.size(), nch = H->chunks.size();
  if ((rc = dalloc(H, &H->d_alpha, B)) || (rc = dalloc(H, &H->d_cfac, B)) ||
      (rc = dalloc(H, &H->d_g, B * H->gstride)) || (rc = dalloc(H, &H->d_Lf, B * H->lf_stride)) ||
      (rc = dalloc(H, &H->d_Lraw, B * H->lraw_stride)) || (rc = dalloc(H, &H->d_rank, B * std::max(1, L))) ||
      (rc = dalloc(H, &H->d_colofs, B * (L + 1))) || (rc = dalloc(H, &H->d_dp, B * n)) ||
      (rc = dalloc(H, &H->d_dm, B * n)) ||
      (rc = dalloc(H, &H->d_LU, B * H->lustride)) || (rc = dalloc(H, &H->d_P, B * H->pstride_inst)) ||
      (rc = dalloc(H, &H->d_tasks, std::max<size_t>(1, ntask))) ||
      (rc = dalloc(H, &H->d_chunks, std::max<size_t>(1, nch))) ||
      (rc = dalloc(H, &H->d_ctr, std::max<size_t>(1, ntask))) ||
      (rc = dalloc(H, &H->d_glseg, B * (size_t)((n + 1 + GLS_SEG - 1) / GLS_SEG))) ||
      (rc = dalloc(H, &H->d_part, std::max<size_t>(1, nch) * 2 * PSTRIDE)) ||
      (rc = dalloc(H, &H->d_gram_part, std::max<size_t>(1, nch) * KRAW * KRAW)) ||
      (rc = dalloc(H, &H->d_gram, std::max<size_t>(1, ntask) * KRAW * KRAW)) ||
      (rc = dalloc(H, &H->d_vkeep, std::max<size_t>(1, ntask) * KRAW * RCAP)) ||
      (rc = dalloc(H, &H->d_task_kr, std::max<size_t>(1, ntask))) ||
      (rc = dalloc(H, &H->d_task_rank, std::max<size_t>(1, ntask))) ||
      (rc = dalloc(H, &H->d_status, 1)) || (rc = dalloc(H, &H->d_flag, 1)) ||
      (rc = dalloc(H, &H->d_in, 5 * B * n + 8)))
    return fail(rc);
  H->d_rhs = H->d_in + 4 * B * n;
  if (cudaMemcpy(H->d_alpha, alpha, B * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
      (ntask && cudaMemcpy(H->d_tasks, H->tasks.data(), ntask * sizeof(PcTask), cudaMemcpyHostToDevice) != cudaSuccess) ||
      (nch && cudaMemcpy(H->d_chunks, H->chunks.data(), nch * sizeof(PcChunk), cudaMemcpyHostToDevice) != cudaSuccess))
    return fail(set_err(FDE_ECUDA, "upload failed"));
  if (cudaMemsetAsync(H->d_status, 0, sizeof(DevStatus), s) != cudaSuccess ||
      cudaMemsetAsync(H->d_rank, 0, B * std::max(1, L) * sizeof(int), s) != cudaSuccess ||
      cudaMemsetAsync(H->d_colofs, 0, B * (L + 1) * sizeof(int), s) != cudaSuccess)
    return fail(set_err(FDE_ECUDA, "memset failed"));
  if (dp && cudaMemcpyAsync(H->d_dp, dp, B * n * sizeof(double), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return fail(set_err(FDE_ECUDA, "copy d_plus failed"));
  if (dm && cudaMemcpyAsync(H->d_dm, dm, B * n * sizeof(double), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return fail(set_err(FDE_ECUDA, "copy d_minus failed"));
  if ((flags & FDE_CHECK) && dp && dm && (rc = check_nonneg(H, H->d_dp, H->d_dm, s)) != FDE_OK) return fail(rc);
  if ((rc = set_dt(H, dt, s)) != FDE_OK) return fail(rc);
  // S1: GL weights
  if ((rc = launch_gl(H, s)) != FDE_OK) return fail(rc);
  // S2: compression
  if ((rc = run_compression(H, s)) != FDE_OK) return fail(rc);
  if (flags & FDE_COMPRESS_ONLY) {                  // S1-S2 only (rank studies): no factor layout
    H->compress_only = true;
    H->last_stream = s;
    *out = H;
    return FDE_OK;
  }
  // one synchronisation per build: the ranks fix the column layout of the factorisation
  if ((rc = finalize_layout(H, s)) != FDE_OK) return fail(rc);
  H->last_stream = s;
  if ((flags & FDE_SYNC) && (rc = sync_and_status(H, s)) != FDE_OK) return fail(rc);
  *out = H;
  return FDE_OK;
}

// One k_step launch over a part of the step (StepArgs in k_step.cuh): leaves [lf0, lf1), tree
// levels [mlo, mhi) (restricted to the part's nodes or all), leaf tasks and/or finals.
struct StepPart { int lf0, lf1, mlo, mhi, restrict_nodes, do_leaf, do_final; };

static int launch_step(fde_hodlr* H, const LeafArgs& la, const StepPart& pt, double* u_next, cudaStream_t s,
                       const char* prof_name = "k_step") {
  const int L = H->L;
  StepArgs sa{};
  sa.la = la;
  TrArgs& a = sa.ta;
  a = H->tr_geo;
  a.L = L; a.NC = H->xcol[L]; a.nleaf = H->nleaf; a.batch = H->batch; a.kmaxc = H->kmax;
  for (int l = 0; l <= L; ++l) a.xc[l] = H->xcol[l];
  for (int m = 0; m < L; ++m) { a.rc[m] = H->trc[m]; a.slev[m] = H->slev[m]; }
  for (int m = 1; m <= L; ++m) a.qlev[m] = H->qlev[m];
  a.qinst = H->qinst; a.sinst = H->sinst;
  a.Qleaf = H->d_Q + H->qlev[L]; a.Q = H->d_Q; a.Sst = H->d_S;
  a.X = H->d_X; a.xstride = H->xstride; a.n = H->n;
  a.leaf_r0 = H->tree.leaf_r0; a.leaf_n = H->tree.leaf_n;
  a.u = u_next; a.bar = H->d_bar; a.st = H->d_status; a.trace = nullptr;
  sa.ctr = reinterpret_cast<unsigned*>(H->d_done);
  sa.done = H->d_done;
  for (int l = 0; l <= L; ++l) sa.dofs[l] = H->dofs[l];
  sa.lofs = H->lofs;
  sa.lf0 = pt.lf0; sa.lf1 = pt.lf1; sa.mlo = pt.mlo; sa.mhi = pt.mhi;
  sa.restrict_nodes = pt.restrict_nodes; sa.do_leaf = pt.do_leaf; sa.do_final = pt.do_final;
  static unsigned long long* step_trace = nullptr;
  if (fde_dbg_env("FDE_TRACE_STEP")) {
    if (!step_trace) CU(cudaMalloc(&step_trace, 16384 * sizeof(unsigned long long)));
    CU(cudaMemsetAsync(step_trace, 0, 16384 * sizeof(unsigned long long), s));
    sa.trace = step_trace;
  }
  CU(cudaMemsetAsync(H->d_done, 0, H->ndone * sizeof(int), s));
  void* args[] = {&sa};
  { PROF(prof_name); CU(cudaLaunchCooperativeKernel((void*)k_step, dim3(H->step_grid), dim3(TR_THREADS), args, H->step_smem, s)); }
  LAUNCHED();
  if (sa.trace) {
    std::vector<unsigned long long> h(16384);
    CU(cudaStreamSynchronize(s));
    CU(cudaMemcpy(h.data(), sa.trace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    FILE* fo = fopen(fde_dbg_env("FDE_TRACE_STEP"), "w");
    if (fo) {
      for (int i = 0; i < 4000; ++i)
        if (h[4 * i + 1]) fprintf(fo, "%d %llu %llu %llu %llu\n", i, h[4 * i], h[4 * i + 1], h[4 * i + 2], h[4 * i + 3]);
      fclose(fo);
    }
  }
  return FDE_OK;
}

// factor (nf = 0) or fused factor + solve of one rhs column (nf = 1: b = u + dt f -> u_next)
static int factor_impl(fde_hodlr* H, const double* dp, const double* dm, int nf, const double* u_prev,
                       const double* f, double* u_next, int keep, cudaStream_t s) {
  const int L = H->L, B = H->batch;
  if (L == 0 && nf == 0 && !keep) return FDE_OK;
  LeafArgs la{};
  la.tree = H->tree; la.mode = 0; la.shift = H->shift; la.cfac = H->d_cfac; la.dt = H->dt;
  la.g = H->d_g; la.gstride = H->gstride; la.dp = dp; la.dm = dm;
  la.Lf = H->d_Lf; la.lf_stride = H->lf_stride; la.rank = H->d_rank;
  for (int l = 0; l < L; ++l) { la.kl[l] = H->kl[l]; la.xcol[l] = H->xcol[l]; }
  la.xcol[L] = H->xcol[L];
  la.X = H->d_X; la.xstride = H->xstride; la.LU = H->d_LU; la.lustride = H->lustride;
  la.keep = keep; la.nf = nf; la.u_prev = u_prev; la.f = f; la.st = H->d_status;
  la.lmap = H->tma_ok ? H->d_tmaps : nullptr;
  la.xmap = H->tma_ok ? H->d_tmaps + (size_t)B * L : nullptr;
  TRY(trace_reset(s));
  la.trace = g_trace;
  const bool tree = nf == 1 && !keep && H->tree_ok && !fde_dbg_env("FDE_LEVEL_PASSES");
  if (tree) {
    la.Q = H->d_Q + H->qlev[L]; la.qinst = H->qinst;
    la.qstride = (long long)(H->xcol[L] - 1) * H->xcol[L];
  }
  if (tree && !fde_dbg_env("FDE_SPLIT_KERNELS")) {
    // one persistent dataflow launch: leaves -> tree levels -> u = X v (k_step.cuh)
    StepPart whole{0, H->nleaf, 0, L, 0, 1, 1};
    return launch_step(H, la, whole, u_next, s);
  }
  { PROF("k_leaf"); k_leaf<<<dim3(H->nleaf, B), LEAF_THREADS, LEAF_SMEM, s>>>(la); }
  LAUNCHED();
  if (tree) return launch_tree(H, u_next, s);
  TRY(launch_levels(H, 0, nf, nullptr, 0, 1, s));
  if (nf) {
    const long long tot = (long long)B * H->n;
    { PROF("k_copy_col0"); k_copy_col0<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(H->d_X, H->xstride, H->n, u_next, B); }
    LAUNCHED();
  }
  return FDE_OK;
}

// solve with the kept factor: y = A^{-1}(b + dt f) (f may be NULL), nrhs columns, ld
// (k_solve.cuh: explicit leaf inverses, then one streaming pass per level)
static int solve_impl(fde_hodlr* H, const double* b, const double* f, double* y, int nrhs, int ld,
                      cudaStream_t s) {
  const int L = H->L, B = H->batch;
  SaArgs sa{};
  sa.tree = H->tree; sa.Ainv = H->d_LU; sa.lustride = H->lustride; sa.b = b; sa.f = f; sa.dt = H->dt;
  sa.y = y; sa.nrhs = nrhs; sa.ld = ld;
  { PROF("k_leaf_apply"); k_leaf_apply<<<dim3(H->nleaf, B, std::max(1, std::min((nrhs + SA_COLS - 1) / SA_COLS, 16))), SA_THREADS, 0, s>>>(sa); }
  LAUNCHED();
  SlArgs sl{};
  sl.tree = H->tree; sl.Lf = H->d_Lf; sl.lf_stride = H->lf_stride; sl.rank = H->d_rank;
  sl.X = H->d_X; sl.xstride = H->xstride; sl.Kst = H->d_Kst; sl.kstride_inst = H->kstride_inst;
  sl.Y = y; sl.nrhs = nrhs; sl.ld = ld;
  for (int l = L - 1; l >= 0; --l) {
    sl.level = l; sl.k = H->kl[l]; sl.xcol = H->xcol[l]; sl.kofs = H->kofs[l];
    const long long nodes = (long long)B << l;
    const int node_rows = H->n >> l;
    // large nodes (>= 4096 rows) are cut into chunks of ~2048 rows, whatever the batch: an
    // instance's arithmetic must not depend on how many instances share the launch (the sharded
    // cfg4 slices are bitwise equal to the full batch, tests/test_parity_full.py)
    if (node_rows < 4096) {
      { PROF("k_solve_level"); k_solve_level<<<dim3(1 << l, B, std::max(1, std::min(nrhs, 32))), SL_THREADS, (size_t)3 * sl.k * sl.k * sizeof(double), s>>>(sl); }
      LAUNCHED();
      continue;
    }
    // few large nodes: several CTAs per node (k_solve_dots / _small / _update)
    SlSplitArgs sp{};
    sp.a = sl;
    sp.nch = node_rows / 2048;
    const size_t need = (size_t)nodes * sp.nch * 2 * KCAP + (size_t)nodes * 2 * KCAP;
    if (need > H->solve_split_cap) {
      if (H->d_solve_split) { cudaStreamSynchronize(s); cudaFree(H->d_solve_split); H->allocs.erase(std::find(H->allocs.begin(), H->allocs.end(), (void*)H->d_solve_split)); H->d_solve_split = nullptr; }
      TRY(dalloc(H, &H->d_solve_split, need));
      H->solve_split_cap = need;
    }
    sp.part = H->d_solve_split;
    sp.sv = H->d_solve_split + (size_t)nodes * sp.nch * 2 * KCAP;
    for (int c = 0; c < nrhs; ++c) {
      sp.c = c;
      { PROF("k_solve_dots"); k_solve_dots<<<dim3((1 << l) * sp.nch, B), SL_THREADS, 0, s>>>(sp); }
      LAUNCHED();
      { PROF("k_solve_small"); k_solve_small<<<dim3(1 << l, B), 32, 0, s>>>(sp); }
      LAUNCHED();
      { PROF("k_solve_update"); k_solve_update<<<dim3((1 << l) * sp.nch, B), SL_THREADS, 0, s>>>(sp); }
      LAUNCHED();
    }
  }
  return FDE_OK;
}

// y = A x with the HODLR representation
static int matvec_impl(fde_hodlr* H, const double* x, double* y, int nrhs, int ld, cudaStream_t s) {
  const int L = H->L, B = H->batch;
  MvArgs ma{};
  ma.tree = H->tree; ma.shift = H->shift; ma.cfac = H->d_cfac; ma.g = H->d_g; ma.gstride = H->gstride;
  ma.dp = H->d_dp; ma.dm = H->d_dm; ma.Lf = H->d_Lf; ma.lf_stride = H->lf_stride; ma.rank = H->d_rank;
  ma.x = x; ma.y = y; ma.nrhs = nrhs; ma.ld = ld; ma.ystride = (long long)ld * nrhs;
  ma.Ppart = H->d_P; ma.pstride_seg = H->pstride_seg; ma.pstride_inst = H->pstride_inst;
  { PROF("k_mv_leaf"); k_mv_leaf<<<dim3(H->nleaf, B), MV_THREADS, MV_LEAF_SMEM, s>>>(ma); }
  LAUNCHED();
  LevelArgs lv{};
  lv.tree = H->tree; lv.mode = 1; lv.Lf = H->d_Lf; lv.lf_stride = H->lf_stride;
  lv.rank = H->d_rank; lv.colofs = H->d_colofs;
  lv.Y = const_cast<double*>(x); lv.ld = ld; lv.nrhs = nrhs; lv.ystride = (long long)ld * nrhs;
  lv.Ppart = H->d_P; lv.pstride_seg = H->pstride_seg; lv.pstride_inst = H->pstride_inst;
  for (int l = L - 1; l >= 0; --l) {
    // levels are independent for a product, but the partial buffer is shared: sequential
    lv.level = l; ma.level = l;
    const int nseg = H->seg_ofs[l + 1] - H->seg_ofs[l];
    { PROF("k_lvl_reduce"); k_lvl_reduce<<<dim3(nseg, B), LVL_THREADS, SMEM_REDUCE, s>>>(lv); }
    LAUNCHED();
    { PROF("k_mv_update"); k_mv_update<<<dim3(nseg, B), MV_THREADS, SMEM_MV_UPDATE, s>>>(ma); }
    LAUNCHED();
  }
  return FDE_OK;
}

// ---------------------------------------------------------------------------------------
// ---- TMA tensor maps (cuTensorMapEncodeTiled through the runtime's driver entry point) ----
static PFN_cuTensorMapEncodeTiled_v12000 g_tmap_encode = nullptr;
static bool tmap_encode(CUtensorMap* m, int rank, void* base, const cuuint64_t* dims,
                        const cuuint64_t* strides_bytes, const cuuint32_t* box) {
  if (!g_tmap_encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      return false;
    }
    g_tmap_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint32_t estr[3] = {1, 1, 1};
  return g_tmap_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)rank, base, dims, strides_bytes, box,
                       estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// X map of one panel buffer (slot B*L or B*L+1 of d_tmaps)
static bool tmap_x(fde_hodlr* H, int slot, double* X, CUtensorMap* out) {
  const int NC = H->xcol[H->L];
  if ((H->n & 1) || (reinterpret_cast<unsigned long long>(X) & 15)) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)H->n, (cuuint64_t)NC, (cuuint64_t)H->batch};
  const cuuint64_t str[2] = {(cuuint64_t)H->n * 8, (cuuint64_t)H->xstride * 8};
  const cuuint32_t box[3] = {(cuuint32_t)LEAF_LDV, 16, 1};
  (void)slot;
  return tmap_encode(out, 3, X, dims, str, box);
}
// All maps of a handle after the layout (ranks known): L maps + the X map of d_X (+ d_X2 if any).
static int tmaps_build(fde_hodlr* H, const std::vector<int>& rk) {
  const int L = H->L, B = H->batch;
  H->tma_ok = false;
  if (L == 0) return FDE_OK;
  std::vector<CUtensorMap> m((size_t)B * L + 2);
  bool ok = true;
  for (int b = 0; b < B && ok; ++b)
    for (int l = 0; l < L && ok; ++l) {
      const int r = rk[(size_t)b * L + l], ml = H->lev_m[l];
      if (r == 0) continue;
      double* base = H->d_Lf + (long long)b * H->lf_stride + H->lev_lofs[l];
      if ((ml & 1) || (reinterpret_cast<unsigned long long>(base) & 15)) { ok = false; break; }
      const cuuint64_t dims[2] = {(cuuint64_t)ml, (cuuint64_t)r};
      const cuuint64_t str[1] = {(cuuint64_t)ml * 8};
      const cuuint32_t box[2] = {(cuuint32_t)LEAF_LDV, (cuuint32_t)r};
      ok = tmap_encode(&m[(size_t)b * L + l], 2, base, dims, str, box);
    }
  ok = ok && tmap_x(H, B * L, H->d_X, &m[(size_t)B * L]);
  if (ok && H->d_X2) ok = tmap_x(H, B * L + 1, H->d_X2, &m[(size_t)B * L + 1]);
  if (!ok) return FDE_OK;                            // (the cp.async projection is used)
  if (!H->d_tmaps) {
    void* q = nullptr;
    CU(cudaMalloc(&q, m.size() * sizeof(CUtensorMap)));
    H->allocs.push_back(q);
    H->d_tmaps = reinterpret_cast<CUtensorMap*>(q);
  }
  CU(cudaMemcpy(H->d_tmaps, m.data(), m.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  H->tma_ok = true;
  return FDE_OK;
}
// the map of X2 once the pipelined run allocates it
static int tmaps_add_x2(fde_hodlr* H) {
  if (!H->tma_ok) return FDE_OK;
  CUtensorMap mx;
  if (!tmap_x(H, H->batch * H->L + 1, H->d_X2, &mx)) { H->tma_ok = false; return FDE_OK; }
  CU(cudaMemcpy(H->d_tmaps + (size_t)H->batch * H->L + 1, &mx, sizeof(mx), cudaMemcpyHostToDevice));
  return FDE_OK;
}

// C-ABI
// One k_run launch of K <= RUN_KMAX pipelined steps: u_out[m] = A_m^{-1}(u^(m-1) + dt f^(m)),
// u^(-1) = u0 (the caller's chunk base pointers).
// inv: the coefficients are the same every step (coef_stride 0, no FDE_REFACTOR): factor once at
// step 0, then only the rhs column per step (k_run.cuh, RunArgs::inv).
static int run_chunk(fde_hodlr* H, int K, double dt, const double* d_plus, const double* d_minus,
                     long long coef_stride, const double* f, long long f_stride, const double* u0,
                     double* u_out, bool inv, cudaStream_t s) {
  const size_t cnt = (size_t)H->batch * H->n;
  const int L = H->L, B = H->batch;
  // second buffer set + stored leaf LUs (allocated once per handle)
  if (!H->d_X2) {
    TRY(dalloc(H, &H->d_X2, (size_t)B * H->xstride));
    TRY(dalloc(H, &H->d_Q2, (size_t)B * H->qinst));
    TRY(dalloc(H, &H->d_S2, (size_t)B * H->sinst));
    H->lurstride = (long long)H->nleaf * LEAF_RSLOT;
    TRY(dalloc(H, &H->d_LUr[0], (size_t)B * H->lurstride));
    TRY(dalloc(H, &H->d_LUr[1], (size_t)B * H->lurstride));
    TRY(tmaps_add_x2(H));
  }
  if (!H->d_Kr[0]) {                                 // split units: [C | Sc^-1 | G] per node, 2 parities
    long long ko = 0;
    for (int m = 0; m < L; ++m) { H->krlev[m] = ko; ko += (1LL << m) * 3LL * H->kl[m] * H->kl[m]; }
    H->krinst = std::max(1LL, ko);
    TRY(dalloc(H, &H->d_Kr[0], (size_t)B * H->krinst));
    TRY(dalloc(H, &H->d_Kr[1], (size_t)B * H->krinst));
  }
  // per-step counters: A done [n_leaf], B' done [n_leaf], pair counters [B 2^(L-1)], per
  // level m: chunk completions [B 2^m] and completed children [B 2^m]; ready queue: one slot
  // per tree unit of the run
  const long long n_leaf = (long long)B * H->nleaf;
  RunArgs ra{};
  // split tree units: per node a U unit (all columns but the right-hand side, off the
  // step-to-step chain) and an R unit (the right-hand-side column, on it) -- k_tree.cuh tr_unit_R.
  // It shortens the chain of latency-bound runs and costs ~25 us of SM time per step (511 more
  // small tasks at cfg3): measured (tools/small_cfgs.py, us/step, unsplit -> split) cfg1 64 -> 53,
  // cfg2 153 -> 117, n=8192 138 -> 124, n=16384 194 -> 167, n=32768 287 -> 288, cfg3 618 -> 638;
  // so split while the run has fewer than 2 leaves per SM.
  {
    int dev = 0, nsm = 148;
    CU(cudaGetDevice(&dev));
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    ra.split = (long long)B * H->nleaf < 2LL * nsm;
  }
  if (const char* e = fde_dbg_env("FDE_RUN_SPLIT")) ra.split = atoi(e) != 0;   // (diagnostics build)
  // whole tree units: the projection (B) runs inside the B' task of the same leaf (one V staging,
  // Q[:, 0] from it); split units keep B separate (its U unit stays off the step chain)
  ra.fuse = ra.split ? 0 : 1;
  if (const char* e = fde_dbg_env("FDE_RUN_FUSE")) ra.fuse = !ra.split && atoi(e) != 0;   // (diagnostics)
  // factor once: the later steps are the rhs column alone, which needs the U / R unit split
  ra.inv = inv ? 1 : 0;
  if (inv) { ra.split = 1; ra.fuse = 0; }
  long long o = 0, units = 0;
  ra.o_A = o; o += n_leaf;
  ra.o_R = o; o += n_leaf;
  for (int m = 0; m < L; ++m) {
    ra.o_lvl[m] = o; o += (long long)B << m;
    ra.o_ku[m] = o; o += (long long)B << m;
    ra.o_kr[m] = o; o += (long long)B << m;
    units += ((long long)B << m) * (ra.split ? 2 : 1);
  }
  ra.per_step = o;
  const long long need = 4 + (long long)K * o;
  if (need > H->runctr_cap) {
    if (H->d_runctr) { cudaStreamSynchronize(s); cudaFree(H->d_runctr); H->allocs.erase(std::find(H->allocs.begin(), H->allocs.end(), (void*)H->d_runctr)); }
    TRY(dalloc(H, &H->d_runctr, (size_t)need));
    H->runctr_cap = need;
  }
  const long long nrq = (long long)K * units;
  if (nrq > H->runrq_cap) {
    if (H->d_runrq) { cudaStreamSynchronize(s); cudaFree(H->d_runrq); H->allocs.erase(std::find(H->allocs.begin(), H->allocs.end(), (void*)H->d_runrq)); }
    TRY(dalloc(H, &H->d_runrq, (size_t)nrq));
    H->runrq_cap = nrq;
  }
  CU(cudaMemsetAsync(H->d_runctr, 0, need * sizeof(int), s));
  CU(cudaMemsetAsync(H->d_runrq, 0, nrq * sizeof(unsigned long long), s));
  ra.heads = reinterpret_cast<unsigned*>(H->d_runctr);
  ra.done = H->d_runctr + 4;
  ra.rq = H->d_runrq;
  ra.rq_cap = nrq;
  ra.use_rq = ra.split;
  // per-step argument blocks (k_run.cuh RunArgs), copied to the device once per call
  LeafArgs la{};
  la.tree = H->tree; la.mode = 0; la.shift = H->shift; la.cfac = H->d_cfac; la.dt = dt;
  la.g = H->d_g; la.gstride = H->gstride;
  la.Lf = H->d_Lf; la.lf_stride = H->lf_stride; la.rank = H->d_rank;
  for (int l = 0; l < L; ++l) { la.kl[l] = H->kl[l]; la.xcol[l] = H->xcol[l]; }
  la.xcol[L] = H->xcol[L];
  la.xstride = H->xstride; la.lustride = H->lurstride; la.keep = 0; la.st = H->d_status;
  la.qinst = H->qinst; la.qstride = (long long)(H->xcol[L] - 1) * H->xcol[L];
  la.trace = nullptr; la.nf = 0; la.store_lu = 1;
  TrArgs a = H->tr_geo;
  a.L = L; a.NC = H->xcol[L]; a.nleaf = H->nleaf; a.batch = B; a.kmaxc = H->kmax;
  for (int l = 0; l <= L; ++l) a.xc[l] = H->xcol[l];
  for (int m = 0; m < L; ++m) { a.rc[m] = H->trc[m]; a.slev[m] = H->slev[m]; }
  for (int m = 1; m <= L; ++m) a.qlev[m] = H->qlev[m];
  a.qinst = H->qinst; a.sinst = H->sinst;
  a.n = H->n; a.xstride = H->xstride;
  a.leaf_r0 = H->tree.leaf_r0; a.leaf_n = H->tree.leaf_n;
  a.bar = H->d_bar; a.st = H->d_status; a.trace = nullptr;
  double* Xp[2] = {H->d_X, H->d_X2};
  double* Qp[2] = {H->d_Q, H->d_Q2};
  double* Sp[2] = {H->d_S, H->d_S2};
  H->run_las.resize(K);
  H->run_tas.resize(K);
  for (int m = 0; m < K; ++m) {
    const int p = inv ? 0 : (m & 1);                 // (factor once: one buffer set, k_run.cuh)
    LeafArgs& lm = H->run_las[m];
    lm = la;
    lm.dp = d_plus + m * coef_stride; lm.dm = d_minus + m * coef_stride; lm.f = f + m * f_stride;
    lm.u_prev = m == 0 ? u0 : u_out + (m - 1) * cnt;
    lm.X = Xp[p]; lm.LU = H->d_LUr[p]; lm.Q = Qp[p] + H->qlev[L];
    lm.lmap = H->tma_ok ? H->d_tmaps : nullptr;
    lm.xmap = H->tma_ok ? H->d_tmaps + (size_t)B * L + p : nullptr;
    TrArgs& tm = H->run_tas[m];
    tm = a;
    // one unit per node in the pipelined run: the row-chunk split that shortens k_step's exposed
    // tree chain would put the extra chunks in the ready queue, where they wait for a CTA to
    // come free from leaf work; measured 630 vs 663 us/step at cfg3
    for (int l = 0; l < L; ++l) tm.rc[l] = 1;
    tm.Q = Qp[p]; tm.Qleaf = Qp[p] + H->qlev[L]; tm.Sst = Sp[p]; tm.X = Xp[p];
    // B' prefetches X^(m-1) of its leaf into L2 (k_final.cuh) when the X buffer cannot stay
    // L2-resident for a step (> 48 MB; 126 MB L2 shared with the stored LU, Q, S traffic):
    // A/B (tools/gpu_s39.sh) cfg3 541 -> 538 us/step, cfg4 pipelined refactor 486 -> 483 ms;
    // cfg1 (88 KB of X) +1 us/step with it, so small buffers skip it
    tm.xmap = (double)B * H->xstride * 8.0 > 48e6 ? lm.xmap : nullptr;
    tm.Kr = ra.split ? H->d_Kr[p] : nullptr; tm.krinst = H->krinst;
    for (int l = 0; l < L; ++l) tm.krlev[l] = H->krlev[l];
    tm.u = u_out + m * cnt;
  }
  static unsigned long long* run_trace = nullptr;
  const long long run_trace_len = 4 + 4 * 262144;
  if (fde_dbg_env("FDE_TRACE_RUN")) {
    if (!run_trace) CU(cudaMalloc(&run_trace, run_trace_len * sizeof(unsigned long long)));
    CU(cudaMemsetAsync(run_trace, 0, run_trace_len * sizeof(unsigned long long), s));
    ra.trace = run_trace; ra.trace_cap = 262144;
    static unsigned long long* run_prof = nullptr;
    if (!run_prof) CU(cudaMalloc(&run_prof, 1200 * sizeof(unsigned long long)));
    CU(cudaMemsetAsync(run_prof, 0, 1200 * sizeof(unsigned long long), s));
    ra.prof = run_prof;
    for (int m = 0; m < K; ++m) { H->run_las[m].prof = run_prof + 16; H->run_tas[m].trace = run_prof; }
  }
  const size_t args_bytes = (size_t)K * (sizeof(LeafArgs) + sizeof(TrArgs));
  if (args_bytes > H->run_args_cap) {
    if (H->d_run_args) { cudaStreamSynchronize(s); cudaFree(H->d_run_args); H->allocs.erase(std::find(H->allocs.begin(), H->allocs.end(), H->d_run_args)); }
    H->d_run_args = nullptr;
    CU(cudaMalloc(&H->d_run_args, args_bytes));
    H->allocs.push_back(H->d_run_args);
    H->run_args_cap = args_bytes;
  }
  // (host blocks are owned by the handle: they stay valid while the asynchronous copy reads them)
  CU(cudaMemcpyAsync(H->d_run_args, H->run_las.data(), K * sizeof(LeafArgs), cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync((char*)H->d_run_args + K * sizeof(LeafArgs), H->run_tas.data(), K * sizeof(TrArgs),
                     cudaMemcpyHostToDevice, s));
  ra.las = reinterpret_cast<const LeafArgs*>(H->d_run_args);
  ra.tas = reinterpret_cast<const TrArgs*>((char*)H->d_run_args + K * sizeof(LeafArgs));
  ra.K = K;
  ra.smem_doubles = (int)(H->step_smem / sizeof(double));
  CU(cudaFuncSetAttribute(k_run, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)H->step_smem));
  void* args[] = {&ra};
  { PROF("k_run"); CU(cudaLaunchCooperativeKernel((void*)k_run, dim3(H->step_grid), dim3(TR_THREADS), args, H->step_smem, s)); }
  LAUNCHED();
  if (ra.trace) {                                 // FDE_TRACE_RUN=<file>: task timeline
    std::vector<unsigned long long> h(run_trace_len);
    CU(cudaStreamSynchronize(s));
    CU(cudaMemcpy(h.data(), ra.trace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    std::vector<unsigned long long> pf(1200);
    CU(cudaMemcpy(pf.data(), ra.prof, 1200 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    for (int g = 0; g < 2; ++g) {
      const unsigned long long* q = pf.data() + 1100 + 8 * g;
      const double c = (double)std::max(1ULL, q[7]) * 1965.0;
      fprintf(stderr, "k_run tree %s units (%llu): stage %.2f sc+T %.2f gj %.2f S %.2f Qupd %.2f (issue %.2f wait %.2f) us\n",
              g ? "upper" : "bottom", q[7], q[0] / c, q[1] / c, q[2] / c, q[3] / c, q[4] / c, q[5] / c, q[6] / c);
    }
    {
      const double c = (double)K * B * H->nleaf * 1965.0;
      fprintf(stderr, "k_run A phases (us avg per leaf): build+gj0 %.2f lu+store %.2f panel %.2f\n",
              pf[16] / c, pf[17] / c, pf[20] / c);
      fprintf(stderr, "k_run A panel, warp 0 (us avg per leaf): gather+scale %.2f acc-init %.2f solve %.2f store %.2f\n",
              pf[21] / c, pf[22] / c, pf[23] / c, pf[24] / c);
      fprintf(stderr, "k_run A panel, warp 0 first-stripe gather+scale %.2f us\n", pf[25] / c);
      const double cb = (double)std::max(1ULL, pf[27]) * 1965.0;
      fprintf(stderr, "k_run B phases (us avg over %llu): V+X staging %.2f dmma %.2f\n",
              pf[27], pf[25] / cb, pf[26] / cb);
      fprintf(stderr, "k_run B tma (warp 1, us avg): setup %.2f Vwait+swap %.2f compute %.2f fullwait %.2f tail-sync %.2f\n",
              pf[28] / cb, pf[29] / cb, pf[30] / cb, pf[31] / cb, pf[32] / cb);
    }
    for (int g = 0; g < 2; ++g) {
      const double c = (double)std::max(1ULL, pf[8 * g + 7]);
      fprintf(stderr, "k_run %s phases (us avg over %llu): issue %.2f S %.2f v %.2f Xv %.2f LUwait %.2f solve %.2f x0+Q0 %.2f\n",
              g ? "final-only" : "B'", pf[8 * g + 7], pf[8 * g + 6] / c / 1965.0, pf[8 * g + 1] / c / 1965.0, pf[8 * g + 2] / c / 1965.0,
              pf[8 * g + 3] / c / 1965.0, pf[8 * g + 4] / c / 1965.0, pf[8 * g + 5] / c / 1965.0, pf[8 * g] / c / 1965.0);
    }
    FILE* fo = fopen(fde_dbg_env("FDE_TRACE_RUN"), "w");
    if (fo) {
      const long long ne = std::min<long long>((long long)h[0], ra.trace_cap);
      for (long long e = 0; e < ne; ++e)
        fprintf(fo, "%llu %llu %llu %llu\n", h[4 + 4 * e], h[5 + 4 * e], h[6 + 4 * e], h[7 + 4 * e]);
      fclose(fo);
    }
  }
  return FDE_OK;
}

extern "C" {

const char* fde_last_error(void) { return g_last_error.c_str(); }

void fde_profile_enable(int on) {
  if (!on) {
    for (auto& r : g_prof_recs) { g_ev_free.push_back(r.a); g_ev_free.push_back(r.b); }
    g_prof_recs.clear();
  }
  g_prof = on != 0;
}

int fde_profile_dump(char* buf, int len) {
  // aggregate per kernel name: {"name": [launches, total_ms], ...}; clears the records
  std::vector<std::pair<std::string, std::pair<long long, double>>> agg;
  for (auto& r : g_prof_recs) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    bool found = false;
    for (auto& e : agg)
      if (e.first == r.name) { e.second.first++; e.second.second += ms; found = true; break; }
    if (!found) agg.push_back({r.name, {1, (double)ms}});
    g_ev_free.push_back(r.a);
    g_ev_free.push_back(r.b);
  }
  g_prof_recs.clear();
  std::string out = "{";
  for (size_t i = 0; i < agg.size(); ++i) {
    char tmp[256];
    snprintf(tmp, sizeof(tmp), "%s\"%s\": [%lld, %.6f]", i ? ", " : "", agg[i].first.c_str(),
             agg[i].second.first, agg[i].second.second);
    out += tmp;
  }
  out += "}";
  if (!buf || len <= (int)out.size()) return -(int)out.size() - 1;
  memcpy(buf, out.c_str(), out.size() + 1);
  return (int)out.size();
}
long long fde_launch_count(void) { return g_launches.load(); }

int hodlr_build(int batch, int n, const double* alpha, double h, double dt, const double* d_plus,
                const double* d_minus, double shift, double tol, int leaf, unsigned flags, void* stream,
                fde_hodlr_t* out) {
  g_last_error.clear();
  if (!d_plus || !d_minus) return set_err(FDE_EDOMAIN, "d_plus / d_minus is NULL");
  return build_impl(batch, n, alpha, h, dt, d_plus, d_minus, shift, tol, leaf, flags,
                    (cudaStream_t)stream, out);
}

int hodlr_update(fde_hodlr_t H, double dt, const double* d_plus, const double* d_minus, unsigned flags,
                 void* stream) {
  g_last_error.clear();
  if (!H) return set_err(FDE_EDOMAIN, "handle is NULL");
  if (H->compress_only) return set_err(FDE_EDIM, "handle built with FDE_COMPRESS_ONLY");
  if (!(dt >= 0.0) || !std::isfinite(dt)) return set_err(FDE_EDOMAIN, "dt=%g must be >= 0", dt);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bytes = (size_t)H->batch * H->n * sizeof(double);
  if (d_plus) CU(cudaMemcpyAsync(H->d_dp, d_plus, bytes, cudaMemcpyDeviceToDevice, s));
  if (d_minus) CU(cudaMemcpyAsync(H->d_dm, d_minus, bytes, cudaMemcpyDeviceToDevice, s));
  if (flags & FDE_CHECK) TRY(check_nonneg(H, H->d_dp, H->d_dm, s));
  TRY(set_dt(H, dt, s));
  H->factored = false;
  H->last_stream = s;
  if (flags & FDE_SYNC) return sync_and_status(H, s);
  return FDE_OK;
}

int hodlr_factor(fde_hodlr_t H, unsigned flags, void* stream) {
  g_last_error.clear();
  if (!H) return set_err(FDE_EDOMAIN, "handle is NULL");
  if (H->compress_only) return set_err(FDE_EDIM, "handle built with FDE_COMPRESS_ONLY");
  cudaStream_t s = (cudaStream_t)stream;
  TRY(factor_impl(H, H->d_dp, H->d_dm, 0, nullptr, nullptr, nullptr, 1, s));
  H->factored = true;
  H->last_stream = s;
  if (flags & FDE_SYNC) return sync_and_status(H, s);
  return FDE_OK;
}

int hodlr_solve(fde_hodlr_t H, const double* b, double* x, int nrhs, int ld, unsigned flags, void* stream) {
  g_last_error.clear();
  if (!H) return set_err(FDE_EDOMAIN, "handle is NULL");
  if (H->compress_only) return set_err(FDE_EDIM, "handle built with FDE_COMPRESS_ONLY");
  if (!H->factored) return set_err(FDE_EDOMAIN, "hodlr_solve before hodlr_factor");
  if (!b || !x) return set_err(FDE_EDOMAIN, "b / x is NULL");
  if (nrhs < 1 || nrhs > NRHS_MAX) return set_err(FDE_EDIM, "nrhs=%d outside [1, %d]", nrhs, NRHS_MAX);
  if (ld < H->n) return set_err(FDE_EDIM, "ld=%d < n=%d", ld, H->n);
  cudaStream_t s = (cudaStream_t)stream;
  TRY(solve_impl(H, b, nullptr, x, nrhs, ld, s));
  H->last_stream = s;
  if (flags & FDE_SYNC) return sync_and_status(H, s);
  return FDE_OK;
}

int hodlr_matvec(fde_hodlr_t H, const double* x, double* y, int nrhs, int ld, unsigned flags, void* stream) {
  g_last_error.clear();
  if (!H) return set_err(FDE_EDOMAIN, "handle is NULL");
  if (H->compress_only) return set_err(FDE_EDIM, "handle built with FDE_COMPRESS_ONLY");
  if (!x || !y) return set_err(FDE_EDOMAIN, "x / y is NULL");
  if (x == y) return set_err(FDE_EDOMAIN, "y must not alias x");
  if (nrhs < 1 || nrhs > NRHS_MAX) return set_err(FDE_EDIM, "nrhs=%d outside [1, %d]", nrhs, NRHS_MAX);
  if (ld < H->n) return set_err(FDE_EDIM, "ld=%d < n=%d", ld, H->n);
  cudaStream_t s = (cudaStream_t)stream;
  TRY(matvec_impl(H, x, y, nrhs, ld, s));
  H->last_stream = s;
  if (flags & FDE_SYNC) return sync_and_status(H, s);
  return FDE_OK;
}

int hodlr_status(fde_hodlr_t H, int* where) {
  if (!H) return set_err(FDE_EDOMAIN, "handle is NULL");
  DevStatus st{};
  CU(cudaStreamSynchronize(H->last_stream));
  TRY(read_status(H, &st));
  if (where) *where = st.where;
  return st.code;
}

int hodlr_ranks(fde_hodlr_t H, int inst, int* ranks, int max_levels, int* levels) {
  if (!H) return set_err(FDE_EDOMAIN, "handle is NULL");
  if (inst < 0 || inst >= H->batch) return set_err(FDE_EDOMAIN, "inst=%d outside [0, %d)", inst, H->batch);
  if (levels) *levels = H->L;
  if (H->L == 0) return FDE_OK;
  if (!ranks || max_levels < H->L) return set_err(FDE_EDIM, "ranks buffer holds %d < L=%d", max_levels, H->L);
  CU(cudaStreamSynchronize(H->last_stream));
  CU(cudaMemcpy(ranks, H->d_rank + (size_t)inst * H->L, H->L * sizeof(int), cudaMemcpyDeviceToHost));
  return FDE_OK;
}

void hodlr_destroy(fde_hodlr_t H) {
  if (!H) return;
  cudaStreamSynchronize(H->last_stream);
  free_handle(H);
}

int fde1d_step(int batch, int n, const double* alpha, double h, double dt, const double* d_plus_m,
               const double* d_minus_m, const double* f_m, const double* u_prev, double* u_next, double tol,
               int leaf, int coeffs_changed, unsigned flags, fde_hodlr_t* cache, void* stream) {
  g_last_error.clear();
  TRY(check_common(batch, n, alpha, h, dt, tol, leaf));
  if (!d_plus_m || !d_minus_m || !f_m || !u_prev || !u_next)
    return set_err(FDE_EDOMAIN, "NULL array argument");
  cudaStream_t s = (cudaStream_t)stream;
  fde_hodlr* H = cache ? *cache : nullptr;
  bool fresh = false;
  if (H) {
    bool same = H->batch == batch && H->n == n && H->h == h && H->leaf == leaf && H->tol == tol &&
                H->shift == 1.0;
    for (int b = 0; same && b < batch; ++b) same = H->alpha[b] == alpha[b];
    if (!same) { hodlr_destroy(H); H = nullptr; if (cache) *cache = nullptr; }
  }
  const size_t cnt = (size_t)batch * n, bytes = cnt * sizeof(double);
  const double *dp = d_plus_m, *dm = d_minus_m, *f = f_m, *u = u_prev;
  double* un = u_next;
  if (!H) {
    TRY(build_impl(batch, n, alpha, h, dt, nullptr, nullptr, 1.0, tol, leaf, 0, s, &H));
    fresh = true;
    if (cache) *cache = H;
  }
  if (flags & FDE_HOST_PTRS) {
    double* st = H->d_in;
    CU(cudaMemcpyAsync(st, d_plus_m, bytes, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(st + cnt, d_minus_m, bytes, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(st + 2 * cnt, f_m, bytes, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(st + 3 * cnt, u_prev, bytes, cudaMemcpyHostToDevice, s));
    dp = st; dm = st + cnt; f = st + 2 * cnt; u = st + 3 * cnt;
    un = st + 3 * cnt;                                     // in place in the staging area
  }
  if ((flags & FDE_CHECK)) TRY(check_nonneg(H, dp, dm, s));
  if ((flags & FDE_RECOMPRESS) && !fresh) {               // S1 + S2 again, same workspaces
    TRY(launch_gl(H, s));
    TRY(run_compression(H, s));
  }
  int rc;
  if (coeffs_changed || fresh || !H->factored || H->dt != dt) {   // A_m depends on dt too
    if (H->dt != dt || fresh) TRY(set_dt(H, dt, s));
    const int keep = (flags & FDE_NO_KEEP) ? 0 : 1;
    rc = factor_impl(H, dp, dm, 1, u, f, un, keep, s);
    H->factored = keep && rc == FDE_OK;
  } else {
    rc = solve_impl(H, u, f, un, 1, n, s);                 // LU reuse
  }
  if (rc != FDE_OK) { if (!cache) hodlr_destroy(H); return rc; }
  if (flags & FDE_HOST_PTRS) CU(cudaMemcpyAsync(u_next, un, bytes, cudaMemcpyDeviceToHost, s));
  H->last_stream = s;
  if ((flags & FDE_SYNC) || !cache || (flags & FDE_HOST_PTRS)) rc = sync_and_status(H, s);
  if (!cache) hodlr_destroy(H);
  return rc;
}

int fde1d_step_split(int world, int rank, fde_allgather_fn gather, void* ctx, int n, double alpha, double h,
                     double dt, const double* d_plus_m, const double* d_minus_m, const double* f_m,
                     const double* u_prev, double* u_next, double tol, int leaf, unsigned flags,
                     fde_hodlr_t* cache, void* stream) {
  g_last_error.clear();
  TRY(check_common(1, n, &alpha, h, dt, tol, leaf));
  if (world < 1 || (world & (world - 1))) return set_err(FDE_EDOMAIN, "world=%d must be a power of two", world);
  if (rank < -1 || rank >= world) return set_err(FDE_EDOMAIN, "rank=%d outside [-1, %d)", rank, world);
  if (rank >= 0 && world > 1 && !gather) return set_err(FDE_EDOMAIN, "world > 1 needs an all-gather callback");
  if (!d_plus_m || !d_minus_m || !f_m || !u_prev || !u_next) return set_err(FDE_EDOMAIN, "NULL array argument");
  if (u_next == u_prev) return set_err(FDE_EDOMAIN, "u_next must not alias u_prev");
  cudaStream_t s = (cudaStream_t)stream;
  fde_hodlr* H = cache ? *cache : nullptr;
  if (H) {
    const bool same = H->batch == 1 && H->n == n && H->h == h && H->leaf == leaf && H->tol == tol &&
                      H->shift == 1.0 && H->alpha[0] == alpha && !H->compress_only;
    if (!same) { hodlr_destroy(H); H = nullptr; if (cache) *cache = nullptr; }
  }
  if (!H) {
    TRY(build_impl(1, n, &alpha, h, dt, nullptr, nullptr, 1.0, tol, leaf, 0, s, &H));
    if (cache) *cache = H;
  }
  auto out = [&](int rc) { if (!cache) hodlr_destroy(H); return rc; };
  int p = 0;
  while ((1 << p) < world) ++p;
  const int L = H->L, NL = H->nleaf;
  if (!H->tree_ok || L < p || NL % world != 0)
    return out(set_err(FDE_EDIM, "the split needs the tree path with L >= log2(world) (L=%d, world=%d)", L, world));
  for (int i = 1; i < NL; ++i)
    if (H->leaf_n[i] != H->leaf_n[0]) return out(set_err(FDE_EDIM, "the split needs equal leaves (n = leaves x leaf)"));
  if (H->dt != dt) { const int rc = set_dt(H, dt, s); if (rc) return out(rc); }
  LeafArgs la{};
  la.tree = H->tree; la.mode = 0; la.shift = H->shift; la.cfac = H->d_cfac; la.dt = dt;
  la.g = H->d_g; la.gstride = H->gstride; la.dp = d_plus_m; la.dm = d_minus_m;
  la.Lf = H->d_Lf; la.lf_stride = H->lf_stride; la.rank = H->d_rank;
  for (int l = 0; l < L; ++l) { la.kl[l] = H->kl[l]; la.xcol[l] = H->xcol[l]; }
  la.xcol[L] = H->xcol[L];
  la.X = H->d_X; la.xstride = H->xstride; la.LU = H->d_LU; la.lustride = H->lustride;
  la.keep = 0; la.nf = 1; la.u_prev = u_prev; la.f = f_m; la.st = H->d_status;
  la.Q = H->d_Q + H->qlev[L]; la.qinst = H->qinst; la.qstride = (long long)(H->xcol[L] - 1) * H->xcol[L];
  const int per = NL / world;
  int rc = FDE_OK;
  if (rank < 0) {
    // every part in this process, one after the other (no part waits on another's launch):
    // the same launches the ranks of a world-sized split run, for checking and per-part timing
    for (int g = 0; g < world && rc == FDE_OK; ++g)
      rc = launch_step(H, la, StepPart{g * per, (g + 1) * per, p, L, 1, 1, 0}, nullptr, s, "k_step_part");
    if (rc == FDE_OK) rc = launch_step(H, la, StepPart{0, NL, 0, p, 0, 0, 1}, u_next, s, "k_step_top");
  } else {
    if (!H->d_split) {
      const long long qs = (long long)(H->xcol[p] - 1) * H->xcol[p];
      rc = dalloc(H, &H->d_split, (size_t)std::max<long long>(qs, n));
    }
    // 1. the part's leaves and its subtree (levels p .. L-1)
    if (rc == FDE_OK) rc = launch_step(H, la, StepPart{rank * per, (rank + 1) * per, p, L, 1, 1, 0}, nullptr, s, "k_step_part");
    // 2. the level-p projected matrices of the subtree roots, node g from rank g (P:1169-1177:
    //    every lower block is a sub-block of the top-level ones; the top levels couple the parts
    //    only through these (xc_p - 1) x xc_p matrices)
    if (rc == FDE_OK && world > 1) {
      const long long qs = (long long)(H->xcol[p] - 1) * H->xcol[p];
      double* Qp = H->d_Q + H->qlev[p];
      if (cudaMemcpyAsync(H->d_split, Qp + rank * qs, qs * sizeof(double), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        rc = set_err(FDE_ECUDA, "split staging copy failed");
      else if (gather(ctx, H->d_split, Qp, qs, s) != 0)
        rc = set_err(FDE_ECUDA, "split exchange callback failed");
    }
    // 3. the top levels 0 .. p-1 (every rank, same data: same S) and the part's finals
    if (rc == FDE_OK) rc = launch_step(H, la, StepPart{rank * per, (rank + 1) * per, 0, p, 0, 0, 1}, u_next, s, "k_step_top");
    // 4. u_next rows of every part
    if (rc == FDE_OK && world > 1) {
      const long long rows = (long long)n / world;
      if (cudaMemcpyAsync(H->d_split, u_next + rank * rows, rows * sizeof(double), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        rc = set_err(FDE_ECUDA, "split staging copy failed");
      else if (gather(ctx, H->d_split, u_next, rows, s) != 0)
        rc = set_err(FDE_ECUDA, "split exchange callback failed");
    }
  }
  if (rc != FDE_OK) return out(rc);
  H->last_stream = s;
  H->factored = false;
  if ((flags & FDE_SYNC) || !cache) rc = sync_and_status(H, s);
  return out(rc);
}

int fde1d_run(int batch, int n, const double* alpha, double h, double dt, int K, const double* d_plus,
              const double* d_minus, long long coef_stride, const double* f, long long f_stride,
              const double* u0, double* u_out, double tol, int leaf, unsigned flags, fde_hodlr_t* cache,
              void* stream) {
  g_last_error.clear();
  TRY(check_common(batch, n, alpha, h, dt, tol, leaf));
  if (K < 1) return set_err(FDE_EDOMAIN, "K=%d must be >= 1", K);
  if (!d_plus || !d_minus || !f || !u0 || !u_out) return set_err(FDE_EDOMAIN, "NULL array argument");
  if (coef_stride < 0 || f_stride < 0) return set_err(FDE_EDOMAIN, "negative stride");
  cudaStream_t s = (cudaStream_t)stream;
  fde_hodlr* H = cache ? *cache : nullptr;
  if (H) {
    bool same = H->batch == batch && H->n == n && H->h == h && H->leaf == leaf && H->tol == tol &&
                H->shift == 1.0;
    for (int b = 0; same && b < batch; ++b) same = H->alpha[b] == alpha[b];
    if (!same) { hodlr_destroy(H); H = nullptr; if (cache) *cache = nullptr; }
  }
  if (!H) {
    TRY(build_impl(batch, n, alpha, h, dt, nullptr, nullptr, 1.0, tol, leaf, 0, s, &H));
    if (cache) *cache = H;
  }
  const size_t cnt = (size_t)batch * n;
  int rc = FDE_OK;
  if (flags & FDE_HOST_PTRS) {
    // host arrays: stage them on the device (H2D on `stream`), run, copy every step's solution back
    if ((coef_stride != 0 && coef_stride != (long long)cnt) || (f_stride != 0 && f_stride != (long long)cnt)) {
      if (!cache) hodlr_destroy(H);
      return set_err(FDE_EDIM, "FDE_HOST_PTRS: strides must be 0 or batch*n");
    }
    const size_t lc = coef_stride ? (size_t)K : 1, lf = f_stride ? (size_t)K : 1;
    const size_t need = (2 * lc + lf + 1 + (size_t)K) * cnt;
    if (need > H->hstage_cap) {
      if (H->d_hstage) { cudaStreamSynchronize(s); cudaFree(H->d_hstage); H->allocs.erase(std::find(H->allocs.begin(), H->allocs.end(), (void*)H->d_hstage)); H->d_hstage = nullptr; }
      TRY(dalloc(H, &H->d_hstage, need));
      H->hstage_cap = need;
    }
    double *sdp = H->d_hstage, *sdm = sdp + lc * cnt, *sf = sdm + lc * cnt, *su0 = sf + lf * cnt, *sout = su0 + cnt;
    if (coef_stride != 0 && K >= 24) {
      // Long runs with per-step coefficients: three launches (head, body, tail).  Only the head's
      // coefficients are copied before the first launch; the rest of the H2D runs on a second
      // stream behind the head launch, and every chunk's solutions go back on a third stream
      // behind the next launch, so of the copies only the head's H2D and the tail's D2H are
      // exposed (cfg3, K = 64: 68 MB in, 34 MB out).  Chunk c starts from the last solution of
      // chunk c-1 (as the RUN_KMAX chunks below); each chunk boundary drains the step pipeline once.
      const int Kh = std::max(4, K / 16);
      const int m0s[4] = {0, Kh, K - Kh, K};
      cudaStream_t csi = nullptr, cso = nullptr;
      cudaEvent_t ev[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
      auto done = [&](int r) {
        if (csi) { cudaStreamSynchronize(csi); cudaStreamDestroy(csi); }
        if (cso) { cudaStreamSynchronize(cso); cudaStreamDestroy(cso); }
        for (auto& e : ev) if (e) cudaEventDestroy(e);
        if (cache) *cache = H; else hodlr_destroy(H);
        return r;
      };
#define CUD(call) do { const cudaError_t e_ = (call); if (e_ != cudaSuccess) return done(set_err(FDE_ECUDA, "%s: %s", #call, cudaGetErrorString(e_))); } while (0)
      CUD(cudaStreamCreateWithFlags(&csi, cudaStreamNonBlocking));
      CUD(cudaStreamCreateWithFlags(&cso, cudaStreamNonBlocking));
      for (auto& e : ev) CUD(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      auto h2d_steps = [&](cudaStream_t q, int a, int b) -> cudaError_t {   // steps [a, b) of the strided arrays
        const size_t o = (size_t)a * cnt, nb = (size_t)(b - a) * cnt * 8;
        cudaError_t e = cudaMemcpyAsync(sdp + o, d_plus + o, nb, cudaMemcpyHostToDevice, q);
        if (e == cudaSuccess) e = cudaMemcpyAsync(sdm + o, d_minus + o, nb, cudaMemcpyHostToDevice, q);
        if (e == cudaSuccess && f_stride) e = cudaMemcpyAsync(sf + o, f + o, nb, cudaMemcpyHostToDevice, q);
        return e;
      };
      CUD(cudaEventRecord(ev[0], s));                     // (the staging area is free once `s` gets here)
      CUD(cudaStreamWaitEvent(csi, ev[0], 0));
      CUD(cudaStreamWaitEvent(cso, ev[0], 0));
      CUD(cudaMemcpyAsync(su0, u0, cnt * 8, cudaMemcpyHostToDevice, s));
      if (!f_stride) CUD(cudaMemcpyAsync(sf, f, cnt * 8, cudaMemcpyHostToDevice, s));
      CUD(h2d_steps(s, m0s[0], m0s[1]));
      CUD(h2d_steps(csi, m0s[1], m0s[2]));
      CUD(cudaEventRecord(ev[1], csi));
      CUD(h2d_steps(csi, m0s[2], m0s[3]));
      CUD(cudaEventRecord(ev[2], csi));
      for (int c = 0; c < 3 && rc == FDE_OK; ++c) {
        const int a = m0s[c], b = m0s[c + 1];
        if (c > 0) CUD(cudaStreamWaitEvent(s, ev[c], 0));
        rc = fde1d_run(batch, n, alpha, h, dt, b - a, sdp + (size_t)a * cnt, sdm + (size_t)a * cnt, coef_stride,
                       sf + (size_t)a * f_stride, f_stride, a == 0 ? su0 : sout + (size_t)(a - 1) * cnt,
                       sout + (size_t)a * cnt, tol, leaf, flags & ~(FDE_HOST_PTRS | FDE_SYNC), &H, stream);
        if (rc != FDE_OK) break;
        CUD(cudaEventRecord(ev[3 + c], s));
        CUD(cudaStreamWaitEvent(cso, ev[3 + c], 0));
        CUD(cudaMemcpyAsync(u_out + (size_t)a * cnt, sout + (size_t)a * cnt, (size_t)(b - a) * cnt * 8,
                            cudaMemcpyDeviceToHost, cso));
      }
      if (rc == FDE_OK) {
        CUD(cudaEventRecord(ev[6], cso));
        CUD(cudaStreamWaitEvent(s, ev[6], 0));
        rc = sync_and_status(H, s);
      }
#undef CUD
      return done(rc);
    }
    CU(cudaMemcpyAsync(sdp, d_plus, lc * cnt * 8, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(sdm, d_minus, lc * cnt * 8, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(sf, f, lf * cnt * 8, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(su0, u0, cnt * 8, cudaMemcpyHostToDevice, s));
    rc = fde1d_run(batch, n, alpha, h, dt, K, sdp, sdm, coef_stride, sf, f_stride, su0, sout, tol, leaf,
                   flags & ~(FDE_HOST_PTRS | FDE_SYNC), &H, stream);
    if (rc == FDE_OK) {
      CU(cudaMemcpyAsync(u_out, sout, (size_t)K * cnt * 8, cudaMemcpyDeviceToHost, s));
      rc = sync_and_status(H, s);
    }
    if (cache) *cache = H; else hodlr_destroy(H);
    return rc;
  }
  // Same coefficients every step (the LU computed once): factor once.  Two factor-once
  // paths -- the pipelined launch (k_run inv mode: the later steps are B' + R units, latency-bound
  // per leaf) and the kept-factor per-step path (fde1d_step: factor with step 1, then streaming
  // solves at HBM rate).  Measured (tools/time_invariant.py, K = 16, ms): 512 leaves 2.0 vs 4.9,
  // 2048 leaves 7.6 vs 7.9, 8192 leaves 30 vs 21, 32768 leaves 120 vs 75; without the projected
  // tree the pipelined launch does not exist (n = 65536, alpha 1.5, tol 1e-12: 28.5 ms refactoring
  // vs 9.8 kept).  Hence the kept path above 16 leaves per SM and without the tree path.
  const bool once = coef_stride == 0 && !(flags & FDE_REFACTOR);
  if (once) {
    int dev = 0, nsm = 148;
    CU(cudaGetDevice(&dev));
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    if (!H->tree_ok || H->L < 1 || (long long)batch * H->nleaf > 16LL * nsm) {
      for (int m = 0; m < K && rc == FDE_OK; ++m)
        rc = fde1d_step(batch, n, alpha, h, dt, d_plus, d_minus, f + m * f_stride,
                        m == 0 ? u0 : u_out + (m - 1) * cnt, u_out + m * cnt, tol, leaf, m == 0,
                        flags & ~(FDE_REFACTOR | FDE_NO_KEEP | FDE_SYNC), &H, stream);
      if (rc == FDE_OK) {
        H->last_stream = s;
        if ((flags & FDE_SYNC) || !cache) rc = sync_and_status(H, s);
        if (!cache) hodlr_destroy(H);
        return rc;
      }
      if (rc != FDE_EDIM) { if (!cache) hodlr_destroy(H); return rc; }
      rc = FDE_OK;                                  // (kept-factor workspace too large: refactor below)
      g_last_error.clear();
    }
  }
  if (!H->tree_ok || H->L < 1) {                  // no pipelined path: one fused step at a time
    for (int m = 0; m < K && rc == FDE_OK; ++m)
      rc = fde1d_step(batch, n, alpha, h, dt, d_plus + m * coef_stride, d_minus + m * coef_stride,
                      f + m * f_stride, m == 0 ? u0 : u_out + (m - 1) * cnt, u_out + m * cnt, tol, leaf, 1,
                      (flags & ~FDE_REFACTOR) | FDE_NO_KEEP, &H, stream);
    if (!cache) hodlr_destroy(H);
    return rc;
  }
  if (H->dt != dt) TRY(set_dt(H, dt, s));
  const bool inv = once;                            // (factor once per launch, k_run inv mode)
  // chunks of at most RUN_KMAX steps per launch (the step index is a 16-bit field of the tree
  // task ids, k_run.cuh rn_tid; the counters and argument blocks are sized per chunk); chunk c
  // starts from the last solution of chunk c-1
  for (int m0 = 0; m0 < K && rc == FDE_OK; m0 += RUN_KMAX) {
    const int Kc = std::min(RUN_KMAX, K - m0);
    rc = run_chunk(H, Kc, dt, d_plus + m0 * coef_stride, d_minus + m0 * coef_stride, coef_stride,
                   f + m0 * f_stride, f_stride, m0 == 0 ? u0 : u_out + (size_t)(m0 - 1) * cnt,
                   u_out + (size_t)m0 * cnt, inv, s);
  }
  if (rc != FDE_OK) { if (!cache) hodlr_destroy(H); return rc; }
  H->last_stream = s;
  H->factored = false;
  if ((flags & FDE_SYNC) || !cache) rc = sync_and_status(H, s);
  if (!cache) hodlr_destroy(H);
  return rc;
}

}  // extern "C"

#include "fde2d.cuh"

// ---------------------------------------------------------------------------------------
// PGMRES with the tridiagonal preconditioners P1 / P2 (k_pgmres.cuh)
#include "k_pgmres.cuh"

namespace {
struct FftPlan { int M1, M2, lg1, lg2; long long M; };
FftPlan fft_plan(long long Mmin) {
  int lg = 4;
  while ((1LL << lg) < Mmin) ++lg;
  FftPlan p;
  p.lg1 = (lg + 1) / 2; p.lg2 = lg - p.lg1;
  p.M1 = 1 << p.lg1; p.M2 = 1 << p.lg2; p.M = 1LL << lg;
  return p;
}
int fft(const FftPlan& p, const double2* x, double2* tmp, double2* X, double sign, double scale, cudaStream_t s) {
  { PROF("k_fft_cols"); k_fft_cols<<<p.M1 / FFT_G, FFT_T, (size_t)(FFT_G + 1) * p.M2 * 16, s>>>(x, tmp, p.M1, p.M2, p.lg2, sign); }
  LAUNCHED();
  { PROF("k_fft_rows"); k_fft_rows<<<p.M2 / FFT_G, FFT_T, (size_t)(FFT_G + 1) * p.M1 * 16, s>>>(tmp, X, p.M1, p.lg1, p.M2, sign, scale); }
  LAUNCHED();
  return FDE_OK;
}
}  // namespace

// A PGMRES plan: the operator's FFT spectra, the preconditioner's block factors and the GMRES
// workspace (Krylov basis of maxit + 1 columns), built once per (alpha, n, h, dt, d+-, precond) and
// reused by every solve (the coefficients are time-invariant in the paper's comparison).
struct fde_pgmres {
  int n = 0, precond = 0, K = 0, nb = 0, nparts = 1;
  double c = 0;
  FftPlan fp{};
  double* base = nullptr;
  size_t oG, oST, oSTt, oZ, oZ1, oZ2, oTmp, oV, oW, oR, oLo, oDi, oUp, oCp, oDd, oSv, oSw, oY, oAb, oRw, oH, oGs, oHp,
      oPart, oSc, oYv, oA, oDp, oDm;
};

extern "C" int fde1d_pgmres_plan(int n, double alpha, double h, double dt, const double* d_plus,
                                 const double* d_minus, int precond, int maxit, void* stream, fde_pgmres_t* out) {
  g_last_error.clear();
  TRY(check_common(1, n, &alpha, h, dt, 0.5, 2));
  if (!d_plus || !d_minus || !out) return set_err(FDE_EDOMAIN, "NULL argument");
  if (precond < 0 || precond > 2) return set_err(FDE_EDOMAIN, "precond=%d (0 none, 1 P1, 2 P2)", precond);
  if (maxit < 1 || maxit > 127) return set_err(FDE_EDOMAIN, "maxit=%d outside 1..127", maxit);
  if (n > (1 << 19)) return set_err(FDE_EDIM, "n=%d exceeds the FFT plan (2^19)", n);
  cudaStream_t s = (cudaStream_t)stream;
  {
    int dev = 0;
    CU(cudaGetDevice(&dev));
    CU(cudaFuncSetAttribute(k_fft_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, (FFT_G + 1) * 1024 * 16));
    CU(cudaFuncSetAttribute(k_fft_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (FFT_G + 1) * 1024 * 16));
  }
  fde_pgmres* P = new fde_pgmres();
  P->n = n; P->precond = precond; P->K = maxit; P->c = dt / std::pow(h, alpha);
  P->fp = fft_plan(2LL * n);
  P->nb = (n + TD_M - 1) / TD_M;
  P->nparts = std::min(148, std::max(1, n / 1024));
  const long long M = P->fp.M;
  size_t o = 0;
  auto carve = [&](size_t d) { const size_t r = o; o += (d + 31) & ~(size_t)31; return r; };
  P->oG = carve(n + 2); P->oST = carve(2 * M); P->oSTt = carve(2 * M); P->oZ = carve(2 * M); P->oZ1 = carve(2 * M);
  P->oZ2 = carve(2 * M); P->oTmp = carve(2 * M); P->oV = carve((size_t)n * (maxit + 1)); P->oW = carve(n);
  P->oR = carve(n); P->oLo = carve(n); P->oDi = carve(n); P->oUp = carve(n); P->oCp = carve(n); P->oDd = carve(n);
  P->oSv = carve(n); P->oSw = carve(n); P->oY = carve(n); P->oAb = carve(2 * P->nb); P->oRw = carve(6 * P->nb);
  P->oH = carve(128 * 129); P->oGs = carve(3 * 128); P->oHp = carve(128); P->oPart = carve(128 * (size_t)P->nparts);
  P->oSc = carve(8); P->oYv = carve(128); P->oA = carve(1); P->oDp = carve(n); P->oDm = carve(n);
  if (cudaMalloc(reinterpret_cast<void**>(&P->base), o * sizeof(double)) != cudaSuccess) {
    cudaGetLastError(); delete P; return set_err(FDE_ENOMEM, "pgmres workspace allocation failed");
  }
  double* base = P->base;
  auto D = [&](size_t off) { return base + off; };
  auto Z = [&](size_t off) { return reinterpret_cast<double2*>(base + off); };
  auto bad = [&](int rc) { cudaFree(P->base); delete P; return rc; };
#define PK(call) do { call; const cudaError_t e_ = cudaGetLastError(); g_launches++; if (e_ != cudaSuccess) return bad(set_err(FDE_ECUDA, "%s", cudaGetErrorString(e_))); } while (0)
  const unsigned gb = (unsigned)((M + 255) / 256), gn = (unsigned)((n + 255) / 256);
  if (cudaMemcpyAsync(D(P->oDp), d_plus, (size_t)n * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(D(P->oDm), d_minus, (size_t)n * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(D(P->oA), &alpha, sizeof(double), cudaMemcpyHostToDevice, s) != cudaSuccess)
    return bad(set_err(FDE_ECUDA, "pgmres plan copies failed"));
  // GL weights (S1) and the spectra of the two circulant embeddings (T and T^T)
  PK((k_gl_weights<<<1, GL_THREADS, 0, s>>>(D(P->oA), n + 2, D(P->oG), n + 2)));
  PK((k_embed_T<<<gb, 256, 0, s>>>(D(P->oG), n, M, Z(P->oZ1), Z(P->oZ2))));
  if (fft(P->fp, Z(P->oZ1), Z(P->oTmp), Z(P->oST), -1.0, 1.0, s) != FDE_OK ||
      fft(P->fp, Z(P->oZ2), Z(P->oTmp), Z(P->oSTt), -1.0, 1.0, s) != FDE_OK)
    return bad(FDE_ECUDA);
  if (precond) {
    PK((k_prec_coeffs<<<gn, 256, 0, s>>>(n, precond, P->c, D(P->oDp), D(P->oDm), D(P->oLo), D(P->oDi), D(P->oUp))));
    PK((k_td_block_setup<<<(P->nb + 127) / 128, 128, 0, s>>>(n, D(P->oLo), D(P->oDi), D(P->oUp), D(P->oCp), D(P->oDd),
                                                             D(P->oSv), D(P->oSw))));
  }
#undef PK
  *out = P;
  return FDE_OK;
}

extern "C" void fde1d_pgmres_destroy(fde_pgmres_t P) {
  if (!P) return;
  cudaDeviceSynchronize();
  cudaFree(P->base);
  delete P;
}

extern "C" int fde1d_pgmres_solve(fde_pgmres_t P, const double* b, double* x, double tol, int* iters,
                                  double* relres, void* stream) {
  g_last_error.clear();
  if (!P || !b || !x) return set_err(FDE_EDOMAIN, "NULL argument");
  if (!(tol > 0.0 && tol < 1.0)) return set_err(FDE_EDOMAIN, "tol=%g outside (0, 1)", tol);
  cudaStream_t s = (cudaStream_t)stream;
  const int n = P->n, nb = P->nb, nparts = P->nparts, K = P->K, precond = P->precond;
  const long long M = P->fp.M;
  const FftPlan& fp = P->fp;
  double* base = P->base;
  auto D = [&](size_t off) { return base + off; };
  auto Z = [&](size_t off) { return reinterpret_cast<double2*>(base + off); };
#define PK(call) do { call; const cudaError_t e_ = cudaGetLastError(); g_launches++; if (e_ != cudaSuccess) return set_err(FDE_ECUDA, "%s", cudaGetErrorString(e_)); } while (0)
  const unsigned gb = (unsigned)((M + 255) / 256), gn = (unsigned)((n + 255) / 256);
  auto apply_A = [&](const double* xin, double* yout) -> int {
    PK((k_pad_complex<<<gb, 256, 0, s>>>(xin, n, M, Z(P->oZ))));
    TRY(fft(fp, Z(P->oZ), Z(P->oTmp), Z(P->oZ), -1.0, 1.0, s));
    PK((k_spec_mul<<<gb, 256, 0, s>>>(Z(P->oZ), Z(P->oST), Z(P->oSTt), M, Z(P->oZ1), Z(P->oZ2))));
    TRY(fft(fp, Z(P->oZ1), Z(P->oTmp), Z(P->oZ1), 1.0, 1.0 / (double)M, s));
    TRY(fft(fp, Z(P->oZ2), Z(P->oTmp), Z(P->oZ2), 1.0, 1.0 / (double)M, s));
    PK((k_apply_combine<<<gn, 256, 0, s>>>(n, xin, Z(P->oZ1), Z(P->oZ2), D(P->oDp), D(P->oDm), P->c, yout)));
    return FDE_OK;
  };
  auto apply_Pinv = [&](const double* r, double* out) -> int {
    if (!precond) { CU(cudaMemcpyAsync(out, r, (size_t)n * 8, cudaMemcpyDeviceToDevice, s)); return FDE_OK; }
    PK((k_td_block_solve<<<(nb + 127) / 128, 128, 0, s>>>(n, D(P->oLo), D(P->oCp), D(P->oDd), r, D(P->oY))));
    PK((k_td_reduced<<<1, 32, 0, s>>>(n, nb, D(P->oSv), D(P->oSw), D(P->oY), D(P->oAb), D(P->oRw))));
    PK((k_td_reconstruct<<<gn, 256, 0, s>>>(n, nb, D(P->oY), D(P->oSv), D(P->oSw), D(P->oAb), out)));
    return FDE_OK;
  };
  auto nrm = [&](const double* v, double* out) -> int {     // out = ||v||
    PK((k_gm_dots<<<nparts, GM_T, 0, s>>>(n, 1, v, v, D(P->oPart))));
    PK((k_gm_sum<<<1, 128, 0, s>>>(1, nparts, D(P->oPart), out)));
    PK((k_sqrt1<<<1, 1, 0, s>>>(out)));
    return FDE_OK;
  };
  double* V = D(P->oV);
  double* H = D(P->oH);
  // r0 = P^{-1} b (x0 = 0), beta, v_0
  TRY(apply_Pinv(b, D(P->oR)));
  TRY(nrm(D(P->oR), D(P->oSc)));
  PK((k_gm_scale<<<gn, 256, 0, s>>>(n, D(P->oR), D(P->oSc), V)));
  PK((k_gm_setg<<<1, 1, 0, s>>>(D(P->oGs), D(P->oSc))));
  CU(cudaMemsetAsync(H, 0, 128 * 129 * sizeof(double), s));
  double beta = 0.0, res = 1.0;
  CU(cudaMemcpyAsync(&beta, D(P->oSc), sizeof(double), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  int k = 0;
  if (beta > 0.0) {
    for (k = 0; k < K; ++k) {
      TRY(apply_A(V + (size_t)k * n, D(P->oR)));
      TRY(apply_Pinv(D(P->oR), D(P->oW)));
      // classical Gram-Schmidt twice: h = V^T w, w -= V h (x2), H[:, k] = h1 + h2
      double* Hc = H + (size_t)k * 128;
      for (int pass = 0; pass < 2; ++pass) {
        PK((k_gm_dots<<<nparts, GM_T, 0, s>>>(n, k + 1, V, D(P->oW), D(P->oPart))));
        PK((k_gm_sum<<<1, 128, 0, s>>>(k + 1, nparts, D(P->oPart), D(P->oHp))));
        PK((k_gm_axpy<<<gn, 256, 0, s>>>(n, k + 1, V, D(P->oHp), D(P->oW))));
        PK((k_add_vec<<<1, 128, 0, s>>>(k + 1, D(P->oHp), Hc)));
      }
      TRY(nrm(D(P->oW), Hc + k + 1));
      PK((k_gm_scale<<<gn, 256, 0, s>>>(n, D(P->oW), Hc + k + 1, V + (size_t)(k + 1) * n)));
      PK((k_gm_givens<<<1, 1, 0, s>>>(k, Hc, D(P->oGs), D(P->oSc) + 1)));
      CU(cudaMemcpyAsync(&res, D(P->oSc) + 1, sizeof(double), cudaMemcpyDeviceToHost, s));
      CU(cudaStreamSynchronize(s));
      if (res <= tol * beta) { ++k; break; }
    }
    if (k > K) k = K;
    PK((k_gm_backsolve<<<1, 1, 0, s>>>(k, H, D(P->oGs), D(P->oYv))));
    CU(cudaMemsetAsync(x, 0, (size_t)n * 8, s));
    PK((k_gm_axpy_neg<<<gn, 256, 0, s>>>(n, k, V, D(P->oYv), x)));
  } else {
    CU(cudaMemsetAsync(x, 0, (size_t)n * 8, s));
  }
  CU(cudaStreamSynchronize(s));
#undef PK
  if (iters) *iters = k;
  if (relres) *relres = beta > 0.0 ? res / beta : 0.0;
  if (beta > 0.0 && res > tol * beta)
    return set_err(FDE_ENOCONV, "PGMRES: preconditioned relative residual %.3e > tol %.1e after %d iterations",
                   res / beta, tol, k);
  return FDE_OK;
}

extern "C" int fde1d_pgmres(int n, double alpha, double h, double dt, const double* d_plus, const double* d_minus,
                            const double* b, double* x, int precond, double tol, int maxit, int* iters,
                            double* relres, unsigned flags, void* stream) {
  fde_pgmres_t P = nullptr;
  TRY(fde1d_pgmres_plan(n, alpha, h, dt, d_plus, d_minus, precond, maxit, stream, &P));
  const int rc = fde1d_pgmres_solve(P, b, x, tol, iters, relres, stream);
  const std::string err = g_last_error;
  fde1d_pgmres_destroy(P);
  g_last_error = err;
  (void)flags;
  return rc;
}

// y = A_m x with the exact operator (Eq. 2.5, shift I): T x and T^T x by circulant embedding + FFT
// -- the matrix-free operator of the PGMRES comparison and of residual checks.
extern "C" int fde1d_apply_exact(int n, double alpha, double h, double dt, const double* d_plus,
                                 const double* d_minus, const double* x, double* y, void* stream) {
  g_last_error.clear();
  TRY(check_common(1, n, &alpha, h, dt, 0.5, 2));
  if (!d_plus || !d_minus || !x || !y) return set_err(FDE_EDOMAIN, "NULL array argument");
  if (x == y) return set_err(FDE_EDOMAIN, "y must not alias x");
  if (n > (1 << 19)) return set_err(FDE_EDIM, "n=%d exceeds the FFT plan (2^19)", n);
  cudaStream_t s = (cudaStream_t)stream;
  {
    int dev = 0;
    CU(cudaGetDevice(&dev));
    CU(cudaFuncSetAttribute(k_fft_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, (FFT_G + 1) * 1024 * 16));
    CU(cudaFuncSetAttribute(k_fft_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (FFT_G + 1) * 1024 * 16));
  }
  const FftPlan fp = fft_plan(2LL * n);
  const long long M = fp.M;
  size_t o = 0;
  auto carve = [&](size_t d) { const size_t r = o; o += (d + 31) & ~(size_t)31; return r; };
  const size_t oG = carve(n + 2), oST = carve(2 * M), oSTt = carve(2 * M), oZ = carve(2 * M), oZ1 = carve(2 * M),
               oZ2 = carve(2 * M), oTmp = carve(2 * M), oA = carve(1);
  double* base = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&base), o * sizeof(double), s) != cudaSuccess) {
    cudaGetLastError(); return set_err(FDE_ENOMEM, "workspace allocation failed");
  }
  auto Z = [&](size_t off) { return reinterpret_cast<double2*>(base + off); };
  const unsigned gb = (unsigned)((M + 255) / 256), gn = (unsigned)((n + 255) / 256);
  CU(cudaMemcpyAsync(base + oA, &alpha, sizeof(double), cudaMemcpyHostToDevice, s));
  k_gl_weights<<<1, GL_THREADS, 0, s>>>(base + oA, n + 2, base + oG, n + 2); LAUNCHED();
  k_embed_T<<<gb, 256, 0, s>>>(base + oG, n, M, Z(oZ1), Z(oZ2)); LAUNCHED();
  TRY(fft(fp, Z(oZ1), Z(oTmp), Z(oST), -1.0, 1.0, s));
  TRY(fft(fp, Z(oZ2), Z(oTmp), Z(oSTt), -1.0, 1.0, s));
  k_pad_complex<<<gb, 256, 0, s>>>(x, n, M, Z(oZ)); LAUNCHED();
  TRY(fft(fp, Z(oZ), Z(oTmp), Z(oZ), -1.0, 1.0, s));
  k_spec_mul<<<gb, 256, 0, s>>>(Z(oZ), Z(oST), Z(oSTt), M, Z(oZ1), Z(oZ2)); LAUNCHED();
  TRY(fft(fp, Z(oZ1), Z(oTmp), Z(oZ1), 1.0, 1.0 / (double)M, s));
  TRY(fft(fp, Z(oZ2), Z(oTmp), Z(oZ2), 1.0, 1.0 / (double)M, s));
  k_apply_combine<<<gn, 256, 0, s>>>(n, x, Z(oZ1), Z(oZ2), d_plus, d_minus, dt / std::pow(h, alpha), y); LAUNCHED();
  CU(cudaFreeAsync(base, s));
  return FDE_OK;
}
