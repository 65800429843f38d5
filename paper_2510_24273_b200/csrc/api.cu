// Host side of the C ABI (include/sals.h): argument validation, workspace
// carving, path / grid planning and stream-ordered launches (programmatic
// dependent launch, thread-block clusters).  Never allocates, never syncs.
#include <dlfcn.h>
#include <nccl.h>

#include <atomic>
#include <cstring>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "../../include/sals.h"
#include "kernels.h"
#include "recon_attn_tc.h"
#include "once.h"

using namespace sals;

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

// Optional per-stage event recorder (sals_decode_profile only).
enum { kStQproj = 0, kStScore, kStTopk, kStReconAttn, kStFlash, kStMerge, kNumStages };
constexpr int kStExchange = kNumStages + 1;   // (sharded) the NCCL all-gathers; bit kNumStages is the append
constexpr int kStShardSelect = kNumStages + 2; // (sharded) global selection + owned list
struct StageTimer {
  cudaEvent_t ev[kNumStages + 1];
  float ms[kNumStages];
  bool used[kNumStages];
};
thread_local StageTimer* g_timer = nullptr;
// Stage mask (sals_profile_stage_mask): bit i enables stage i; bit kNumStages the append.
thread_local uint32_t g_stage_mask = 0xffffffffu;
// TMA score kernel for bf16 (SALS_SCORE_LSU=1 in the environment selects the LSU kernel).
// single-CTA top-k for <= 8192 entries (SALS_TOPK_CLUSTER=1 forces the cluster kernel)
const bool g_topk_cluster = [] { const char* e = getenv("SALS_TOPK_CLUSTER"); return e && e[0] == '1'; }();
const bool g_fused_merge = [] { const char* e = getenv("SALS_FUSED_MERGE"); return e && e[0] == '1'; }();
const bool g_score_tma = [] { const char* e = getenv("SALS_SCORE_LSU"); return !(e && e[0] == '1'); }();
inline bool on(int stage) { return (g_stage_mask >> stage) & 1u; }
void mark_begin(cudaStream_t st) { if (g_timer) cudaEventRecord(g_timer->ev[kNumStages], st); }
void mark(int stage, cudaStream_t st) {
  if (!g_timer) return;
  cudaEventRecord(g_timer->ev[stage], st);
  g_timer->used[stage] = true;
}

sals_status fail(sals_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

template <typename... KArgs, typename... Args>
cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                   int cluster, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[na].val.programmaticStreamSerializationAllowed = 1;
  ++na;
  if (cluster >= 1) {
    attrs[na].id = cudaLaunchAttributeClusterDimension;
    attrs[na].val.clusterDim.x = cluster;
    attrs[na].val.clusterDim.y = 1;
    attrs[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

#define SALS_CUDA_TRY(expr)                                                          \
  do {                                                                               \
    cudaError_t e_ = (expr);                                                         \
    if (e_ != cudaSuccess) return fail(SALS_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

int next_pow2(int v) { int p = 1; while (p < v) p <<= 1; return p; }
size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// quantised value cache: bits per value (0 = dtype values)
inline int vq_bits(const sals_config* c) { return (c->v_bits == 4 || c->v_bits == 2) ? c->v_bits : 0; }
// high-precision recent window of the quantised value cache (8-bit ring of cfg->recent rows)
inline int hp_window(const sals_config* c) { return vq_bits(c) ? c->recent : 0; }
inline size_t hp_row_bytes(const sals_config* c) { return (size_t)c->num_kv_heads * (128 + 16); }
inline size_t v_row_bytes(const sals_config* c) {
  const int d = c->head_dim, nkv = c->num_kv_heads;
  if (vq_bits(c)) return (size_t)nkv * ((size_t)d * c->v_bits / 8 + (size_t)(d / 32) * 4);
  return (size_t)nkv * d * (c->dtype == SALS_BF16 ? 2 : 4);
}

sals_status validate(const sals_config* c) {
  if (!c) return fail(SALS_ERR_INVALID_ARGUMENT, "cfg is NULL");
  if (c->num_q_heads < 1 || c->num_kv_heads < 1 || c->num_q_heads % c->num_kv_heads)
    return fail(SALS_ERR_INVALID_ARGUMENT, "num_q_heads (%d) must be a positive multiple of num_kv_heads (%d)",
                c->num_q_heads, c->num_kv_heads);
  const int G = c->num_q_heads / c->num_kv_heads;
  if (G != 1 && G != 2 && G != 4 && G != 8) return fail(SALS_ERR_UNSUPPORTED, "GQA group %d not in {1,2,4,8}", G);
  const int d = c->head_dim;
  if (d != 16 && d != 32 && d != 64 && d != 128 && d != 256)
    return fail(SALS_ERR_UNSUPPORTED, "head_dim %d not in {16,32,64,128,256}", d);
  if (c->dtype != SALS_F32 && c->dtype != SALS_BF16) return fail(SALS_ERR_INVALID_ARGUMENT, "bad dtype %d", c->dtype);
  if (c->dtype == SALS_F32 && d > 128) return fail(SALS_ERR_UNSUPPORTED, "fp32 supports head_dim <= 128");
  const int D = c->num_kv_heads * d;
  if (D > 8192) return fail(SALS_ERR_UNSUPPORTED, "n_kv*d = %d > 8192", D);
  if (c->rank < 8 || c->rank > D || c->rank % 8)
    return fail(SALS_ERR_INVALID_ARGUMENT, "rank %d must be a multiple of 8 in [8, D=%d]", c->rank, D);
  if (c->score_rank < 8 || c->score_rank > c->rank || c->score_rank % 8)
    return fail(SALS_ERR_INVALID_ARGUMENT, "score_rank %d must be a multiple of 8 in [8, rank]", c->score_rank);
  const int epc = c->dtype == SALS_BF16 ? 8 : 4;
  if (c->score_rank / epc > 128) return fail(SALS_ERR_UNSUPPORTED, "score_rank too large");
  if (c->top_k < 1) return fail(SALS_ERR_INVALID_ARGUMENT, "top_k must be >= 1");
  if (c->sink < 0 || c->recent < 0 || c->sink + c->recent > c->top_k)
    return fail(SALS_ERR_INVALID_ARGUMENT, "need 0 <= sink, recent and sink + recent <= top_k");
  if (!(c->rope_base > 0.f)) return fail(SALS_ERR_INVALID_ARGUMENT, "rope_base must be > 0");
  if (c->rope_style != SALS_ROPE_HALF && c->rope_style != SALS_ROPE_INTERLEAVED)
    return fail(SALS_ERR_INVALID_ARGUMENT, "bad rope_style");
  if (c->softmax_scale < 0.f) return fail(SALS_ERR_INVALID_ARGUMENT, "softmax_scale must be >= 0");
  if (c->path < SALS_PATH_AUTO || c->path > SALS_PATH_TCGEN05) return fail(SALS_ERR_INVALID_ARGUMENT, "bad path");
  if (c->v_bits != 0 && c->v_bits != 16 && c->v_bits != 4 && c->v_bits != 2)
    return fail(SALS_ERR_INVALID_ARGUMENT, "v_bits %d not in {0, 16, 4, 2}", c->v_bits);
  if (vq_bits(c) && (c->dtype != SALS_BF16 || d != 128))
    return fail(SALS_ERR_UNSUPPORTED, "quantised values need bf16 and head_dim 128");
  return SALS_OK;
}

RopeTable make_rope(const sals_config* c) {
  RopeTable t{};
  t.half = c->head_dim / 2;
  t.style = c->rope_style;
  for (int p = 0; p < t.half; ++p) {
    t.theta[p] = std::pow((double)c->rope_base, -2.0 * p / c->head_dim);
    t.th_hi[p] = (float)t.theta[p];
    t.th_lo[p] = (float)(t.theta[p] - (double)t.th_hi[p]);
  }
  return t;
}

float scale_log2(const sals_config* c) {
  const float sc = c->softmax_scale > 0.f ? c->softmax_scale : 1.0f / std::sqrt((float)c->head_dim);
  return sc * kLog2e;
}

size_t esize(const sals_config* c) { return c->dtype == SALS_BF16 ? 2 : 4; }

// ---------------------------------------------------------------- planning
struct Plan {
  int D, G, kmax;
  bool tc;                 // fused tcgen05 reconstruct + attention
  int nsplit, chunk;       // flash split (SIMT) / 128-row tiles (tc v1) / chunks + tiles per CTA (tc v2)
  bool tc2;
  int tk_cs, tk_slice;     // top-k cluster size / slice
  int tk_nt, tk_cap;       // threads per CTA, candidate capacity (histogram-assisted kernel)
  int tk_n;                // entries per request (upper bound)
  size_t tk_smem;
  int proj_cs, proj_rows;
  // workspace offsets
  size_t off_qtil, off_qrope, off_scores, off_sel, off_count, off_ccount, off_kr, off_part, off_hist, total;
  int hist_words;          // histogram + (tcgen05 v2) split-merge counters, zeroed by the query projection
  int64_t score_stride;
};

bool tc_eligible(const sals_config* c, int batch, int kmax) {
  const int D = c->num_kv_heads * c->head_dim;
  return c->dtype == SALS_BF16 && (int64_t)batch * kmax >= 128 && tc_supported(c->head_dim, D, c->rank,
         c->num_q_heads / c->num_kv_heads);
}

// Top-k cluster plan of the histogram-assisted kernel (K4 / K8).
constexpr size_t kTopkDynSmem = 190 * 1024;
// 16-CTA cluster x 23808-entry slices: slice * 8 B + 1024 candidates x 4 B = 190 KB (plan_topk)
constexpr int kMaxSeqLen = 16 * 23808;
sals_status plan_topk(int n_entries, Plan& p) {
  static const int slice_env = [] { const char* e = getenv("SALS_TOPK_SLICE"); return e ? atoi(e) : 0; }();
  const int target = (slice_env >= 256 && slice_env <= 16384) ? slice_env : 2048;   // experiment override
  int cs = 1;
  while (cs < 16 && ceil_div(n_entries, cs) > target) cs <<= 1;
  int slice = ceil_div(n_entries, cs);
  slice = (int)align_up(std::max(slice, 4), 4);
  if (slice > 24576) return fail(SALS_ERR_UNSUPPORTED, "top-k over %d entries exceeds the cluster limit", n_entries);
  p.tk_cs = cs;
  p.tk_slice = slice;
  p.tk_n = n_entries;
  p.tk_nt = slice >= 4096 ? 1024 : 512;
  // signed: the staged slice (8 B per entry) plus a candidate area of at least
  // kMinCand entries must fit the kernel's dynamic shared memory
  constexpr int64_t kMinCand = 1024;
  const int64_t avail = (int64_t)kTopkDynSmem - (int64_t)slice * 8;
  if (avail < kMinCand * 4)
    return fail(SALS_ERR_UNSUPPORTED, "top-k over %d entries exceeds the cluster's shared memory", n_entries);
  p.tk_cap = (int)std::min<int64_t>(kCandCap, avail / 4);
  p.tk_smem = (size_t)slice * 8 + (size_t)p.tk_cap * 4;
  return SALS_OK;
}

void plan_flash(int batch, int n_kv, int ntok, int tpw_unr, int& nsplit, int& chunk) {
  const int target = 148 * 48;   // warps: ~48 per SM keep enough K/V rows in flight
  int ns = std::max(1, ceil_div(target, (int64_t)batch * n_kv));
  ns = std::min(ns, 512);   // merge_kernel's two-round-trip path holds <= 512 splits
  ns = std::min(ns, std::max(1, ceil_div(ntok, tpw_unr)));
  chunk = (int)align_up(ceil_div(ntok, ns), tpw_unr);
  chunk = std::max(chunk, tpw_unr);
  nsplit = std::max(1, ceil_div(ntok, chunk));
}

int flash_tpw_unr(const sals_config* c) {
  const int epl = c->dtype == SALS_BF16 ? 8 : 4;
  const int lpt = c->head_dim / epl;
  const int G = c->num_q_heads / c->num_kv_heads;
  return (32 / lpt) * (G <= 2 ? 4 : 2);   // flash_decode_kernel TPW * UNR
}

// Rows of U per CTA of the projection cluster: a multiple of 8 (16-byte vectors),
// at most 512 (the CTA's U slice, rows x 128 B, is staged in shared memory
// before the PDL wait).  Measured (bench stage times, c2 D = 4096 / c3 D = 1024):
// 8-CTA clusters beat 16 (a 16-CTA cluster needs 16 free SMs of one GPC) and 4.
void plan_proj(Plan& p, bool query) {
  (void)query;
  static const int cs_env = [] { const char* e = getenv("SALS_PROJ_CS"); return e ? atoi(e) : 0; }();
  int cs = std::min(8, std::max(1, ceil_div(p.D, 64)));
  while (ceil_div(p.D, cs) > 512) cs *= 2;
  if (cs_env >= 1 && cs_env <= 16 && ceil_div(p.D, cs_env) <= 512) cs = cs_env;   // experiment override
  p.proj_rows = (int)align_up(ceil_div(p.D, cs), 8);
  p.proj_cs = ceil_div(p.D, p.proj_rows);
}

sals_status make_plan(const sals_config* c, int batch, int max_s, Plan& p, bool for_size) {
  p.D = c->num_kv_heads * c->head_dim;
  p.G = c->num_q_heads / c->num_kv_heads;
  p.kmax = std::min(c->top_k, max_s);
  const bool want_tc = c->path == SALS_PATH_TCGEN05 || (c->path == SALS_PATH_AUTO);
  p.tc = want_tc && tc_eligible(c, batch, p.kmax);
  if (c->path == SALS_PATH_TCGEN05 && !p.tc && !for_size)
    return fail(SALS_ERR_UNSUPPORTED, "tcgen05 path needs bf16, B*k >= 128, d in {64,128,256}, D %% 256 == 0");
  p.tc2 = p.tc && tc2_supported(c->head_dim, p.D, c->rank, p.G);
  if (vq_bits(c) && !p.tc2 && !for_size)
    return fail(SALS_ERR_UNSUPPORTED, "quantised values need the tcgen05 v2 path (bf16, d = 128, B*k >= 128)");
  if (p.tc2) {
    const int ntiles = ceil_div(p.kmax, kTcRows);
    const int64_t units = (int64_t)batch * (p.D / 256) * ntiles;
    const int tpc = std::max(1, ceil_div(units, 148));
    p.chunk = tpc;
    p.nsplit = ceil_div(ntiles, tpc);
  } else if (p.tc) {
    p.nsplit = ceil_div(p.kmax, kTcRows);
    p.chunk = kTcRows;
  } else {
    plan_flash(batch, c->num_kv_heads, p.kmax, flash_tpw_unr(c), p.nsplit, p.chunk);
  }
  sals_status st = plan_topk(max_s, p);
  if (st != SALS_OK) return st;
  plan_proj(p, true);
  const size_t es = esize(c);
  p.score_stride = (int64_t)align_up(max_s, 4);
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
  p.off_qtil = take((size_t)batch * c->score_rank * 4);
  p.off_qrope = take((size_t)batch * c->num_q_heads * c->head_dim * 4);
  p.off_scores = take((size_t)batch * p.score_stride * 4);
  p.off_sel = take((size_t)batch * c->top_k * 4);
  p.off_count = take((size_t)batch * 4);
  p.off_ccount = take((size_t)batch * 4);   // (sharded) valid local candidates per request
  p.off_kr = take(p.tc ? 0 : (size_t)batch * c->top_k * p.D * es);
  p.off_part = take((size_t)batch * c->num_q_heads * p.nsplit * (c->head_dim + 2) * 4);
  p.hist_words = batch * kH0Bins + (p.tc2 ? batch * (p.D / 256) : 0);
  p.off_hist = take((size_t)p.hist_words * 4);
  p.total = off;
  return SALS_OK;
}

// ------------------------------------------------------------ dispatchers
// mode 0 append, 1 query projection (+ query RoPE role), 2 both (fused append + decode)
template <typename T>
sals_status launch_project(const sals_config* c, const Plan& p, int mode, ProjectArgs& a, cudaStream_t st) {
  a.rows_per_cta = p.proj_rows;
  const int cpb = 8 * (16 / (int)sizeof(T));
  int gy;
  if (mode == 0) gy = ceil_div(a.ncols, cpb);
  else if (mode == 1) gy = ceil_div(a.ncols, cpb) + 1;
  else { a.n_append_blocks = ceil_div(a.ncols_a, cpb); gy = a.n_append_blocks + ceil_div(a.ncols, cpb) + 1; }
  dim3 grid(p.proj_cs, gy);
  static DeviceOnce once;
  SALS_CUDA_TRY(once.run([] {
    cudaError_t e = cudaSuccess;
    auto set = [&](auto k) {
      if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
    };
    set(project_kernel<T, 0, 256>); set(project_kernel<T, 1, 256>); set(project_kernel<T, 2, 256>);
    set(project_kernel<T, 0, 512>); set(project_kernel<T, 1, 512>); set(project_kernel<T, 2, 512>);
    return e;
  }));
  // 512 threads when a CTA owns 512 rows of U (c2: 6.3 -> 6.1 us), else 256 (c3: 3.8 vs 4.6 us)
  const int nt = p.proj_rows >= 512 ? 512 : 256;
  // the CTA's U slice (rows x 128 B), then the per-warp partials [warps][8][8 * 16 B / elem]
  const size_t smem = (size_t)p.proj_rows * 128 + (size_t)(nt / 32) * 8 * (8 * (16 / sizeof(T))) * 4;
  if (nt == 512) {
    if (mode == 0) SALS_CUDA_TRY(launch(project_kernel<T, 0, 512>, grid, dim3(512), smem, st, p.proj_cs, a));
    else if (mode == 1) SALS_CUDA_TRY(launch(project_kernel<T, 1, 512>, grid, dim3(512), smem, st, p.proj_cs, a));
    else SALS_CUDA_TRY(launch(project_kernel<T, 2, 512>, grid, dim3(512), smem, st, p.proj_cs, a));
  } else {
    if (mode == 0) SALS_CUDA_TRY(launch(project_kernel<T, 0, 256>, grid, dim3(256), smem, st, p.proj_cs, a));
    else if (mode == 1) SALS_CUDA_TRY(launch(project_kernel<T, 1, 256>, grid, dim3(256), smem, st, p.proj_cs, a));
    else SALS_CUDA_TRY(launch(project_kernel<T, 2, 256>, grid, dim3(256), smem, st, p.proj_cs, a));
  }
  return SALS_OK;
}

template <typename T>
sals_status launch_score(const sals_config* c, ScoreArgs a, int batch, int max_len, cudaStream_t st) {
  if (sizeof(T) == 2 && g_score_tma) {
    int nsm = 0;
    SALS_CUDA_TRY(device_sm_count(&nsm));
    cudaError_t e = launch_score_tma(a, batch, max_len, st, nsm);
    if (e == cudaSuccess) { g_launches.fetch_add(1, std::memory_order_relaxed); return SALS_OK; }
    if (e != cudaErrorNotSupported) return fail(SALS_ERR_CUDA, "score_tma launch: %s", cudaGetErrorString(e));
  }
  const int epc = sizeof(T) == 2 ? 8 : 4;
  const int V = c->score_rank / epc;
  int LG, CPL;
  if (V <= 32) { LG = next_pow2(V); CPL = 1; }
  else if (V <= 64) { LG = 32; CPL = 2; }
  else { LG = 32; CPL = 4; }
  const int tpw = 32 / LG;
  const int unr = CPL == 1 ? 8 : (CPL == 2 ? 4 : 2);
  const int step = 8 * tpw * unr;
  const int64_t work = (int64_t)batch * max_len;
  int tpc = (int)align_up(std::max<int64_t>(step, (work + 599) / 600), step);
  a.tokens_per_cta = tpc;
  dim3 grid(std::max(1, ceil_div(max_len, tpc)), batch);
  void (*k)(ScoreArgs) = nullptr;
  switch (LG * 10 + CPL) {
    case 11: k = latent_score_kernel<T, 1, 1>; break;
    case 21: k = latent_score_kernel<T, 2, 1>; break;
    case 41: k = latent_score_kernel<T, 4, 1>; break;
    case 81: k = latent_score_kernel<T, 8, 1>; break;
    case 161: k = latent_score_kernel<T, 16, 1>; break;
    case 321: k = latent_score_kernel<T, 32, 1>; break;
    case 322: k = latent_score_kernel<T, 32, 2>; break;
    case 324: k = latent_score_kernel<T, 32, 4>; break;
    default: return fail(SALS_ERR_UNSUPPORTED, "score rank layout");
  }
  SALS_CUDA_TRY(launch(k, grid, dim3(kScoreThreads), 0, st, 0, a));
  return SALS_OK;
}

sals_status launch_topk(TopkArgs a, int batch, const Plan& p, cudaStream_t st) {
  static DeviceOnce once;
  SALS_CUDA_TRY(once.run([] {
    auto* k512 = topk_hist_kernel<512>;
    auto* k1024 = topk_hist_kernel<1024>;
    cudaError_t e = cudaFuncSetAttribute(k512, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTopkDynSmem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k512, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k1024, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTopkDynSmem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k1024, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return e;
  }));
  // cluster attribute even for cs == 1 (the kernels use cluster barriers / DSMEM)
  if (p.tk_n <= 8192 && !g_topk_cluster) {
    cudaError_t e = launch_topk_cta(a, batch, p.tk_n, st);
    if (e != cudaSuccess) return fail(SALS_ERR_CUDA, "topk_cta launch: %s", cudaGetErrorString(e));
    g_launches.fetch_add(1, std::memory_order_relaxed);
  } else {
    a.cand_cap = p.tk_cap;
    if (p.tk_nt == 1024)
      SALS_CUDA_TRY(launch(topk_hist_kernel<1024>, dim3(batch * p.tk_cs), dim3(1024), p.tk_smem, st, p.tk_cs, a));
    else
      SALS_CUDA_TRY(launch(topk_hist_kernel<512>, dim3(batch * p.tk_cs), dim3(512), p.tk_smem, st, p.tk_cs, a));
  }
  return SALS_OK;
}

template <typename T>
sals_status launch_recon_simt(const sals_config* c, ReconArgs a, int batch, int kmax, cudaStream_t st) {
  const int DH = c->head_dim;
  const size_t smem = (size_t)(32 * 33 + DH * 33 + 32 * DH) * 4;
  static DeviceOnce once;
  SALS_CUDA_TRY(once.run([] {
    return cudaFuncSetAttribute(recon_rope_simt_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  }));
  dim3 grid(ceil_div(kmax, 32), c->num_kv_heads, batch);
  SALS_CUDA_TRY(launch(recon_rope_simt_kernel<T>, grid, dim3(256), smem, st, 0, a));
  return SALS_OK;
}

template <typename T, bool DENSE>
sals_status launch_flash(const sals_config* c, FlashArgs a, int batch, cudaStream_t st) {
  const int G = c->num_q_heads / c->num_kv_heads;
  void (*k)(FlashArgs) = nullptr;
#define SALS_FD_CASE(DH)                                                     \
  case DH:                                                                   \
    switch (G) {                                                             \
      case 1: k = flash_decode_kernel<T, DH, 1, DENSE>; break;               \
      case 2: k = flash_decode_kernel<T, DH, 2, DENSE>; break;               \
      case 4: k = flash_decode_kernel<T, DH, 4, DENSE>; break;               \
      case 8: k = flash_decode_kernel<T, DH, 8, DENSE>; break;               \
    }                                                                        \
    break;
  if (sizeof(T) == 2) {
    switch (c->head_dim) { SALS_FD_CASE(16) SALS_FD_CASE(32) SALS_FD_CASE(64) SALS_FD_CASE(128) SALS_FD_CASE(256) }
  } else {
    switch (c->head_dim) { SALS_FD_CASE(16) SALS_FD_CASE(32) SALS_FD_CASE(64) SALS_FD_CASE(128) }
  }
#undef SALS_FD_CASE
  if (!k) return fail(SALS_ERR_UNSUPPORTED, "flash decode shape");
  // one CTA = one split x up to 8 consecutive KV heads (their row segments are contiguous)
  int hpc = 8;
  while (c->num_kv_heads % hpc) hpc >>= 1;
  dim3 grid(a.nsplit, c->num_kv_heads / hpc, batch);
  SALS_CUDA_TRY(launch(k, grid, dim3(32 * hpc), 0, st, 0, a));
  return SALS_OK;
}

template <typename T>
sals_status launch_merge(const sals_config* c, MergeArgs a, int batch, cudaStream_t st) {
  // head_dim x SG threads (SG <= 8): SG split streams per dim when there are many splits
  // (the dense comparator's ~148 at B = 1, the fused kernel's 8-32 chunks at c3 / c4)
  int sgs = a.nsplit >= 128 ? 8 : (a.nsplit >= 64 ? 4 : (a.nsplit >= 16 ? 2 : 1));
  while (sgs > 1 && c->head_dim * sgs > 1024) sgs >>= 1;
  const int nt = std::max(32, c->head_dim * sgs);
  SALS_CUDA_TRY(launch(merge_kernel<T>, dim3(batch * c->num_q_heads), dim3(nt), 0, st, 0, a));
  return SALS_OK;
}

// Shared tail of decode: reconstruct + RoPE + attention + merge over a token
// list sel/count (local rows), producing either y (T) or one fp32 partial per
// (b, h) when `partial_out` is set.
template <typename T>
sals_status attend_list(const sals_config* c, const Plan& p, const void* U, const void* latent,
                        const void* v_cache, int64_t cap, int batch, int64_t pos_base, const int* sel,
                        const int* count, char* ws, void* out, float* partial_out, cudaStream_t st,
                        const int* seq_len_hp = nullptr) {
  float* part = reinterpret_cast<float*>(ws + p.off_part);
  const float* qrope = reinterpret_cast<const float*>(ws + p.off_qrope);
  if (p.tc) {
    TcArgs t{};
    t.latent = latent; t.cap = cap; t.r = c->rank; t.U = U; t.v_cache = v_cache;
    t.v_bits = vq_bits(c); t.v_row_bytes = (int)v_row_bytes(c);
    t.hp_window = seq_len_hp ? hp_window(c) : 0;
    t.hp_ring_off = (int64_t)batch * cap * (int64_t)v_row_bytes(c); t.seq_len = seq_len_hp;
    t.sel = sel; t.count = count; t.k_stride = c->top_k; t.D = p.D; t.head_dim = c->head_dim;
    t.G = p.G; t.n_q = c->num_q_heads; t.pos_base = pos_base; t.rope = make_rope(c);
    t.qrope = qrope; t.scale_log2 = scale_log2(c); t.partials = part; t.ntiles = p.nsplit;
    t.tiles_per_cta = p.tc2 ? p.chunk : 0;
    // v2 writes y itself: directly for one chunk, else the last chunk CTA merges
    // measured: the separate merge kernel beats the in-kernel last-CTA merge
    // (SALS_FUSED_MERGE=1) at c3 / c4, so by default only a single chunk writes y directly
    const bool direct = p.tc2 && !partial_out &&
                        (p.nsplit == 1 || (g_fused_merge && p.nsplit <= tc2_merge_max_splits(p.G)));
    t.direct_out = direct ? out : nullptr;
    t.counters = (direct && p.nsplit > 1)
                     ? reinterpret_cast<unsigned*>(ws + p.off_hist) + (size_t)batch * kH0Bins : nullptr;
    if (on(kStReconAttn)) {
      sals_status s = launch_recon_attn_tc(t, batch, st);
      if (s != SALS_OK) return fail(s, "%s", tc_last_error());
      g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    mark(kStReconAttn, st);
    if (direct) return SALS_OK;   // y written by the fused kernel
  } else {
    ReconArgs r{};
    r.latent = latent; r.cap = cap; r.r = c->rank; r.U = U; r.sel = sel; r.count = count;
    r.k_stride = c->top_k; r.D = p.D; r.head_dim = c->head_dim; r.pos_base = pos_base;
    r.rope = make_rope(c); r.kr = ws + p.off_kr;
    sals_status s = on(kStReconAttn) ? launch_recon_simt<T>(c, r, batch, p.kmax, st) : SALS_OK;
    if (s != SALS_OK) return s;
    mark(kStReconAttn, st);
    FlashArgs f{};
    f.qrope = qrope; f.kbase = ws + p.off_kr; f.v_cache = v_cache; f.sel = sel; f.count = count;
    f.cap = cap; f.D = p.D; f.k_stride = c->top_k; f.n_q = c->num_q_heads; f.n_kv = c->num_kv_heads;
    f.nsplit = p.nsplit; f.chunk = p.chunk; f.scale_log2 = scale_log2(c); f.partials = part;
    s = on(kStFlash) ? launch_flash<T, false>(c, f, batch, st) : SALS_OK;
    if (s != SALS_OK) return s;
    mark(kStFlash, st);
  }
  MergeArgs m{};
  m.partials = part;
  m.bh_stride = (int64_t)p.nsplit * (c->head_dim + 2);
  m.s_stride = c->head_dim + 2;
  m.nsplit = p.nsplit; m.n_q = c->num_q_heads; m.head_dim = c->head_dim;
  m.out = partial_out ? (void*)partial_out : out;
  m.normalize = partial_out ? 0 : 1;
  if (!on(kStMerge)) return SALS_OK;
  sals_status ms = partial_out ? launch_merge<float>(c, m, batch, st) : launch_merge<T>(c, m, batch, st);
  mark(kStMerge, st);
  return ms;
}

// k_new / v_new non-null: fused append + decode (sals_append_decode): one projection
// launch writes the new latent / value rows (slot seq_len - 1) and projects the query.
template <typename T>
sals_status decode_impl(const sals_config* c, const void* U, const void* q, const void* latent,
                        const void* v_cache, int64_t cap, int batch, const int* seq_len, int max_s,
                        void* out, int* sel_out, float* scores_out, char* ws, const Plan& p,
                        cudaStream_t st, const void* k_new = nullptr, const void* v_new = nullptr) {
  float* qtil = reinterpret_cast<float*>(ws + p.off_qtil);
  float* qrope = reinterpret_cast<float*>(ws + p.off_qrope);
  int* sel = reinterpret_cast<int*>(ws + p.off_sel);
  int* count = reinterpret_cast<int*>(ws + p.off_count);
  float* scores = scores_out ? scores_out : reinterpret_cast<float*>(ws + p.off_scores);
  const int64_t sstride = scores_out ? max_s : p.score_stride;

  ProjectArgs pa{};
  pa.U = U; pa.x = q; pa.x_stride = c->num_q_heads * c->head_dim; pa.D = p.D; pa.r = c->rank;
  pa.ncols = c->score_rank; pa.B = batch; pa.head_dim = c->head_dim; pa.group = p.G;
  pa.n_q = c->num_q_heads; pa.out_f32 = qtil; pa.qrope = qrope; pa.seq_len = seq_len; pa.rope = make_rope(c);
  uint32_t* hist = reinterpret_cast<uint32_t*>(ws + p.off_hist);
  pa.hist0_zero = hist; pa.hist0_words = p.hist_words;
  mark_begin(st);
  const bool fused = k_new != nullptr;
  sals_status s = SALS_OK;
  if (fused) {
    pa.xa = k_new; pa.ncols_a = c->rank; pa.v_new = v_new; pa.pos = nullptr;
    pa.v_bits = vq_bits(c); pa.v_row_bytes = (int)v_row_bytes(c);
    pa.hp_window = hp_window(c); pa.hp_ring_off = (int64_t)batch * cap * (int64_t)v_row_bytes(c);
    pa.latent = const_cast<void*>(latent); pa.v_cache = const_cast<void*>(v_cache); pa.cap = cap;
    Plan pf = p;
    plan_proj(pf, false);   // the append's cluster shape (more column blocks)
    s = on(kStQproj) ? launch_project<T>(c, pf, 2, pa, st) : SALS_OK;
  } else if (on(kStQproj)) {
    s = launch_project<T>(c, p, 1, pa, st);
  }
  if (s != SALS_OK) return s;
  mark(kStQproj, st);

  ScoreArgs sa{};
  sa.latent = latent; sa.cap = cap; sa.r = c->rank; sa.rstar = c->score_rank; sa.qtil = qtil;
  sa.len = seq_len; sa.scores = scores; sa.stride = sstride;
  sa.hist0 = hist; sa.seq_len = seq_len; sa.idx_base = 0; sa.sink = c->sink; sa.recent = c->recent;
  sa.stream_after_wait = fused ? 1 : 0;   // the new latent row comes from the kernel just before
  s = on(kStScore) ? launch_score<T>(c, sa, batch, max_s, st) : SALS_OK;
  if (s != SALS_OK) return s;
  mark(kStScore, st);

  TopkArgs ta{};
  ta.scores = scores; ta.score_stride = sstride; ta.seq_len = seq_len; ta.idx_base = 0;
  ta.k = c->top_k; ta.sink = c->sink; ta.recent = c->recent; ta.mode = 0; ta.slice = p.tk_slice;
  ta.sel_out = sel; ta.sel_stride = c->top_k; ta.sel_count = count; ta.pad_to = c->top_k;
  ta.sel_out2 = sel_out;
  ta.hist0 = hist;
  s = on(kStTopk) ? launch_topk(ta, batch, p, st) : SALS_OK;
  if (s != SALS_OK) return s;
  mark(kStTopk, st);

  return attend_list<T>(c, p, U, latent, v_cache, cap, batch, 0, sel, count, ws, out, nullptr, st, seq_len);
}

}  // namespace

// =====================================================================  C ABI
extern "C" {

const char* sals_status_string(sals_status s) {
  switch (s) {
    case SALS_OK: return "SALS_OK";
    case SALS_ERR_INVALID_ARGUMENT: return "SALS_ERR_INVALID_ARGUMENT";
    case SALS_ERR_UNSUPPORTED: return "SALS_ERR_UNSUPPORTED";
    case SALS_ERR_WORKSPACE_TOO_SMALL: return "SALS_ERR_WORKSPACE_TOO_SMALL";
    case SALS_ERR_CUDA: return "SALS_ERR_CUDA";
    case SALS_ERR_NCCL: return "SALS_ERR_NCCL";
  }
  return "SALS_ERR_UNKNOWN";
}

const char* sals_last_error(void) { return g_err.c_str(); }

size_t sals_v_row_bytes(const sals_config* cfg) {
  if (validate(cfg) != SALS_OK) return 0;
  return v_row_bytes(cfg);
}

size_t sals_v_cache_bytes(const sals_config* cfg, int32_t batch, int64_t cap) {
  if (validate(cfg) != SALS_OK || batch < 1 || cap < 1) return 0;
  return (size_t)batch * cap * v_row_bytes(cfg) + (size_t)batch * hp_window(cfg) * hp_row_bytes(cfg);
}

uint32_t sals_profile_stage_mask(uint32_t mask) {
  const uint32_t old = g_stage_mask;
  g_stage_mask = mask;
  return old;
}

uint64_t sals_launch_count(int32_t reset) {
  return reset ? g_launches.exchange(0) : g_launches.load();
}

sals_status sals_workspace_selection_offsets(const sals_config* cfg, int32_t batch, int32_t max_seq_len,
                                             size_t* off_sel, size_t* off_count) {
  sals_status s = validate(cfg);
  if (s != SALS_OK) return s;
  if (!off_sel || !off_count || batch < 1 || max_seq_len < 1) return fail(SALS_ERR_INVALID_ARGUMENT, "bad arguments");
  Plan p{};
  s = make_plan(cfg, batch, max_seq_len, p, true);
  if (s != SALS_OK) return s;
  *off_sel = p.off_sel;
  *off_count = p.off_count;
  return SALS_OK;
}

size_t sals_workspace_bytes(const sals_config* cfg, int32_t batch, int32_t max_seq_len) {
  if (validate(cfg) != SALS_OK || batch < 1 || max_seq_len < 1) return 0;
  Plan p{};
  if (make_plan(cfg, batch, max_seq_len, p, true) != SALS_OK) return 0;
  return p.total;
}

sals_status sals_append_latent(const sals_config* cfg, const void* U, const void* k_new, const void* v_new,
                               int32_t batch, const int32_t* d_pos, void* latent_cache, void* v_cache,
                               int64_t cap, void* stream) {
  sals_status s = validate(cfg);
  if (s != SALS_OK) return s;
  if (!U || !k_new || !v_new || !d_pos || !latent_cache || !v_cache)
    return fail(SALS_ERR_INVALID_ARGUMENT, "NULL tensor argument");
  if (batch < 1 || batch > 65535 || cap < 1) return fail(SALS_ERR_INVALID_ARGUMENT, "bad batch / cap");
  Plan p{};
  p.D = cfg->num_kv_heads * cfg->head_dim;
  plan_proj(p, false);
  ProjectArgs a{};
  a.U = U; a.x = k_new; a.x_stride = p.D; a.D = p.D; a.r = cfg->rank; a.ncols = cfg->rank; a.B = batch;
  a.head_dim = cfg->head_dim; a.group = 1; a.n_q = cfg->num_q_heads; a.latent = latent_cache; a.cap = cap;
  a.pos = d_pos; a.v_new = v_new; a.v_cache = v_cache;
  a.v_bits = vq_bits(cfg); a.v_row_bytes = (int)v_row_bytes(cfg);
  a.hp_window = hp_window(cfg); a.hp_ring_off = (int64_t)batch * cap * (int64_t)v_row_bytes(cfg);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!on(kNumStages)) return SALS_OK;
  if (cfg->dtype == SALS_BF16) return launch_project<__nv_bfloat16>(cfg, p, 0, a, st);
  return launch_project<float>(cfg, p, 0, a, st);
}

sals_status sals_decode(const sals_config* cfg, const void* U, const void* q, const void* latent_cache,
                        const void* v_cache, int64_t cap, int32_t batch, const int32_t* d_seq_len,
                        int32_t max_seq_len, void* out, int32_t* sel_idx_out, float* scores_out,
                        void* workspace, size_t ws_bytes, void* stream) {
  sals_status s = validate(cfg);
  if (s != SALS_OK) return s;
  if (!U || !q || !latent_cache || !v_cache || !d_seq_len || !out || !workspace)
    return fail(SALS_ERR_INVALID_ARGUMENT, "NULL tensor argument");
  if (batch < 1 || batch > 65535) return fail(SALS_ERR_UNSUPPORTED, "batch %d outside [1, 65535]", batch);
  if (max_seq_len < 1 || max_seq_len > cap) return fail(SALS_ERR_INVALID_ARGUMENT, "need 1 <= max_seq_len <= cap");
  if (max_seq_len > kMaxSeqLen) return fail(SALS_ERR_UNSUPPORTED, "max_seq_len > %d", kMaxSeqLen);
  if (reinterpret_cast<uintptr_t>(workspace) % 256) return fail(SALS_ERR_INVALID_ARGUMENT, "workspace not 256-B aligned");
  Plan p{};
  s = make_plan(cfg, batch, max_seq_len, p, false);
  if (s != SALS_OK) return s;
  if (ws_bytes < p.total) return fail(SALS_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu", ws_bytes, p.total);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  char* ws = reinterpret_cast<char*>(workspace);
  if (cfg->dtype == SALS_BF16)
    return decode_impl<__nv_bfloat16>(cfg, U, q, latent_cache, v_cache, cap, batch, d_seq_len, max_seq_len, out,
                                      sel_idx_out, scores_out, ws, p, st);
  return decode_impl<float>(cfg, U, q, latent_cache, v_cache, cap, batch, d_seq_len, max_seq_len, out,
                            sel_idx_out, scores_out, ws, p, st);
}

int sals_prefill_impl(const sals_config* cfg, const void* U, const void* k, const void* v, int32_t batch,
                      int32_t n_tokens, int64_t start, void* latent_cache, void* v_cache, int64_t cap, void* stream,
                      int do_latent, int do_v);
const char* sals_prefill_last_error(void);

size_t sals_calibrate_ws_impl(int D);
int sals_calibrate_impl(const sals_config* cfg, const void* K, int64_t n_rows, void* U_out, float* eig_out,
                        void* workspace, size_t ws_bytes, void* stream);

size_t sals_calibrate_workspace_bytes(const sals_config* cfg) {
  if (validate(cfg) != SALS_OK) return 0;
  return sals_calibrate_ws_impl(cfg->num_kv_heads * cfg->head_dim);
}

sals_status sals_calibrate(const sals_config* cfg, const void* K, int64_t n_rows, void* U_out, float* eigvals_out,
                           void* workspace, size_t ws_bytes, void* stream) {
  sals_status s = validate(cfg);
  if (s != SALS_OK) return s;
  if (!K || !U_out || !workspace) return fail(SALS_ERR_INVALID_ARGUMENT, "NULL argument");
  if (n_rows < 1 || n_rows > 0x7fffffff) return fail(SALS_ERR_INVALID_ARGUMENT, "n_rows out of range");
  const int rc = sals_calibrate_impl(cfg, K, n_rows, U_out, eigvals_out, workspace, ws_bytes, stream);
  if (rc == 3) return fail(SALS_ERR_WORKSPACE_TOO_SMALL, "%s", sals_prefill_last_error());
  if (rc != 0) return fail(SALS_ERR_CUDA, "%s", sals_prefill_last_error());
  return SALS_OK;
}

sals_status sals_append_latent_bulk(const sals_config* cfg, const void* U, const void* k, const void* v,
                                    int32_t batch, int32_t n_tokens, int64_t start, void* latent_cache,
                                    void* v_cache, int64_t cap, void* stream) {
  sals_status s = validate(cfg);
  if (s != SALS_OK) return s;
  if (!U || !k || !v || !latent_cache || !v_cache) return fail(SALS_ERR_INVALID_ARGUMENT, "NULL tensor argument");
  if (batch < 1 || n_tokens < 1 || cap < 1 || start < 0 || start + n_tokens > cap)
    return fail(SALS_ERR_INVALID_ARGUMENT, "need batch, n_tokens >= 1 and 0 <= start, start + n_tokens <= cap");
  if (vq_bits(cfg) && (cfg->dtype != SALS_BF16 || cfg->head_dim != 128))
    return fail(SALS_ERR_UNSUPPORTED, "quantised value rows need bf16 and head_dim 128");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // latent rows: the tcgen05 GEMM (prefill_tc.cu), cuBLAS outside its shapes
  cudaError_t e = launch_prefill_tc(cfg, U, k, batch, n_tokens, start, latent_cache, cap, st);
  if (e != cudaSuccess && e != cudaErrorNotSupported) return fail(SALS_ERR_CUDA, "prefill_tc: %s", cudaGetErrorString(e));
  const bool latent_done = e == cudaSuccess;
  if (latent_done) g_launches.fetch_add(1, std::memory_order_relaxed);
  // value rows: quantised in a kernel (the append's rule), else copied by the fallback
  if (vq_bits(cfg)) {
    e = launch_prefill_vq(cfg, v, batch, n_tokens, start, v_cache, cap, (int)v_row_bytes(cfg), hp_window(cfg),
                          (int64_t)batch * cap * (int64_t)v_row_bytes(cfg), st);
    if (e != cudaSuccess) return fail(SALS_ERR_CUDA, "prefill_vq: %s", cudaGetErrorString(e));
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  if ((!latent_done || !vq_bits(cfg)) &&
      sals_prefill_impl(cfg, U, k, v, batch, n_tokens, start, latent_cache, v_cache, cap, stream, latent_done ? 0 : 1,
                        vq_bits(cfg) ? 0 : 1) != 0)
    return fail(SALS_ERR_CUDA, "%s", sals_prefill_last_error());
  return SALS_OK;
}

sals_status sals_append_decode(const sals_config* cfg, const void* U, const void* k_new, const void* v_new,
                               const void* q, void* latent_cache, void* v_cache, int64_t cap, int32_t batch,
                               const int32_t* d_seq_len, int32_t max_seq_len, void* out, int32_t* sel_idx_out,
                               float* scores_out, void* workspace, size_t ws_bytes, void* stream) {
  sals_status s = validate(cfg);
  if (s != SALS_OK) return s;
  if (!U || !k_new || !v_new || !q || !latent_cache || !v_cache || !d_seq_len || !out || !workspace)
    return fail(SALS_ERR_INVALID_ARGUMENT, "NULL tensor argument");
  if (batch < 1 || batch > 65535) return fail(SALS_ERR_UNSUPPORTED, "batch %d outside [1, 65535]", batch);
  if (max_seq_len < 1 || max_seq_len > cap) return fail(SALS_ERR_INVALID_ARGUMENT, "need 1 <= max_seq_len <= cap");
  if (max_seq_len > kMaxSeqLen) return fail(SALS_ERR_UNSUPPORTED, "max_seq_len > %d", kMaxSeqLen);
  if (reinterpret_cast<uintptr_t>(workspace) % 256) return fail(SALS_ERR_INVALID_ARGUMENT, "workspace not 256-B aligned");
  Plan p{};
  s = make_plan(cfg, batch, max_seq_len, p, false);
  if (s != SALS_OK) return s;
  if (ws_bytes < p.total) return fail(SALS_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu", ws_bytes, p.total);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  char* ws = reinterpret_cast<char*>(workspace);
  if (cfg->dtype == SALS_BF16)
    return decode_impl<__nv_bfloat16>(cfg, U, q, latent_cache, v_cache, cap, batch, d_seq_len, max_seq_len, out,
                                      sel_idx_out, scores_out, ws, p, st, k_new, v_new);
  return decode_impl<float>(cfg, U, q, latent_cache, v_cache, cap, batch, d_seq_len, max_seq_len, out,
                            sel_idx_out, scores_out, ws, p, st, k_new, v_new);
}

sals_status sals_decode_profile(const sals_config* cfg, const void* U, const void* q, const void* latent_cache,
                                const void* v_cache, int64_t cap, int32_t batch, const int32_t* d_seq_len,
                                int32_t max_seq_len, void* out, void* workspace, size_t ws_bytes, int32_t iters,
                                float* stage_ms, void* stream) {
  if (!stage_ms || iters < 1) return fail(SALS_ERR_INVALID_ARGUMENT, "stage_ms / iters");
  StageTimer t{};
  for (int i = 0; i <= kNumStages; ++i) SALS_CUDA_TRY(cudaEventCreate(&t.ev[i]));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  sals_status s = SALS_OK;
  for (int it = 0; it < iters && s == SALS_OK; ++it) {
    g_timer = &t;
    s = sals_decode(cfg, U, q, latent_cache, v_cache, cap, batch, d_seq_len, max_seq_len, out, nullptr, nullptr,
                    workspace, ws_bytes, stream);
    g_timer = nullptr;
    if (s != SALS_OK) break;
    if (cudaStreamSynchronize(st) != cudaSuccess) { s = fail(SALS_ERR_CUDA, "profile sync"); break; }
    cudaEvent_t prev = t.ev[kNumStages];
    for (int k = 0; k < kNumStages; ++k) {
      if (!t.used[k]) continue;
      float ms = 0.f;
      cudaEventElapsedTime(&ms, prev, t.ev[k]);
      t.ms[k] += ms;
      prev = t.ev[k];
    }
  }
  for (int k = 0; k < kNumStages; ++k) stage_ms[k] = t.used[k] ? t.ms[k] / iters : 0.f;
  for (int i = 0; i <= kNumStages; ++i) cudaEventDestroy(t.ev[i]);
  return s;
}

// ------------------------------------------------------------ dense baseline
// The TMA-streamed kernel (dense_tma.cu) where its shapes allow (bf16, d = 128,
// n_kv a multiple of 8), else flash_decode_kernel; SALS_DENSE_LSU=1 forces the latter.
static bool use_dense_tma(const sals_config* cfg) {
  static const bool force_lsu = [] { const char* e = getenv("SALS_DENSE_LSU"); return e && e[0] == '1'; }();
  return !force_lsu && dense_tma_supported(cfg->head_dim, cfg->num_kv_heads, cfg->num_q_heads / cfg->num_kv_heads,
                                           cfg->dtype == SALS_BF16 ? 2 : 4);
}
static void plan_dense(const sals_config* cfg, int batch, int max_seq_len, int& nsplit, int& chunk) {
  if (use_dense_tma(cfg)) {
    int nsm = 0;
    if (device_sm_count(&nsm) != cudaSuccess || nsm < 1) nsm = 148;
    dense_tma_plan(batch, max_seq_len, cfg->head_dim, cfg->num_kv_heads, nsm, nsplit, chunk);
  } else {
    plan_flash(batch, cfg->num_kv_heads, max_seq_len, flash_tpw_unr(cfg), nsplit, chunk);
  }
}

// threads of the dense append / query-RoPE kernels: one per rotation pair and per
// 16-byte vector of a head row
static int dense_rope_threads(const sals_config* cfg) {
  const int half = cfg->head_dim / 2, nvec = cfg->head_dim * (int)esize(cfg) / 16;
  return (int)align_up((size_t)std::max(half, nvec), 32);
}

size_t sals_dense_workspace_bytes(const sals_config* cfg, int32_t batch, int32_t max_seq_len) {
  if (validate(cfg) != SALS_OK || batch < 1 || max_seq_len < 1) return 0;
  int nsplit, chunk;
  plan_dense(cfg, batch, max_seq_len, nsplit, chunk);
  return align_up((size_t)batch * cfg->num_q_heads * cfg->head_dim * 4, 256) +
         align_up((size_t)batch * cfg->num_q_heads * nsplit * (cfg->head_dim + 2) * 4, 256);
}

sals_status sals_dense_append(const sals_config* cfg, const void* k_new, const void* v_new, int32_t batch,
                              const int32_t* d_pos, void* k_cache, void* v_cache, int64_t cap, void* stream) {
  sals_status s = validate(cfg);
  if (s != SALS_OK) return s;
  if (!k_new || !v_new || !d_pos || !k_cache || !v_cache) return fail(SALS_ERR_INVALID_ARGUMENT, "NULL tensor argument");
  if (batch < 1 || batch > 65535) return fail(SALS_ERR_INVALID_ARGUMENT, "bad batch");
  DenseAppendArgs a{};
  a.k_new = k_new; a.v_new = v_new; a.pos = d_pos; a.k_cache = k_cache; a.v_cache = v_cache; a.cap = cap;
  a.D = cfg->num_kv_heads * cfg->head_dim; a.head_dim = cfg->head_dim; a.n_kv = cfg->num_kv_heads;
  a.rope = make_rope(cfg);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const dim3 grid(cfg->num_kv_heads, batch), block(dense_rope_threads(cfg));
  if (cfg->dtype == SALS_BF16) SALS_CUDA_TRY(launch(dense_append_kernel<__nv_bfloat16>, grid, block, 0, st, 0, a));
  else SALS_CUDA_TRY(launch(dense_append_kernel<float>, grid, block, 0, st, 0, a));
  return SALS_OK;
}

sals_status sals_dense_decode(const sals_config* cfg, const void* q, const void* k_cache, const void* v_cache,
                              int64_t cap, int32_t batch, const int32_t* d_seq_len, int32_t max_seq_len,
                              void* out, void* workspace, size_t ws_bytes, void* stream) {
  sals_status s = validate(cfg);
  if (s != SALS_OK) return s;
  if (!q || !k_cache || !v_cache || !d_seq_len || !out || !workspace)
    return fail(SALS_ERR_INVALID_ARGUMENT, "NULL tensor argument");
  if (batch < 1 || batch > 65535 || max_seq_len < 1 || max_seq_len > cap)
    return fail(SALS_ERR_INVALID_ARGUMENT, "bad batch / max_seq_len");
  if (ws_bytes < sals_dense_workspace_bytes(cfg, batch, max_seq_len))
    return fail(SALS_ERR_WORKSPACE_TOO_SMALL, "dense workspace too small");
  int nsplit, chunk;
  plan_dense(cfg, batch, max_seq_len, nsplit, chunk);
  const bool tma = use_dense_tma(cfg);
  char* ws = reinterpret_cast<char*>(workspace);
  float* qrope = reinterpret_cast<float*>(ws);
  float* part = reinterpret_cast<float*>(ws + align_up((size_t)batch * cfg->num_q_heads * cfg->head_dim * 4, 256));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Plan p{};
  p.D = cfg->num_kv_heads * cfg->head_dim;
  p.G = cfg->num_q_heads / cfg->num_kv_heads;
  // query RoPE at s_b - 1 (fp32): one CTA per (query head, request)
  DenseAppendArgs ra{};
  ra.k_new = q; ra.head_dim = cfg->head_dim; ra.rope = make_rope(cfg);
  const dim3 rgrid(cfg->num_q_heads, batch), rblock(dense_rope_threads(cfg));
  FlashArgs f{};
  f.qrope = qrope; f.kbase = k_cache; f.v_cache = v_cache; f.count = d_seq_len; f.cap = cap; f.D = p.D;
  f.k_stride = 0; f.n_q = cfg->num_q_heads; f.n_kv = cfg->num_kv_heads; f.nsplit = nsplit; f.chunk = chunk;
  f.scale_log2 = scale_log2(cfg); f.partials = part;
  MergeArgs m{};
  m.partials = part; m.bh_stride = (int64_t)nsplit * (cfg->head_dim + 2); m.s_stride = cfg->head_dim + 2;
  m.nsplit = nsplit; m.n_q = cfg->num_q_heads; m.head_dim = cfg->head_dim; m.out = out; m.normalize = 1;
  if (cfg->dtype == SALS_BF16) {
    SALS_CUDA_TRY(launch(dense_qrope_kernel<__nv_bfloat16>, rgrid, rblock, 0, st, 0, ra, d_seq_len, qrope,
                         (int)cfg->num_q_heads));
    if (tma) {
      SALS_CUDA_TRY(launch_dense_tma(f, batch, cfg->head_dim, p.G, st));
      g_launches.fetch_add(1, std::memory_order_relaxed);
    } else {
      s = launch_flash<__nv_bfloat16, true>(cfg, f, batch, st);
    }
    if (s != SALS_OK) return s;
    return launch_merge<__nv_bfloat16>(cfg, m, batch, st);
  }
  SALS_CUDA_TRY(launch(dense_qrope_kernel<float>, rgrid, rblock, 0, st, 0, ra, d_seq_len, qrope,
                       (int)cfg->num_q_heads));
  s = launch_flash<float, true>(cfg, f, batch, st);
  if (s != SALS_OK) return s;
  return launch_merge<float>(cfg, m, batch, st);
}

// ------------------------------------------------------------ sharded decode
size_t sals_shard_workspace_bytes(const sals_config* cfg, int32_t batch, int32_t max_local_len, int32_t world) {
  if (validate(cfg) != SALS_OK || batch < 1 || max_local_len < 1 || world < 1) return 0;
  Plan p{};
  if (make_plan(cfg, batch, std::max(max_local_len, 1), p, true) != SALS_OK) return 0;
  return align_up(p.total, 256);
}

// (k_new != nullptr: the new token's latent / value rows are appended in the query
// projection's launch, on the shard that holds position s_b - 1; sals_append_decode_sharded)
static sals_status shard_candidates_impl(const sals_config* cfg, const void* U, const void* q,
                                         const void* latent_shard, int64_t cap_local, int32_t batch,
                                         int64_t shard_start, const int32_t* d_local_len, int32_t max_local_len,
                                         const int32_t* d_seq_len, float* cand_score, int32_t* cand_idx,
                                         void* workspace, size_t ws_bytes, void* stream, const void* k_new,
                                         const void* v_new, void* v_shard) {
  sals_status s = validate(cfg);
  if (s != SALS_OK) return s;
  if (!U || !q || !latent_shard || !d_local_len || !d_seq_len || !cand_score || !cand_idx || !workspace)
    return fail(SALS_ERR_INVALID_ARGUMENT, "NULL tensor argument");
  if (batch < 1 || max_local_len < 1 || max_local_len > cap_local || shard_start < 0)
    return fail(SALS_ERR_INVALID_ARGUMENT, "bad shard geometry");
  Plan p{};
  s = make_plan(cfg, batch, max_local_len, p, false);
  if (s != SALS_OK) return s;
  if (ws_bytes < sals_shard_workspace_bytes(cfg, batch, max_local_len, 1))
    return fail(SALS_ERR_WORKSPACE_TOO_SMALL, "shard workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  char* ws = reinterpret_cast<char*>(workspace);
  float* qtil = reinterpret_cast<float*>(ws + p.off_qtil);
  float* scores = reinterpret_cast<float*>(ws + p.off_scores);
  ProjectArgs pa{};
  pa.U = U; pa.x = q; pa.x_stride = cfg->num_q_heads * cfg->head_dim; pa.D = p.D; pa.r = cfg->rank;
  pa.ncols = cfg->score_rank; pa.B = batch; pa.head_dim = cfg->head_dim; pa.group = p.G; pa.n_q = cfg->num_q_heads;
  pa.out_f32 = qtil; pa.qrope = reinterpret_cast<float*>(ws + p.off_qrope); pa.seq_len = d_seq_len;
  pa.rope = make_rope(cfg);
  uint32_t* hist = reinterpret_cast<uint32_t*>(ws + p.off_hist);
  pa.hist0_zero = hist; pa.hist0_words = p.hist_words;
  const bool fused = k_new != nullptr;
  if (fused) {   // append role in the same launch: one read of U (as sals_append_decode)
    pa.xa = k_new; pa.ncols_a = cfg->rank; pa.v_new = v_new; pa.pos = nullptr;
    pa.v_bits = vq_bits(cfg); pa.v_row_bytes = (int)v_row_bytes(cfg);
    pa.latent = const_cast<void*>(latent_shard); pa.v_cache = v_shard; pa.cap = cap_local;
    pa.append_len = d_local_len; pa.append_base = shard_start;
  }
  const int mode = fused ? 2 : 1;
  ScoreArgs sa{};
  sa.latent = latent_shard; sa.cap = cap_local; sa.r = cfg->rank; sa.rstar = cfg->score_rank; sa.qtil = qtil;
  sa.len = d_local_len; sa.scores = scores; sa.stride = p.score_stride;
  sa.hist0 = hist; sa.seq_len = d_seq_len; sa.idx_base = shard_start; sa.sink = cfg->sink; sa.recent = cfg->recent;
  sa.stream_after_wait = fused ? 1 : 0;   // the new latent row comes from the kernel just before
  if (cfg->dtype == SALS_BF16) {
    if (on(kStQproj)) s = launch_project<__nv_bfloat16>(cfg, p, mode, pa, st);
    if (s == SALS_OK && on(kStScore)) s = launch_score<__nv_bfloat16>(cfg, sa, batch, max_local_len, st);
  } else {
    if (on(kStQproj)) s = launch_project<float>(cfg, p, mode, pa, st);
    if (s == SALS_OK && on(kStScore)) s = launch_score<float>(cfg, sa, batch, max_local_len, st);
  }
  if (s != SALS_OK) return s;
  TopkArgs ta{};
  ta.scores = scores; ta.score_stride = p.score_stride; ta.n_entries = d_local_len; ta.seq_len = d_seq_len;
  ta.idx_base = shard_start; ta.k = cfg->top_k; ta.sink = cfg->sink; ta.recent = cfg->recent; ta.mode = 1;
  ta.slice = p.tk_slice; ta.sel_out = cand_idx; ta.sel_stride = cfg->top_k; ta.sel_score = cand_score;
  ta.pad_to = cfg->top_k;
  ta.sel_count = reinterpret_cast<int*>(ws + p.off_ccount);   // read by the selection (shard.cu)
  ta.hist0 = hist;
  return on(kStTopk) ? launch_topk(ta, batch, p, st) : SALS_OK;
}

sals_status sals_shard_candidates(const sals_config* cfg, const void* U, const void* q, const void* latent_shard,
                                  int64_t cap_local, int32_t batch, int64_t shard_start,
                                  const int32_t* d_local_len, int32_t max_local_len, const int32_t* d_seq_len,
                                  float* cand_score, int32_t* cand_idx, void* workspace, size_t ws_bytes,
                                  void* stream) {
  return shard_candidates_impl(cfg, U, q, latent_shard, cap_local, batch, shard_start, d_local_len, max_local_len,
                               d_seq_len, cand_score, cand_idx, workspace, ws_bytes, stream, nullptr, nullptr,
                               nullptr);
}

sals_status sals_shard_attend(const sals_config* cfg, const void* U, const void* q, const void* latent_shard,
                              const void* v_shard, int64_t cap_local, int32_t batch, int64_t shard_start,
                              const int32_t* d_local_len, int32_t max_local_len, const int32_t* d_seq_len,
                              const float* cand_all_score, const int32_t* cand_idx, int32_t world, int32_t rank,
                              float* partial, void* workspace, size_t ws_bytes, void* stream) {
  sals_status s = validate(cfg);
  if (s != SALS_OK) return s;
  if (!U || !q || !latent_shard || !v_shard || !d_local_len || !d_seq_len || !cand_all_score || !cand_idx ||
      !partial || !workspace)
    return fail(SALS_ERR_INVALID_ARGUMENT, "NULL tensor argument");
  if (world < 1 || rank < 0 || rank >= world || batch < 1 || max_local_len < 1 || max_local_len > cap_local)
    return fail(SALS_ERR_INVALID_ARGUMENT, "bad shard geometry");
  if (hp_window(cfg)) return fail(SALS_ERR_UNSUPPORTED, "the quantised values' recent window is not sharded");
  Plan p{};
  s = make_plan(cfg, batch, max_local_len, p, false);
  if (s != SALS_OK) return s;
  if (ws_bytes < sals_shard_workspace_bytes(cfg, batch, max_local_len, world))
    return fail(SALS_ERR_WORKSPACE_TOO_SMALL, "shard workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  char* ws = reinterpret_cast<char*>(workspace);
  int* own = reinterpret_cast<int*>(ws + p.off_sel);
  int* own_count = reinterpret_cast<int*>(ws + p.off_count);
  // global selection from the gathered scores fused with this rank's owned list (shard.cu)
  ShardSelectArgs sa{};
  sa.all_score = cand_all_score; sa.own_idx = cand_idx; sa.world = world; sa.rank = rank; sa.batch = batch;
  sa.kc = cfg->top_k; sa.seq_len = d_seq_len; sa.local_len = d_local_len; sa.shard_start = shard_start;
  sa.k = cfg->top_k; sa.sink = cfg->sink; sa.recent = cfg->recent; sa.own_sel = own; sa.own_count = own_count;
  sa.cand_count = reinterpret_cast<const int*>(ws + p.off_ccount);
  // one rank: the selection is every local candidate -- a parallel copy over kSelCopyCtas CTAs
  if (on(kStShardSelect))
    SALS_CUDA_TRY(launch(shard_select_kernel, dim3(batch, world == 1 ? kSelCopyCtas : 1), dim3(1024), 0, st, 0, sa));
  if (cfg->dtype == SALS_BF16)
    return attend_list<__nv_bfloat16>(cfg, p, U, latent_shard, v_shard, cap_local, batch, shard_start, own,
                                      own_count, ws, nullptr, partial, st);
  return attend_list<float>(cfg, p, U, latent_shard, v_shard, cap_local, batch, shard_start, own, own_count, ws,
                            nullptr, partial, st);
}

sals_status sals_merge_partials(const sals_config* cfg, const float* partial_all, int32_t world, int32_t batch,
                                void* out, void* stream) {
  sals_status s = validate(cfg);
  if (s != SALS_OK) return s;
  if (!partial_all || !out || world < 1 || batch < 1) return fail(SALS_ERR_INVALID_ARGUMENT, "bad merge arguments");
  MergeArgs m{};
  m.partials = partial_all; m.bh_stride = cfg->head_dim + 2;
  m.s_stride = (int64_t)batch * cfg->num_q_heads * (cfg->head_dim + 2);
  m.nsplit = world; m.n_q = cfg->num_q_heads; m.head_dim = cfg->head_dim; m.out = out; m.normalize = 1;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (cfg->dtype == SALS_BF16) return launch_merge<__nv_bfloat16>(cfg, m, batch, st);
  return launch_merge<float>(cfg, m, batch, st);
}

}  // extern "C"

// ------------------------------------------- sharded decode with its own NCCL
// the whole sharded layer-step in one call -- the three device
// phases above around two in-place NCCL all-gathers on the caller's stream
// (NVLink / NVSwitch between the GPUs of a node).  NCCL is resolved at run time
// (dlopen of libnccl.so.2: the copy torch already loaded if there is one), so
// the library has no link-time NCCL dependency.
namespace {
struct NcclFns {
  decltype(&ncclGetUniqueId) get_id = nullptr;
  decltype(&ncclCommInitRank) init = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) err = nullptr;
  bool ok = false;
};
const NcclFns& nccl() {
  static const NcclFns f = [] {
    NcclFns n{};
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return n;
    n.get_id = reinterpret_cast<decltype(n.get_id)>(dlsym(h, "ncclGetUniqueId"));
    n.init = reinterpret_cast<decltype(n.init)>(dlsym(h, "ncclCommInitRank"));
    n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(h, "ncclCommDestroy"));
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(dlsym(h, "ncclAllGather"));
    n.group_start = reinterpret_cast<decltype(n.group_start)>(dlsym(h, "ncclGroupStart"));
    n.group_end = reinterpret_cast<decltype(n.group_end)>(dlsym(h, "ncclGroupEnd"));
    n.err = reinterpret_cast<decltype(n.err)>(dlsym(h, "ncclGetErrorString"));
    n.ok = n.get_id && n.init && n.destroy && n.all_gather && n.group_start && n.group_end && n.err;
    return n;
  }();
  return f;
}
struct SalsComm {
  ncclComm_t comm;
  int32_t world, rank;
};
#define SALS_NCCL_TRY(expr)                                                              \
  do {                                                                                   \
    ncclResult_t r_ = (expr);                                                            \
    if (r_ != ncclSuccess) return fail(SALS_ERR_NCCL, "%s: %s", #expr, nccl().err(r_)); \
  } while (0)
struct ShardLayout {
  size_t base, cand_s, cand_i, part, part_all, total;
};
ShardLayout shard_layout(const sals_config* cfg, int32_t batch, int32_t max_local_len, int32_t world) {
  ShardLayout L{};
  L.base = align_up(sals_shard_workspace_bytes(cfg, batch, max_local_len, world), 256);
  const size_t cand = align_up((size_t)world * batch * cfg->top_k * 4, 256);
  const size_t part = (size_t)batch * cfg->num_q_heads * (cfg->head_dim + 2) * 4;
  L.cand_s = L.base;                                                  // [P, B, k] gathered scores
  L.cand_i = L.cand_s + cand;                                         // [B, k] this rank's indices
  L.part_all = L.cand_i + align_up((size_t)batch * cfg->top_k * 4, 256);
  L.total = L.part_all + align_up(part * world, 256);
  return L;
}
}  // namespace

extern "C" {

sals_status sals_comm_unique_id(void* id_out) {
  if (!id_out) return fail(SALS_ERR_INVALID_ARGUMENT, "NULL id buffer");
  if (!nccl().ok) return fail(SALS_ERR_NCCL, "libnccl.so.2 not found");
  SALS_NCCL_TRY(nccl().get_id(reinterpret_cast<ncclUniqueId*>(id_out)));
  return SALS_OK;
}

sals_status sals_comm_init(const void* nccl_unique_id, int32_t world, int32_t rank, void** comm) {
  if (!nccl_unique_id || !comm || world < 1 || rank < 0 || rank >= world)
    return fail(SALS_ERR_INVALID_ARGUMENT, "bad communicator arguments");
  if (!nccl().ok) return fail(SALS_ERR_NCCL, "libnccl.so.2 not found");
  ncclUniqueId id;
  memcpy(&id, nccl_unique_id, sizeof(id));
  ncclComm_t c = nullptr;
  SALS_NCCL_TRY(nccl().init(&c, world, id, rank));
  *comm = new SalsComm{c, world, rank};
  return SALS_OK;
}

sals_status sals_comm_destroy(void* comm) {
  if (!comm) return SALS_OK;
  SalsComm* c = reinterpret_cast<SalsComm*>(comm);
  ncclResult_t r = nccl().destroy(c->comm);
  delete c;
  if (r != ncclSuccess) return fail(SALS_ERR_NCCL, "ncclCommDestroy: %s", nccl().err(r));
  return SALS_OK;
}

size_t sals_decode_sharded_workspace_bytes(const sals_config* cfg, int32_t batch, int32_t max_local_len,
                                           int32_t world) {
  if (sals_shard_workspace_bytes(cfg, batch, max_local_len, world) == 0) return 0;
  return shard_layout(cfg, batch, max_local_len, world).total;
}

static sals_status decode_sharded_impl(const sals_config* cfg, void* comm, const void* U, const void* q,
                                       const void* latent_shard, const void* v_shard, int64_t cap_local,
                                       int32_t batch, int64_t shard_start, const int32_t* d_local_len,
                                       int32_t max_local_len, const int32_t* d_seq_len, void* out, void* workspace,
                                       size_t ws_bytes, void* stream, const void* k_new, const void* v_new) {
  sals_status s = validate(cfg);
  if (s != SALS_OK) return s;
  // everything the later phases check, checked before the first one enqueues work
  if (!comm) return fail(SALS_ERR_INVALID_ARGUMENT, "NULL communicator");
  if (!U || !q || !latent_shard || !v_shard || !d_local_len || !d_seq_len || !out || !workspace)
    return fail(SALS_ERR_INVALID_ARGUMENT, "NULL tensor argument");
  if (batch < 1 || max_local_len < 1 || max_local_len > cap_local || shard_start < 0)
    return fail(SALS_ERR_INVALID_ARGUMENT, "bad shard geometry");
  if (hp_window(cfg)) return fail(SALS_ERR_UNSUPPORTED, "the quantised values' recent window is not sharded");
  const SalsComm* c = reinterpret_cast<const SalsComm*>(comm);
  const int P = c->world, me = c->rank;
  if (ws_bytes < sals_decode_sharded_workspace_bytes(cfg, batch, max_local_len, P))
    return fail(SALS_ERR_WORKSPACE_TOO_SMALL, "sharded workspace too small");
  const ShardLayout L = shard_layout(cfg, batch, max_local_len, P);
  char* ws = reinterpret_cast<char*>(workspace);
  const size_t nc = (size_t)batch * cfg->top_k;
  const size_t np = (size_t)batch * cfg->num_q_heads * (cfg->head_dim + 2);
  float* cand_s = reinterpret_cast<float*>(ws + L.cand_s);
  int32_t* cand_i = reinterpret_cast<int32_t*>(ws + L.cand_i);
  float* part_all = reinterpret_cast<float*>(ws + L.part_all);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // 1. local candidates: scores straight into this rank's slot of the gather buffer,
  //    global indices kept locally (the gathered order (rank, position) is the index order)
  s = shard_candidates_impl(cfg, U, q, latent_shard, cap_local, batch, shard_start, d_local_len, max_local_len,
                            d_seq_len, cand_s + me * nc, cand_i, workspace, L.base, stream, k_new, v_new,
                            const_cast<void*>(v_shard));
  if (s != SALS_OK) return s;
  // 2. in-place all-gather of the candidate scores (rank order)
  if (on(kStExchange)) SALS_NCCL_TRY(nccl().all_gather(cand_s + me * nc, cand_s, nc, ncclFloat32, c->comm, st));
  // 3. global selection + owned list (one kernel), attention over the owned tokens -> partial slot
  s = sals_shard_attend(cfg, U, q, latent_shard, v_shard, cap_local, batch, shard_start, d_local_len, max_local_len,
                        d_seq_len, cand_s, cand_i, P, me, part_all + me * np, workspace, L.base, stream);
  if (s != SALS_OK) return s;
  // 4. in-place all-gather of the partials, 5. merge on every rank
  if (on(kStExchange)) SALS_NCCL_TRY(nccl().all_gather(part_all + me * np, part_all, np, ncclFloat32, c->comm, st));
  return on(kStMerge) ? sals_merge_partials(cfg, part_all, P, batch, out, stream) : SALS_OK;
}

sals_status sals_decode_sharded(const sals_config* cfg, void* comm, const void* U, const void* q,
                                const void* latent_shard, const void* v_shard, int64_t cap_local, int32_t batch,
                                int64_t shard_start, const int32_t* d_local_len, int32_t max_local_len,
                                const int32_t* d_seq_len, void* out, void* workspace, size_t ws_bytes,
                                void* stream) {
  return decode_sharded_impl(cfg, comm, U, q, latent_shard, v_shard, cap_local, batch, shard_start, d_local_len,
                             max_local_len, d_seq_len, out, workspace, ws_bytes, stream, nullptr, nullptr);
}

sals_status sals_append_decode_sharded(const sals_config* cfg, void* comm, const void* U, const void* k_new,
                                       const void* v_new, const void* q, void* latent_shard, void* v_shard,
                                       int64_t cap_local, int32_t batch, int64_t shard_start,
                                       const int32_t* d_local_len, int32_t max_local_len, const int32_t* d_seq_len,
                                       void* out, void* workspace, size_t ws_bytes, void* stream) {
  if (!k_new || !v_new) return fail(SALS_ERR_INVALID_ARGUMENT, "NULL tensor argument");
  return decode_sharded_impl(cfg, comm, U, q, latent_shard, v_shard, cap_local, batch, shard_start, d_local_len,
                             max_local_len, d_seq_len, out, workspace, ws_bytes, stream, k_new, v_new);
}

}  // extern "C"
