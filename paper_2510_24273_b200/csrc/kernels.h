// Kernel argument structs and declarations shared by the kernels and the
// host launcher (api.cu).  Internal to the library; the public boundary is
// include/sals.h.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "sals.h"

namespace sals {

// Block sizes shared by kernels and launcher.
constexpr int kScoreThreads = 256;
// First radix digit of the top-k, built by the score kernel: the top 11 bits of
// the order-preserving float key of every ranked score.
constexpr int kH0Bits = 11, kH0Bins = 1 << kH0Bits, kH0Shift = 32 - kH0Bits;
constexpr int kCandCap = 12288;   // threshold-bin candidate keys held by every top-k CTA (48 KB)

struct ProjectArgs {
  const void* U;        // [D, r]
  const void* x;        // append: k_new [B, D]; qproj: q [B, n_q*d]
  int x_stride;
  int D, r, ncols;      // ncols = r (append) or r* (qproj)
  int B, head_dim, group, n_q;
  int rows_per_cta;
  // qproj outputs
  float* out_f32;       // [B, r*]
  float* qrope;         // [B, n_q, d]
  const int* seq_len;   // [B]
  RopeTable rope;
  // append outputs
  void* latent; int64_t cap; const int* pos;
  const void* v_new; void* v_cache;
  uint32_t* hist0_zero; int hist0_words;   // qproj: zero the score histogram (rope-role CTAs)
  // fused append + query projection (MODE 2): append role's input / columns / block count;
  // pos == nullptr -> the new token's slot is seq_len[b] - 1
  const void* xa; int ncols_a; int n_append_blocks;
  // (sharded) append_len != nullptr: the new token's local slot is seq_len[b] - 1 - append_base,
  // written only when it is this shard's last row (append_len[b] - 1), else skipped
  const int* append_len; int64_t append_base;
  int v_bits, v_row_bytes;   // value row format (0: dtype values; 4 / 2: quantised, head_dim 128)
  int hp_window;             // > 0: the last hp_window tokens also kept at 8 bits in a ring after the main rows
  int64_t hp_ring_off;       // bytes from v_cache to the ring [B, hp_window, n_kv * 144]
};

struct ScoreArgs {
  const void* latent;   // [B, cap, r]
  int64_t cap; int r, rstar;
  const float* qtil;    // [B, r*]
  const int* len;       // [B] tokens to score (s_b, or the shard's local length)
  float* scores;        // [B, stride]
  int64_t stride;
  int tokens_per_cta;
  uint32_t* hist0;      // nullable [B, kH0Bins]: top-digit histogram of the ranked scores (zeroed upstream)
  const int* seq_len;   // [B] global s_b (ranked range [sink, s_b - recent))
  int64_t idx_base;     // global index of local token 0
  int sink, recent;
  int stream_after_wait;  // 1: the latent rows may have been written by the previous kernel (fused append)
};

struct TopkArgs {
  const float* scores; int64_t score_stride;  // [B, stride]
  const int* n_entries;   // nullable: entries of request b (else seq_len[b])
  const int* seq_len;     // [B] global s_b
  int64_t idx_base;       // global index of entry 0 (shard start)
  int k, sink, recent;
  int mode;               // 0 = full Alg. 1 selection; 1 = ranked-range candidates only
  int slice;              // entries per CTA
  int* sel_out; int64_t sel_stride;
  float* sel_score;       // nullable
  int* sel_count;         // nullable [B]
  int pad_to;             // -1 padding up to this many entries
  int* sel_out2;          // nullable second copy of sel_out (user buffer), stride sel_stride
  const uint32_t* hist0;  // nullable [B, kH0Bins] from the score kernel: histogram-assisted path
  int cand_cap;           // histogram-assisted path: capacity of the cluster-wide candidate array
};

struct ReconArgs {        // SIMT reconstruct + RoPE (path S)
  const void* latent; int64_t cap; int r;
  const void* U;
  const int* sel; const int* count; int k_stride;
  int D, head_dim;
  int64_t pos_base;       // global position of latent row 0 (shards)
  RopeTable rope;
  void* kr;               // [B*k_stride, D]
};

struct FlashArgs {        // split-K flash decode over a token list (sparse or dense)
  const float* qrope;     // [B, n_q, d]
  const void* kbase;      // dense: k_cache [B, cap, D]; sparse: K^R_C [B*k_stride, D]
  const void* v_cache;    // [B, cap, D]
  const int* sel;         // sparse: [B, k_stride] (local rows into v_cache)
  const int* count;       // [B]
  int64_t cap; int D, k_stride, n_q, n_kv, nsplit, chunk;
  float scale_log2;
  float* partials;        // [B, n_q, nsplit, d+2]
  int64_t sel_row_base;   // subtract from sel entries to get the local v_cache row
};

struct MergeArgs {
  const float* partials;
  int64_t bh_stride, s_stride;
  int nsplit, n_q, head_dim;
  void* out;              // normalize: y [B, n_q*d] (T); else fp32 partial [B, n_q, d+2] (m, l, o)
  int normalize;
};

struct DenseAppendArgs {
  const void* k_new; const void* v_new; const int* pos;
  void* k_cache; void* v_cache; int64_t cap;
  int D, head_dim, n_kv;
  RopeTable rope;
};

struct ShardSelectArgs {   // sharded: global selection from the gathered scores + owned list (shard.cu)
  const float* all_score;   // [P, B, kc] all-gathered candidate scores (rank order, -inf padded)
  const int* own_idx;       // [B, kc] this rank's candidates (global index, ascending, -1 padded)
  int world, rank, batch, kc;
  const int* seq_len; const int* local_len; int64_t shard_start;
  int k, sink, recent;
  int* own_sel; int* own_count;   // [B, k] local rows ascending, [B]
  const int* cand_count;          // [B] valid entries of own_idx (a prefix: the list is compacted)
};
cudaError_t launch_prefill_tc(const sals_config* c, const void* U, const void* k, int batch, int n, int64_t start,
                              void* latent, int64_t cap, cudaStream_t st);
cudaError_t launch_prefill_vq(const sals_config* c, const void* v, int batch, int n, int64_t start, void* v_cache,
                              int64_t cap, int v_row_bytes, int hp_window, int64_t hp_ring_off, cudaStream_t st);
constexpr int kSelCopyCtas = 16;   // CTAs per request of the one-rank (copy) selection
__global__ void shard_select_kernel(ShardSelectArgs a);


template <typename T, int MODE, int NT> __global__ void project_kernel(ProjectArgs a);
template <typename T, int LG, int CPL> __global__ void latent_score_kernel(ScoreArgs a);
// TMA-streamed bf16 scoring (score_tma.cu); cudaErrorNotSupported outside its shapes.
// Single-CTA histogram-assisted top-k for <= 8192 entries per request (topk_cta.cu).
cudaError_t launch_topk_cta(const TopkArgs& a, int batch, int max_entries, cudaStream_t st);
cudaError_t launch_score_tma(const ScoreArgs& a, int batch, int max_len, cudaStream_t st, int nsm);
// TMA-streamed dense comparator (dense_tma.cu); cudaErrorNotSupported outside its shapes.
bool dense_tma_supported(int head_dim, int n_kv, int G, int dtype_bytes);
void dense_tma_plan(int batch, int max_len, int head_dim, int n_kv, int nsm, int& nsplit, int& chunk);
cudaError_t launch_dense_tma(const FlashArgs& a, int batch, int head_dim, int G, cudaStream_t st);
template <int NT> __global__ void topk_hist_kernel(TopkArgs a);
template <typename T> __global__ void recon_rope_simt_kernel(ReconArgs a);
template <typename T, int DH, int G, bool DENSE> __global__ void flash_decode_kernel(FlashArgs a);
template <typename T> __global__ void merge_kernel(MergeArgs a);
template <typename T> __global__ void dense_append_kernel(DenseAppendArgs a);
template <typename T> __global__ void dense_qrope_kernel(DenseAppendArgs a, const int* seq_len, float* qrope, int n_q);

}  // namespace sals
