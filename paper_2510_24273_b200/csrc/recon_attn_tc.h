// Fused tcgen05 reconstruct + RoPE + sparse attention (path T) — launcher interface.
#pragma once
#include "kernels.h"
#include "../../include/sals.h"

namespace sals {

constexpr int kTcRows = 128;   // selected tokens per tile (UMMA M)

struct TcArgs {
  const void* latent; int64_t cap; int r;
  const void* U;
  const void* v_cache;
  const int* sel; const int* count; int k_stride;
  int D, head_dim, G, n_q;
  int64_t pos_base;
  RopeTable rope;
  const float* qrope;
  float scale_log2;
  float* partials;        // [B, n_q, ntiles, d+2]
  int ntiles;             // v1: tiles per request = ceil(k / 128); v2: chunks per request
  int tiles_per_cta;      // v2: tiles of 128 tokens per CTA (chunk length)
  void* direct_out;       // v2: write y [B, n_q*d] directly (no merge kernel): one chunk, or
                          // several with `counters` (the last chunk CTA of a (request, column
                          // block) merges the partials, deterministic split order)
  unsigned* counters;     // v2, nullable: [B, D/256] arrival counters, zero on entry
  int v_bits;             // 0: dtype values; 4 / 2: quantised value rows (v2 only)
  int v_row_bytes;        // bytes of one token's value row
  int hp_window;          // > 0: positions >= s_b - hp_window read their 8-bit ring rows (DESIGN R15)
  int64_t hp_ring_off;    // bytes from v_cache to the ring [B, hp_window, n_kv * 144]
  const int* seq_len;     // [B] (hp window)
};

bool tc_supported(int head_dim, int D, int rank, int G);
bool tc2_supported(int head_dim, int D, int rank, int G);   // persistent v2 (d = 128, G <= 4)
int tc2_merge_max_splits(int G);
bool tc2_pair_enabled();                                       // SALS_TC2_CG=2: cta_group::2 MHA variant                             // in-kernel split merge limit
sals_status launch_recon_attn_tc(const TcArgs& a, int batch, cudaStream_t st);
const char* tc_last_error();
// cuTensorMapEncodeTiled (driver entry point, resolved once), or nullptr.
void* tma_encoder_fn();

}  // namespace sals
