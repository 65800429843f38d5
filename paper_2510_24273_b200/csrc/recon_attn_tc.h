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
  int ntiles;             // tiles per request = ceil(k / 128)
};

bool tc_supported(int head_dim, int D, int rank, int G);
sals_status launch_recon_attn_tc(const TcArgs& a, int batch, cudaStream_t st);
const char* tc_last_error();

}  // namespace sals
