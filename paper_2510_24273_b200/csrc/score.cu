// K3: latent scoring  p'_j = q~_{:r*} . K~[b, j, :r*]   (Alg. 1 line 4)
//
// HBM-bound stream over the first r* coordinates of every latent row
// (B * s * r* * sizeof(T) bytes; Sec. 4.5 "read s r* elements").
// LG lanes cover one token with 16-byte ld.global.nc loads (CPL 16-B chunks
// per lane); each lane keeps its slice of q~ in registers, so the only
// traffic is the latent stream.  Each warp keeps UNR tokens' loads in flight
// before reducing.  The per-token reduction order (chunk-sequential in a lane,
// then an xor butterfly over LG lanes) does not depend on the grid, so a
// sequence shard scores its tokens bit-identically.
#include "common.cuh"
#include "kernels.h"

namespace sals {


template <typename T, int LG, int CPL>
__global__ void __launch_bounds__(kScoreThreads)
latent_score_kernel(ScoreArgs a) {
  constexpr int EPC = Elem<T>::kPer16;
  constexpr int TPW = 32 / LG;
  constexpr int UNR = (CPL == 1) ? 8 : (CPL == 2 ? 4 : 2);
  const int b = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / LG, li = lane % LG;
  const int V = a.rstar / EPC;  // 16-B chunks per token
  __shared__ uint32_t hs[kH0Bins];
  if (a.hist0)
    for (int i = threadIdx.x; i < kH0Bins; i += kScoreThreads) hs[i] = 0;
  __syncthreads();

  pdl_wait();
  float qreg[CPL][EPC];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int ch = li + c * LG;
#pragma unroll
    for (int e = 0; e < EPC; ++e) qreg[c][e] = (ch < V) ? a.qtil[(size_t)b * a.rstar + ch * EPC + e] : 0.f;
  }
  const int len = a.len[b];
  const int t0 = blockIdx.x * a.tokens_per_cta;
  const int t1 = min(t0 + a.tokens_per_cta, len);
  const char* base = reinterpret_cast<const char*>(a.latent) + (size_t)b * a.cap * a.r * sizeof(T);
  const size_t row_bytes = (size_t)a.r * sizeof(T);
  float* out = a.scores + (size_t)b * a.stride;
  constexpr int kWarps = kScoreThreads / 32;
  // ranked range (global indices) for the top-digit histogram
  const int64_t s_glob = a.hist0 ? a.seq_len[b] : 0;
  const int64_t r_lo = a.sink, r_hi = s_glob - a.recent;

  for (int tb = t0 + warp * TPW * UNR; tb < t1; tb += kWarps * TPW * UNR) {
    uint4 raw[UNR][CPL];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int t = tb + u * TPW + sub;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int ch = li + c * LG;
        raw[u][c] = (t < t1 && ch < V) ? ld_nc_v4(base + (size_t)t * row_bytes + ch * 16)
                                       : make_uint4(0, 0, 0, 0);
      }
    }
    float acc[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      acc[u] = 0.f;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        float f[EPC];
        Elem<T>::unpack(raw[u][c], f);
#pragma unroll
        for (int e = 0; e < EPC; ++e) acc[u] = fmaf(f[e], qreg[c][e], acc[u]);
      }
#pragma unroll
      for (int off = LG / 2; off > 0; off >>= 1) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], off);
    }
    // every lane of a token group holds the token's score after the butterfly:
    // lane li writes (and histograms) the tokens u with u % LG == li, in parallel
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (u % LG != li) continue;
      const int t = tb + u * TPW + sub;
      if (t < t1) {
        out[t] = acc[u];
        const int64_t g = a.idx_base + t;
        if (a.hist0 && g >= r_lo && g < r_hi) atomicAdd(&hs[float_key(acc[u]) >> kH0Shift], 1u);
      }
    }
  }
  if (a.hist0) {
    __syncthreads();
    uint32_t* gh = a.hist0 + (size_t)b * kH0Bins;
    for (int i = threadIdx.x; i < kH0Bins; i += kScoreThreads)
      if (hs[i]) atomicAdd(&gh[i], hs[i]);
  }
  pdl_launch_dependents();
}

#define SALS_SCORE_INST(T)                                              \
  template __global__ void latent_score_kernel<T, 1, 1>(ScoreArgs);     \
  template __global__ void latent_score_kernel<T, 2, 1>(ScoreArgs);     \
  template __global__ void latent_score_kernel<T, 4, 1>(ScoreArgs);     \
  template __global__ void latent_score_kernel<T, 8, 1>(ScoreArgs);     \
  template __global__ void latent_score_kernel<T, 16, 1>(ScoreArgs);    \
  template __global__ void latent_score_kernel<T, 32, 1>(ScoreArgs);    \
  template __global__ void latent_score_kernel<T, 32, 2>(ScoreArgs);    \
  template __global__ void latent_score_kernel<T, 32, 4>(ScoreArgs);
SALS_SCORE_INST(float)
SALS_SCORE_INST(__nv_bfloat16)

}  // namespace sals
