// K4, single-CTA variant for requests of at most 8192 entries (c2's 4K, the
// c5 sweep's 4K / 8K): C = TopK(p', k) (Alg. 1 line 5) with the sink /
// critical / recent policy and ties to the lower index (reading
// R5), identical output to topk_hist_kernel (cluster variant) and the oracle.
//
// One 1024-thread CTA per request, no cluster.  Thread t owns the EPT
// consecutive entries [t EPT, t EPT + EPT) in registers (float4 loads), so
// thread order is index order and every ordered step is a block scan:
//  P0  threshold bin of the top 11 key bits from the score kernel's histogram
//      hist0 (one descending block scan over 2048 bins, 2 per thread);
//  P1-P3  radix passes over key bits [20:13], [12:5], [4:0] of the ranked
//      entries that share the prefix (smem histogram of 256 bins, digit found
//      by one warp) -> the threshold key T and need_eq, the number of entries
//      equal to T to take; the passes stop as soon as every entry with the
//      resolved prefix is taken (T is then compared at that prefix's bits);
//  E   block scan of the per-thread counts of entries equal to T (index order)
//      -> which ties are taken (the lowest indices);
//  S   block scan of the per-thread selected counts -> ascending output.
// Keys are the order-preserving uint32 images of the fp32 scores (larger score
// => larger key), so selection by key is selection by score.
#include "common.cuh"
#include "kernels.h"

namespace sals {
namespace tkc {
#ifdef SALS_TKC_TRACE
__device__ long long g_tkc_t[16];
#define TKC_T(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_tkc_t[i] = clock64(); } while (0)
#else
#define TKC_T(i) do {} while (0)
#endif

constexpr int NT = 1024;   // 32 warps (block_excl_scan relies on it)

// Block-wide exclusive scan of one int per thread (thread order): .x = the
// exclusive prefix, .y = the block total.  Two __syncthreads.
__device__ __forceinline__ int2 block_excl_scan(int v, int* wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += n;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int w = wsum[lane];   // NW == 32
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += n;
    }
    wsum[32 + lane] = wi - w;   // exclusive warp offsets
    if (lane == 31) wsum[64] = wi;
  }
  __syncthreads();
  return make_int2(wsum[32 + warp] + incl - v, wsum[64]);
}

// Every warp: the digit d of a 256-bin histogram h (descending) such that the
// entries in bins > d number < need <= those in bins >= d, need minus the entries
// in bins > d, and the entries in bin d.  Register-only result (ballot + shuffle
// broadcast), so no shared flag and no second barrier.
__device__ __forceinline__ int3 digit_search_all(const uint32_t* h, int need) {
  const int lane = threadIdx.x & 31;
  // bins 255 - 8 lane - j, j < 8: two 16-byte loads per lane (conflict-free, the
  // 1 KB histogram in 8 wavefronts; a scalar lane-strided read would be 8-way conflicted)
  const uint4 hi4 = reinterpret_cast<const uint4*>(h)[63 - 2 * lane];
  const uint4 lo4 = reinterpret_cast<const uint4*>(h)[62 - 2 * lane];
  const int c[8] = {(int)hi4.w, (int)hi4.z, (int)hi4.y, (int)hi4.x, (int)lo4.w, (int)lo4.z, (int)lo4.y, (int)lo4.x};
  int t = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) t += c[j];
  int incl = t;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += n;
  }
  int excl = incl - t;
  const bool mine = excl < need && need <= incl;
  const unsigned m = __ballot_sync(0xffffffffu, mine);
  int d = 0, r = need, cb = -1;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (mine && excl < need && need <= excl + c[j]) { d = 255 - 8 * lane - j; r = need - excl; cb = c[j]; }
    excl += c[j];
  }
  const int src = m ? __ffs(m) - 1 : 0;
  return make_int3(__shfl_sync(0xffffffffu, d, src), __shfl_sync(0xffffffffu, r, src),
                   __shfl_sync(0xffffffffu, cb, src));
}

template <int EPT>
__global__ void __launch_bounds__(NT, 1) topk_cta_kernel(TopkArgs a) {
  __shared__ __align__(16) uint32_t hist[3][256];   // one histogram per radix pass (no reuse, no extra barrier)
  __shared__ int wsum[3][65];   // one scratch per block scan
  __shared__ volatile int s_digit, s_need, s_cnt;
  __shared__ int3 s_dr[3];
  const int tid = threadIdx.x;
  const int b = blockIdx.x;
  if (tid < 256) { hist[0][tid] = 0; hist[1][tid] = 0; hist[2][tid] = 0; }

  TKC_T(0);
  pdl_wait();
  TKC_T(1);
  pdl_launch_dependents();   // the reconstruction kernel's prologue may start (see topk_hist.cu)
  const int s = a.seq_len[b];
  const int n = a.n_entries ? a.n_entries[b] : s;
  const int x = a.sink, z = a.recent;
  const bool mode0 = a.mode == 0;
  const bool all_mode0 = mode0 && (s <= a.k);
  const int ib32 = (int)a.idx_base;

  // ---- loads: this thread's EPT scores and 2 histogram bins (one round) ----
  const int e0 = tid * EPT;
  float sc[EPT];
  const float* row = a.scores + (size_t)b * a.score_stride;
  if (EPT >= 4 && (a.score_stride & 3) == 0) {
#pragma unroll
    for (int v = 0; v < EPT / 4; ++v) {
      const float4 f = (e0 + 4 * v < n) ? *reinterpret_cast<const float4*>(row + e0 + 4 * v)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
      sc[4 * v] = f.x; sc[4 * v + 1] = f.y; sc[4 * v + 2] = f.z; sc[4 * v + 3] = f.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < EPT; ++j) sc[j] = (e0 + j < n) ? row[e0 + j] : 0.f;
  }
  const uint32_t* hg = a.hist0 + (size_t)b * kH0Bins;
  const int c0 = (int)hg[kH0Bins - 1 - 2 * tid], c1 = (int)hg[kH0Bins - 2 - 2 * tid];

  uint32_t key[EPT];
  bool rk[EPT], fc[EPT];     // entry j ranked / forced
#pragma unroll
  for (int j = 0; j < EPT; ++j) {
    // 32-bit index arithmetic (positions < 2^31; checked by the launcher)
    const int i = e0 + j;
    const int gi = ib32 + i;
    const int valid = (i < n) & (gi < s);
    const int inr = (gi >= x) & (gi < s - z) & (all_mode0 ? 0 : 1);
    key[j] = float_key(sc[j]);
    rk[j] = (valid & inr) != 0;
    fc[j] = (valid & (inr ^ 1) & (mode0 ? 1 : 0)) != 0;
  }

  TKC_T(2);
  // ---- P0: threshold bin (descending scan of the 2048 top-digit bins) ----
  const int2 sc0 = block_excl_scan(c0 + c1, wsum[0]);
  const int excl0 = sc0.x, nr = sc0.y;
  // nd = clamp(want, 0, nr), with the two special cases decided by direct compares:
  // ptxas (CUDA 12.9, sm_100a) derived `clamp(...) == nr` from the select predicate of
  // a VIMNMX.RELU and got it wrong, so nothing below compares the clamped value
  const int want = all_mode0 ? 0 : a.k - x - z;
  const bool take_all = want >= nr;        // every ranked entry selected (also nr == 0)
  const bool take_none = want <= 0;
  const int nd = take_all ? nr : (take_none ? 0 : want);
  if (tid == 0) { s_digit = -2; s_need = 0; s_cnt = -1; }
  __syncthreads();
  if (nd > 0 && nd < nr) {
    if (excl0 < nd && nd <= excl0 + c0) { s_digit = kH0Bins - 1 - 2 * tid; s_need = nd - excl0; s_cnt = c0; }
    else if (excl0 + c0 < nd && nd <= excl0 + c0 + c1) {
      s_digit = kH0Bins - 2 - 2 * tid; s_need = nd - excl0 - c0; s_cnt = c1;
    }
  }
  __syncthreads();
  // T: every ranked key > T is selected, keys == T up to need_eq (index order).
  // The radix passes run unconditionally (block-uniform control flow around the
  // barriers); their result is ignored when no / every ranked entry is taken.
  const bool all_ranked = take_all;   // (includes nr == 0)
  if (take_none || nr == 0) {                 // no ranked entry selected
#pragma unroll
    for (int j = 0; j < EPT; ++j) rk[j] = false;
  }
  uint32_t prefix = (uint32_t)max(s_digit, 0) << kH0Shift;
  int rem = s_need;
  // tsh: the key bits below it are not resolved; the passes stop early (block-uniform:
  // every thread reads the same shared values) once every key with the resolved prefix
  // is taken (rem == the bin's count), and the selection then compares prefixes
  int tsh = s_cnt == rem ? kH0Shift : 0;
  TKC_T(3);
  // ---- P1-P3: radix passes over the ranked keys that share the prefix ----
#pragma unroll
  for (int ps = 0; ps < 3; ++ps) {
    if (tsh == 0) {
      const int sh = ps == 0 ? 13 : (ps == 1 ? 5 : 0);
      const uint32_t dmask = ps == 2 ? 31u : 255u;
      const int hi = sh + (ps == 2 ? 5 : 8);        // bits above this digit are fixed by the prefix
      uint32_t* h = hist[ps];
#pragma unroll
      for (int j = 0; j < EPT; ++j)
        if (rk[j] && (key[j] >> hi) == (prefix >> hi)) atomicAdd(&h[(key[j] >> sh) & dmask], 1u);
      __syncthreads();
      if (tid < 32) {   // one warp searches, the result is broadcast through shared memory
        const int3 dr = digit_search_all(h, rem);
        if (tid == 0) s_dr[ps] = dr;
      }
      __syncthreads();
      prefix |= (uint32_t)s_dr[ps].x << sh;
      rem = s_dr[ps].y;
      if (sh > 0 && s_dr[ps].z == rem) tsh = sh;
    }
  }
  // T (compared at bits >= tsh): keys above T are selected, keys equal to T up to need_eq
  const uint32_t T = prefix >> tsh;
  const int need_eq = rem;

  TKC_T(4);
  // ---- E + S in ONE block scan: per thread the ties (key == T) and the definite
  // picks (forced, or key > T, or every ranked entry); the ties taken before
  // thread t are min(ties before t, need_eq), so its first output slot is
  // (definite before t) + min(ties before t, need_eq).  Packed 16 + 16 bits
  // (counts <= 8192).
  int my_eq = 0, my_def = 0;
#pragma unroll
  for (int j = 0; j < EPT; ++j) {
    const bool eq = !all_ranked && rk[j] && (key[j] >> tsh) == T;
    const bool def = fc[j] || (rk[j] && (all_ranked || (key[j] >> tsh) > T));
    my_eq += eq ? 1 : 0;
    my_def += def ? 1 : 0;
  }
  TKC_T(5);
  const int2 scs = block_excl_scan((my_eq << 16) | my_def, wsum[1]);
  const int eq_before = scs.x >> 16, def_before = scs.x & 0xffff;
  const int count = (scs.y & 0xffff) + min(scs.y >> 16, need_eq);
  int pos = def_before + min(eq_before, need_eq);
  bool sl[EPT];
  {
    int e = eq_before;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const bool eq = !all_ranked && rk[j] && (key[j] >> tsh) == T;
      sl[j] = fc[j] || (rk[j] && (all_ranked || (key[j] >> tsh) > T)) || (eq && e < need_eq);
      e += eq ? 1 : 0;
    }
  }
  int* out = a.sel_out + (size_t)b * a.sel_stride;
  int* out2 = a.sel_out2 ? a.sel_out2 + (size_t)b * a.sel_stride : nullptr;
  float* osc = a.sel_score ? a.sel_score + (size_t)b * a.sel_stride : nullptr;
#pragma unroll
  for (int j = 0; j < EPT; ++j) {
    if (sl[j] && pos < a.pad_to) {   // (bound: an inconsistent histogram must not write out of row)
      const int gi = ib32 + e0 + j;
      out[pos] = gi;
      if (out2) out2[pos] = gi;
      if (osc) osc[pos] = key_float(key[j]);
      ++pos;
    }
  }
  for (int i = count + tid; i < a.pad_to; i += NT) {
    out[i] = -1;
    if (out2) out2[i] = -1;
    if (osc) osc[i] = -INFINITY;
  }
  if (tid == 0 && a.sel_count) a.sel_count[b] = min(count, a.pad_to);
  TKC_T(6);
}

}  // namespace tkc

cudaError_t launch_topk_cta(const TopkArgs& a, int batch, int max_entries, cudaStream_t st) {
  void (*k)(TopkArgs) = nullptr;
  if (max_entries <= 1024) k = tkc::topk_cta_kernel<1>;
  else if (max_entries <= 2048) k = tkc::topk_cta_kernel<2>;
  else if (max_entries <= 4096) k = tkc::topk_cta_kernel<4>;
  else if (max_entries <= 8192) k = tkc::topk_cta_kernel<8>;
  else return cudaErrorNotSupported;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(batch);
  cfg.blockDim = dim3(tkc::NT);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, a);
}

}  // namespace sals
