// K4 / K9: TopK selection  C = TopK(p', k)   (Alg. 1 line 5)
// with the sink / critical / recent policy and ties to the lower
// index (reading R5).  One thread-block CLUSTER per request.
//
// Each CTA of the cluster holds a contiguous slice of the request's scores in
// shared memory as order-preserving uint32 keys.  The threshold key T (the
// need-th largest ranked key) is found by radix selection; a final ordered
// compaction writes, in ascending index order, every forced entry, every
// ranked entry with key > T and the first (need - #{key > T}) entries equal to
// T.  Ordered work is done warp-wise on 32 consecutive entries at a time
// (ballot + popc), so shared-memory accesses are conflict-free.
//
// This is the GENERIC kernel, used for K9 (global selection over the
// all-gathered shard candidates): four 8-bit cluster-wide radix passes
// (per-warp histograms pushed to every peer with DSMEM stores).  The decode
// path (K4) and the shard-local selection (K8) use the histogram-assisted
// kernel in topk_hist.cu.
//
// mode 0 (sals_decode): entry e is token e; forced = [0,x) u [s-z,s); the
//   k-x-z best of [x, s-z) are ranked; all s tokens when s <= k.
// mode 1 (sharded): entries carry global indices (cand_idx, or idx_base + e);
//   only the ranked range [x, s-z) takes part; up to k-x-z are selected.
#include "common.cuh"
#include "kernels.h"

namespace sals {

constexpr int kTopkWarps = kTopkThreads / 32;
constexpr int kMaxCluster = 16;

#ifdef SALS_TC_TRACE
__device__ unsigned long long g_tk_trace[32];
#define TK_STAMP(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_tk_trace[(i)] = clock64(); } while (0)
#else
#define TK_STAMP(i) do {} while (0)
#endif

// Inclusive scan of one value per thread across the block; *total receives the
// block-wide sum (same value in every thread).
__device__ __forceinline__ int block_incl_scan(int v, int* warp_tot, int* total = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  if (lane == 31) warp_tot[warp] = v;
  __syncthreads();
  if (warp == 0) {
    int t = (lane < kTopkWarps) ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int n = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += n;
    }
    if (lane < kTopkWarps) warp_tot[lane] = t;   // inclusive warp prefix
  }
  __syncthreads();
  const int add = (warp > 0) ? warp_tot[warp - 1] : 0;
  const int r = v + add;
  if (total) *total = warp_tot[kTopkWarps - 1];
  __syncthreads();
  return r;
}

// Exclusive prefix over the warps of per-warp counts wc[w][q0..q0+NQ) in place
// (warp 0), totals into tot[q].  Caller synchronises before and after.
template <int NQ>
__device__ __forceinline__ void warp_counts_exclusive(int (*wc)[4], int q0, int* tot) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
#pragma unroll
    for (int q = q0; q < q0 + NQ; ++q) {
      const int v = lane < kTopkWarps ? wc[lane][q] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += n;
      }
      if (lane < kTopkWarps) wc[lane][q] = incl - v;
      if (lane == 31) tot[q] = incl;
    }
  }
}

// Warp-level digit search: lane l owns bins 255 - 8l - j (descending); find the
// bin holding the rem-th largest and the count still needed inside it.
__device__ __forceinline__ void warp_digit_search(const uint32_t* hist, int rem, int* s_digit, int* s_need) {
  const int lane = threadIdx.x & 31;
  int c8[8], tot = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) { c8[j] = (int)hist[255 - 8 * lane - j]; tot += c8[j]; }
  int incl = tot;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int nb = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += nb;
  }
  int excl = incl - tot;
  if (excl < rem && rem <= incl) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (excl < rem && rem <= excl + c8[j]) { *s_digit = 255 - 8 * lane - j; *s_need = rem - excl; }
      excl += c8[j];
    }
  }
}

__global__ void __launch_bounds__(kTopkThreads)
topk_cluster_kernel(TopkArgs a) {
  extern __shared__ __align__(16) uint8_t tk_smem[];
  __shared__ uint32_t inc_hist[2][kMaxCluster][256];   // generic path: [pass parity][source rank][digit]
  __shared__ uint32_t s_tot[256];
  __shared__ int inc_cnt[kMaxCluster][8];              // [source rank]: ranked, def, eq, def0, cand
  __shared__ int wcnt[kTopkWarps][4];                   // per-warp counts -> exclusive warp bases
  __shared__ int s_ctot[4];
  __shared__ int warp_tot[32];
  __shared__ int s_digit, s_need, s_nranked;

  const int CS = (int)cluster_nctarank();
  const int rank = (int)cluster_ctarank();
  const int b = blockIdx.x / CS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const int slice = a.slice;
  uint32_t* keys = reinterpret_cast<uint32_t*>(tk_smem);
  uint8_t* cls = tk_smem + (size_t)slice * 4;   // 0 none, 1 forced, 2 ranked
  const size_t gidx_off = ((size_t)slice * 5 + 15) / 16 * 16;
  int* gidx = a.cand_idx ? reinterpret_cast<int*>(tk_smem + gidx_off) : nullptr;
  uint32_t (*whist)[256] = reinterpret_cast<uint32_t (*)[256]>(
      tk_smem + gidx_off + (a.cand_idx ? (size_t)slice * 4 : 0));

  TK_STAMP(0);
  pdl_wait();
  TK_STAMP(1);
  const int s = a.seq_len[b];
  const int n = a.n_entries ? a.n_entries[b] : (a.cand_idx ? a.n_const : s);
  const int e0 = rank * slice;
  const int nloc = max(0, min(slice, n - e0));
  const int x = a.sink, z = a.recent;
  const bool all_mode0 = (a.mode == 0) && (s <= a.k);
  // warp w owns the ordered chunk [w0, w1) of the slice, processed 32 entries per round
  const int wc = ((nloc + kTopkWarps - 1) / kTopkWarps + 31) / 32 * 32;
  const int w0 = min(nloc, warp * wc), w1 = min(nloc, w0 + wc);

  // ---- load slice -> keys / classes (8 independent loads in flight per thread) ----
  int my_ranked = 0;
  for (int i0 = tid; i0 < nloc; i0 += 8 * kTopkThreads) {
    float sc[8];
    int ix[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * kTopkThreads;
      sc[u] = 0.f;
      ix[u] = -1;
      if (i < nloc) {
        const int e = e0 + i;
        const size_t off = a.seg_len > 0 ? (size_t)(e / a.seg_len) * a.seg_stride + (size_t)b * a.seg_len + e % a.seg_len
                                         : (size_t)b * a.score_stride + e;
        ix[u] = a.cand_idx ? a.cand_idx[off] : (int)(a.idx_base + e);
        sc[u] = a.scores[off];
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * kTopkThreads;
      if (i >= nloc) continue;
      const int idx = ix[u];
      uint8_t c = 0;
      if (idx >= 0 && idx < s) {
        const bool in_rank = (idx >= x) && (idx < s - z);
        if (a.mode == 0) c = (all_mode0 || !in_rank) ? 1 : 2;
        else c = in_rank ? 2 : 0;
      }
      keys[i] = (c == 2) ? float_key(sc[u]) : 0u;
      cls[i] = c;
      if (gidx) gidx[i] = idx;
      my_ranked += (c == 2);
    }
  }
  __syncthreads();
  TK_STAMP(2);

  // Results of either selection path: threshold key T, ties taken (lowest
  // indices first), and the cross-CTA counts that place this CTA's output.
  uint32_t T = 0xffffffffu;
  int need_eq = 0;
  int def_before = 0, eq_before = 0, def_total = 0, eq_total = 0, eq_local = 0;
  {
    // four cluster-wide 8-bit radix passes
    {
      int tot;
      block_incl_scan(my_ranked, warp_tot, &tot);
      if (tid < CS) st_dsmem_u32(mapa_shared(smem_u32(&inc_cnt[rank][0]), tid), (uint32_t)tot);
    }
    cluster_sync_all();
    if (tid == 0) {
      int nr = 0;
      for (int c = 0; c < CS; ++c) nr += inc_cnt[c][0];
      int nd = (a.mode == 0) ? (all_mode0 ? 0 : a.k - x - z) : (a.k - x - z);
      s_nranked = nr;
      s_need = max(0, min(nd, nr));
    }
    __syncthreads();
    const int n_ranked = s_nranked;
    const int need = s_need;
    __syncthreads();
    T = 0xffffffffu;
    need_eq = 0;
    if (need == n_ranked && need > 0) {
      T = 0u; need_eq = n_ranked;          // every ranked entry is selected
    } else if (need > 0) {
      uint32_t prefix = 0;
      int rem = need;
      for (int i = tid; i < kTopkWarps * 256; i += kTopkThreads) (&whist[0][0])[i] = 0;
      __syncthreads();
      for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        for (int i = tid; i < nloc; i += kTopkThreads) {
          if (cls[i] != 2) continue;
          const uint32_t key = keys[i];
          if (pass > 0 && ((key ^ prefix) >> (shift + 8)) != 0) continue;
          atomicAdd(&whist[warp][(key >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (tid < 256) {
          uint32_t t = 0;
#pragma unroll
          for (int w = 0; w < kTopkWarps; ++w) { t += whist[w][tid]; whist[w][tid] = 0; }
          const uint32_t addr = smem_u32(&inc_hist[pass & 1][rank][tid]);
          for (int c = 0; c < CS; ++c) st_dsmem_u32(mapa_shared(addr, c), t);
        }
        cluster_sync_all();
        if (tid < 256) {
          uint32_t t = 0;
          for (int c = 0; c < CS; ++c) t += inc_hist[pass & 1][c][tid];
          s_tot[tid] = t;
        }
        __syncthreads();
        if (warp == 0) warp_digit_search(s_tot, rem, &s_digit, &s_need);
        __syncthreads();
        prefix |= (uint32_t)s_digit << shift;
        rem = s_need;
        __syncthreads();
      }
      T = prefix;
      need_eq = rem;
    }
    // per-CTA definite / tie counts, exchanged
    {
      int dcnt = 0, ecnt = 0;
      for (int base = w0; base < w1; base += 32) {
        const int i = base + lane;
        bool d = false, e = false;
        if (i < w1) {
          const uint8_t c = cls[i];
          d = (c == 1) || (c == 2 && keys[i] > T);
          e = (c == 2 && keys[i] == T);
        }
        dcnt += __popc(__ballot_sync(0xffffffffu, d));
        ecnt += __popc(__ballot_sync(0xffffffffu, e));
      }
      if (lane == 0) { wcnt[warp][2] = dcnt; wcnt[warp][3] = ecnt; }
    }
    __syncthreads();
    if (tid == 0) {
      int d = 0, e = 0;
      for (int w = 0; w < kTopkWarps; ++w) { d += wcnt[w][2]; e += wcnt[w][3]; }
      s_ctot[2] = d;
      s_ctot[3] = e;
    }
    __syncthreads();
    if (tid < CS) {
      st_dsmem_u32(mapa_shared(smem_u32(&inc_cnt[rank][1]), tid), (uint32_t)s_ctot[2]);
      st_dsmem_u32(mapa_shared(smem_u32(&inc_cnt[rank][2]), tid), (uint32_t)s_ctot[3]);
    }
    cluster_sync_all();
    for (int c = 0; c < CS; ++c) {
      const int dc = inc_cnt[c][1], ec = inc_cnt[c][2];
      if (c < rank) { def_before += dc; eq_before += ec; }
      def_total += dc; eq_total += ec;
    }
    eq_local = inc_cnt[rank][2];
  }
  TK_STAMP(9);

  // ---- ordered compaction (shared by both paths) ----------------------------
  const int take_local = max(0, min(need_eq - eq_before, eq_local));
  const int out_base = def_before + min(need_eq, eq_before);
  const int count = def_total + min(need_eq, eq_total);
  {
    int dcnt = 0, ecnt = 0;
    for (int base = w0; base < w1; base += 32) {
      const int i = base + lane;
      bool d = false, e = false;
      if (i < w1) {
        const uint8_t c = cls[i];
        d = (c == 1) || (c == 2 && keys[i] > T);
        e = (c == 2 && keys[i] == T);
      }
      dcnt += __popc(__ballot_sync(0xffffffffu, d));
      ecnt += __popc(__ballot_sync(0xffffffffu, e));
    }
    if (lane == 0) { wcnt[warp][2] = dcnt; wcnt[warp][3] = ecnt; }
  }
  __syncthreads();
  warp_counts_exclusive<2>(wcnt, 2, s_ctot);
  __syncthreads();
  int* out = a.sel_out + (size_t)b * a.sel_stride;
  int* out2 = a.sel_out2 ? a.sel_out2 + (size_t)b * a.sel_stride : nullptr;
  float* osc = a.sel_score ? a.sel_score + (size_t)b * a.sel_stride : nullptr;
  {
    int rd = wcnt[warp][2], re = wcnt[warp][3];     // running definite / tie counts before the round
    for (int base = w0; base < w1; base += 32) {
      const int i = base + lane;
      bool d = false, e = false;
      if (i < w1) {
        const uint8_t c = cls[i];
        d = (c == 1) || (c == 2 && keys[i] > T);
        e = (c == 2 && keys[i] == T);
      }
      const uint32_t dm = __ballot_sync(0xffffffffu, d), em = __ballot_sync(0xffffffffu, e);
      const int db = rd + __popc(dm & lt_mask);      // definite entries before i in this CTA
      const int eb = re + __popc(em & lt_mask);      // ties before i in this CTA
      if (d || (e && eb < take_local)) {
        const int pos = out_base + db + min(eb, take_local);
        const int gi = gidx ? gidx[i] : (int)(a.idx_base + e0 + i);
        out[pos] = gi;
        if (out2) out2[pos] = gi;
        if (osc) osc[pos] = key_float(keys[i]);
      }
      rd += __popc(dm);
      re += __popc(em);
    }
  }
  if (rank == CS - 1) {
    for (int i = count + tid; i < a.pad_to; i += kTopkThreads) {
      out[i] = -1;
      if (out2) out2[i] = -1;
      if (osc) osc[i] = -INFINITY;
    }
    if (tid == 0 && a.sel_count) a.sel_count[b] = count;
  }
  TK_STAMP(10);
  cluster_sync_all();   // keep shared memory alive until every peer finished its DSMEM reads
  TK_STAMP(11);
  pdl_launch_dependents();
}

}  // namespace sals

extern "C" int sals_debug_topk_trace(unsigned long long* out) {
#ifdef SALS_TC_TRACE
  return (int)cudaMemcpyFromSymbol(out, sals::g_tk_trace, sizeof(sals::g_tk_trace));
#else
  (void)out;
  return -1;
#endif
}
