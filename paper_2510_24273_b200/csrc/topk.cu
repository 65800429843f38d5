// K4 / K9: TopK selection  C = TopK(p', k)   (Alg. 1 line 5)
// with the sink / critical / recent policy and ties to the lower
// index (reading R5).  One thread-block CLUSTER per request.
//
// Each CTA of the cluster loads a contiguous slice of the request's scores
// into shared memory as order-preserving uint32 keys.  Four 8-bit radix
// passes find the threshold key T (the need-th largest ranked key): per-warp
// shared-memory histograms -> CTA histogram -> summed across the cluster
// through DSMEM, and every CTA picks the same digit.  A final ordered
// compaction writes, in ascending index order, every forced entry, every
// ranked entry with key > T, and the first (need - #{key > T}) entries with
// key == T (lowest indices first, counted across CTAs in rank order).
//
// mode 0 (sals_decode): entry e is token e; forced = [0,x) u [s-z,s); the
//   k-x-z best of [x, s-z) are ranked; all s tokens when s <= k.
// mode 1 (sharded): entries carry global indices (cand_idx, or idx_base + e);
//   only the ranked range [x, s-z) takes part; up to k-x-z are selected.
//   Used for a shard's local candidates and for the global select (K9) over
//   the all-gathered candidates, which arrive in ascending index order.
#include "common.cuh"
#include "kernels.h"

namespace sals {

constexpr int kTopkWarps = kTopkThreads / 32;
constexpr int kMaxCluster = 16;

// Inclusive scan of one value per thread across the 512-thread block; *total
// receives the block-wide sum (same value in every thread).
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

__global__ void __launch_bounds__(kTopkThreads)
topk_cluster_kernel(TopkArgs a) {
  extern __shared__ __align__(16) uint8_t tk_smem[];
  // Cluster exchange is push-based: every CTA stores its values into a slot of
  // EVERY peer's shared memory (fire-and-forget st.shared::cluster), so after
  // the cluster barrier all reads are local.
  __shared__ uint32_t inc_hist[2][kMaxCluster][256];   // [pass parity][source rank][digit]
  __shared__ uint32_t s_tot[256];
  __shared__ int inc_cnt[kMaxCluster][4];              // [source rank]: ranked, definite, ties
  __shared__ int warp_tot[32];
  __shared__ int s_digit, s_need, s_nranked;

  const int CS = (int)cluster_nctarank();
  const int rank = (int)cluster_ctarank();
  const int b = blockIdx.x / CS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int slice = a.slice;
  uint32_t* keys = reinterpret_cast<uint32_t*>(tk_smem);
  uint8_t* cls = tk_smem + (size_t)slice * 4;   // 0 none, 1 forced, 2 ranked
  // global indices are only stored when they come from a candidate list
  const size_t gidx_off = ((size_t)slice * 5 + 15) / 16 * 16;
  int* gidx = a.cand_idx ? reinterpret_cast<int*>(tk_smem + gidx_off) : nullptr;
  // per-warp digit histograms after the key / class / index arrays
  uint32_t (*whist)[256] = reinterpret_cast<uint32_t (*)[256]>(
      tk_smem + gidx_off + (a.cand_idx ? (size_t)slice * 4 : 0));

  pdl_wait();
  const int s = a.seq_len[b];
  const int n = a.n_entries ? a.n_entries[b] : (a.cand_idx ? a.n_const : s);
  const int e0 = rank * slice;
  const int nloc = max(0, min(slice, n - e0));
  const int x = a.sink, z = a.recent;
  const bool all_mode0 = (a.mode == 0) && (s <= a.k);

  // ---- load slice -> keys / classes (4 independent loads in flight per thread) ----
  int my_ranked = 0;
  for (int i0 = tid; i0 < nloc; i0 += 4 * kTopkThreads) {
    float sc[4];
    int ix[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
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
    for (int u = 0; u < 4; ++u) {
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
  {
    int tot;
    block_incl_scan(my_ranked, warp_tot, &tot);
    if (tid >= kTopkThreads - 32 && tid - (kTopkThreads - 32) < CS)
      st_dsmem_u32(mapa_shared(smem_u32(&inc_cnt[rank][0]), tid - (kTopkThreads - 32)), (uint32_t)tot);
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

  // ---- radix select of the threshold key T (4 x 8-bit passes) ------------
  uint32_t T = 0xffffffffu;
  int need_eq = 0;
  if (need == n_ranked && need > 0) {
    T = 0u; need_eq = n_ranked;          // every ranked entry is selected
  } else if (need > 0) {
    uint32_t prefix = 0;
    int rem = need;
    for (int i = tid; i < kTopkWarps * 256; i += kTopkThreads) (&whist[0][0])[i] = 0;
    __syncthreads();
    for (int pass = 0; pass < 4; ++pass) {
      const int shift = 24 - 8 * pass;
      // per-warp histogram of the digit (shared-memory atomics; a fully conflicting
      // warp costs ~32 cycles, cheaper than aggregating with match.any)
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
      if (warp == 0) {
        // lane l owns digits 255 - 8l - j, j = 0..7 (descending)
        int c8[8], tot = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) { c8[j] = (int)s_tot[255 - 8 * lane - j]; tot += c8[j]; }
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
            if (excl < rem && rem <= excl + c8[j]) { s_digit = 255 - 8 * lane - j; s_need = rem - excl; }
            excl += c8[j];
          }
        }
      }
      __syncthreads();
      prefix |= (uint32_t)s_digit << shift;
      rem = s_need;
    }
    T = prefix;
    need_eq = rem;
  }

  // ---- ordered compaction ------------------------------------------------
  const int run = (nloc + kTopkThreads - 1) / kTopkThreads;
  const int i0 = min(nloc, tid * run), i1 = min(nloc, i0 + run);
  int n_def = 0, n_eq = 0;
  for (int i = i0; i < i1; ++i) {
    const uint8_t c = cls[i];
    if (c == 1 || (c == 2 && keys[i] > T)) ++n_def;
    else if (c == 2 && keys[i] == T) ++n_eq;
  }
  int def_cta, eq_cta;
  const int def_incl = block_incl_scan(n_def, warp_tot, &def_cta);
  const int eq_incl = block_incl_scan(n_eq, warp_tot, &eq_cta);
  if (tid >= kTopkThreads - 32 && tid - (kTopkThreads - 32) < CS) {
    const int c = tid - (kTopkThreads - 32);
    st_dsmem_u32(mapa_shared(smem_u32(&inc_cnt[rank][1]), c), (uint32_t)def_cta);
    st_dsmem_u32(mapa_shared(smem_u32(&inc_cnt[rank][2]), c), (uint32_t)eq_cta);
  }
  cluster_sync_all();
  int def_before = 0, eq_before = 0, def_total = 0, eq_total = 0;
  for (int c = 0; c < CS; ++c) {
    const int dc = inc_cnt[c][1];
    const int ec = inc_cnt[c][2];
    if (c < rank) { def_before += dc; eq_before += ec; }
    def_total += dc; eq_total += ec;
  }
  const int eq_local = inc_cnt[rank][2];
  const int take_local = max(0, min(need_eq - eq_before, eq_local));
  const int out_base = def_before + min(need_eq, eq_before);
  const int count = def_total + min(need_eq, eq_total);

  int pos = out_base + (def_incl - n_def) + min(eq_incl - n_eq, take_local);
  int eq_rank = eq_incl - n_eq;
  int* out = a.sel_out + (size_t)b * a.sel_stride;
  int* out2 = a.sel_out2 ? a.sel_out2 + (size_t)b * a.sel_stride : nullptr;
  float* osc = a.sel_score ? a.sel_score + (size_t)b * a.sel_stride : nullptr;
  for (int i = i0; i < i1; ++i) {
    const uint8_t c = cls[i];
    bool take = false;
    if (c == 1 || (c == 2 && keys[i] > T)) take = true;
    else if (c == 2 && keys[i] == T) { take = eq_rank < take_local; ++eq_rank; }
    if (take) {
      const int gi = gidx ? gidx[i] : (int)(a.idx_base + e0 + i);
      out[pos] = gi;
      if (out2) out2[pos] = gi;
      if (osc) osc[pos] = key_float(keys[i]);
      ++pos;
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
  cluster_sync_all();   // keep shared memory alive until every peer finished its DSMEM reads
  pdl_launch_dependents();
}

}  // namespace sals
