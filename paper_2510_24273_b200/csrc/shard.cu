// Sequence-sharded decode: the global selection of one rank from the
// all-gathered candidate SCORES, fused with its owned-token list.
//
// Every rank p holds the contiguous positions [lo_p, hi_p) of a request and has
// contributed its local top-min(k-x-z, n) candidates of the ranked range [x, s-z)
// (ascending global index, -inf padded) to the all-gathered array [P][B][kc].
// The global TopK (Alg. 1 line 5; ties -> lower index, DESIGN R5) takes the
// kr = k-x-z largest of their union.  Because the shards are contiguous and each
// rank's list is ascending, the global index order of the gathered entries is
// (rank, position): the indices never need to travel, only the scores.
//
// One CTA per request finds the exact kr-th largest key T among the P*kc entries
// by a three-pass radix select (11 + 11 + 10 bits of the order-preserving uint32
// key) and the quota of entries equal to T that the selection takes, then keeps
// THIS rank's candidates with key > T plus its share of the ties (ranks before it
// take theirs first) and writes the owned list:  owned sinks | owned picks |
// owned recents, as local rows, ascending.  When the union has <= kr entries
// (one rank, or short shards) every candidate is selected without a search.
#include "common.cuh"
#include "kernels.h"

namespace sals {

constexpr int kSelThreads = 1024;
constexpr int kSelBins = 2048;

// suffix count of the histogram: the digit d with cnt(> d) < need <= cnt(>= d);
// returns d and cnt(> d).  Every thread calls it (block barriers inside).
__device__ int select_digit(const unsigned* hist, int nbins, int need, int* s_warp, int* s_res, int* above) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = nbins / kSelThreads;   // 2 or 1 bins per thread, in descending digit order
  // thread t owns digits [nbins - per (t+1), nbins - per t) (descending across threads)
  int local = 0;
  for (int j = 0; j < per; ++j) local += (int)hist[nbins - 1 - (tid * per + j)];
  int incl = local;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += v;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = lane < kSelThreads / 32 ? s_warp[lane] : 0;
    int wi = w;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, wi, off);
      if (lane >= off) wi += v;
    }
    if (lane < kSelThreads / 32) s_warp[lane] = wi - w;   // exclusive warp offsets
  }
  __syncthreads();
  int before = s_warp[warp] + incl - local;   // count of digits above this thread's first digit
  for (int j = 0; j < per; ++j) {
    const int d = nbins - 1 - (tid * per + j);
    const int c = (int)hist[d];
    if (before < need && need <= before + c) { s_res[0] = d; s_res[1] = before; }
    before += c;
  }
  __syncthreads();
  *above = s_res[1];
  return s_res[0];
}

// Block-wide exclusive prefix sum of one int per thread; *total = the sum.  All threads call.
__device__ int block_excl_scan(int v, int* s_warp, int* total) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += t;
  }
  __syncthreads();   // s_warp free (a previous use has been read)
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int w = s_warp[lane];   // kSelThreads / 32 == 32 warps
    int wi = w;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, wi, off);
      if (lane >= off) wi += t;
    }
    s_warp[lane] = wi - w;
    if (lane == 31) s_warp[32] = wi;
  }
  __syncthreads();
  *total = s_warp[32];
  return s_warp[warp] + incl - v;
}

__global__ void __launch_bounds__(kSelThreads) shard_select_kernel(ShardSelectArgs a) {
  __shared__ unsigned hist[kSelBins];
  __shared__ int s_warp[kSelThreads / 32 + 1], s_res[2], s_cnt[2];
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_wait();
  const int s = a.seq_len[b];
  const int64_t lo = a.shard_start;
  const int64_t hi = min((int64_t)s, lo + (int64_t)a.local_len[b]);
  int* own = a.own_sel + (size_t)b * a.k;
  if (s <= a.k) {   // every token is selected (R3): the owned list is the whole local range
    if (blockIdx.y != 0) { pdl_launch_dependents(); return; }
    const int n = (int)max((int64_t)0, hi - lo);
    for (int i = tid; i < n; i += kSelThreads) own[i] = i;
    if (tid == 0) a.own_count[b] = n;
    pdl_launch_dependents();
    return;
  }
  const int x = min(a.sink, s), z0 = max(x, s - a.recent);
  const int kr = a.k - x - (s - z0);   // >= 0 (sink + recent <= k); 0: the forced tokens only
  const int kc = a.kc, P = a.world, me = a.rank;
  if (P == 1) {
    // one rank: the union is this rank's list, at most kr entries -- all selected; the valid
    // entries are the list's prefix, so every CTA of the request copies its share directly
    const int64_t sk1_ = min(hi, (int64_t)x), rc0_ = max(lo, (int64_t)z0);
    const int nsk_ = (int)max((int64_t)0, sk1_ - lo), nrc_ = (int)max((int64_t)0, hi - rc0_);
    const int n = kr > 0 ? a.cand_count[b] : 0;
    const int* midx_ = a.own_idx + (size_t)b * kc;
    const int per = (n + gridDim.y - 1) / gridDim.y;
    const int j1 = min(n, ((int)blockIdx.y + 1) * per);
    for (int j = (int)blockIdx.y * per + tid; j < j1; j += kSelThreads) own[nsk_ + j] = (int)(midx_[j] - lo);
    if (blockIdx.y == 0) {
      for (int i = tid; i < nsk_; i += kSelThreads) own[i] = i;                       // lo == 0 holds the sinks
      for (int i = tid; i < nrc_; i += kSelThreads) own[nsk_ + n + i] = (int)(rc0_ + i - lo);
      if (tid == 0) a.own_count[b] = nsk_ + n + nrc_;
    }
    pdl_launch_dependents();
    return;
  }
  const size_t bs = (size_t)a.batch * kc;               // rank stride of the gathered array
  const float* all = a.all_score + (size_t)b * kc;      // entry (p, j) at all[p * bs + j]
  const float* mine = all + (size_t)me * bs;
  const int* midx = a.own_idx + (size_t)b * kc;

  // ---- exact kr-th largest key of the union (radix select), tie quota
  uint32_t prefix = 0, pmask = 0;
  int need = kr;
  // the union's valid entries: <= kr -> every candidate is selected (one rank, short shards;
  // a single rank's list holds at most kr entries by construction)
  if (P > 1) {
    if (tid == 0) s_cnt[0] = 0;
    __syncthreads();
    int c = 0;
    if ((kc & 3) == 0 && (bs & 3) == 0) {   // 16-byte loads, all issued before the sums
      const int n4 = kc >> 2;
      for (int p = 0; p < P; ++p) {
        const float4* a4 = reinterpret_cast<const float4*>(all + (size_t)p * bs);
        for (int j0 = 0; j0 < n4; j0 += 4 * kSelThreads) {
          float4 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = j0 + u * kSelThreads + tid;
            v[u] = j < n4 ? __ldcg(a4 + j) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            c += (v[u].x != -INFINITY) + (v[u].y != -INFINITY) + (v[u].z != -INFINITY) + (v[u].w != -INFINITY);
        }
      }
    } else {
      for (int p = 0; p < P; ++p)
        for (int j = tid; j < kc; j += kSelThreads) c += all[(size_t)p * bs + j] != -INFINITY;
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) atomicAdd(&s_cnt[0], c);
    __syncthreads();
  }
  const bool take_all = P == 1 || s_cnt[0] <= kr;
  const int shifts[3] = {21, 10, 0}, widths[3] = {11, 11, 10};
  for (int pass = 0; pass < ((kr > 0 && !take_all) ? 3 : 0); ++pass) {
    const int nb = 1 << widths[pass], sh = shifts[pass];
    for (int i = tid; i < kSelBins; i += kSelThreads) hist[i] = 0u;
    __syncthreads();
    for (int p = 0; p < P; ++p)
      for (int j0 = 0; j0 < kc; j0 += kSelThreads) {
        const int j = j0 + tid;
        const float v = j < kc ? all[(size_t)p * bs + j] : -INFINITY;
        const uint32_t key = float_key(v);
        const bool in = v != -INFINITY && (key & pmask) == prefix;
        const uint32_t bin = in ? (key >> sh) & (nb - 1) : 0xffffffffu;
        // warp-aggregated increments: scores of one request share few top digits, and
        // per-entry shared-memory atomics on the same bin serialise
        const uint32_t peers = __match_any_sync(0xffffffffu, bin);
        if (in && (__ffs(peers) - 1) == lane) atomicAdd(&hist[bin], (unsigned)__popc(peers));
      }
    __syncthreads();
    int above = 0;
    const int d = select_digit(hist, kSelBins, need, s_warp, s_res, &above);
    need -= above;
    prefix |= (uint32_t)d << sh;
    pmask |= (uint32_t)(nb - 1) << sh;
    __syncthreads();
  }
  const uint32_t T = prefix;
  // ties: entries == T on ranks before this one take theirs first
  int take_eq = 0;
  if (!take_all && kr > 0) {
    __syncthreads();
    if (tid == 0) { s_cnt[0] = 0; s_cnt[1] = 0; }
    __syncthreads();
    int before = 0, mine_eq = 0;
    for (int p = 0; p <= me; ++p)
      for (int j = tid; j < kc; j += kSelThreads) {
        const float v = all[(size_t)p * bs + j];
        if (v != -INFINITY && float_key(v) == T) { if (p < me) ++before; else ++mine_eq; }
      }
    before = __reduce_add_sync(0xffffffffu, before);
    mine_eq = __reduce_add_sync(0xffffffffu, mine_eq);
    if (lane == 0) { atomicAdd(&s_cnt[0], before); atomicAdd(&s_cnt[1], mine_eq); }
    __syncthreads();
    take_eq = max(0, min(need - s_cnt[0], s_cnt[1]));
  }

  // ---- owned list: sinks | picks (ordered compaction of this rank's candidates) | recents
  const int64_t sk0 = max(lo, (int64_t)0), sk1 = min(hi, (int64_t)x);
  const int64_t rc0 = max(lo, (int64_t)z0), rc1 = hi;
  const int nsk = (int)max((int64_t)0, sk1 - sk0), nrc = (int)max((int64_t)0, rc1 - rc0);
  for (int i = tid; i < nsk; i += kSelThreads) own[i] = (int)(sk0 + i - lo);
  // rounds of kSelThreads * 4 candidates staged in shared memory by coalesced 16-byte
  // loads; thread t then owns the contiguous run [4t, 4t + 4) of the round (ascending index
  // order is kept): one block scan for the tie ranks, one for the output positions
  constexpr int kSelPer = 4, kRound = kSelThreads * kSelPer;
  __shared__ __align__(16) float sv[kRound];                             // the round's scores
  __shared__ __align__(16) int sg[kRound];                               // and global indices
  int base = nsk, ebase = 0;
  for (int r0 = 0; r0 < kc; r0 += kRound) {
    __syncthreads();   // the previous round's readers of sv / sg are done
    if ((kc & 3) == 0 && r0 + 4 * tid + 4 <= kc) {
      const float4 f = __ldcg(reinterpret_cast<const float4*>(mine + r0) + tid);
      const int4 g = __ldcg(reinterpret_cast<const int4*>(midx + r0) + tid);
      reinterpret_cast<float4*>(sv)[tid] = f;
      reinterpret_cast<int4*>(sg)[tid] = g;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = r0 + 4 * tid + e;
        sv[4 * tid + e] = j < kc ? mine[j] : -INFINITY;
        sg[4 * tid + e] = j < kc ? midx[j] : -1;
      }
    }
    __syncthreads();
    uint32_t keys[kSelPer];
    int gis[kSelPer];
    int neq = 0;
#pragma unroll
    for (int e = 0; e < kSelPer; ++e) {
      const float v = sv[kSelPer * tid + e];
      gis[e] = sg[kSelPer * tid + e];
      const bool valid = v != -INFINITY && gis[e] >= 0;
      keys[e] = valid ? float_key(v) : 0u;
      if (!valid) gis[e] = -1;
      neq += (valid && !take_all && kr > 0 && keys[e] == T) ? 1 : 0;
    }
    int etot = 0;
    int erank = ebase + block_excl_scan(neq, s_warp, &etot);
    int nsel = 0;
    uint32_t selm = 0;
#pragma unroll
    for (int e = 0; e < kSelPer; ++e) {
      const bool valid = gis[e] >= 0;
      const bool gt = valid && kr > 0 && (take_all || keys[e] > T);
      const bool eq = valid && !take_all && kr > 0 && keys[e] == T;
      const bool sel = gt || (eq && erank < take_eq);
      erank += eq ? 1 : 0;
      if (sel) { selm |= 1u << e; ++nsel; }
    }
    int stot = 0;
    int pos = base + block_excl_scan(nsel, s_warp, &stot);
#pragma unroll
    for (int e = 0; e < kSelPer; ++e)
      if (selm >> e & 1u) own[pos++] = (int)(gis[e] - lo);
    base += stot;
    ebase += etot;
  }
  for (int i = tid; i < nrc; i += kSelThreads) own[base + i] = (int)(rc0 + i - lo);
  if (tid == 0) a.own_count[b] = base + nrc;
  pdl_launch_dependents();
}

}  // namespace sals
