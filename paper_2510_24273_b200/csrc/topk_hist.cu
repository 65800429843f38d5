// K4 (and the shard-local half of K8): TopK selection  C = TopK(p', k)
// (Alg. 1 line 5) with the sink / critical / recent policy
// and ties to the lower index (reading R5) -- histogram-assisted
// kernel.  One thread-block CLUSTER of CS CTAs per request; CTA `rank` owns the
// contiguous slice [rank*slice, (rank+1)*slice) of the request's entries.
//
// The score kernel (K3) already built hist0[b], the histogram of the top 11
// bits of the order-preserving keys of the RANKED scores, on all SMs.  So:
//  A. every CTA scans hist0 (no exchange) for the threshold bin digit0 and the
//     count rem0 still needed inside it, while its score loads are in flight;
//     then, in one pass over the loaded scores, each warp stages -- in index
//     order, compacted with ballot/popc -- only the entries that can be
//     selected: "definite" ones (forced, or ranked with top digit > digit0)
//     and "candidates" (ranked, top digit == digit0).  Everything else is
//     dropped here and never touched again.
//  B. per-warp counts -> CTA counts -> pushed to every peer (DSMEM), barrier 1.
//  C. fast path (<= cand_cap candidates cluster-wide, segments padded to 16 B):
//     every CTA compacts its candidates' keys into its own segment of the
//     cluster-wide candidate array (rank order) and bulk-copies that segment
//     (cp.async.bulk shared::cta -> shared::cluster, one issuing thread per
//     peer) into every peer, completing on the peer's mbarrier -- no second
//     cluster barrier.  Each CTA then selects the remaining 21 bits locally:
//     one 8-bit radix pass, then an exact count-select over the (typically a
//     few dozen) survivors, or two more radix passes when many keys are
//     nearly equal; totals come from the histograms, and the counts that
//     place this CTA from the lower ranks' segments -- no further exchange.
//     overflow path: three cluster-wide radix passes over the staged
//     candidates (histograms pushed to every peer), then one count exchange.
//  D. ordered compaction over the staged list only (a few % of the slice).
// Output: ascending index order, -1 padded to pad_to; identical to the generic
// kernel's (topk.cu) and to the oracle's selection (reading R5).
#include "common.cuh"
#include "kernels.h"
#include <climits>

namespace sals {

namespace {

constexpr int kMaxCluster = 16;
constexpr uint32_t kDefFlag = 0x80000000u;   // staged index flag: definite entry

#ifdef SALS_TC_TRACE
__device__ unsigned long long g_tkh_trace[32];
#define TKH_STAMP(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_tkh_trace[(i)] = clock64(); } while (0)
#else
#define TKH_STAMP(i) do {} while (0)
#endif

// Exclusive prefix over the NW warps of wc[w][q] (q in [q0, q0+NQ)) in place,
// totals into tot[q].  Run by warp 0; caller synchronises before and after.
template <int NW, int NQ>
__device__ __forceinline__ void warp_prefix(int (*wc)[4], int q0, int* tot) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
#pragma unroll
    for (int q = q0; q < q0 + NQ; ++q) {
      const int v = lane < NW ? wc[lane][q] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += n;
      }
      if (lane < NW) wc[lane][q] = incl - v;
      if (lane == 31) tot[q] = incl;
    }
  }
}

// Warp 0: lane l owns bins 255-8l-j (descending); find the bin holding the
// rem-th largest entry and the count still needed inside it.
__device__ __forceinline__ void digit_search256(const uint32_t* hist, int rem, int* s_digit, int* s_need,
                                                int* s_cnt) {
  const int lane = threadIdx.x & 31;
  // the lane's 8 bins are 32 contiguous bytes: two 16-byte loads (a per-bin
  // strided read would put 8 lanes on each bank)
  const uint4* h4 = reinterpret_cast<const uint4*>(hist) + (248 - 8 * lane) / 4;
  const uint4 lo = h4[0], hi = h4[1];
  const int c8[8] = {(int)hi.w, (int)hi.z, (int)hi.y, (int)hi.x, (int)lo.w, (int)lo.z, (int)lo.y, (int)lo.x};
  int tot = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) tot += c8[j];
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
      if (excl < rem && rem <= excl + c8[j]) { *s_digit = 255 - 8 * lane - j; *s_need = rem - excl; *s_cnt = c8[j]; }
      excl += c8[j];
    }
  }
}

__device__ __forceinline__ bool tk_mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  return ok != 0;
}

}  // namespace

template <int NT>
__global__ void __launch_bounds__(NT)
topk_hist_kernel(TopkArgs a) {
  constexpr int NW = NT / 32;
  constexpr int kBatch = 8;                        // 32-entry rounds per warp with loads in flight
  constexpr int kSurvMax = 128;                    // exact brute-force select below this many survivors
  extern __shared__ __align__(16) uint8_t tk_smem[];
  __shared__ uint32_t inc_hist[2][kMaxCluster][256];   // overflow path: [pass parity][source rank][digit]
  __shared__ __align__(16) uint32_t hist[2][256];
  __shared__ uint32_t surv[kSurvMax];
  __shared__ __align__(8) uint64_t cand_bar;           // peers' candidate segments landed (bulk copies)
  __shared__ int inc_cnt[kMaxCluster][4];              // [source rank]: def0, cand, gt, eq
  __shared__ int wcnt[NW][4];                          // per warp: def0, cand, gt, eq -> exclusive prefixes
  __shared__ int s_ctot[4];
  __shared__ int warp_tot[32];
  __shared__ int s_red[2];
  __shared__ int s_digit, s_need, s_cnt, s_nsurv;
  __shared__ uint32_t s_T;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t bar_addr = smem_u32(&cand_bar);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_addr) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_nsurv = 0;
  }
  if (tid < 2) s_red[tid] = 0;
  if (tid < 256) { hist[0][tid] = 0; hist[1][tid] = 0; }
  // every CTA of the cluster must be running (and its barrier initialised)
  // before a peer writes its shared memory: arrive now, wait before the first
  // DSMEM store
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");

  const int CS = (int)cluster_nctarank();
  const int rank = (int)cluster_ctarank();
  const int b = blockIdx.x / CS;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const int slice = a.slice;
  uint32_t* st_idx = reinterpret_cast<uint32_t*>(tk_smem);   // [slice] staged global index | kDefFlag
  uint32_t* st_key = st_idx + slice;                          // [slice] staged key (0 for forced)
  uint32_t* cand = st_key + slice;                            // [cand_cap] cluster-wide candidate keys
  const uint32_t cand_addr = smem_u32(cand);

  TKH_STAMP(0);
  pdl_wait();
  // the reconstruction kernel may launch now: before its own wait it only sets up
  // barriers / TMEM and stages q^R (written two kernels upstream)
  pdl_launch_dependents();
  const int s = a.seq_len[b];
  const int n = a.n_entries ? a.n_entries[b] : s;
  const int e0 = rank * slice;
  const int nloc = max(0, min(slice, n - e0));
  const int x = a.sink, z = a.recent;
  const bool all_mode0 = (a.mode == 0) && (s <= a.k);
  const int wc = ((nloc + NW - 1) / NW + 31) / 32 * 32;    // warp w owns [w0, w1) of the slice
  const int w0 = min(nloc, warp * wc), w1 = min(nloc, w0 + wc);
  const float* sc_b = a.scores + (size_t)b * a.score_stride + e0;
  const int gbase = (int)(a.idx_base + e0);                // global index of slice entry 0
  // slice-local bounds: valid (global index < s) and ranked ([x, s - z))
  const int i_valid = min(w1, s - gbase);
  const int i_lo = all_mode0 ? INT_MAX : x - gbase;
  const int i_hi = s - z - gbase;
  const bool forced_mode = (a.mode == 0);

  // ---- A. loads of the first batch in flight, threshold bin from hist0 ----
  float sc[kBatch];
#pragma unroll
  for (int u = 0; u < kBatch; ++u) {
    const int i = w0 + u * 32 + lane;
    sc[u] = (i < w1) ? __ldg(sc_b + i) : 0.f;
  }
  int digit0, rem0;
  {
    constexpr int BPT = kH0Bins / NT;                       // bins per thread, descending
    const uint32_t* hg = a.hist0 + (size_t)b * kH0Bins;
    int cb[BPT], t = 0;
#pragma unroll
    for (int j = 0; j < BPT; ++j) { cb[j] = (int)hg[kH0Bins - 1 - BPT * tid - j]; t += cb[j]; }
    int v = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int nb = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += nb;
    }
    if (lane == 31) warp_tot[warp] = v;
    __syncthreads();
    int wexcl = 0, nr = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) { const int wt = warp_tot[w]; wexcl += (w < warp) ? wt : 0; nr += wt; }
    const int incl = v + wexcl;
    int nd = all_mode0 ? 0 : a.k - x - z;                   // ranked entries still to choose
    // no equality test on the clamped value (see topk_cta.cu: ptxas derived
    // `clamp == nr` from a VIMNMX select predicate and got it wrong there)
    const bool take_all = nd >= nr, take_none = nd <= 0;
    nd = take_all ? nr : (take_none ? 0 : nd);
    if (tid == 0) { s_digit = (!take_none && nr > 0 && take_all) ? -1 : kH0Bins; s_need = 0; }   // all ranked / none
    __syncthreads();
    if (nd > 0 && nd < nr) {
      int excl = incl - t;
      if (excl < nd && nd <= incl) {
#pragma unroll
        for (int j = 0; j < BPT; ++j) {
          if (excl < nd && nd <= excl + cb[j]) { s_digit = kH0Bins - 1 - BPT * tid - j; s_need = nd - excl; }
          excl += cb[j];
        }
      }
    }
    __syncthreads();
    digit0 = s_digit;
    rem0 = s_need;
  }
  TKH_STAMP(1);

  // ---- A'. classify + stage (index order, ballot compaction) ----
  int n_def = 0, n_st = 0;   // warp-uniform running counts
  for (int r0 = 0; w0 + r0 * 32 < w1; r0 += kBatch) {
    if (r0 > 0) {
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int i = w0 + (r0 + u) * 32 + lane;
        sc[u] = (i < w1) ? __ldg(sc_b + i) : 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      if (w0 + (r0 + u) * 32 >= w1) break;                  // warp-uniform
      const int i = w0 + (r0 + u) * 32 + lane;
      const bool valid = i < i_valid;
      const bool ranked = valid && i >= i_lo && i < i_hi;
      const uint32_t key = ranked ? float_key(sc[u]) : 0u;
      const int top = (int)(key >> kH0Shift);
      const bool def = ranked ? (top > digit0) : (valid && forced_mode);
      const bool keep = def || (ranked && top == digit0);
      const uint32_t km = __ballot_sync(0xffffffffu, keep);
      const uint32_t dm = __ballot_sync(0xffffffffu, def);
      if (keep) {
        const int p = w0 + n_st + __popc(km & lt_mask);
        st_idx[p] = (uint32_t)(gbase + i) | (def ? kDefFlag : 0u);
        st_key[p] = key;
      }
      n_st += __popc(km);
      n_def += __popc(dm);
    }
  }
  if (lane == 0) { wcnt[warp][0] = n_def; wcnt[warp][1] = n_st - n_def; }
  __syncthreads();
  warp_prefix<NW, 2>(wcnt, 0, s_ctot);
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");   // every peer is running
  __syncthreads();
  // ---- B. CTA counts to every peer, barrier 1 ----
  if (tid < CS) {
    st_dsmem_u32(mapa_shared(smem_u32(&inc_cnt[rank][0]), tid), (uint32_t)s_ctot[0]);
    st_dsmem_u32(mapa_shared(smem_u32(&inc_cnt[rank][1]), tid), (uint32_t)s_ctot[1]);
  }
  TKH_STAMP(2);
  cluster_sync_all();
  TKH_STAMP(3);
  // candidate segments are padded to 16 bytes (bulk-copy granularity)
  int off_pad = 0, total_pad = 0, d0_before = 0, d0_total = 0;
  for (int c = 0; c < CS; ++c) {
    const int dc = inc_cnt[c][0], cp = (inc_cnt[c][1] + 3) & ~3;
    if (c < rank) { off_pad += cp; d0_before += dc; }
    total_pad += cp;
    d0_total += dc;
  }
  const int own_cnt = inc_cnt[rank][1];
  const int own_pad = (own_cnt + 3) & ~3;
  const int st_lo = w0, st_hi = w0 + n_st;                  // this warp's staged list
  uint32_t T;
  int need_eq = 0, gt_before = 0, eq_before = 0, gt_total = 0, eq_total = 0;
  const bool fast = total_pad <= a.cand_cap;                // uniform across the cluster
  if (fast) {
    // ---- C. own candidates -> own segment, bulk-copied into every peer ----
    {
      int run = off_pad + wcnt[warp][1];
      for (int base = st_lo; base < st_hi; base += 32) {
        const int p = base + lane;
        const bool cnd = p < st_hi && !(st_idx[p] & kDefFlag);
        const uint32_t m = __ballot_sync(0xffffffffu, cnd);
        if (cnd) cand[run + __popc(m & lt_mask)] = st_key[p];
        run += __popc(m);
      }
      // pad keys never match the threshold bin's top digit
      if (tid < own_pad - own_cnt) cand[off_pad + own_cnt + tid] = (digit0 == 0) ? 0xffffffffu : 0u;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_addr),
                   "r"((uint32_t)(total_pad - own_pad) * 4u) : "memory");
    if (tid < CS && tid != rank && own_pad > 0) {     // one issuing thread per peer
      const uint32_t src = cand_addr + 4u * (uint32_t)off_pad;
      asm volatile(
          "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          ::"r"(mapa_shared(src, tid)), "r"(src), "r"((uint32_t)own_pad * 4u), "r"(mapa_shared(bar_addr, tid))
          : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    while (!tk_mbar_try_wait(bar_addr, 0)) {}
    TKH_STAMP(4);
    // ---- local selection of the remaining 21 bits ----
    if (rem0 > 0) {
      const uint32_t d0 = (uint32_t)digit0;
      // pass 1: bits 20..13
      for (int i = tid; i < total_pad; i += NT) {
        const uint32_t key = cand[i];
        if ((key >> kH0Shift) == d0) atomicAdd(&hist[0][(key >> 13) & 255u], 1u);
      }
      __syncthreads();
      if (warp == 0) digit_search256(hist[0], rem0, &s_digit, &s_need, &s_cnt);
      __syncthreads();
      const uint32_t p19 = (d0 << 8) | (uint32_t)s_digit;    // top 19 bits of T
      const int rem1 = s_need, m = s_cnt;                    // m keys share p19
      if (m <= kSurvMax) {
        // survivors: exact select by counting (m is small)
        for (int i = tid; i < total_pad; i += NT) {
          const uint32_t key = cand[i];
          if ((key >> 13) == p19) surv[atomicAdd(&s_nsurv, 1)] = key;
        }
        __syncthreads();
        if (tid < m) {
          const uint32_t v = surv[tid];
          int g = 0, e = 0;
          for (int j = 0; j < m; ++j) { const uint32_t u = surv[j]; g += u > v; e += u == v; }
          if (g < rem1 && rem1 <= g + e) { s_T = v; s_need = rem1 - g; s_cnt = e; }   // same values from every tie
        }
        __syncthreads();
        T = s_T;
        need_eq = s_need;
        eq_total = s_cnt;
      } else {
        // many near-equal keys: two more radix passes (bits 12..5, 4..0)
        uint32_t prefix = p19 << 13;
        int rem = rem1;
#pragma unroll 1
        for (int ps = 1; ps < 3; ++ps) {
          const int sh = ps == 1 ? 5 : 0;
          const uint32_t dmask = ps == 1 ? 255u : 31u;
          uint32_t* h = hist[ps & 1];
          uint32_t* h_next = hist[(ps + 1) & 1];
          for (int i = tid; i < total_pad; i += NT) {
            const uint32_t key = cand[i];
            if ((key >> (sh + (ps == 1 ? 8 : 5))) == (prefix >> (sh + (ps == 1 ? 8 : 5))))
              atomicAdd(&h[(key >> sh) & dmask], 1u);
          }
          if (tid < 256) h_next[tid] = 0;                    // read by the previous search only
          __syncthreads();
          if (warp == 0) digit_search256(h, rem, &s_digit, &s_need, &s_cnt);
          __syncthreads();
          prefix |= (uint32_t)s_digit << sh;
          rem = s_need;
        }
        T = prefix;
        need_eq = rem;
        eq_total = s_cnt;
      }
      gt_total = rem0 - need_eq;
    } else {
      T = (digit0 < 0) ? 0u : 0xffffffffu;                   // all ranked definite / none
    }
    TKH_STAMP(5);
  } else {
    // ---- C'. overflow: cluster-wide radix passes over the staged candidates ----
    uint32_t prefix = (uint32_t)digit0 << kH0Shift;
    int rem = rem0;
    if (rem0 > 0) {
#pragma unroll 1
      for (int ps = 0; ps < 3; ++ps) {
        const int sh = ps == 0 ? 13 : (ps == 1 ? 5 : 0);
        const uint32_t dmask = ps == 2 ? 31u : 255u;
        const uint32_t hi_mask = ~((dmask << sh) | ((1u << sh) - 1u));
        uint32_t* h = hist[ps & 1];
        for (int p = st_lo + lane; p < st_hi; p += 32) {
          if (st_idx[p] & kDefFlag) continue;
          const uint32_t key = st_key[p];
          if ((key & hi_mask) == prefix) atomicAdd(&h[(key >> sh) & dmask], 1u);
        }
        __syncthreads();
        if (tid < 256) {
          const uint32_t addr = smem_u32(&inc_hist[ps & 1][rank][tid]);
          const uint32_t hv = h[tid];
          for (int c = 0; c < CS; ++c) st_dsmem_u32(mapa_shared(addr, c), hv);
          hist[(ps + 1) & 1][tid] = 0;
        }
        cluster_sync_all();
        if (tid < 256) {
          uint32_t t = 0;
          for (int c = 0; c < CS; ++c) t += inc_hist[ps & 1][c][tid];
          h[tid] = t;
        }
        __syncthreads();
        if (warp == 0) digit_search256(h, rem, &s_digit, &s_need, &s_cnt);
        __syncthreads();
        prefix |= (uint32_t)s_digit << sh;
        rem = s_need;
      }
      T = prefix;
      need_eq = rem;
    } else {
      T = (digit0 < 0) ? 0u : 0xffffffffu;
    }
  }
  // ---- per-warp gt / eq counts over the staged candidates; (fast path) the
  //      candidates of lower ranks, which precede this CTA's ----
  {
    int gcnt = 0, ecnt = 0;
    for (int base = st_lo; base < st_hi; base += 32) {
      const int p = base + lane;
      bool gt = false, eq = false;
      if (p < st_hi && !(st_idx[p] & kDefFlag)) { const uint32_t k = st_key[p]; gt = k > T; eq = k == T; }
      gcnt += __popc(__ballot_sync(0xffffffffu, gt));
      ecnt += __popc(__ballot_sync(0xffffffffu, eq));
    }
    if (lane == 0) { wcnt[warp][2] = gcnt; wcnt[warp][3] = ecnt; }
    if (fast && off_pad > 0 && rem0 > 0) {
      int gb = 0, eb = 0;
      const uint32_t d0 = (uint32_t)digit0;
      for (int i = tid; i < off_pad; i += NT) {
        const uint32_t key = cand[i];
        const bool in_bin = (key >> kH0Shift) == d0;
        gb += in_bin && key > T;
        eb += key == T;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        gb += __shfl_xor_sync(0xffffffffu, gb, off);
        eb += __shfl_xor_sync(0xffffffffu, eb, off);
      }
      if (lane == 0 && (gb | eb)) { atomicAdd(&s_red[0], gb); atomicAdd(&s_red[1], eb); }
    }
  }
  __syncthreads();
  warp_prefix<NW, 2>(wcnt, 2, s_ctot);
  __syncthreads();
  if (fast) {
    gt_before = s_red[0];
    eq_before = s_red[1];
  } else {
    // exchange the CTA's gt / eq totals
    if (tid < CS) {
      st_dsmem_u32(mapa_shared(smem_u32(&inc_cnt[rank][2]), tid), (uint32_t)s_ctot[2]);
      st_dsmem_u32(mapa_shared(smem_u32(&inc_cnt[rank][3]), tid), (uint32_t)s_ctot[3]);
    }
    cluster_sync_all();
    for (int c = 0; c < CS; ++c) {
      const int gc = inc_cnt[c][2], ec = inc_cnt[c][3];
      if (c < rank) { gt_before += gc; eq_before += ec; }
      gt_total += gc; eq_total += ec;
    }
  }
  TKH_STAMP(6);

  // ---- D. ordered compaction over the staged list ----
  const int eq_local = s_ctot[3];
  const int take_local = max(0, min(need_eq - eq_before, eq_local));
  const int out_base = d0_before + gt_before + min(need_eq, eq_before);
  const int count = d0_total + gt_total + min(need_eq, eq_total);
  int* out = a.sel_out + (size_t)b * a.sel_stride;
  int* out2 = a.sel_out2 ? a.sel_out2 + (size_t)b * a.sel_stride : nullptr;
  float* osc = a.sel_score ? a.sel_score + (size_t)b * a.sel_stride : nullptr;
  {
    int rd = wcnt[warp][0] + wcnt[warp][2];   // definite entries of this CTA before the warp's round
    int re = wcnt[warp][3];                   // ties of this CTA before the warp's round
    for (int base = st_lo; base < st_hi; base += 32) {
      const int p = base + lane;
      bool d = false, e = false;
      uint32_t si = 0, key = 0;
      if (p < st_hi) {
        si = st_idx[p];
        key = st_key[p];
        d = (si & kDefFlag) || key > T;
        e = !(si & kDefFlag) && key == T;
      }
      const uint32_t dm = __ballot_sync(0xffffffffu, d), em = __ballot_sync(0xffffffffu, e);
      const int db = rd + __popc(dm & lt_mask);
      const int eb = re + __popc(em & lt_mask);
      if (d || (e && eb < take_local)) {
        const int pos = out_base + db + min(eb, take_local);
        const int gi = (int)(si & ~kDefFlag);
        out[pos] = gi;
        if (out2) out2[pos] = gi;
        if (osc) osc[pos] = key_float(key);
      }
      rd += __popc(dm);
      re += __popc(em);
    }
  }
  if (rank == CS - 1) {
    for (int i = count + tid; i < a.pad_to; i += NT) {
      out[i] = -1;
      if (out2) out2[i] = -1;
      if (osc) osc[i] = -INFINITY;
    }
    if (tid == 0 && a.sel_count) a.sel_count[b] = count;
  }
  // the bulk copies out of this CTA's shared memory must have read it before exit;
  // no DSMEM access follows the last cluster barrier / mbarrier wait otherwise
  if (fast && tid < CS && tid != rank && own_pad > 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  TKH_STAMP(7);
  pdl_launch_dependents();
}

template __global__ void topk_hist_kernel<512>(TopkArgs);
template __global__ void topk_hist_kernel<1024>(TopkArgs);

}  // namespace sals

extern "C" int sals_debug_topk_hist_trace(unsigned long long* out) {
#ifdef SALS_TC_TRACE
  return (int)cudaMemcpyFromSymbol(out, sals::g_tkh_trace, sizeof(sals::g_tkh_trace));
#else
  (void)out;
  return -1;
#endif
}
