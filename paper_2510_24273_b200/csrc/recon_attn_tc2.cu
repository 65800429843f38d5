// Path T v2: persistent, warp-specialised fused reconstruction + RoPE + sparse
// attention (Alg. 1 lines 6-9; Eq. 6) for head_dim 128.
//
// One CTA per (request b, 256-column block = 2 KV heads, chunk of up to
// `tpc` tiles of 128 selected tokens).  The CTA streams its tiles:
//   warp 0      : U tiles (B operand) by TMA, 3-stage mbarrier ring
//   warps 4-7   : gathered latent rows (A operand) by cp.async into SWIZZLE_128B
//   warp 1      : TMEM allocation + the single tcgen05.mma issuer; the 128 x 256
//                 fp32 accumulator is DOUBLE-BUFFERED in TMEM (2 x 256 columns),
//                 so the MMA of tile i+1 runs while tile i is in the epilogue
//   warp 2      : the tile's V rows (512 contiguous bytes each) by cp.async.bulk
//   warps 8-15  : epilogue.  Warp w reads TMEM lanes 32 (w % 4).. (its 32
//                 tokens); half h = (w-8)/4 rotates pairs [32h, 32h+32) of both
//                 KV heads at each token's original position and forms partial
//                 logits for the G query heads of each; the halves exchange
//                 partial logits through shared memory, then half h owns KV
//                 head h: tile max / sum, online-softmax rescale, P V over the
//                 staged V rows.  Logits and K_C never leave the SM.
// After its last tile the CTA writes y directly (single chunk) or one
// (m, l, o) partial per (query head, chunk) for merge_kernel.
//
// MHA batches of >= 4 requests (CG = 2, tc2_pair_axis): the CTAs of requests 2j and
// 2j + 1 (same column block and chunk) form a cluster and compute M = 256 rows with
// tcgen05.mma.cta_group::2, issued by the even CTA into both CTAs' TMEM: each CTA
// stages its own 128 latent rows and HALF of the 256 U columns per stage (a 4-deep
// ring of 32 KB instead of 3 x 48 KB, half the L2 reads of U); a relay thread per CTA
// turns "my stage landed" into a (relaxed) remote arrive on the even CTA's pfull
// barrier, MMA completion is multicast to both CTAs' empty / tfull barriers, and both
// epilogues release the accumulator with remote arrives on the even CTA's tempty.
#include <cuda.h>
#include <type_traits>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "recon_attn_tc.h"
#include "once.h"

namespace sals {
namespace tc2 {

constexpr int kRows = 128, kBK = 64, kBN = 256, kStages = 3, kDH = 128;
constexpr int kStages2 = 4;   // cta_group::2 (MHA): 16 KB A + 16 KB U half per stage
constexpr int kThreads = 512;
constexpr int kABytes = kRows * kBK * 2;   // 16 KB
constexpr int kBBytes = kBN * kBK * 2;     // 32 KB
constexpr int kVBytes = kRows * kBN * 2;   // 64 KB
constexpr int kPS = kRows + 4;             // sP row stride (floats): the two KV-head halves of a warp hit different banks

__host__ __device__ constexpr int smem_bytes(int G, int CG = 1);
static_assert(1024 + 3 * (128 * 64 * 2 + 256 * 64 * 2) + 128 * 256 * 2 + 8 * 64 * 8 + 16 * 128 * 4 + 8 * (128 + 4) * 4 + 1024 <=
                  232448, "G = 4 shared memory over the 227 KB limit");
__host__ __device__ constexpr int smem_bytes(int G, int CG) {
  return 1024 + (CG == 2 ? kStages2 * (kABytes + kBBytes / 2) : kStages * (kABytes + kBBytes)) + kVBytes + 2 * G * 64 * 8 /*sQ*/ + 2 * 2 * G * kRows * 4 /*sL*/ +
         (2 * G * kPS * 4 > 4096 ? 2 * G * kPS * 4 : 4096) /*sP*/ + 1024 /*misc: sRed, sAl, sIdxV, barriers, TMEM slot (< 1 KB)*/;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void cp_async_16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* map, int col, int r0, int r1, int r2,
                                            int r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void bar_epi() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ void bar_half(int h) { asm volatile("bar.sync %0, 128;" ::"r"(2 + h) : "memory"); }

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kBN >> 3) << 17) |
                            ((uint32_t)(kRows >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accum)
      : "memory");
}
// ---- cta_group::2 (a CTA pair computes M = 256 rows: each CTA its 128 token rows and
// half of the 256 U columns; the even CTA issues the MMAs into both CTAs' TMEM)
constexpr uint32_t kIdesc2 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kBN >> 3) << 17) |
                             ((uint32_t)(256 >> 4) << 24);
__device__ __forceinline__ void mma_bf16_cg2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc2), "r"(accum)
      : "memory");
}
// arrive on the barrier at this offset in both CTAs of the pair
__device__ __forceinline__ void mma_commit_cg2(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"((uint16_t)3)
               : "memory");
}
// shared::cluster address of this CTA's `p` in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_rank(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
#ifndef SALS_RELAY_RELEASE
#define SALS_RELAY_RELEASE 0
#endif
// relay / accumulator-release arrive: the stage's bytes were written by the async proxy
// (TMA / cp.async) and are complete (the local full barrier), the TMEM reads of an
// epilogue warp are complete (tcgen05.wait::ld); relaxed avoids a cluster-scope release
// fence per arrive, measured ~1.3k cycles each (SALS_RELAY_RELEASE=1: the release form)
__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint32_t cluster_addr) {
#if SALS_RELAY_RELEASE
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
#else
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
#endif
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld8_nowait(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
template <int N>
__device__ __forceinline__ void tmem_ldn_nowait(uint32_t taddr, float* v) {
  if constexpr (N == 16) tmem_ld16_nowait(taddr, v); else tmem_ld8_nowait(taddr, v);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// P V on tcgen05 (bf16 values): A = the staged V tile as an MN-major SWIZZLE_128B
// operand (M = 128 dims of one KV head, K = 16 tokens per instruction: 64-dim blocks
// LBO = 16 KB apart, 8-token row groups SBO = 1 KB apart), B = P^T as a K-major
// SWIZZLE_128B operand (N = 8 rows = query heads, K = tokens), D = O_tile^T in TMEM
// (lane = dim, column = query head), fp32.
__device__ __forceinline__ uint64_t sw128_mn_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)(16384 >> 4) << 16;   // LBO: next 64-element block along M
  d |= (uint64_t)(1024 >> 4) << 32;    // SBO: next 8-row group along K
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
constexpr uint32_t kIdescPV = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) /*A MN-major*/ | ((uint32_t)(8 >> 3) << 17) |
                              ((uint32_t)(128 >> 4) << 24);
__device__ __forceinline__ void mma_bf16_pv(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdescPV), "r"(accum)
      : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}

struct KArgs {
  TcArgs a;
};

// Split merge fused into the kernel: every chunk CTA of (request b, column block
// nb) has written its (m, l, o) partials and fenced them; the CTA that arrives
// last merges the gridDim.x partials of its NQH query heads in split order
// (log-sum-exp, two passes: max, then weighted sums) and writes y.  All threads
// of the CTA call this.
template <int NQH>
__device__ __forceinline__ void merge_if_last(const TcArgs& a, int b, int nb, int tid, float* scratch) {
  __shared__ int s_last;
  __syncthreads();
  if (tid == 0) {
    const unsigned old = atomicAdd(&a.counters[(size_t)b * gridDim.y + nb], 1u);   // after the partials' fences
    s_last = old == (unsigned)a.ntiles - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (tid == 0) a.counters[(size_t)b * gridDim.y + nb] = 0;   // every chunk CTA has arrived: re-arm
  const int ns = a.ntiles;   // chunks per request
  // the NQH heads' partials [NQH][ns][d+2] are one contiguous block: stage it in
  // shared memory with a single round of independent 8-byte loads, then merge
  // (log-sum-exp, split order) from shared memory
  const int blk = NQH * ns * (kDH + 2);
  const float2* src = reinterpret_cast<const float2*>(a.partials + ((size_t)b * a.n_q + nb * NQH) * ns * (kDH + 2));
  float2* dst = reinterpret_cast<float2*>(scratch);
  for (int i = tid; i < blk / 2; i += kThreads) dst[i] = __ldcg(src + i);
  float* sw = scratch + blk;          // [NQH][ns] normalised weights
  __syncthreads();
  if (tid < NQH) {
    const float* ph = scratch + tid * ns * (kDH + 2);
    float M = -INFINITY;
    for (int sp = 0; sp < ns; ++sp) M = fmaxf(M, ph[sp * (kDH + 2)]);
    float L = 0.f;
    for (int sp = 0; sp < ns; ++sp) {
      const float ms = ph[sp * (kDH + 2)];
      const float w = ms == -INFINITY ? 0.f : exp2f(ms - M);
      sw[tid * ns + sp] = w;
      L = fmaf(ph[sp * (kDH + 2) + 1], w, L);
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    for (int sp = 0; sp < ns; ++sp) sw[tid * ns + sp] *= inv;
  }
  __syncthreads();
  for (int o = tid; o < NQH * kDH; o += kThreads) {
    const int qh = o / kDH, n = o - qh * kDH;
    const float* ph = scratch + qh * ns * (kDH + 2) + 2 + n;
    const float* w = sw + qh * ns;
    float acc = 0.f;
    for (int sp = 0; sp < ns; ++sp) acc = fmaf(w[sp], ph[sp * (kDH + 2)], acc);
    __nv_bfloat16* y = reinterpret_cast<__nv_bfloat16*>(a.direct_out) + ((size_t)b * a.n_q + nb * NQH + qh) * kDH;
    y[n] = __float2bfloat16_rn(acc);
  }
}

#ifdef SALS_TC_TRACE
__device__ unsigned long long g_trace[128];
#define TSTAMP(slot)                                                                          \
  do {                                                                                        \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) g_trace[(slot)] = clock64();   \
  } while (0)
#else
#define TSTAMP(slot) do {} while (0)
#endif
#ifdef SALS_TC_CTATIME
// per-CTA globaltimer stamps (ns): [cta][0 start, 1 after the PDL wait, 2 last MMA issued, 3 end]
__device__ unsigned long long g_ctatime[1024][4];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define CTIME(slot)                                                                                         \
  do {                                                                                                      \
    const unsigned cid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);                    \
    if (cid < 1024) g_ctatime[cid][(slot)] = gtimer();                                                      \
  } while (0)
#else
#define CTIME(slot) do {} while (0)
#endif

// VBH: 16 = dtype (bf16) value rows; 4 / 2 = quantised value rows (DESIGN R15):
// per KV head 128*VB/8 code bytes then 4 (bf16 scale, bf16 zero) pairs;
// 40 / 20 = the same with the 8-bit recent window (a compile-time variant so the
// kernels without the window carry none of its code).
template <int G, int STYLE, int VBH, int CG>
__global__ void __launch_bounds__(kThreads, 1)
recon_attn_tc2_kernel(const __grid_constant__ CUtensorMap tmap_u, const __grid_constant__ CUtensorMap tmap_lat,
                      const __grid_constant__ CUtensorMap tmap_v, const __grid_constant__ CUtensorMap tmap_vh,
                      const __grid_constant__ KArgs ka) {
  constexpr int NQH = 2 * G;             // query heads of this CTA (2 KV heads)
  constexpr int VB = VBH >= 20 ? VBH / 10 : VBH;
  constexpr bool HPW = VBH >= 20;        // recent-window variant
  // bf16 values with GQA (G >= 2): P V on tcgen05 (P rounded to bf16, fp32 accumulation
  // in TMEM), issued by the MMA warp between the reconstruction chunks of the next tile.
  // MHA (G = 1: 1 FFMA2 per token and dim pair) and quantised values (dequantisation in
  // the loop) keep the CUDA-core P V over TMA-gathered rows.  Measured (bench stage
  // times): c3 / c4 31.9 -> 28.0 us, c2 22.8 -> 23.8 us (the 16-byte V copies compete
  // with the A operand's cp.async), hence G >= 2 only.
  constexpr bool TPV = VB == 16 && G >= 2;
  // CG = 2: MHA with dtype values only (every tcgen05 op of a kernel uses one cta_group,
  // and the GQA P V runs per CTA)
  constexpr bool C2 = CG == 2;
  static_assert(!C2 || (G == 1 && VBH == 16), "cta_group::2 variant: MHA, bf16 values");
  constexpr int ST = C2 ? kStages2 : kStages;             // operand ring depth
  constexpr int kBHalf = C2 ? kBBytes / 2 : kBBytes;       // U bytes per stage in this CTA
  constexpr int kVHead = VB == 16 ? kDH * 2 : kDH * VB / 8 + (kDH / 32) * 4;   // value bytes per head-token
  constexpr int kVRow = 2 * kVHead;                                           // bytes of a V tile row (2 heads)
  constexpr int kVRowH = 2 * 144;   // (quantised) 8-bit recent-window row of the 2 heads (DESIGN R15)
  constexpr int kHGrp = 1280;       // smem of 4 such rows: [4 x 144 B head 0 | pad to 640 | 4 x 144 B head 1 | pad]
                                    // (TMA destinations 128-B aligned)
  const TcArgs& a = ka.a;
  extern __shared__ uint8_t smem_raw[];
  // align with pointer arithmetic on the __shared__ array so the compiler keeps the shared
  // address space (an integer round trip would turn every access into a generic load)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = sA + ST * kABytes;
  uint8_t* sV = sB + ST * kBHalf;
  float2* sQ = reinterpret_cast<float2*>(sV + kVBytes);          // [NQH][64] (q_lo, q_hi) per pair
  float* sL = reinterpret_cast<float*>(sQ + NQH * 64);           // [2 halves][NQH][128] partial logits
  float* sP = sL + 2 * NQH * kRows;                              // [NQH][kPS] probabilities
  float* sRed = sP + (NQH * kPS > 1024 ? NQH * kPS : 1024);       // [2 kinds][2 halves][4][G]
  float* sAl = sRed + 2 * 2 * 4 * G;                             // [NQH] online-softmax rescale of the tile
  int* sIdxV = reinterpret_cast<int*>(sAl + NQH);                // [128] global rows of the V tile
  uint64_t* bars = reinterpret_cast<uint64_t*>(sIdxV + kRows);
  uint64_t* full = bars;                 // [stages]
  uint64_t* empty = bars + ST;           // [stages]
  uint64_t* tfull = bars + 2 * ST;       // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint64_t* vfull = tempty + 2;
  uint64_t* vempty = vfull + 1;
  uint64_t* pready = vempty + 1;          // (TPV) [2] P of the tile written (epilogue -> MMA warp)
  uint64_t* pvfull = pready + 2;          // (TPV) [2] O_tile in TMEM (tcgen05.commit -> epilogue)
  uint64_t* pfull = pvfull + 2;           // (C2, even CTA) [stages] both CTAs' stage landed (2 relays)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pfull + ST);
  int* s_thp = reinterpret_cast<int*>(tmem_slot + 1);   // first tile token read from the 8-bit recent window
  uint8_t* sVh = sV + kRows * kVRow;                      // (quantised) 8-bit rows of the recent window
  static_assert(VB == 16 || kRows * kVRow + 32 * 1280 <= kVBytes, "recent-window staging exceeds the V tile");

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // (C2, pair of requests: the cluster pairs along x, which a cta_group::2 launch needs,
  // so x = 2 chunk + (b & 1), z = b / 2)
  const bool zpair = C2;
  const int chunk = zpair ? (int)(blockIdx.x >> 1) : (int)blockIdx.x, nb = blockIdx.y;
  const int b = zpair ? (int)(2 * blockIdx.z + (blockIdx.x & 1)) : (int)blockIdx.z;
  const int n0 = nb * kBN;
  if (tid == 0) CTIME(0);

  // Prologue before griddepcontrol.wait (overlaps the top-k kernel, which triggers
  // its dependents early): barriers, TMEM allocation and the rotated queries
  // (q^R comes from the query projection, which completed before the top-k's
  // upstream did).  Only the selection (sel / count) is read after the wait.
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) { mbar_init(&full[s], 128 + 1); mbar_init(&empty[s], 1); mbar_init(&pfull[s], 2); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], C2 ? 16 : 8); }
    mbar_init(vfull, TPV ? 256 : 1);   // TPV: the 256 epilogue threads' cp.async; else one expect_tx
    mbar_init(vempty, 1);
    for (int i = 0; i < 2; ++i) { mbar_init(&pready[i], 1); mbar_init(&pvfull[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if constexpr (TPV) {   // P^T operands [2 heads][2 token blocks][8 rows x 128 B]: rows >= G stay zero
    for (int i = tid; i < 4096 / 16; i += kThreads) reinterpret_cast<uint4*>(sP)[i] = make_uint4(0, 0, 0, 0);
  }
  if (warp == 1) {
    if constexpr (C2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if (warp >= 8) {   // rotated, scaled queries: sQ4[qh][p/2] = (q_lo(p), q_lo(p+1), q_hi(p), q_hi(p+1))
    float4* sQ4 = reinterpret_cast<float4*>(sQ);
    for (int i = tid - 256; i < NQH * 32; i += 256) {
      const int qh = i >> 5, p = 2 * (i & 31);
      const int lo0 = STYLE == 0 ? p : 2 * p, hi0 = STYLE == 0 ? p + 64 : 2 * p + 1;
      const int lo1 = STYLE == 0 ? p + 1 : 2 * p + 2, hi1 = STYLE == 0 ? p + 65 : 2 * p + 3;
      const float* qr = a.qrope + ((size_t)b * a.n_q + nb * NQH + qh) * kDH;
      const float sc = a.scale_log2;
      sQ4[i] = make_float4(qr[lo0] * sc, qr[lo1] * sc, qr[hi0] * sc, qr[hi1] * sc);
    }
  }
  if (tid == 0) TSTAMP(80);
  pdl_wait();
  if (tid == 0) TSTAMP(82);
  if (tid == 0) CTIME(1);
  const int cnt = a.count[b];
  const int ntiles_b = (cnt + kRows - 1) / kRows;
  const int t_begin = chunk * a.tiles_per_cta;
  const int t_end = min(ntiles_b, t_begin + a.tiles_per_cta);
  const int ntile = max(0, t_end - t_begin);
  const int* selb = a.sel + (size_t)b * a.k_stride;
  // (C2) both CTAs of the pair run the same number of pair steps: the larger tile count;
  // a CTA past its own tiles contributes zero rows and skips their epilogue
  const uint32_t crank = C2 ? cluster_ctarank() : 0u;
  int ntile_pair = ntile;
  if constexpr (C2) {
    const int pcnt = a.count[b ^ 1];   // the partner request, same chunk
    const int pt0 = chunk * a.tiles_per_cta;
    const int pt1 = min((pcnt + kRows - 1) / kRows, pt0 + a.tiles_per_cta);
    ntile_pair = max(ntile, pt1 - pt0);
  }

  if (ntile_pair == 0) {   // no selected tokens for this chunk: empty partials (m = -inf, l = 0, o = 0)
    tc_fence_before();
    __syncthreads();
    if constexpr (C2) cluster_sync_all();
    if (warp == 1) {
      tc_fence_after();
      if constexpr (C2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(*tmem_slot), "r"(512));
      else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_slot), "r"(512));
    }
    for (int i = tid; i < NQH * (kDH + 2); i += kThreads) {
      const int qh = i / (kDH + 2), j = i - qh * (kDH + 2);
      a.partials[(((size_t)b * a.n_q + nb * NQH + qh) * a.ntiles + chunk) * (kDH + 2) + j] = j == 0 ? -INFINITY : 0.f;
    }
    if (a.counters) __threadfence();
    if (a.counters) merge_if_last<NQH>(a, b, nb, tid, reinterpret_cast<float*>(smem));
    pdl_launch_dependents();
    return;
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (C2) cluster_sync_all();   // the peer's barriers / TMEM exist before any remote use
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nk = a.r / kBK;

  if (warp == 0) {
    // ================= U (B operand) producer: one TMA per K chunk =================
    if (lane == 0) {
      // (C2: this CTA's half, the U columns n0 + 128 crank .. +128, from a 128-row box map)
      int u = 0;
      for (int it = 0; it < ntile_pair; ++it)
        for (int kc = 0; kc < nk; ++kc, ++u) {
          const int s = u % ST;
          if (u >= ST) mbar_wait(&empty[s], ((u / ST) - 1) & 1);
#ifdef SALS_EXP_NO_U   // experiment (trace builds only): U fetched for the first stages only
          if (u >= ST) { mbar_arrive(&full[s]); continue; }
#endif
          mbar_arrive_expect_tx(&full[s], kBHalf);
          tma_load_2d(smem_u32(sB + s * kBHalf), &tmap_u, kc * kBK, n0 + (int)crank * (kBN / 2), &full[s]);
        }
      if constexpr (C2) {   // the even CTA's last commits (multicast) have reached this CTA's slots
        for (int v = max(0, u - ST); v < u; ++v) mbar_wait(&empty[v % ST], (v / ST) & 1);
      }
    }
  } else if (C2 && warp == 1) {
    // ================= MMA issuer (cta_group::2): the even CTA, M = 256 over the pair =================
    if (lane == 0 && crank == 0) {
      int u = 0;
      for (int it = 0; it < ntile_pair; ++it) {
        const int buf = it & 1;
        if (it >= 2) mbar_wait_cluster(&tempty[buf], ((it >> 1) - 1) & 1);   // both CTAs' epilogues
        TSTAMP(0 + it);
        tc_fence_after();
        const uint32_t acc = tmem + buf * kBN;
        for (int kc = 0; kc < nk; ++kc, ++u) {
          const int s = u % ST;
          mbar_wait_cluster(&pfull[s], (u / ST) & 1);
          if (kc == 0) TSTAMP(88 + it);
          tc_fence_after();
          const uint32_t ab = smem_u32(sA + s * kABytes), bb = smem_u32(sB + s * kBHalf);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            mma_bf16_cg2(acc, sw128_desc(ab + k * 32), sw128_desc(bb + k * 32), (kc | k) ? 1u : 0u);
          mma_commit_cg2(&empty[s]);
        }
        mma_commit_cg2(&tfull[buf]);
        TSTAMP(8 + it);
      }
      CTIME(2);
      pdl_launch_dependents();
    }
  } else if (C2 && warp == 3) {
    // ================= (C2) relay: this CTA's stage landed -> the even CTA's pfull =================
    if (lane == 0) {
      int u = 0;
      for (int it = 0; it < ntile_pair; ++it)
        for (int kc = 0; kc < nk; ++kc, ++u) {
          const int s = u % ST;
          mbar_wait(&full[s], (u / ST) & 1);
          fence_proxy_async();   // the cp.async-written A rows -> the tensor core's proxy
          mbar_arrive_remote_relaxed(mapa_rank(&pfull[s], 0));
          if (it == 0 && kc < 8) TSTAMP(96 + kc);
        }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    if (lane == 0) {
      int u = 0;
      int pv = 0;   // (TPV) next tile whose P V is to be issued
      // P V of tile pv: 2 KV heads x 8 k-steps of 16 tokens into columns buf * 256 + kh * 8
      // one tile per call; returns whether it issued (block: wait for the tile's P)
      auto issue_pv = [&](bool block) -> bool {
        if constexpr (TPV) {
          if (pv < ntile) {
            const int pb = pv & 1;
            if (!block && !mbar_test(&pready[pb], (pv >> 1) & 1)) return false;
            mbar_wait(&pready[pb], (pv >> 1) & 1);
            tc_fence_after();
            fence_proxy_async();
#pragma unroll
            for (int kh = 0; kh < 2; ++kh) {
              const uint32_t va = smem_u32(sV + 2 * kh * (kRows * 128));
              const uint32_t pa = smem_u32(sP) + kh * 2048;
#pragma unroll
              for (int kt = 0; kt < kRows / 16; ++kt)
                mma_bf16_pv(tmem + pb * kBN + kh * 8, sw128_mn_desc(va + kt * 2048),
                            sw128_desc(pa + (kt >> 2) * 1024 + (kt & 3) * 32), kt ? 1u : 0u);
            }
            mma_commit(&pvfull[pb]);
            ++pv;
            return true;
          }
        }
        return false;
      };
      for (int it = 0; it < ntile; ++it) {
        const int buf = it & 1;
        if (it >= 2) {
          if constexpr (TPV) { while (pv <= it - 2) issue_pv(true); }   // the epilogue frees buf only after P V
          mbar_wait(&tempty[buf], ((it >> 1) - 1) & 1);
        }
        TSTAMP(0 + it);
        tc_fence_after();
        const uint32_t acc = tmem + buf * kBN;
        for (int kc = 0; kc < nk; ++kc, ++u) {
          const int s = u % ST;
          if constexpr (TPV) {
            while (!mbar_test(&full[s], (u / ST) & 1)) issue_pv(false);
          }
          mbar_wait(&full[s], (u / ST) & 1);
          tc_fence_after();
          fence_proxy_async();
          const uint32_t ab = smem_u32(sA + s * kABytes), bb = smem_u32(sB + s * kBHalf);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            mma_bf16(acc, sw128_desc(ab + k * 32), sw128_desc(bb + k * 32), (kc | k) ? 1u : 0u);
          mma_commit(&empty[s]);
        }
        mma_commit(&tfull[buf]);
        TSTAMP(8 + it);
        while (issue_pv(false)) {}
      }
      if constexpr (TPV) { while (pv < ntile) issue_pv(true); }
      CTIME(2);
      // all MMAs issued: the next kernel may launch and run its pre-wait prologue
      // (the projection stages U, a weight) while this CTA's last epilogue runs
      pdl_launch_dependents();
    }
  } else if (TPV && (warp == 2 || warp == 3)) {
    // (TPV: the epilogue warps stage the V tiles themselves)
  } else if (warp == 2) {
    // ======== V rows producer: 32 TMA tile::gather4 of 4 x 512-B rows per tile; also
    // warms L2 with the next tile's V and latent rows ========
    const char* vb = reinterpret_cast<const char*>(a.v_cache);
    int* idx = sIdxV;
    const int hp_lim = (HPW && a.hp_window > 0) ? max(0, a.seq_len[b] - a.hp_window) : -1;
    for (int it = 0; it < ntile; ++it) {
      const int tile = t_begin + it;
      const int nv = min(kRows, cnt - tile * kRows);
      int gi[4];   // the tile's gather rows, loaded BEFORE waiting for sV (the L2 round trip overlaps the P V)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int t = lane + 32 * j;
        gi[j] = t < nv ? b * (int)a.cap + selb[tile * kRows + t] : -1;
      }
      if (it >= 1) mbar_wait(vempty, (it - 1) & 1);     // previous tile's P V done with sV (and sIdxV)
#pragma unroll
      for (int j = 0; j < 4; ++j) idx[lane + 32 * j] = gi[j];
      __syncwarp();
      // quantised values with a recent window: tokens at positions >= s_b - w (a suffix of
      // the ascending tile) are read from the 8-bit ring (slot pos % w) into sVh
      int thp = nv;
      if constexpr (HPW) {
        if (hp_lim >= 0) {   // positions from the indices just staged (no second global read)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int t = lane + 32 * j;
            if (t < nv && idx[t] - b * (int)a.cap >= hp_lim) thp = min(thp, t);
          }
          thp = __reduce_min_sync(0xffffffffu, thp);
        }
      }
      const bool hp_lane = HPW && thp < nv && 4 * lane + 3 >= thp && 4 * lane < nv;
      const int n_hp = __popc(__ballot_sync(0xffffffffu, hp_lane));
      if (lane == 0) {
        *s_thp = thp;
        mbar_arrive_expect_tx(vfull, (uint32_t)(kRows * kVRow + n_hp * 4 * kVRowH));
      }
      __syncwarp();
      tma_gather4(smem_u32(sV + lane * 4 * kVRow), &tmap_v, VB == 16 ? n0 : nb * kVRow, idx[4 * lane],
                  idx[4 * lane + 1], idx[4 * lane + 2], idx[4 * lane + 3], vfull);
      if (hp_lane) {
        int ri[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int t = 4 * lane + e;
          ri[e] = (t >= thp && t < nv) ? b * a.hp_window + (idx[t] - b * (int)a.cap) % a.hp_window : -1;
        }
        // box rows are <= 256 bytes: one gather per KV head (4 rows x 144 B each)
        tma_gather4(smem_u32(sVh + lane * kHGrp), &tmap_vh, nb * kVRowH, ri[0], ri[1], ri[2], ri[3], vfull);
        tma_gather4(smem_u32(sVh + lane * kHGrp + kHGrp / 2), &tmap_vh, nb * kVRowH + 144, ri[0], ri[1], ri[2],
                    ri[3], vfull);
      }
      if (it + 1 < ntile) {   // next tile's V rows -> L2 via the LSU (keeps the TMA queue for loads)
        const int ntl = tile + 1;
        const int nnv = min(kRows, cnt - ntl * kRows);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int t = lane + 32 * j;
          if (t < nnv) {
            const char* vr = VB == 16 ? vb + (((size_t)b * a.cap + selb[ntl * kRows + t]) * a.D + n0) * 2
                                      : vb + ((size_t)b * a.cap + selb[ntl * kRows + t]) * a.v_row_bytes + nb * kVRow;
#pragma unroll
            for (int c = 0; c < (kVRow + 127) / 128; ++c) prefetch_l2(vr + c * 128);
          }
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ======== A producers: gathered latent rows by 16-byte cp.async into the
    // SWIZZLE_128B K-major tile (8 lanes per 128-B row chunk, 4 rows per instruction) ========
    const char* latent = reinterpret_cast<const char*>(a.latent);
    const int aw = warp - 4, ch = lane & 7;
    int u = 0;
    // gather indices of tile it+1 are loaded while tile it's chunks are issued
    auto load_rows = [&](int tile, int* rows) {
      const int nv = min(kRows, cnt - tile * kRows);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int rl = aw * 32 + i * 4 + (lane >> 3);
        rows[i] = rl < nv ? selb[tile * kRows + rl] : -1;
      }
    };
    int rows[8], rows_nx[8];
    load_rows(t_begin, rows);
    for (int it = 0; it < ntile_pair; ++it) {   // (C2: past this CTA's tiles no row is valid -> zero fill)
      if (it + 1 < ntile_pair) load_rows(t_begin + it + 1, rows_nx);
      for (int kc = 0; kc < nk; ++kc, ++u) {
        const int s = u % ST;
        if (u >= ST) mbar_wait(&empty[s], ((u / ST) - 1) & 1);
        const uint32_t base = smem_u32(sA + s * kABytes);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rl = aw * 32 + i * 4 + (lane >> 3);
          const int row = rows[i];
          const char* src = latent + (((size_t)b * a.cap + (row >= 0 ? row : 0)) * a.r + kc * kBK + ch * 8) * 2;
          cp_async_16(base + rl * 128 + ((ch ^ (rl & 7)) << 4), src, row >= 0 ? 16u : 0u);
        }
        cp_async_arrive_noinc(&full[s]);
        if (aw == 0 && lane == 0 && kc == 0) TSTAMP(64 + it);
      }
      if (aw == 0 && lane == 0) TSTAMP(72 + it);
#pragma unroll
      for (int i = 0; i < 8; ++i) rows[i] = rows_nx[i];
    }
  } else if (warp >= 8) {
    // ================= epilogue =================
    const int ew = warp - 8, rq = warp & 3, hf = ew >> 2;
    const int m = rq * 32 + lane;                  // token row of the tile (TMEM lane)
    const int n = rq * 32 + lane;                  // dim of KV head hf in the final write
    // P V mapping: warp ew owns tokens [16 ew, 16 ew + 16) of every tile; lane owns
    // dims [8 (lane & 15), +8) of KV head kh = lane >> 4 (one 16-B V vector per token)
    const int kh = lane >> 4;
    float m_run[G], l_run[G], lp[G];   // lp: this warp's share of the softmax denominator of head kh*G+g
    float ot[G], lt[G];                 // (TPV) o (dim n of KV head hf) and softmax denominator per query head
#pragma unroll
    for (int g = 0; g < G; ++g) { ot[g] = 0.f; lt[g] = 0.f; }
    float2 ov[G][4];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      m_run[g] = -INFINITY; l_run[g] = 0.f; lp[g] = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) ov[g][e] = make_float2(0.f, 0.f);
    }
    const uint32_t tl = tmem + ((uint32_t)(rq * 32) << 16);
    // the token row of tile it+1 is loaded during tile it (its L2 round trip would
    // otherwise sit in front of the first RoPE angle of every tile)
    int row_nx = m < min(kRows, cnt - t_begin * kRows) ? selb[t_begin * kRows + m] : -1;
    for (int it = 0; it < ntile_pair; ++it) {
      const int tile = t_begin + it, buf = it & 1;
      if (C2 && it >= ntile) {   // the partner's tile: release the accumulator, nothing to compute
        mbar_wait(&tfull[buf], (it >> 1) & 1);
        tc_fence_after();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote_relaxed(mapa_rank(&tempty[buf], 0));   // (TMEM reads waited: wait::ld)
        continue;
      }
      const int nv = min(kRows, cnt - tile * kRows);
      const int row = row_nx;
      if (it + 1 < ntile) row_nx = m < min(kRows, cnt - (tile + 1) * kRows) ? selb[(tile + 1) * kRows + m] : -1;
      const int pos = (int)a.pos_base + (row >= 0 ? row : 0);
      if constexpr (TPV) {
        // ---- stage the tile's V rows (the previous tile's P V has completed): this warp's 32
        // tokens x the 256 bytes of KV head hf, 16-byte cp.async into the SWIZZLE_128B
        // MN-major operand layout [64-dim block][token][128 B] (chunk c of token t at c ^ (t % 8));
        // two tokens (256 contiguous bytes each) per instruction, in flight during the logits
        const int cj = lane & 15;
        const int dim = hf * kDH + 8 * cj;
        const uint32_t vdst = smem_u32(sV) + (dim >> 6) * (kRows * 128);
        const int ch = (dim & 63) >> 3;
        const char* vsrc = reinterpret_cast<const char*>(a.v_cache) + ((size_t)n0 + dim) * 2;
#pragma unroll 4
        for (int q = 0; q < 16; ++q) {
          const int tl = 2 * q + (lane >> 4);
          const int t = rq * 32 + tl;
          const int r = __shfl_sync(0xffffffffu, row, tl);
          cp_async_16(vdst + t * 128 + ((ch ^ (t & 7)) << 4), vsrc + ((size_t)b * a.cap + (r >= 0 ? r : 0)) * a.D * 2,
                      r >= 0 ? 16u : 0u);
        }
        cp_async_arrive_noinc(vfull);
      }
      mbar_wait(&tfull[buf], (it >> 1) & 1);
      if (ew == 0 && lane == 0) TSTAMP(16 + it);
      tc_fence_after();
      float2 part[2][G];         // packed (even pair, odd pair) partial logits per (KV head, query head)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int g = 0; g < G; ++g) part[j][g] = make_float2(0.f, 0.f);
      const uint32_t tacc = tl + buf * kBN;
      const float4* sQ4 = reinterpret_cast<const float4*>(sQ);
      // pairs per TMEM chunk: 8 for G = 4 (register pressure), else 16
      constexpr int PW = G >= 4 ? 8 : 16;
#pragma unroll   // (fully unrolled: the next chunk's angles are scheduled across the TMEM waits)
      for (int pc = 0; pc < 32 / PW; ++pc) {
        const int p0 = 32 * hf + PW * pc;
        float xl[2][PW], xh[2][PW];
        // issue all four TMEM loads of the chunk, one wait
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if (STYLE == 0) {
            tmem_ldn_nowait<PW>(tacc + j * kDH + p0, xl[j]);
            tmem_ldn_nowait<PW>(tacc + j * kDH + 64 + p0, xh[j]);
          } else {
            tmem_ldn_nowait<PW>(tacc + j * kDH + 2 * p0, xl[j]);
            tmem_ldn_nowait<PW>(tacc + j * kDH + 2 * p0 + PW, xh[j]);
          }
        }
        float cs[PW], sn[PW];
#pragma unroll
        for (int i = 0; i < PW; ++i) rope_cs_fast(a.rope.th_hi[p0 + i], a.rope.th_lo[p0 + i], pos, cs[i], sn[i]);
        tmem_wait_ld();
        if (STYLE == 1) {   // de-interleave (2i, 2i+1) pairs
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            float t0[PW], t1[PW];
#pragma unroll
            for (int i = 0; i < PW; ++i) { t0[i] = xl[j][i]; t1[i] = xh[j][i]; }
#pragma unroll
            for (int i = 0; i < PW / 2; ++i) {
              xl[j][i] = t0[2 * i]; xh[j][i] = t0[2 * i + 1];
              xl[j][PW / 2 + i] = t1[2 * i]; xh[j][PW / 2 + i] = t1[2 * i + 1];
            }
          }
        }
#pragma unroll
        for (int i = 0; i < PW; i += 2) {
          const float2 c2 = make_float2(cs[i], cs[i + 1]);
          const float2 s2 = make_float2(sn[i], sn[i + 1]);
          const float2 ns2 = make_float2(-sn[i], -sn[i + 1]);
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const float2 xl2 = make_float2(xl[j][i], xl[j][i + 1]);
            const float2 xh2 = make_float2(xh[j][i], xh[j][i + 1]);
            const float2 rl = __ffma2_rn(xl2, c2, __fmul2_rn(xh2, ns2));   // x_lo c - x_hi s
            const float2 rh = __ffma2_rn(xl2, s2, __fmul2_rn(xh2, c2));    // x_lo s + x_hi c
#pragma unroll
            for (int g = 0; g < G; ++g) {
              const float4 q = sQ4[(j * G + g) * 32 + ((p0 + i) >> 1)];
              part[j][g] = __ffma2_rn(make_float2(q.x, q.y), rl, __ffma2_rn(make_float2(q.z, q.w), rh, part[j][g]));
            }
          }
        }
      }
      if constexpr (!TPV) {   // (TPV: the buffer also receives the tile's P V; released after it)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {                               // this warp is done with the accumulator
          if constexpr (C2) mbar_arrive_remote_relaxed(mapa_rank(&tempty[buf], 0));   // (TMEM reads waited: wait::ld)
          else mbar_arrive(&tempty[buf]);
        }
      }
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int g = 0; g < G; ++g) sL[(hf * NQH + j * G + g) * kRows + m] = part[j][g].x + part[j][g].y;
      bar_epi();
      if (ew == 0 && lane == 0) TSTAMP(24 + it);
      // ---- half hf owns KV head hf: full logits, tile softmax, online rescale
      float lg[G], mnew[G], alpha[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int q = hf * G + g;
        lg[g] = (row >= 0) ? sL[q * kRows + m] + sL[(NQH + q) * kRows + m] : -INFINITY;
        float v = lg[g];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
        if (lane == 0) sRed[(hf * 4 + rq) * G + g] = v;
      }
      bar_half(hf);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float* r = sRed + hf * 4 * G + g;
        const float mt = fmaxf(fmaxf(r[0], r[G]), fmaxf(r[2 * G], r[3 * G]));
        mnew[g] = fmaxf(m_run[g], mt);
        alpha[g] = exp2f(m_run[g] - mnew[g]);        // m_run = -inf -> 0
        const float p = (row >= 0) ? exp2f(lg[g] - mnew[g]) : 0.f;
        if constexpr (TPV) {
          // bf16 P^T operand of KV head hf: [2 token blocks of 64][8 rows = query heads][128 B],
          // SWIZZLE_128B (16-byte chunk (m % 64) / 8 of row g at chunk ^ g); the denominator
          // sums the same rounded p the P V uses
          const __nv_bfloat16 pb = __float2bfloat16_rn(p);
          reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<uint8_t*>(sP) + hf * 2048 + (m >> 6) * 1024 + g * 128 +
                                           ((((m & 63) >> 3) ^ g) << 4))[m & 7] = pb;
          float ps = __bfloat162float(pb);
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
          if (lane == 0) sRed[2 * 4 * G + (hf * 4 + rq) * G + g] = ps;
        } else {
          sP[(hf * G + g) * kPS + m] = p;
        }
        m_run[g] = mnew[g];
        if (rq == 0 && lane == 0) sAl[hf * G + g] = alpha[g];
      }
      // (the softmax denominator is summed by the P V lanes, which read every p anyway)
      bar_epi();                                       // sP / sAl of both halves visible
      mbar_wait(vfull, it & 1);
      if (ew == 0 && lane == 0) TSTAMP(32 + it);
      if constexpr (TPV) {
        // ---- P V on tcgen05: P^T (smem) and the V tile are complete -> the MMA warp issues the
        // tile's 2 x 8 MMAs between its reconstruction chunks; O_tile^T (lane = dim n of KV head
        // hf, column = query head) lands in columns buf * 256 + hf * 8 of the drained buffer
        fence_proxy_async();   // this thread's P writes -> the tensor core's (async) proxy
        bar_epi();
        if (ew == 0 && lane == 0) mbar_arrive(&pready[buf]);
        float tsum[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float* r = sRed + 2 * 4 * G + hf * 4 * G + g;
          tsum[g] = (r[0] + r[G]) + (r[2 * G] + r[3 * G]);
          const float al = sAl[hf * G + g];
          lt[g] = lt[g] * al + tsum[g];
          ot[g] *= al;
        }
        mbar_wait(&pvfull[buf], (it >> 1) & 1);
        tc_fence_after();
        float od[8];
        tmem_ld8_nowait(tl + buf * kBN + hf * 8, od);
        tmem_wait_ld();
#pragma unroll
        for (int g = 0; g < G; ++g) ot[g] += od[g];
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);     // accumulator buffer (and its P V columns) free
      } else
      // ---- P V: 16 tokens of this warp x 8 dims of KV head kh per lane, one 16-B V vector per token
      {
        float al[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          al[g] = sAl[kh * G + g];
          lp[g] *= al[g];
#pragma unroll
          for (int e = 0; e < 4; ++e) { ov[g][e].x *= al[g]; ov[g][e].y *= al[g]; }
        }
        const uint4* vrow = reinterpret_cast<const uint4*>(sV) + lane;   // (VB 16) row t at vrow[t * 32]
        const uint8_t* qrow = sV + kh * kVHead;                            // (quantised) row t at qrow[t * kVRow]
        const int thp = *s_thp;                                            // tokens >= thp: 8-bit window rows
        const float* pp = sP + kh * G * kPS;
        const int tb = 16 * ew;
        // the window branch only in warps whose 16 tokens reach it (warp-uniform:
        // thp is per CTA), so the other warps run the plain quantised loop
        auto pv = [&](auto win) {
          constexpr bool W = decltype(win)::value;
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const int t0 = tb + 4 * q4;
            if (t0 >= nv) break;
            float4 p4[G];
#pragma unroll
            for (int g = 0; g < G; ++g) p4[g] = *reinterpret_cast<const float4*>(pp + g * kPS + t0);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if (t0 + j < nv) {
                float2 vv[4];   // the lane's 8 values (dims 8 (lane & 15) .. + 8 of KV head kh)
                if constexpr (VB == 16) {
                  const uint4 v = vrow[(t0 + j) * 32];
                  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                  for (int e = 0; e < 4; ++e) vv[e] = make_float2(__uint_as_float(w[e] << 16), __uint_as_float(w[e] & 0xffff0000u));
                } else if (W && t0 + j >= thp) {   // 8-bit recent-window row
                  // group of 4 tokens: [4 x 144 B of head 0 | pad][4 x 144 B of head 1 | pad]
                  const int tt = t0 + j;
                  const uint8_t* rh = sVh + (tt >> 2) * kHGrp + kh * (kHGrp / 2) + (tt & 3) * 144;
                  const int l8 = lane & 15;
                  const uint32_t par = *reinterpret_cast<const uint32_t*>(rh + 128 + 4 * (l8 >> 2));
                  const float sf = __uint_as_float(par << 16), zf = __uint_as_float(par & 0xffff0000u);
                  const uint2 cw = *reinterpret_cast<const uint2*>(rh + 8 * l8);
                  const uint32_t w2[2] = {cw.x, cw.y};
#pragma unroll
                  for (int e = 0; e < 4; ++e)
                    vv[e] = make_float2(fmaf(sf, (float)((w2[e >> 1] >> (16 * (e & 1))) & 255u), zf),
                                        fmaf(sf, (float)((w2[e >> 1] >> (16 * (e & 1) + 8)) & 255u), zf));
                } else {
                  const uint8_t* rq = qrow + (t0 + j) * kVRow;
                  const int l8 = lane & 15;
                  const uint32_t par = *reinterpret_cast<const uint32_t*>(rq + 128 * VB / 8 + 4 * (l8 >> 2));
                  const float sf = __uint_as_float(par << 16), zf = __uint_as_float(par & 0xffff0000u);
                  uint32_t cw;
                  if constexpr (VB == 4) cw = *reinterpret_cast<const uint32_t*>(rq + 4 * l8);
                  else cw = *reinterpret_cast<const uint16_t*>(rq + 2 * l8);
                  constexpr uint32_t m = (1u << VB) - 1;
#pragma unroll
                  for (int e = 0; e < 4; ++e)
                    vv[e] = make_float2(fmaf(sf, (float)((cw >> (2 * e * VB)) & m), zf),
                                        fmaf(sf, (float)((cw >> ((2 * e + 1) * VB)) & m), zf));
                }
#pragma unroll
                for (int g = 0; g < G; ++g) {
                  const float pj = j == 0 ? p4[g].x : j == 1 ? p4[g].y : j == 2 ? p4[g].z : p4[g].w;
                  lp[g] += pj;
                  const float2 p2 = make_float2(pj, pj);
#pragma unroll
                  for (int e = 0; e < 4; ++e) ov[g][e] = __ffma2_rn(p2, vv[e], ov[g][e]);
                }
              }
            }
          }
        };
        if constexpr (HPW) {
          if (tb + 16 <= thp) pv(std::false_type{});
          else pv(std::true_type{});
        } else if constexpr (VB == 16) {
          if (tb + 16 <= nv) {
            // all 16 of the warp's tokens valid (every full tile): no per-token guards, the
            // V vectors and probabilities of 8 tokens are loaded before their FFMA2s
#pragma unroll
            for (int h8 = 0; h8 < 2; ++h8) {
              uint4 vr[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) vr[j] = vrow[(tb + 8 * h8 + j) * 32];
              float4 pa[G], pb[G];
#pragma unroll
              for (int g = 0; g < G; ++g) {
                pa[g] = *reinterpret_cast<const float4*>(pp + g * kPS + tb + 8 * h8);
                pb[g] = *reinterpret_cast<const float4*>(pp + g * kPS + tb + 8 * h8 + 4);
              }
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const uint32_t w[4] = {vr[j].x, vr[j].y, vr[j].z, vr[j].w};
                float2 vv[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) vv[e] = make_float2(__uint_as_float(w[e] << 16), __uint_as_float(w[e] & 0xffff0000u));
#pragma unroll
                for (int g = 0; g < G; ++g) {
                  const float4 p4 = j < 4 ? pa[g] : pb[g];
                  const int jj = j & 3;
                  const float pj = jj == 0 ? p4.x : jj == 1 ? p4.y : jj == 2 ? p4.z : p4.w;
                  lp[g] += pj;
                  const float2 p2 = make_float2(pj, pj);
#pragma unroll
                  for (int e = 0; e < 4; ++e) ov[g][e] = __ffma2_rn(p2, vv[e], ov[g][e]);
                }
              }
            }
          } else {
            pv(std::false_type{});
          }
        } else {
          pv(std::false_type{});
        }
      }
      bar_epi();                                       // sV / sP / sL / sRed / sAl free
      if (ew == 0 && lane == 0) TSTAMP(40 + it);
      if (ew == 0 && lane == 0) mbar_arrive(vempty);
    }
    float o[G];
    if constexpr (TPV) {
#pragma unroll
      for (int g = 0; g < G; ++g) { o[g] = ot[g]; l_run[g] = lt[g]; }
    } else {
    // ---- reduce the 8 token groups' partial P V (sV is free: the V producer is done)
    float* red = reinterpret_cast<float*>(sV);   // [8 warps][NQH][128]
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int e = 0; e < 4; ++e)
        *reinterpret_cast<float2*>(red + ((size_t)ew * NQH + kh * G + g) * kDH + 8 * (lane & 15) + 2 * e) = ov[g][e];
    float* lred = red + 8 * NQH * kDH;           // [8 warps][NQH] denominators
    if ((lane & 15) == 0)
#pragma unroll
      for (int g = 0; g < G; ++g) lred[ew * NQH + kh * G + g] = lp[g];
    bar_epi();
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float l = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) l += lred[w * NQH + hf * G + g];
      l_run[g] = l;
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float acc = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) acc += red[((size_t)w * NQH + hf * G + g) * kDH + n];
      o[g] = acc;
    }
    }
    // ---- write y (single chunk) or the chunk's partial
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int h = nb * NQH + hf * G + g;
      if (a.direct_out && a.ntiles == 1) {
        __nv_bfloat16* y = reinterpret_cast<__nv_bfloat16*>(a.direct_out) + ((size_t)b * a.n_q + h) * kDH;
        y[n] = __float2bfloat16_rn(l_run[g] > 0.f ? o[g] / l_run[g] : 0.f);
      } else {
        float* dst = a.partials + (((size_t)b * a.n_q + h) * a.ntiles + chunk) * (kDH + 2);
        dst[2 + n] = o[g];
        if (n == 0) { dst[0] = m_run[g]; dst[1] = l_run[g]; }
      }
    }
    if (a.counters && a.ntiles > 1) __threadfence();
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (C2) cluster_sync_all();   // every remote arrive / MMA of the pair has landed
  if (tid == 0) TSTAMP(81);
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    if constexpr (C2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
  if (tid == 0) CTIME(3);
  if (a.counters && a.ntiles > 1) merge_if_last<NQH>(a, b, nb, tid, reinterpret_cast<float*>(smem));
  pdl_launch_dependents();
}

template <int G, int STYLE, int VBH, int CG = 1>
cudaError_t launch_t(const CUtensorMap& map, const CUtensorMap& map_lat, const CUtensorMap& map_v,
                     const CUtensorMap& map_vh, const TcArgs& a, int batch, cudaStream_t st, int axis = 0) {
  auto kern = recon_attn_tc2_kernel<G, STYLE, VBH, CG>;
  static DeviceOnce once;
  cudaError_t e = once.run([&] {
    cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes(G, CG));
    return r;
  });
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = (CG == 2 && axis == 3) ? dim3(2 * a.ntiles, a.D / kBN, batch / 2) : dim3(a.ntiles, a.D / kBN, batch);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem_bytes(G, CG);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = CG == 2 ? 2 : 1;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = CG == 2 ? 2 : 1;
  KArgs ka{a};
  return cudaLaunchKernelEx(&cfg, kern, map, map_lat, map_v, map_vh, ka);
}

// MHA with bf16 values on a CTA pair (cta_group::2, M = 256: each U tile is read once per
// pair instead of once per CTA).  Measured (c5 sweep, 32 layers, one B200, profiles/r2/experiments): with request pairs the
// pair kernel is 1.00-1.10x the one-CTA kernel from B = 4 up (the most at long contexts and
// large batches: half the L2 reads of U, a 4-deep operand ring), 0.95-0.98x at B = 1 / 2
// (chunk pairs / short chains), so it runs for MHA batches of >= 4 requests, paired by
// request (a pair runs max(tiles) of its CTAs: two requests' same chunk).
int tc2_pair_axis(const TcArgs& a, int batch) {
  if (!tc2_pair_enabled() || a.G != 1 || a.v_bits != 0) return 0;
  return (batch >= 4 && batch % 2 == 0) ? 3 : 0;
}

}  // namespace tc2

bool tc2_pair_enabled() {   // SALS_TC2_CG=1: the one-CTA kernel for every shape
  static const bool on = [] { const char* e = getenv("SALS_TC2_CG"); return !(e && e[0] == '1'); }();
  return on;
}

extern "C" int sals_debug_tc_ctatime(unsigned long long* host_out) {
#ifdef SALS_TC_CTATIME
  return (int)cudaMemcpyFromSymbol(host_out, tc2::g_ctatime, sizeof(tc2::g_ctatime));
#else
  (void)host_out;
  return -1;
#endif
}

extern "C" int sals_debug_tc_trace(unsigned long long* host_out) {
#ifdef SALS_TC_TRACE
  return (int)cudaMemcpyFromSymbol(host_out, tc2::g_trace, sizeof(tc2::g_trace));
#else
  (void)host_out;
  return -1;
#endif
}

// Largest split count the in-kernel merge can stage in shared memory.
int tc2_merge_max_splits(int G) {
  return (tc2::smem_bytes(G) - 1024) / (2 * G * (tc2::kDH + 3) * 4);
}

bool tc2_supported(int head_dim, int D, int rank, int G) {
  return head_dim == 128 && D % tc2::kBN == 0 && rank % tc2::kBK == 0 && (G == 1 || G == 2 || G == 4);
}

cudaError_t launch_recon_attn_tc2(const CUtensorMap& map, const CUtensorMap& map_u128, const CUtensorMap& ml,
                                  const CUtensorMap& mv, const CUtensorMap& mvh, const TcArgs& a, int batch,
                                  cudaStream_t st) {
  const int style = a.rope.style;
  const int axis = tc2::tc2_pair_axis(a, batch);
  if (axis) {
    return style ? tc2::launch_t<1, 1, 16, 2>(map_u128, ml, mv, mvh, a, batch, st, axis)
                 : tc2::launch_t<1, 0, 16, 2>(map_u128, ml, mv, mvh, a, batch, st, axis);
  }
#define SALS_TC2_VB(VB)                                                                                         \
  switch (a.G) {                                                                                                \
    case 1: return style ? tc2::launch_t<1, 1, VB>(map, ml, mv, mvh, a, batch, st) : tc2::launch_t<1, 0, VB>(map, ml, mv, mvh, a, batch, st); \
    case 2: return style ? tc2::launch_t<2, 1, VB>(map, ml, mv, mvh, a, batch, st) : tc2::launch_t<2, 0, VB>(map, ml, mv, mvh, a, batch, st); \
    case 4: return style ? tc2::launch_t<4, 1, VB>(map, ml, mv, mvh, a, batch, st) : tc2::launch_t<4, 0, VB>(map, ml, mv, mvh, a, batch, st); \
  }                                                                                                             \
  return cudaErrorInvalidValue;
  if (a.v_bits == 4 && a.hp_window > 0) { SALS_TC2_VB(40) }
  if (a.v_bits == 2 && a.hp_window > 0) { SALS_TC2_VB(20) }
  if (a.v_bits == 4) { SALS_TC2_VB(4) }
  if (a.v_bits == 2) { SALS_TC2_VB(2) }
  SALS_TC2_VB(16)
#undef SALS_TC2_VB
}

}  // namespace sals
