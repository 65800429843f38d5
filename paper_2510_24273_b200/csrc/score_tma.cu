// K3, TMA variant: latent scoring  p'_j = q~_{:r*} . K~[b, j, :r*]
// (Alg. 1 line 4) for bf16 caches with r* in {64, 128, 256}.
//
// The stage is a pure HBM stream of B * s * r* * 2 bytes (Sec. 4.5 "read s r*
// elements"), so the design goal is bytes in flight at minimum
// instruction cost:
//  - persistent grid: one CTA per SM (grid <= 148); the (request, 32-token
//    chunk) items are split evenly and contiguously over the CTAs;
//  - one producer lane streams each chunk's rows [b*cap + t0, +32) x [0, r*)
//    with ONE 2-D TMA box (32 rows x r*·2 bytes; the unread tail r*..r of each
//    latent row is skipped by the box) into an 8-stage mbarrier ring
//    (8 x 16 KB in flight per SM at r* = 256);
//  - 8 consumer warps, each owning whole chunks, read the staged rows from
//    shared memory (LG = r*/8 lanes per token, one 16-byte vector each,
//    conflict-free), q~ in registers, fp32 dot products, then a transposing
//    shuffle reduction (see below).  The per-token reduction order does not
//    depend on the grid, so a sequence shard scores its tokens bit-identically
//    to one GPU;
//  - the top-digit histogram of the ranked scores for the top-k kernel is built
//    in shared memory and flushed once per CTA.
// Programmatic dependent launch: the producer starts streaming BEFORE
// griddepcontrol.wait.  That is safe because every kernel of this library
// triggers its dependents only after its own griddepcontrol.wait, so when this
// grid starts, the kernel two launches up (sals_append_latent, which wrote the
// new latent row) has completed and flushed; only q~ (written by the query
// projection just before) is read after the wait.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.h"
#include "recon_attn_tc.h"
#include "once.h"

namespace sals {
namespace stma {

constexpr int kTok = 32;      // tokens per TMA box
constexpr int kStages = 8;
constexpr int kCons = 8;      // consumer warps
constexpr int kThreads = (kCons + 1) * 32;

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
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// Consumers only (named barrier 1, 256 threads): add the CTA's histogram of one
// request into the global one and clear it (a CTA's item range may straddle requests).
__device__ __forceinline__ void flush_hist(uint32_t* hs, uint32_t* gh, int tid) {
  asm volatile("bar.sync 1, %0;" ::"n"(kCons * 32) : "memory");
  for (int i = tid; i < kH0Bins; i += kCons * 32) {
    const uint32_t v = hs[i];
    if (v) { atomicAdd(&gh[i], v); hs[i] = 0; }
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kCons * 32) : "memory");
}

__host__ __device__ constexpr size_t smem_bytes(int rstar) {
  return 128 + (size_t)kStages * kTok * rstar * 2 + 2 * kStages * 8 + kH0Bins * 4;
}

template <int LG>   // lanes per token = r* / 8
__global__ void __launch_bounds__(kThreads, 1)
score_tma_kernel(const __grid_constant__ CUtensorMap map, const __grid_constant__ ScoreArgs a, int nchunk, int items) {
  constexpr int TPW = 32 / LG;             // tokens per warp instruction
  static_assert(LG >= 8 && LG <= 32 && TPW * LG == kTok, "r* in {64, 128, 256}");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  const int row_bytes = LG * 16;                       // r* * 2
  const int stage_bytes = kTok * row_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * stage_bytes);
  uint64_t* empty = full + kStages;
  uint32_t* hs = reinterpret_cast<uint32_t*>(empty + kStages);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i0 = (int)((int64_t)blockIdx.x * items / gridDim.x);
  const int i1 = (int)((int64_t)(blockIdx.x + 1) * items / gridDim.x);
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (a.hist0)
    for (int i = tid; i < kH0Bins; i += kThreads) hs[i] = 0;
  __syncthreads();

  if (warp == kCons) {
    // ================= producer: one TMA box per (request, 32-token chunk) =================
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&map) : "memory");
      // stream_after_wait: the new token's latent row (slot len - 1) was written by the
      // kernel just before (fused append): the chunk holding it is loaded only after
      // griddepcontrol.wait; every older row streams before it
      bool waited = !a.stream_after_wait;
      int u = 0, b = i0 / nchunk, c = i0 - b * nchunk;
      int len = i0 < i1 ? a.len[b] : 0;
      for (int it = i0; it < i1; ++it) {
        if (c * kTok < len) {
          if (!waited && (c + 1) * kTok >= len) { pdl_wait(); waited = true; }
          const int s = u % kStages;
          if (u >= kStages) mbar_wait(&empty[s], ((u / kStages) - 1) & 1);
          mbar_arrive_expect_tx(&full[s], (uint32_t)stage_bytes);
          tma_load_2d(smem_u32(smem + s * stage_bytes), &map, 0, (int)((int64_t)b * a.cap + c * kTok), &full[s]);
          ++u;
        }
        if (++c == nchunk && it + 1 < i1) { c = 0; ++b; len = a.len[b]; }
      }
    }
  } else {
    // ================= consumers: warp w owns every kCons-th staged chunk =================
    // Lane (sub, li) holds dims [8 li, 8 li + 8) of the chunk's tokens sub + TPW k,
    // k < LG; a transposing reduction over the LG lanes of its group leaves lane li
    // with the full score of token sub + TPW li (log2 LG shuffle rounds for LG
    // tokens instead of one butterfly per token), so the writes and the histogram
    // updates are lane-parallel.  The adds form the same tree for every token (up
    // to commutation, which is exact), so a token's score does not depend on its
    // slot in the chunk or on the grid.
    pdl_wait();   // q~ comes from the query projection
    const int li = lane % LG, sub = lane / LG;
    float q[8];
    int b = i0 / nchunk, c = i0 - b * nchunk, cur_b = -1, len = 0, u = 0;
    int64_t r_lo = 0, r_hi = 0;
    float* out = nullptr;
    for (int it = i0; it < i1; ++it) {
      if (b != cur_b) {
        if (a.hist0 && cur_b >= 0) flush_hist(hs, a.hist0 + (size_t)cur_b * kH0Bins, tid);
        cur_b = b;
        len = a.len[b];
        const float4* qv = reinterpret_cast<const float4*>(a.qtil + (size_t)b * a.rstar + li * 8);
        const float4 q0 = qv[0], q1 = qv[1];
        q[0] = q0.x; q[1] = q0.y; q[2] = q0.z; q[3] = q0.w; q[4] = q1.x; q[5] = q1.y; q[6] = q1.z; q[7] = q1.w;
        out = a.scores + (size_t)b * a.stride;
        const int64_t sg = a.hist0 ? a.seq_len[b] : 0;
        r_lo = a.sink; r_hi = sg - a.recent;
      }
      const int t0 = c * kTok;
      if (++c == nchunk) { c = 0; ++b; }
      if (t0 >= len) continue;
      const int uu = u++;
      if (uu % kCons != warp) continue;
      const int s = uu % kStages;
      mbar_wait(&full[s], (uu / kStages) & 1);
      const uint8_t* st = smem + s * stage_bytes + li * 16;
      float v[LG];
#pragma unroll
      for (int k0 = 0; k0 < LG; k0 += 8) {
        uint4 raw[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) raw[k] = *reinterpret_cast<const uint4*>(st + (sub + TPW * (k0 + k)) * row_bytes);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          float f[8];
          Elem<__nv_bfloat16>::unpack(raw[k], f);
          float acc = 0.f;
#pragma unroll
          for (int e = 0; e < 8; ++e) acc = fmaf(f[e], q[e], acc);
          v[k0 + k] = acc;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);   // the chunk is in registers
#pragma unroll
      for (int off = LG / 2; off > 0; off >>= 1) {
        const bool up = (li & off) != 0;
#pragma unroll
        for (int i = 0; i < off; ++i) {
          const float send = up ? v[i] : v[i + off];
          const float keep = up ? v[i + off] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      const int t = t0 + sub + TPW * li;
      if (t < len) {
        out[t] = v[0];
        const int64_t g = a.idx_base + t;
        if (a.hist0 && g >= r_lo && g < r_hi) atomicAdd(&hs[float_key(v[0]) >> kH0Shift], 1u);
      }
    }
    if (a.hist0 && cur_b >= 0) flush_hist(hs, a.hist0 + (size_t)cur_b * kH0Bins, tid);
  }
  pdl_launch_dependents();
}

}  // namespace stma

// Host launcher.  Returns cudaErrorNotSupported when the shape is outside the
// TMA kernel (the caller then uses the LSU kernel).
cudaError_t launch_score_tma(const ScoreArgs& a, int batch, int max_len, cudaStream_t st, int nsm) {
  if (a.rstar != 64 && a.rstar != 128 && a.rstar != 256) return cudaErrorNotSupported;
  auto* enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tma_encoder_fn());
  if (!enc) return cudaErrorNotSupported;
  const uint64_t rows = (uint64_t)batch * (uint64_t)a.cap;
  if (rows > 0x7fffffffull) return cudaErrorNotSupported;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)a.r, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)a.r * 2};
  cuuint32_t box[2] = {(cuuint32_t)a.rstar, (cuuint32_t)stma::kTok};
  cuuint32_t estr[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a.latent), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  const int nchunk = (max_len + stma::kTok - 1) / stma::kTok;
  const int items = batch * nchunk;
  const size_t smem = stma::smem_bytes(a.rstar);
  void (*k)(CUtensorMap, ScoreArgs, int, int) = nullptr;
  switch (a.rstar) {
    case 64: k = stma::score_tma_kernel<8>; break;
    case 128: k = stma::score_tma_kernel<16>; break;
    default: k = stma::score_tma_kernel<32>; break;
  }
  static DeviceOnce once[3];
  const int ai = a.rstar == 64 ? 0 : (a.rstar == 128 ? 1 : 2);
  cudaError_t e = once[ai].run([&] { return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); });
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(std::max(1, std::min(items, nsm)));
  cfg.blockDim = dim3(stma::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, map, a, nchunk, items);
}

}  // namespace sals
