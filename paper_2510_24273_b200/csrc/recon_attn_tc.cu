// Path T: fused selective reconstruction + RoPE + sparse attention on the
// 5th-generation tensor cores (Alg. 1 lines 6-9; Eq. 6).
//
// One CTA per (request b, tile of 128 selected tokens, block of 256 columns of
// D = 256/d KV heads).  The reconstruction K_C = K~_C U^T is a real dense
// contraction (M = 128 selected rows, N = 256, K = r):
//   * A = the 128 gathered latent rows, staged by 4 producer warps with 16-byte
//     cp.async into the canonical K-major SWIZZLE_128B layout,
//   * B = the U rows of the column block, one 2-D TMA per 64-wide K chunk,
//   * tcgen05.mma.cta_group::1.kind::f16 (bf16 x bf16 -> fp32) issued by one
//     thread into a 128 x 256 fp32 accumulator in TMEM, 3-stage mbarrier ring.
// In parallel one thread streams the 128 gathered V rows (512 contiguous bytes
// each) into shared memory with cp.async.bulk.
// Epilogue (the same 4 warps, thread = selected token = TMEM lane): tcgen05.ld
// the reconstructed key row, rotate it by RoPE at the token's ORIGINAL position
// (reading R8) in fp32, dot it with the rotated queries of the G query heads of
// each KV head (logits never leave registers; K_C never touches HBM), tile
// softmax (max / sum over the 128 rows), then P V from shared memory -> one
// split-K partial (m, l, o) per (query head, tile), merged by merge_kernel.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"
#include "recon_attn_tc.h"
#include "once.h"

namespace sals {

namespace {

constexpr int kBK = 64;             // K chunk = one 128-byte swizzle atom of bf16
constexpr int kBN = 256;            // columns per CTA (UMMA N)
constexpr int kStages = 3;
constexpr int kThreads = 192;       // warps 0-3 producers/epilogue, 4 TMA+TMEM, 5 MMA
constexpr int kABytes = kTcRows * kBK * 2;    // 16 KB
constexpr int kBBytes = kBN * kBK * 2;        // 32 KB
constexpr int kVBytes = kTcRows * kBN * 2;    // 64 KB
constexpr int kSmemBytes = kStages * (kABytes + kBBytes) + kVBytes + 1024 /*align*/ + 2048 /*misc*/;

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
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
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// K-major SWIZZLE_128B shared-memory matrix descriptor (tcgen05 format):
// start>>4 [0,14), LBO>>4 [16,30) (unused for swizzled K-major: 1), SBO>>4
// [32,46) = 1024 B between 8-row groups, version 1 at bit 46, layout 2 (128B) at [61,64).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// Instruction descriptor, kind::f16: D fp32, A/B bf16, both K-major, N, M.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kBN >> 3) << 17) |
                            ((uint32_t)(kTcRows >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// 32 consecutive fp32 columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

struct TcKernelArgs {
  TcArgs a;
};

// DH = head_dim; G = query heads per KV head; STYLE = RoPE pairing.
template <int DH, int G, int STYLE>
__global__ void __launch_bounds__(kThreads, 1)
recon_attn_tc_kernel(const __grid_constant__ CUtensorMap tmap_u, const __grid_constant__ TcKernelArgs ka) {
  constexpr int HPB = kBN / DH;          // KV heads per CTA
  constexpr int NQH = HPB * G;           // query heads per CTA
  constexpr int HALF = DH / 2;
  constexpr int PCH = 32;                // rotation pairs per epilogue chunk
  const TcArgs& a = ka.a;
  extern __shared__ uint8_t smem_raw[];
  // align with pointer arithmetic on the __shared__ array so the compiler keeps the shared
  // address space (an integer round trip would turn every access into a generic load)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                                       // [stages][128][128 B] swizzled
  uint8_t* sB = sA + kStages * kABytes;                     // [stages][256][128 B] swizzled
  uint8_t* sV = sB + kStages * kBBytes;                     // [128][512 B]
  uint8_t* misc = sV + kVBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(misc);       // [stages]
  uint64_t* empty = full + kStages;                         // [stages]
  uint64_t* mma_done = empty + kStages;
  uint64_t* v_full = mma_done + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(v_full + 1);
  int* sRows = reinterpret_cast<int*>(tmem_slot + 4);       // [128]
  float* sRed = reinterpret_cast<float*>(sRows + kTcRows);  // [4][NQH]
  float* sQ = reinterpret_cast<float*>(sA);                 // after the mainloop: [NQH][DH]
  float* sP = reinterpret_cast<float*>(sA + kABytes);       // after the mainloop: [NQH][128]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ti = blockIdx.x, nb = blockIdx.y, b = blockIdx.z;
  const int n0 = nb * kBN;

  pdl_wait();
  const int cnt = a.count[b];
  const int nvalid = min(kTcRows, cnt - ti * kTcRows);
  if (nvalid <= 0) {   // tile past this request's selection: empty partials
    for (int i = tid; i < NQH; i += kThreads) {
      const int h = (nb * HPB) * G + i;
      float* dst = a.partials + (((size_t)b * a.n_q + h) * a.ntiles + ti) * (DH + 2);
      dst[0] = -INFINITY;
      dst[1] = 0.f;
    }
    pdl_launch_dependents();
    return;
  }
  if (tid < kTcRows) sRows[tid] = (tid < nvalid) ? a.sel[(size_t)b * a.k_stride + ti * kTcRows + tid] : -1;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 128 + 1); mbar_init(&empty[s], 1); }
    mbar_init(mma_done, 1);
    mbar_init(v_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nk = a.r / kBK;
  const char* latent = reinterpret_cast<const char*>(a.latent);

  if (warp < 4) {
    // ===== A producer: gathered latent rows -> swizzled K-major tile =====
    for (int kc = 0; kc < nk; ++kc) {
      const int s = kc % kStages;
      if (kc >= kStages) mbar_wait(&empty[s], ((kc / kStages) - 1) & 1);
      const uint32_t base = smem_u32(sA + s * kABytes);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int rl = warp * 32 + i * 4 + (lane >> 3);
        const int ch = lane & 7;
        const int row = sRows[rl];
        const char* src = latent + (((size_t)b * a.cap + (row >= 0 ? row : 0)) * a.r + kc * kBK + ch * 8) * 2;
        cp_async_16(base + rl * 128 + ((ch ^ (rl & 7)) << 4), src, row >= 0 ? 16u : 0u);
      }
      cp_async_arrive_noinc(&full[s]);
    }
  } else if (warp == 4) {
    if (lane == 0) {
      // ===== V rows (bulk copies, 512 contiguous bytes each) then the U pipeline =====
      mbar_arrive_expect_tx(v_full, (uint32_t)nvalid * (kBN * 2));
      const char* vb = reinterpret_cast<const char*>(a.v_cache);
      for (int t = 0; t < nvalid; ++t)
        bulk_load(smem_u32(sV + t * (kBN * 2)), vb + (((size_t)b * a.cap + sRows[t]) * a.D + n0) * 2, kBN * 2, v_full);
      for (int kc = 0; kc < nk; ++kc) {
        const int s = kc % kStages;
        if (kc >= kStages) mbar_wait(&empty[s], ((kc / kStages) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], kBBytes);
        tma_load_2d(smem_u32(sB + s * kBBytes), &tmap_u, kc * kBK, n0, &full[s]);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      // ===== MMA issuer =====
      for (int kc = 0; kc < nk; ++kc) {
        const int s = kc % kStages;
        mbar_wait(&full[s], (kc / kStages) & 1);
        tc_fence_after();
        fence_proxy_async();
        const uint32_t abase = smem_u32(sA + s * kABytes), bbase = smem_u32(sB + s * kBBytes);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k)
          mma_bf16(tmem, sw128_desc(abase + k * 32), sw128_desc(bbase + k * 32), (kc | k) ? 1u : 0u);
        mma_commit(&empty[s]);
      }
      mma_commit(mma_done);
    }
  }

  if (warp < 4) {
    // ===== epilogue: RoPE + logits + softmax + P V =====
    mbar_wait(mma_done, 0);
    tc_fence_after();
    // rotated, scaled queries of this CTA's query heads -> sQ (stage buffers are free now)
    for (int i = tid; i < NQH * DH; i += 128) {
      const int qh = i / DH, j = i % DH;
      const int h = nb * HPB * G + qh;
      sQ[i] = a.qrope[((size_t)b * a.n_q + h) * DH + j] * a.scale_log2;
    }
    epi_bar();
    const int m = tid;                    // row = TMEM lane
    const int row = sRows[m];
    const int64_t pos = a.pos_base + (row >= 0 ? row : 0);
    const uint32_t tbase = tmem + ((uint32_t)(warp * 32) << 16);
    float acc[HPB][G];
#pragma unroll
    for (int j = 0; j < HPB; ++j)
#pragma unroll
      for (int g = 0; g < G; ++g) acc[j][g] = 0.f;
#pragma unroll 1
    for (int p0 = 0; p0 < HALF; p0 += PCH) {
      float cs[PCH], sn[PCH];
#pragma unroll
      for (int i = 0; i < PCH; ++i) rope_cs_fast(a.rope.th_hi[p0 + i], a.rope.th_lo[p0 + i], (int)pos, cs[i], sn[i]);
#pragma unroll
      for (int j = 0; j < HPB; ++j) {
        float xl[PCH], xh[PCH];
        if (STYLE == 0) {
          tmem_ld32(tbase + j * DH + p0, xl);
          tmem_ld32(tbase + j * DH + HALF + p0, xh);
        } else {
          float t0[32], t1[32];
          tmem_ld32(tbase + j * DH + 2 * p0, t0);
          tmem_ld32(tbase + j * DH + 2 * p0 + 32, t1);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            xl[i] = t0[2 * i]; xh[i] = t0[2 * i + 1];
            xl[16 + i] = t1[2 * i]; xh[16 + i] = t1[2 * i + 1];
          }
        }
#pragma unroll
        for (int i = 0; i < PCH; ++i) {
          const float rl = xl[i] * cs[i] - xh[i] * sn[i];
          const float rh = xl[i] * sn[i] + xh[i] * cs[i];
          const int lo = STYLE == 0 ? p0 + i : 2 * (p0 + i);
          const int hi = STYLE == 0 ? HALF + p0 + i : 2 * (p0 + i) + 1;
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const float* q = sQ + (j * G + g) * DH;
            acc[j][g] = fmaf(q[lo], rl, fmaf(q[hi], rh, acc[j][g]));
          }
        }
      }
    }
    // tile softmax over the 128 rows (log2 domain)
    float mx[NQH];
#pragma unroll
    for (int j = 0; j < HPB; ++j)
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float v = (row >= 0) ? acc[j][g] : -INFINITY;
        acc[j][g] = v;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0) sRed[warp * NQH + j * G + g] = v;
      }
    epi_bar();
#pragma unroll
    for (int q = 0; q < NQH; ++q)
      mx[q] = fmaxf(fmaxf(sRed[q], sRed[NQH + q]), fmaxf(sRed[2 * NQH + q], sRed[3 * NQH + q]));
    epi_bar();
#pragma unroll
    for (int j = 0; j < HPB; ++j)
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int q = j * G + g;
        const float p = (row >= 0) ? exp2f(acc[j][g] - mx[q]) : 0.f;
        sP[q * kTcRows + m] = p;
        float v = p;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) sRed[warp * NQH + q] = v;
      }
    mbar_wait(v_full, 0);
    epi_bar();
    // P V: thread owns columns (2 tid, 2 tid + 1) of the 256-column block
    const int n = 2 * tid;
    const int j = n / DH;
    float o0[G], o1[G];
#pragma unroll
    for (int g = 0; g < G; ++g) o0[g] = o1[g] = 0.f;
    const uint32_t* vrow = reinterpret_cast<const uint32_t*>(sV) + tid;
#pragma unroll 4
    for (int t = 0; t < nvalid; ++t) {
      const uint32_t vv = vrow[t * (kBN / 2)];
      const float v0 = __uint_as_float(vv << 16), v1 = __uint_as_float(vv & 0xffff0000u);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float p = sP[(j * G + g) * kTcRows + t];
        o0[g] = fmaf(p, v0, o0[g]);
        o1[g] = fmaf(p, v1, o1[g]);
      }
    }
    const int dl = n - j * DH;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int q = j * G + g;
      const int h = nb * HPB * G + q;
      float* dst = a.partials + (((size_t)b * a.n_q + h) * a.ntiles + ti) * (DH + 2);
      dst[2 + dl] = o0[g];
      dst[3 + dl] = o1[g];
      if (dl == 0) {
        dst[0] = mx[q];
        dst[1] = (sRed[q] + sRed[NQH + q]) + (sRed[2 * NQH + q] + sRed[3 * NQH + q]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
  pdl_launch_dependents();
}

// ---------------------------------------------------------------- host side
thread_local std::string g_tc_err;
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

PFN_cuTensorMapEncodeTiled_v12000 g_encode_drv = nullptr;

// cuTensorMapEncodeTiled is a pure function of its arguments, but a host call of a
// few microseconds; a decode step encodes 4-5 maps per layer per call, which made the
// eager (e2e) path host-bound at c2.  Encoded maps are cached by their full argument
// list (direct-mapped, 1024 entries, under a mutex): a hit is a key compare and a copy.
struct MapKey {
  void* addr;
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5], estr[5];
  uint32_t rank, dt, il, sw, l2, oob;
};
struct MapEntry {
  MapKey key;
  CUtensorMap map;
  bool valid;
};
constexpr int kMapCache = 1024;
MapEntry g_map_cache[kMapCache];
std::mutex g_map_mu;

CUresult encode_cached(CUtensorMap* out, CUtensorMapDataType dt, cuuint32_t rank, void* addr, const cuuint64_t* dims,
                       const cuuint64_t* strides, const cuuint32_t* box, const cuuint32_t* estr,
                       CUtensorMapInterleave il, CUtensorMapSwizzle sw, CUtensorMapL2promotion l2,
                       CUtensorMapFloatOOBfill oob) {
  if (rank < 1 || rank > 5) return g_encode_drv(out, dt, rank, addr, dims, strides, box, estr, il, sw, l2, oob);
  MapKey k;
  std::memset(&k, 0, sizeof(k));
  k.addr = addr; k.rank = rank; k.dt = dt; k.il = il; k.sw = sw; k.l2 = l2; k.oob = oob;
  for (uint32_t i = 0; i < rank; ++i) { k.dims[i] = dims[i]; k.box[i] = box[i]; k.estr[i] = estr[i]; }
  for (uint32_t i = 0; i + 1 < rank; ++i) k.strides[i] = strides[i];
  uint64_t h = 1469598103934665603ull;   // FNV-1a over the key bytes
  const unsigned char* kb = reinterpret_cast<const unsigned char*>(&k);
  for (size_t i = 0; i < sizeof(k); ++i) h = (h ^ kb[i]) * 1099511628211ull;
  MapEntry& e = g_map_cache[h % kMapCache];
  {
    std::lock_guard<std::mutex> lock(g_map_mu);
    if (e.valid && std::memcmp(&e.key, &k, sizeof(k)) == 0) { *out = e.map; return CUDA_SUCCESS; }
  }
  const CUresult r = g_encode_drv(out, dt, rank, addr, dims, strides, box, estr, il, sw, l2, oob);
  if (r == CUDA_SUCCESS) {
    std::lock_guard<std::mutex> lock(g_map_mu);
    e.key = k; e.map = *out; e.valid = true;
  }
  return r;
}

bool get_encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      g_encode_drv = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
      g_encode = &encode_cached;
    }
  });
  return g_encode != nullptr;
}

template <int DH, int G, int STYLE>
cudaError_t launch_t(const CUtensorMap& map, const TcArgs& a, int batch, cudaStream_t st) {
  auto kern = recon_attn_tc_kernel<DH, G, STYLE>;
  static DeviceOnce once;
  cudaError_t e = once.run([&] { return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes); });
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.ntiles, a.D / kBN, batch);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  TcKernelArgs ka{a};
  return cudaLaunchKernelEx(&cfg, kern, map, ka);
}

template <int DH, int STYLE>
cudaError_t launch_g(const CUtensorMap& map, const TcArgs& a, int batch, cudaStream_t st) {
  switch (a.G) {
    case 1: return launch_t<DH, 1, STYLE>(map, a, batch, st);
    case 2: return launch_t<DH, 2, STYLE>(map, a, batch, st);
    case 4: return launch_t<DH, 4, STYLE>(map, a, batch, st);
    case 8: return launch_t<DH, 8, STYLE>(map, a, batch, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_recon_attn_tc2(const CUtensorMap& map, const CUtensorMap& map_u128, const CUtensorMap& ml,
                                  const CUtensorMap& mv, const CUtensorMap& mvh, const TcArgs& a, int batch,
                                  cudaStream_t st);

bool tc_supported(int head_dim, int D, int rank, int G) {
  return (head_dim == 64 || head_dim == 128 || head_dim == 256) && D % kBN == 0 && rank % kBK == 0 &&
         (G == 1 || G == 2 || G == 4 || G == 8) && !(head_dim == 64 && G == 8);
}

const char* tc_last_error() { return g_tc_err.c_str(); }

void* tma_encoder_fn() { return get_encoder() ? reinterpret_cast<void*>(g_encode) : nullptr; }

sals_status launch_recon_attn_tc(const TcArgs& a, int batch, cudaStream_t st) {
  if (!tc_supported(a.head_dim, a.D, a.r, a.G)) { g_tc_err = "shape not supported by the tcgen05 path"; return SALS_ERR_UNSUPPORTED; }
  if (!get_encoder()) { g_tc_err = "cuTensorMapEncodeTiled unavailable"; return SALS_ERR_CUDA; }
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)a.r, (cuuint64_t)a.D};
  cuuint64_t strides[1] = {(cuuint64_t)a.r * 2};
  cuuint32_t box[2] = {kBK, kBN};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = g_encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a.U), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) { g_tc_err = "cuTensorMapEncodeTiled failed (U must be 16-B aligned)"; return SALS_ERR_CUDA; }
  cudaError_t e;
  const int style = a.rope.style;
  if (a.tiles_per_cta > 0) {   // planned for the persistent v2 kernel
    // gather4 maps: latent [B*cap, r] rows of 64-column boxes (SWIZZLE_128B) and
    // V [B*cap, D] rows of 256-column boxes (linear), one row per box
    CUtensorMap ml, mv;
    const cuuint64_t rows = (cuuint64_t)batch * (cuuint64_t)a.cap;
    if (rows > 0x7fffffffull) { g_tc_err = "B*cap exceeds the 2^31 rows of a TMA gather"; return SALS_ERR_UNSUPPORTED; }
    cuuint64_t dl[2] = {(cuuint64_t)a.r, rows}, sl[1] = {(cuuint64_t)a.r * 2};
    cuuint32_t bl[2] = {64, 1};
    // value rows: bf16 [D] per token (256-column boxes), or the quantised byte rows
    // (2 heads' code + parameter bytes per box, DESIGN R15)
    const bool vq = a.v_bits != 0;
    const int vhead = vq ? 128 * a.v_bits / 8 + 16 : 0;
    cuuint64_t dv[2] = {vq ? (cuuint64_t)a.v_row_bytes : (cuuint64_t)a.D, rows};
    cuuint64_t sv[1] = {vq ? (cuuint64_t)a.v_row_bytes : (cuuint64_t)a.D * 2};
    cuuint32_t bv[2] = {vq ? (cuuint32_t)(2 * vhead) : 256u, 1};   // (bf16 rows: used by the v1 kernel only)
    if (g_encode(&ml, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a.latent), dl, sl, bl, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
        g_encode(&mv, vq ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                 const_cast<void*>(a.v_cache), dv, sv, bv, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      g_tc_err = "cuTensorMapEncodeTiled failed for the gather maps";
      return SALS_ERR_CUDA;
    }
    // (quantised values) the 8-bit recent-window ring [B * w, n_kv * 144] after the rows
    CUtensorMap mvh = mv;
    if (vq && a.hp_window > 0) {
      const cuuint64_t hrow = (cuuint64_t)(a.D / 128) * 144;
      cuuint64_t dh[2] = {hrow, (cuuint64_t)batch * (cuuint64_t)a.hp_window}, sh[1] = {hrow};
      cuuint32_t bh[2] = {144u, 1};   // one KV head per box (boxes are <= 256 elements)
      if (g_encode(&mvh, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2,
                   const_cast<char*>(reinterpret_cast<const char*>(a.v_cache)) + a.hp_ring_off, dh, sh, bh, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        g_tc_err = "cuTensorMapEncodeTiled failed for the recent-window map";
        return SALS_ERR_CUDA;
      }
    }
    // (cta_group::2 variant) U boxes of 128 columns: one half of the pair's 256 per CTA
    CUtensorMap mu2 = map;
    cuuint32_t box2[2] = {kBK, kBN / 2};
    if (tc2_pair_enabled() && g_encode(&mu2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a.U), dims, strides, box2, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      g_tc_err = "cuTensorMapEncodeTiled failed for the 128-column U map";
      return SALS_ERR_CUDA;
    }
    e = launch_recon_attn_tc2(map, mu2, ml, mv, mvh, a, batch, st);
    if (e != cudaSuccess) { g_tc_err = cudaGetErrorString(e); return SALS_ERR_CUDA; }
    return SALS_OK;
  }
  switch (a.head_dim) {
    case 64: e = style ? launch_g<64, 1>(map, a, batch, st) : launch_g<64, 0>(map, a, batch, st); break;
    case 128: e = style ? launch_g<128, 1>(map, a, batch, st) : launch_g<128, 0>(map, a, batch, st); break;
    default: e = style ? launch_g<256, 1>(map, a, batch, st) : launch_g<256, 0>(map, a, batch, st); break;
  }
  if (e != cudaSuccess) { g_tc_err = cudaGetErrorString(e); return SALS_ERR_CUDA; }
  return SALS_OK;
}

}  // namespace sals
