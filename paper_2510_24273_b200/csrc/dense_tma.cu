// The dense comparator, TMA-streamed: split-K flash decode over the FULL post-RoPE
// K / V cache (the "dense attention" the paper compares against, "dense
// attention reads 2 s d elements"; Eq. 6 with every token selected).
//
// The stage is a pure HBM stream of 2 B s D 2 bytes, so the design goal is
// bytes in flight at minimum instruction cost (same recipe as score_tma.cu).
// Built for the GQA shapes with 8 KV heads (c3 / c4: D = 1024, G <= 4; other shapes
// use flash_decode_kernel, see dense_tma_supported):
//  - one CTA per SM: grid (nsplit, B) with nsplit * B ~ #SMs; a CTA owns the
//    contiguous token range [split * chunk, +chunk) of request b and ALL KV heads,
//    so its K rows (and its V rows) are ONE contiguous byte range of the cache
//    ([b, t, :] rows of D * 2 bytes are adjacent for consecutive t);
//  - one producer lane streams that range with 1-D bulk copies
//    (cp.async.bulk, 16 KB of K + 16 KB of V per stage = 8 tokens) into a 6-stage
//    mbarrier ring (~160 KB in flight per SM), L2 evict-first;
//  - 8 consumer warps, warp w = KV head w; lane (sub, li) reads dims [8 li, 8 li + 8)
//    of token 2 i + sub of the stage (one 16-byte shared-memory vector per token,
//    conflict-free) and holds the rotated queries of the G query heads in registers.
//    G = 4: FFMA2 dot products, a transposing shuffle reduction (lane li ends with the
//    logit of (pair li / 4, head li % 4)), the online softmax on one value per lane,
//    FFMA2 P V; G = 1 / 2: a butterfly per (pair, head) and one online-softmax state
//    (m, l, o[8]) per query head and token parity, merged at the end;
//  - output: partials [B, n_q, nsplit, d+2] = (m, l, o[d]) for merge_kernel.
// Programmatic dependent launch: the producer streams every stage that does not
// hold the newest token (slot len - 1) before griddepcontrol.wait (the cache rows
// were written at least two launches up, which have completed when this grid
// starts: every kernel of the library triggers its dependents only after its own
// wait); the rotated queries (written by the RoPE kernel just before) are read
// after it.
#include "common.cuh"
#include "kernels.h"
#include "once.h"

namespace sals {
namespace dtma {

constexpr int kStageBytes = 16384;   // per operand (K or V) per stage
constexpr int kStages = 6;
constexpr int kCons = 8;             // consumer warps
constexpr int kThreads = (kCons + 1) * 32;
constexpr int kDH = 128;             // head_dim (16 lanes x 8 bf16)
constexpr size_t kSmem = 128 + (size_t)kStages * 2 * kStageBytes + 2 * kStages * 8;

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
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

template <int G, int HPW>
__global__ void __launch_bounds__(kThreads, 1) dense_tma_kernel(const __grid_constant__ FlashArgs a) {
  // D = 8 HPW x 128, so a stage holds ts = 8 / HPW tokens = NP token pairs
  constexpr int NP = 4 / HPW, ts = 2 * NP;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * 2 * kStageBytes);
  uint64_t* empty = full + kStages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int split = blockIdx.x, b = blockIdx.y;
  const size_t rowb = (size_t)a.D * 2;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], kCons); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int len = a.count[b];
  const int t0 = split * a.chunk;
  const int t1 = min(len, t0 + a.chunk);
  const int nst = t1 > t0 ? (t1 - t0 + ts - 1) / ts : 0;

  if (warp == kCons) {
    // ================= producer: K and V rows of ts tokens per stage =================
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      const char* kb = reinterpret_cast<const char*>(a.kbase) + ((size_t)b * a.cap + t0) * rowb;
      const char* vb = reinterpret_cast<const char*>(a.v_cache) + ((size_t)b * a.cap + t0) * rowb;
      bool waited = false;
      for (int u = 0; u < nst; ++u) {
        const int tt = t0 + u * ts;
        const int nt = min(ts, t1 - tt);
        if (!waited && tt + nt >= len) { pdl_wait(); waited = true; }   // the newest row
        const int s = u % kStages;
        if (u >= kStages) mbar_wait(&empty[s], ((u / kStages) - 1) & 1);
        const uint32_t bytes = (uint32_t)(nt * rowb);
        mbar_arrive_expect_tx(&full[s], 2 * bytes);
        uint8_t* dst = smem + (size_t)s * 2 * kStageBytes;
        bulk_load(smem_u32(dst), kb + (size_t)u * ts * rowb, bytes, &full[s], pol);
        bulk_load(smem_u32(dst + kStageBytes), vb + (size_t)u * ts * rowb, bytes, &full[s], pol);
      }
    }
  } else if constexpr (G == 4 && HPW == 1) {
    // ================= consumers, GQA 4 (c3 / c4): transposed reductions =================
    // Lane (sub, li) holds dims [8 li, +8) of the 4 token pairs' tokens 2 i + sub.  The 16
    // partial logits (pair i, query head g) of a lane are reduced over the 16 lanes of its
    // half with a TRANSPOSING butterfly (15 shuffles instead of 64: each level halves the
    // values a lane keeps), after which lane li holds the full logit of (i, g) = (li / 4,
    // li % 4).  The online softmax then runs one value per lane (group max / sum over the 8
    // lanes of query head g: 3 shuffles each), the rescale factors and the 16 p are
    // broadcast back for the P V.  m and l of head g are kept (group-uniform) by the lanes
    // with li % 4 == g; o by every lane for its 8 dims and its token parity.
    pdl_wait();   // q^R comes from the RoPE kernel just before
    const int sub = lane >> 4, li = lane & 15;
    const int hoff = warp * kDH * 2;
    float2 q2[4][4], o2[4][4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const float4* qv = reinterpret_cast<const float4*>(a.qrope + ((size_t)b * a.n_q + warp * 4 + g) * kDH + li * 8);
      const float4 q0 = qv[0], q1 = qv[1];
      const float sl = a.scale_log2;
      q2[g][0] = make_float2(q0.x * sl, q0.y * sl); q2[g][1] = make_float2(q0.z * sl, q0.w * sl);
      q2[g][2] = make_float2(q1.x * sl, q1.y * sl); q2[g][3] = make_float2(q1.z * sl, q1.w * sl);
#pragma unroll
      for (int e = 0; e < 4; ++e) o2[g][e] = make_float2(0.f, 0.f);
    }
    float m_s = -INFINITY, l_s = 0.f;   // query head li % 4 (group-uniform)
    const int src_half = lane & 16;
    for (int u = 0; u < nst; ++u) {
      const int s = u % kStages;
      const int nt = min(ts, t1 - (t0 + u * ts));
      mbar_wait(&full[s], (u / kStages) & 1);
      const uint8_t* ks = smem + (size_t)s * 2 * kStageBytes + li * 16 + hoff;
      const uint8_t* vs = ks + kStageBytes;
      uint4 kr[4], vr[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int t = 2 * i + sub;
        kr[i] = t < nt ? *reinterpret_cast<const uint4*>(ks + t * rowb) : make_uint4(0, 0, 0, 0);
        vr[i] = t < nt ? *reinterpret_cast<const uint4*>(vs + t * rowb) : make_uint4(0, 0, 0, 0);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);   // the stage is in registers
      float v[16];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t w[4] = {kr[i].x, kr[i].y, kr[i].z, kr[i].w};
        float2 k2[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) k2[e] = make_float2(__uint_as_float(w[e] << 16), __uint_as_float(w[e] & 0xffff0000u));
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          float2 acc = __fmul2_rn(q2[g][0], k2[0]);
#pragma unroll
          for (int e = 1; e < 4; ++e) acc = __ffma2_rn(q2[g][e], k2[e], acc);
          v[i * 4 + g] = acc.x + acc.y;
        }
      }
#pragma unroll
      for (int off = 8, c = 8; off > 0; off >>= 1, c >>= 1) {
        const bool up = (li & off) != 0;
#pragma unroll
        for (int k = 0; k < c; ++k) {
          const float send = up ? v[k] : v[k + c];
          const float keep = up ? v[k + c] : v[k];
          v[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      const bool valid = 2 * (li >> 2) + sub < nt;
      const float sc = valid ? v[0] : -INFINITY;
      float mx = sc;
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
      const float mn = fmaxf(m_s, mx);   // (token 0 of a stage is always valid: mn finite)
      const float alpha = m_s == -INFINITY ? 0.f : exp2f(m_s - mn);
      const float p = valid ? exp2f(sc - mn) : 0.f;
      float ps = p + __shfl_xor_sync(0xffffffffu, p, 4);
      ps += __shfl_xor_sync(0xffffffffu, ps, 8);
      ps += __shfl_xor_sync(0xffffffffu, ps, 16);
      l_s = l_s * alpha + ps;
      m_s = mn;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const float al = __shfl_sync(0xffffffffu, alpha, src_half | g);
        const float2 al2 = make_float2(al, al);
#pragma unroll
        for (int e = 0; e < 4; ++e) o2[g][e] = __fmul2_rn(o2[g][e], al2);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t w[4] = {vr[i].x, vr[i].y, vr[i].z, vr[i].w};
        float2 v2[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) v2[e] = make_float2(__uint_as_float(w[e] << 16), __uint_as_float(w[e] & 0xffff0000u));
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const float pg = __shfl_sync(0xffffffffu, p, src_half | (4 * i + g));
          const float2 p2 = make_float2(pg, pg);
#pragma unroll
          for (int e = 0; e < 4; ++e) o2[g][e] = __ffma2_rn(p2, v2[e], o2[g][e]);
        }
      }
    }
    // the two token parities share m: add their o; write the partials (lanes of half 0)
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      float ov[8];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        ov[2 * e] = o2[g][e].x + __shfl_xor_sync(0xffffffffu, o2[g][e].x, 16);
        ov[2 * e + 1] = o2[g][e].y + __shfl_xor_sync(0xffffffffu, o2[g][e].y, 16);
      }
      float* dst = a.partials + (((size_t)b * a.n_q + warp * 4 + g) * a.nsplit + split) * (kDH + 2);
      if (sub == 0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) dst[2 + li * 8 + e] = ov[e];
        if (li == g) { dst[0] = m_s; dst[1] = l_s; }
      }
    }
  } else {
    // ================= consumers =================
    pdl_wait();   // q^R comes from the RoPE kernel just before
    const int sub = lane >> 4, li = lane & 15;
    float q[HPW][G][8], o[HPW][G][8], m[HPW][G], l[HPW][G];
#pragma unroll
    for (int j = 0; j < HPW; ++j) {
      const int h = warp + kCons * j;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float4* qv = reinterpret_cast<const float4*>(a.qrope + ((size_t)b * a.n_q + h * G + g) * kDH + li * 8);
        const float4 q0 = qv[0], q1 = qv[1];
        q[j][g][0] = q0.x * a.scale_log2; q[j][g][1] = q0.y * a.scale_log2;
        q[j][g][2] = q0.z * a.scale_log2; q[j][g][3] = q0.w * a.scale_log2;
        q[j][g][4] = q1.x * a.scale_log2; q[j][g][5] = q1.y * a.scale_log2;
        q[j][g][6] = q1.z * a.scale_log2; q[j][g][7] = q1.w * a.scale_log2;
        m[j][g] = -INFINITY; l[j][g] = 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e) o[j][g][e] = 0.f;
      }
    }
    for (int u = 0; u < nst; ++u) {
      const int s = u % kStages;
      const int nt = min(ts, t1 - (t0 + u * ts));
      mbar_wait(&full[s], (u / kStages) & 1);
      const uint8_t* ks = smem + (size_t)s * 2 * kStageBytes + li * 16;
      const uint8_t* vs = ks + kStageBytes;
      // the stage's NP token pairs per lane half: logits first, one max / rescale per head
      {
#pragma unroll
        for (int j = 0; j < HPW; ++j) {
          const int hoff = (warp + kCons * j) * kDH * 2;
          uint4 kr[NP];
          bool ok[NP];
#pragma unroll
          for (int i = 0; i < NP; ++i) {
            const int t = 2 * i + sub;
            ok[i] = t < nt;
            kr[i] = ok[i] ? *reinterpret_cast<const uint4*>(ks + t * rowb + hoff) : make_uint4(0, 0, 0, 0);
          }
          float sc[NP][G];
#pragma unroll
          for (int i = 0; i < NP; ++i) {
            float kf[8];
            Elem<__nv_bfloat16>::unpack(kr[i], kf);
#pragma unroll
            for (int g = 0; g < G; ++g) {
              float acc = 0.f;
#pragma unroll
              for (int e = 0; e < 8; ++e) acc = fmaf(q[j][g][e], kf[e], acc);
              sc[i][g] = acc;
            }
          }
#pragma unroll
          for (int off = 8; off > 0; off >>= 1)
#pragma unroll
            for (int i = 0; i < NP; ++i)
#pragma unroll
              for (int g = 0; g < G; ++g) sc[i][g] += __shfl_xor_sync(0xffffffffu, sc[i][g], off);
          uint4 vr[NP];
#pragma unroll
          for (int i = 0; i < NP; ++i) {
            const int t = 2 * i + sub;
            vr[i] = ok[i] ? *reinterpret_cast<const uint4*>(vs + t * rowb + hoff) : make_uint4(0, 0, 0, 0);
          }
#pragma unroll
          for (int g = 0; g < G; ++g) {
            float mx = m[j][g];
#pragma unroll
            for (int i = 0; i < NP; ++i) if (ok[i]) mx = fmaxf(mx, sc[i][g]);
            if (mx == -INFINITY) continue;   // no valid token for this lane half yet
            const float corr = exp2f(m[j][g] - mx);
            l[j][g] *= corr;
#pragma unroll
            for (int e = 0; e < 8; ++e) o[j][g][e] *= corr;
#pragma unroll
            for (int i = 0; i < NP; ++i) {
              const float p = ok[i] ? exp2f(sc[i][g] - mx) : 0.f;
              float vf[8];
              Elem<__nv_bfloat16>::unpack(vr[i], vf);
              l[j][g] += p;
#pragma unroll
              for (int e = 0; e < 8; ++e) o[j][g][e] = fmaf(p, vf[e], o[j][g][e]);
            }
            m[j][g] = mx;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // merge the two token streams (sub = 0 / 1) and write the partials
#pragma unroll
    for (int j = 0; j < HPW; ++j) {
      const int h = warp + kCons * j;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float mo = __shfl_xor_sync(0xffffffffu, m[j][g], 16);
        const float lo = __shfl_xor_sync(0xffffffffu, l[j][g], 16);
        const float mn = fmaxf(m[j][g], mo);
        const float c1 = (m[j][g] == -INFINITY) ? 0.f : exp2f(m[j][g] - mn);
        const float c2 = (mo == -INFINITY) ? 0.f : exp2f(mo - mn);
        float ov[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float oo = __shfl_xor_sync(0xffffffffu, o[j][g][e], 16);
          ov[e] = o[j][g][e] * c1 + oo * c2;
        }
        if (sub == 0) {
          float* dst = a.partials + (((size_t)b * a.n_q + h * G + g) * a.nsplit + split) * (kDH + 2);
          if (li == 0) { dst[0] = mn; dst[1] = l[j][g] * c1 + lo * c2; }
#pragma unroll
          for (int e = 0; e < 8; ++e) dst[2 + li * 8 + e] = ov[e];
        }
      }
    }
  }
  pdl_launch_dependents();
}

}  // namespace dtma

// Host launcher.  cudaErrorNotSupported outside the kernel's shapes (bf16,
// head_dim 128, n_kv a multiple of 8 with n_kv / 8 * G <= 8, 2 D dividing 16 KB):
// the caller then uses flash_decode_kernel.
// Measured (bench dense step, round 2): with 8 KV heads (D = 1024, the GQA shapes c3 / c4)
// this kernel beats flash_decode_kernel (c4 0.50 vs 0.42 of the HBM peak); with 32
// heads (D = 4096, c2) flash_decode_kernel's 8-heads-per-CTA LSU stream is faster
// (0.92 vs 0.84), so the TMA kernel is built for n_kv = 8 only (G <= 4: registers).
bool dense_tma_supported(int head_dim, int n_kv, int G, int dtype_bytes) {
  return dtype_bytes == 2 && head_dim == dtma::kDH && n_kv == dtma::kCons && (G == 1 || G == 2 || G == 4);
}

void dense_tma_plan(int batch, int max_len, int head_dim, int n_kv, int nsm, int& nsplit, int& chunk) {
  const int ts = dtma::kStageBytes / (2 * n_kv * head_dim);
  nsplit = std::max(1, nsm / std::max(1, batch));
  chunk = (max_len + nsplit - 1) / nsplit;
  chunk = ((chunk + ts - 1) / ts) * ts;
  nsplit = std::max(1, (max_len + chunk - 1) / chunk);
}

cudaError_t launch_dense_tma(const FlashArgs& a, int batch, int head_dim, int G, cudaStream_t st) {
  const int n_kv = a.n_kv;
  if (!dense_tma_supported(head_dim, n_kv, G, 2)) return cudaErrorNotSupported;
  const int hpw = n_kv / dtma::kCons;
  void (*k)(FlashArgs) = nullptr;
  int ki = 0;
#define SALS_DT_CASE(H, GG, I) \
  if (hpw == H && G == GG) { k = dtma::dense_tma_kernel<GG, H>; ki = I; }
  SALS_DT_CASE(1, 1, 0) SALS_DT_CASE(1, 2, 1) SALS_DT_CASE(1, 4, 2)
#undef SALS_DT_CASE
  if (!k) return cudaErrorNotSupported;
  static DeviceOnce once[3];
  cudaError_t e = once[ki].run(
      [&] { return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dtma::kSmem); });
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.nsplit, batch);
  cfg.blockDim = dim3(dtma::kThreads);
  cfg.dynamicSmemBytes = dtma::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, a);
}

}  // namespace sals
