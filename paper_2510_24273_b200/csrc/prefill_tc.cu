// Prefill / bulk append on the tensor cores: Eq. 1 /
// Alg. 1 line 3 for a block of n consecutive tokens of every request,
//   latent_cache[b, start + i, :] = U^T k[b, i, :]          (i < n)
// as a tcgen05 GEMM  C[n x r] = K_b[n x D] . U[D x r]  per request:
//   A = key rows [128 tokens x 64 of D] by TMA, K-major SWIZZLE_128B (the tensor map
//       spans all B*n rows; rows past a request's n are computed and not stored)
//   B = U [64 of D x 256 of r] by TMA as four 64-column boxes: an MN-major
//       SWIZZLE_128B operand (64-column blocks LBO = 8 KB apart, 8-row groups SBO = 1 KB)
//   D = 128 x 256 fp32 in TMEM; 4-stage mbarrier ring; one elected thread issues
//       tcgen05.mma.cta_group::1.kind::f16; epilogue warps round to bf16 and store the rows.
// and the value rows of the block: copied as dtype, or (cfg->v_bits 4 / 2) quantised
// per token and 32-channel group with the append's rule (quant.cuh, DESIGN R15), the
// last w tokens also into the 8-bit recent-window ring (slot pos % w).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.h"
#include "once.h"
#include "quant.cuh"

namespace sals {
void* tma_encoder_fn();

namespace ptc {

constexpr int kM = 128, kN = 256, kBK = 64, kStages = 4, kThreads = 256;
constexpr int kABytes = kM * kBK * 2;   // 16 KB
constexpr int kBBytes = kN * kBK * 2;   // 32 KB
constexpr int kSmem = 1024 + kStages * (kABytes + kBBytes) + 256;

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\nPW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra PW_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint64_t desc_k(uint32_t saddr) {   // K-major SWIZZLE_128B (SBO 1 KB)
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
__device__ __forceinline__ uint64_t desc_mn(uint32_t saddr) {  // MN-major SWIZZLE_128B (LBO 8 KB, SBO 1 KB)
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(8192 >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

struct Args {
  void* latent; int64_t cap; int r, D, n, start;
};

// grid (ceil(n / 128), ceil(r / 256), B); N of the tile = min(256, r - n0) (a multiple of 64)
__global__ void __launch_bounds__(kThreads, 1)
prefill_tc_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_u, const Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = sA + kStages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * kBBytes);
  uint64_t* empty = full + kStages;
  uint64_t* done = empty + kStages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.x * kM, n0 = blockIdx.y * kN, b = blockIdx.z;
  const int nn = min(kN, a.r - n0);           // 64 .. 256
  const int nbox = nn / 64;
  const int nk = a.D / kBK;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  pdl_wait();
  if (warp == 0 && lane == 0) {
    for (int kc = 0; kc < nk; ++kc) {
      const int s = kc % kStages;
      if (kc >= kStages) mbar_wait(&empty[s], ((kc / kStages) - 1) & 1);
      mbar_expect(&full[s], (uint32_t)(kABytes + nbox * 8192));
      tma2d(smem_u32(sA + s * kABytes), &tm_k, kc * kBK, b * a.n + m0, &full[s]);
      for (int j = 0; j < nbox; ++j) tma2d(smem_u32(sB + s * kBBytes + j * 8192), &tm_u, n0 + 64 * j, kc * kBK, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) /*B MN-major*/ |
                           ((uint32_t)(nn >> 3) << 17) | ((uint32_t)(kM >> 4) << 24);
    for (int kc = 0; kc < nk; ++kc) {
      const int s = kc % kStages;
      mbar_wait(&full[s], (kc / kStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t aa = smem_u32(sA + s * kABytes), bb = smem_u32(sB + s * kBBytes);
#pragma unroll
      for (int ks = 0; ks < kBK / 16; ++ks) {
        const uint32_t acc = (kc | ks) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(desc_k(aa + ks * 32)), "l"(desc_mn(bb + ks * 2048)), "r"(idesc), "r"(acc)
            : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&empty[s]))
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(done))
                 : "memory");
  } else if (warp >= 4) {
    // epilogue: warp 4 + q reads TMEM lanes 32 q .. (token rows), 32 columns at a time
    const int q = warp - 4, m = m0 + q * 32 + lane;
    mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(a.latent) + ((size_t)b * a.cap + a.start + m) * a.r + n0;
    for (int c0 = 0; c0 < nn; c0 += 32) {
      uint32_t v[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
            "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
            "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(tmem + ((uint32_t)(q * 32) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (m < a.n) {
        uint4 o[4];
        uint32_t* ow = reinterpret_cast<uint32_t*>(o);
#pragma unroll
        for (int i = 0; i < 16; ++i) ow[i] = pack_bf16x2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
#pragma unroll
        for (int i = 0; i < 4; ++i) reinterpret_cast<uint4*>(dst + c0)[i] = o[i];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
  pdl_launch_dependents();
}

// value rows of the block: quantised (v_bits 4 / 2) per (token, 32-channel group);
// the last w tokens of the block (positions >= start + n - w) also into the ring
struct VArgs {
  const void* v; void* v_cache; int64_t cap; int D, n, start, B, bits, v_row_bytes, hp_window;
  int64_t hp_ring_off;
};
__global__ void __launch_bounds__(256) prefill_vq_kernel(VArgs a) {
  pdl_wait();
  const int slices = a.D / 8;
  const int64_t nitems = (int64_t)a.B * a.n * slices;
  const int gph = 128 / 32, hb = 128 * a.bits / 8 + gph * 4;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < nitems; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const bool ok = i < nitems;
    const int64_t tok = ok ? i / slices : 0;            // b * n + t
    const int sl = ok ? (int)(i - tok * slices) : 0;
    const int b = (int)(tok / a.n), t = (int)(tok - (int64_t)b * a.n);
    const int gi = sl >> 2, q = sl & 3, h = gi / gph, gq = gi - h * gph;
    float f[8];
    if (ok) Elem<__nv_bfloat16>::unpack(ld_v4(reinterpret_cast<const char*>(a.v) + ((size_t)tok * a.D + sl * 8) * 2), f);
    else for (int e = 0; e < 8; ++e) f[e] = 0.f;
    const int pos = a.start + t;
    char* row = reinterpret_cast<char*>(a.v_cache) + ((size_t)b * a.cap + pos) * a.v_row_bytes + (size_t)h * hb;
    char* ring = (a.hp_window > 0 && t >= a.n - a.hp_window)
                     ? reinterpret_cast<char*>(a.v_cache) + a.hp_ring_off +
                           ((size_t)b * a.hp_window + pos % a.hp_window) * (size_t)(a.D / 128) * 144 + (size_t)h * 144
                     : nullptr;
    quantize_slice(f, ok, a.bits, row, gq, q, ring);
  }
  pdl_launch_dependents();
}

}  // namespace ptc

// 0 = done on the tensor cores; cudaErrorNotSupported = shape outside the kernel (the
// caller uses cuBLAS); other = launch failure
cudaError_t launch_prefill_tc(const sals_config* c, const void* U, const void* k, int batch, int n, int64_t start,
                              void* latent, int64_t cap, cudaStream_t st) {
  const int D = c->num_kv_heads * c->head_dim, r = c->rank;
  if (c->dtype != SALS_BF16 || D % 64 || r % 64 || n < 1) return cudaErrorNotSupported;
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tma_encoder_fn());
  if (!enc) return cudaErrorNotSupported;
  const cuuint64_t rows = (cuuint64_t)batch * (cuuint64_t)n;
  if (rows > 0x7fffffffull) return cudaErrorNotSupported;
  CUtensorMap tk, tu;
  cuuint64_t dk[2] = {(cuuint64_t)D, rows}, sk[1] = {(cuuint64_t)D * 2};
  cuuint32_t bk[2] = {64, 128}, es[2] = {1, 1};
  cuuint64_t du[2] = {(cuuint64_t)r, (cuuint64_t)D}, su[1] = {(cuuint64_t)r * 2};
  cuuint32_t bu[2] = {64, 64};
  if (enc(&tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(k), dk, sk, bk, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
      enc(&tu, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(U), du, su, bu, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  static DeviceOnce once;
  cudaError_t e = once.run([] {
    return cudaFuncSetAttribute(ptc::prefill_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ptc::kSmem);
  });
  if (e != cudaSuccess) return e;
  ptc::Args a{latent, cap, r, D, n, (int)start};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((n + ptc::kM - 1) / ptc::kM, (r + ptc::kN - 1) / ptc::kN, batch);
  cfg.blockDim = dim3(ptc::kThreads);
  cfg.dynamicSmemBytes = ptc::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, ptc::prefill_tc_kernel, tk, tu, a);
}

cudaError_t launch_prefill_vq(const sals_config* c, const void* v, int batch, int n, int64_t start, void* v_cache,
                              int64_t cap, int v_row_bytes, int hp_window, int64_t hp_ring_off, cudaStream_t st) {
  ptc::VArgs a{v, v_cache, cap, c->num_kv_heads * c->head_dim, n, (int)start, batch, c->v_bits, v_row_bytes,
               hp_window, hp_ring_off};
  const int64_t items = (int64_t)batch * n * (a.D / 8);
  const int grid = (int)std::min<int64_t>((items + 255) / 256, 148 * 16);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(std::max(grid, 1));
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, ptc::prefill_vq_kernel, a);
}

}  // namespace sals
