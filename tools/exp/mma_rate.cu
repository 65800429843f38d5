// Microbenchmark: tcgen05.mma (kind::f16, bf16 in / fp32 accumulate, both operands
// from shared memory, SWIZZLE_128B K-major) issue rate on sm_100a, per CTA shape,
// with and without competing shared-memory traffic from other warps.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_rate mma_rate.cu
//
// Every CTA (one per SM: ~200 KB of dynamic smem) issues NITER K=16 MMAs on the
// same operand tiles into one TMEM accumulator, commits once, waits.  Reported:
// cycles per MMA (clock64 of the issuing thread, median over CTAs) against the
// floor max(M,128) * N / (256 * cta_group) of B300_MICROARCH.md, and the chip's
// TFLOP/s from CUDA events.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <int CG, int M, int N, int NOISE>
__global__ void __launch_bounds__(256, 1) mma_kernel(int niter, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // A: 128 rows x 64 K (16 KB) per CTA; B: N/CG rows x 64 K per CTA
  uint8_t* sA = smem;
  uint8_t* sB = smem + 16384;
  uint8_t* sNoise = smem + 16384 + 32768;   // 64 KB scribbled by the noise warps
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (16384 + 32768) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                   "r"(256));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                   "r"(256));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (CG == 2) cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  const bool leader = CG == 1 || cluster_ctarank() == 0;
  constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  volatile uint32_t stop = 0;
  if (warp == 1 && lane == 0 && leader) {
    const uint32_t ab = smem_u32(sA), bb = smem_u32(sB);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < niter; ++i) {
      const int k = i & 3;
      const uint64_t ad = sw128_desc(ab + k * 32), bd = sw128_desc(bb + k * 32);
      if (CG == 1)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)(i > 0))
            : "memory");
      else
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)(i > 0))
            : "memory");
    }
    if (CG == 1)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                   : "memory");
    else
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(&bar)),
          "h"((uint16_t)3)
          : "memory");
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  } else if (NOISE && warp >= 4) {
    // competing shared-memory traffic: 16-byte stores + loads over 64 KB
    uint4* p = reinterpret_cast<uint4*>(sNoise);
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (int it = 0; it < niter / 4; ++it) {
      for (int j = 0; j < 8; ++j) {
        const int idx = ((it * 8 + j) * 128 + (warp - 4) * 32 + lane) & 4095;
        if (NOISE == 1) p[idx] = make_uint4(it, j, lane, warp);
        else { const uint4 v = p[idx]; acc.x ^= v.x; acc.y += v.y; }
      }
    }
    if (acc.x == 0xdeadbeef) cyc[0] = acc.y;
  }
  if (!leader && warp == 1 && lane == 0) mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (CG == 2) cluster_sync();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
  (void)stop;
}

template <int CG, int M, int N, int NOISE>
void run(const char* name, int nsm) {
  const int niter = 8192;
  auto k = mma_kernel<CG, M, N, NOISE>;
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* d;
  cudaMalloc(&d, nsm * sizeof(unsigned long long));
  cudaMemset(d, 0, nsm * sizeof(unsigned long long));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nsm);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) cudaLaunchKernelEx(&cfg, k, niter, d);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int w = 0; w < reps; ++w) cudaLaunchKernelEx(&cfg, k, niter, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> h(nsm);
  cudaMemcpy(h.data(), d, nsm * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  std::vector<unsigned long long> v;
  for (int i = 0; i < nsm; ++i)
    if (h[i]) v.push_back(h[i]);
  std::sort(v.begin(), v.end());
  const double med = v.empty() ? 0 : (double)v[v.size() / 2] / niter;
  const double flop = 2.0 * M * N * 16 * niter * (nsm / CG) * reps;
  const double floor_cyc = (double)std::max(M, 128) * N / (256.0 * CG);
  printf("%-28s err=%d  cycles/MMA %.1f (floor %.0f, %.0f%%)  chip %.0f TFLOP/s  (%.3f ms/launch)\n", name, (int)err,
         med, floor_cyc, 100.0 * floor_cyc / med, flop / (ms * 1e-3) / 1e12, ms / reps);
  cudaFree(d);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", nsm);
  run<1, 128, 256, 0>("cg1 M128 N256", nsm);
  run<1, 128, 128, 0>("cg1 M128 N128", nsm);
  run<1, 128, 64, 0>("cg1 M128 N64", nsm);
  run<1, 128, 256, 1>("cg1 M128 N256 +st.shared", nsm);
  run<1, 128, 256, 2>("cg1 M128 N256 +ld.shared", nsm);
  run<2, 256, 256, 0>("cg2 M256 N256", nsm);
  run<2, 256, 128, 0>("cg2 M256 N128", nsm);
  run<2, 256, 256, 1>("cg2 M256 N256 +st.shared", nsm);
  run<2, 256, 256, 2>("cg2 M256 N256 +ld.shared", nsm);
  return 0;
}
