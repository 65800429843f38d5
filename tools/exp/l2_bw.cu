// Microbenchmark: L2 -> SM bandwidth on sm_100a with cp.async.bulk (the path the
// fused kernel's U / latent operands take).  Every CTA (one per SM) streams
// ITER chunks of CHUNK bytes from an L2-resident buffer of BUF bytes into a
// 4-stage shared-memory ring (mbarrier complete_tx), a second kernel reads
// scattered 1 KB rows (gather-like) the same way.  Reports chip GB/s and B/clk.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o l2_bw.bin l2_bw.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

#ifndef STAGES
#define STAGES 4
#endif
constexpr int kStages = STAGES;

// ROW = bytes per bulk copy; CHUNK = bytes per stage (CHUNK / ROW copies per stage)
template <int ROW>
__global__ void stream_kernel(const char* buf, size_t buf_bytes, int chunk, int iters, unsigned long long* cyc,
                              const int* perm) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[kStages];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nrows = chunk / ROW;
  const size_t nbuf_rows = buf_bytes / ROW;
  unsigned long long t0 = clock64();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int it = 0; it < iters + kStages; ++it) {
      const int s = it % kStages;
      if (it >= kStages) mbar_wait(&full[s], ((it / kStages) - 1) & 1);   // consume stage (it - kStages)
      if (it < iters) {
        if (lane == 0) mbar_expect(&full[s], chunk);
        __syncwarp();
        for (int r = lane; r < nrows; r += 32) {
          const size_t g = ((size_t)blockIdx.x * 7919 + (size_t)it * nrows + r);
          const size_t row = perm ? (size_t)perm[g % 65536] % nbuf_rows : g % nbuf_rows;
          bulk_load(smem_u32(smem + s * chunk + r * ROW), buf + row * ROW, ROW, &full[s]);
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const size_t big = 1ull << 30;
  char* buf;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 1, big);
  int* perm;
  cudaMalloc(&perm, 65536 * 4);
  {
    int* h = new int[65536];
    uint32_t x = 12345;
    for (int i = 0; i < 65536; ++i) { x = x * 1664525u + 1013904223u; h[i] = (int)(x >> 4); }
    cudaMemcpy(perm, h, 65536 * 4, cudaMemcpyHostToDevice);
    delete[] h;
  }
  unsigned long long* cyc;
  cudaMalloc(&cyc, nsm * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("SMs %d, clock %d MHz\n", nsm, clk_khz / 1000);
  struct Case { const char* name; size_t buf; int chunk; int row; bool scatter; int grid; };
  const Case cases[] = {
      {"seq 4MB chunk16K", 4u << 20, 16384, 16384, false, nsm},
      {"seq 4MB chunk32K", 4u << 20, 32768, 32768, false, nsm},
      {"seq 4MB chunk16K 2/SM", 4u << 20, 16384, 16384, false, 2 * nsm},
      {"seq 4MB chunk16K grid64", 4u << 20, 16384, 16384, false, 64},
      {"rows1K L2 16MB chunk16K", 16u << 20, 16384, 1024, true, nsm},
      {"rows1K HBM 1GB chunk16K", big, 16384, 1024, true, nsm},
      {"seq HBM 1GB chunk16K", big, 16384, 16384, false, nsm},
  };
  for (const Case& c : cases) {
    const int iters = c.buf >= big ? 200 : 2000;
    const size_t smem = (size_t)kStages * c.chunk;
    void (*k)(const char*, size_t, int, int, unsigned long long*, const int*) =
        c.row == 1024 ? stream_kernel<1024> : (c.row == 512 ? stream_kernel<512> : stream_kernel<16384>);
    int row = c.row;
    if (c.row >= 16384) k = stream_kernel<16384>, row = 16384;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k<<<c.grid, 64, smem>>>(buf, c.buf, c.chunk, iters, cyc, c.scatter ? perm : nullptr);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)c.grid * iters * c.chunk;
    const double gbs = bytes / (ms * 1e-3) / 1e9;
    printf("%-28s err=%d  %8.1f GB/s  %6.1f B/clk/chip (at %d MHz)  %5.1f B/clk/SM  (row %d)\n", c.name,
           (int)cudaGetLastError(), gbs, gbs * 1e9 / (clk_khz * 1e3), clk_khz / 1000,
           gbs * 1e9 / (clk_khz * 1e3) / c.grid, row);
  }
  return 0;
}
