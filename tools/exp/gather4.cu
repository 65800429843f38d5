// Experiment: semantics of TMA tile::gather4 box dims (not part of the library).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void k(const __grid_constant__ CUtensorMap map, int r0, int r1, int r2, int r3, unsigned short* out) {
  __shared__ alignas(1024) unsigned short sm[4 * 64 * 4];
  __shared__ alignas(8) uint64_t bar;
  uint32_t sbar = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 1024; ++i) sm[i] = 0xffff;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(512));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                 ::"r"((uint32_t)__cvta_generic_to_shared(sm)), "l"(&map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(sbar) : "memory");
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(sbar));
    for (int i = 0; i < 1024; ++i) out[i] = sm[i];
  }
}

int main() {
  const int R = 64, C = 64;
  std::vector<unsigned short> h(R * C);
  for (int r = 0; r < R; ++r) for (int c = 0; c < C; ++c) h[r * C + c] = (unsigned short)(r * 100 + c);
  unsigned short *d, *o;
  cudaMalloc(&d, h.size() * 2); cudaMalloc(&o, 2048);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  for (int boxr : {1, 4}) {
    for (int sw : {0, 1}) {
      CUtensorMap map;
      cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
      cuuint64_t str[1] = {(cuuint64_t)C * 2};
      cuuint32_t box[2] = {64, (cuuint32_t)boxr};
      cuuint32_t es[2] = {1, 1};
      CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      cudaMemset(o, 0, 2048);
      k<<<1, 32>>>(map, 5, 17, 2, 40, o);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<unsigned short> r(1024);
      cudaMemcpy(r.data(), o, 2048, cudaMemcpyDeviceToHost);
      printf("box rows %d swizzle %d encode %d launch %s\n", boxr, sw, (int)cr, cudaGetErrorString(e));
      for (int row = 0; row < 5; ++row) {
        printf("  smem row %d:", row);
        for (int c = 0; c < 64; c += 8) printf(" %5d", r[row * 64 + c]);
        printf("\n");
      }
      if (e != cudaSuccess) return 0;
    }
  }
  return 0;
}
