// Prefill / bulk append: Eq. 1 / Alg. 1 line 3
// applied to a block of n consecutive tokens of every request:
//   latent_cache[b, start + i, :] = U^T k[b, i, :]      (i < n)
//   v_cache[b, start + i, :]      = v[b, i, :]
// The projection is a plain dense GEMM (B*n x D) x (D x r) with no fused
// epilogue, so it runs on cuBLAS (bf16 in, fp32 accumulate, output written
// straight into the cache rows: one strided-batched call, the batch stride is
// the cache's request pitch); the value rows are one 2-D async copy.  Not on
// the decode hot path.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <string>

#include "../../include/sals.h"

namespace {

thread_local cublasHandle_t g_cublas = nullptr;
thread_local std::string g_prefill_err;

}  // namespace

extern "C" const char* sals_prefill_last_error(void) { return g_prefill_err.c_str(); }

// Returns 0 on success; on failure a message is kept for sals_last_error()
// (api.cu maps the code to a sals_status).
extern "C" int sals_prefill_impl(const sals_config* cfg, const void* U, const void* k, const void* v, int32_t batch,
                                 int32_t n_tokens, int64_t start, void* latent_cache, void* v_cache, int64_t cap,
                                 void* stream) {
  const int D = cfg->num_kv_heads * cfg->head_dim, r = cfg->rank;
  const bool bf16 = cfg->dtype == SALS_BF16;
  const size_t es = bf16 ? 2 : 4;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!g_cublas && cublasCreate(&g_cublas) != CUBLAS_STATUS_SUCCESS) {
    g_prefill_err = "cublasCreate failed";
    return 1;
  }
  if (cublasSetStream(g_cublas, st) != CUBLAS_STATUS_SUCCESS) {
    g_prefill_err = "cublasSetStream failed";
    return 1;
  }
  // column-major view: C[r x n] (ld r) = U_cm[r x D] (ld r) * K_b_cm[D x n] (ld D)
  const float alpha = 1.f, beta = 0.f;
  const cudaDataType_t t = bf16 ? CUDA_R_16BF : CUDA_R_32F;
  char* c0 = reinterpret_cast<char*>(latent_cache) + (size_t)start * r * es;
  cublasStatus_t cs = cublasGemmStridedBatchedEx(
      g_cublas, CUBLAS_OP_N, CUBLAS_OP_N, r, n_tokens, D, &alpha, U, t, r, 0, k, t, D, (long long)n_tokens * D,
      &beta, c0, t, r, (long long)cap * r, batch, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
  if (cs != CUBLAS_STATUS_SUCCESS) {
    g_prefill_err = "cublasGemmStridedBatchedEx failed (" + std::to_string((int)cs) + ")";
    return 1;
  }
  cudaError_t e = cudaMemcpy2DAsync(reinterpret_cast<char*>(v_cache) + (size_t)start * D * es, (size_t)cap * D * es,
                                    v, (size_t)n_tokens * D * es, (size_t)n_tokens * D * es, batch,
                                    cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) {
    g_prefill_err = std::string("value rows copy: ") + cudaGetErrorString(e);
    return 1;
  }
  return 0;
}
