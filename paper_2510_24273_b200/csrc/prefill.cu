// Prefill / bulk append: Eq. 1 / Alg. 1 line 3
// applied to a block of n consecutive tokens of every request:
//   latent_cache[b, start + i, :] = U^T k[b, i, :]      (i < n)
//   v_cache[b, start + i, :]      = v[b, i, :]
// bf16 with D, r multiples of 64 runs on the in-build tcgen05 GEMM
// (prefill_tc.cu); this file is the fallback for the other shapes / fp32: a
// cuBLAS strided-batched GEMM (fp32 accumulate, written straight into the cache
// rows, the batch stride is the cache's request pitch) and the dtype value rows
// as one 2-D async copy.  Not on the decode hot path.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <string>
#include <unordered_map>

#include "../../include/sals.h"

namespace {

// library handles per (calling thread, device): a handle is bound to the device
// that was current when it was created
thread_local std::unordered_map<int, cublasHandle_t> g_cublas;
thread_local std::string g_prefill_err;

cublasHandle_t cublas_handle() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  auto it = g_cublas.find(dev);
  if (it != g_cublas.end()) return it->second;
  cublasHandle_t h = nullptr;
  if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return nullptr;
  g_cublas[dev] = h;
  return h;
}

}  // namespace

extern "C" const char* sals_prefill_last_error(void) { return g_prefill_err.c_str(); }

// Returns 0 on success; on failure a message is kept for sals_last_error()
// (api.cu maps the code to a sals_status).
extern "C" int sals_prefill_impl(const sals_config* cfg, const void* U, const void* k, const void* v, int32_t batch,
                                 int32_t n_tokens, int64_t start, void* latent_cache, void* v_cache, int64_t cap,
                                 void* stream, int do_latent, int do_v) {
  const int D = cfg->num_kv_heads * cfg->head_dim, r = cfg->rank;
  const bool bf16 = cfg->dtype == SALS_BF16;
  const size_t es = bf16 ? 2 : 4;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (do_latent) {
  cublasHandle_t hb = cublas_handle();
  if (!hb) {
    g_prefill_err = "cublasCreate failed";
    return 1;
  }
  if (cublasSetStream(hb, st) != CUBLAS_STATUS_SUCCESS) {
    g_prefill_err = "cublasSetStream failed";
    return 1;
  }
  // column-major view: C[r x n] (ld r) = U_cm[r x D] (ld r) * K_b_cm[D x n] (ld D)
  const float alpha = 1.f, beta = 0.f;
  const cudaDataType_t t = bf16 ? CUDA_R_16BF : CUDA_R_32F;
  char* c0 = reinterpret_cast<char*>(latent_cache) + (size_t)start * r * es;
  cublasStatus_t cs = cublasGemmStridedBatchedEx(
      hb, CUBLAS_OP_N, CUBLAS_OP_N, r, n_tokens, D, &alpha, U, t, r, 0, k, t, D, (long long)n_tokens * D,
      &beta, c0, t, r, (long long)cap * r, batch, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
  if (cs != CUBLAS_STATUS_SUCCESS) {
    g_prefill_err = "cublasGemmStridedBatchedEx failed (" + std::to_string((int)cs) + ")";
    return 1;
  }
  }
  if (!do_v) return 0;
  cudaError_t e = cudaMemcpy2DAsync(reinterpret_cast<char*>(v_cache) + (size_t)start * D * es, (size_t)cap * D * es,
                                    v, (size_t)n_tokens * D * es, (size_t)n_tokens * D * es, batch,
                                    cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) {
    g_prefill_err = std::string("value rows copy: ") + cudaGetErrorString(e);
    return 1;
  }
  return 0;
}

// ---------------------------------------------------------------------------
// Offline calibration (§4.2): C = K^T K over the
// stacked pre-RoPE calibration keys K [N, D], eigen-decomposition C = U S U^T,
// U_r = the leading r eigenvectors (descending eigenvalue order, which is what
// makes the first r* columns the score subspace).  Library primitives: the
// Gram matrix on cuBLAS (fp32 accumulate), the symmetric eigensolver on
// cuSOLVER (syevd, fp32); one kernel reorders / sign-normalises the columns
// (the largest-magnitude component of each column is made positive, first such
// index on ties) and converts to the storage type.
#include <cusolverDn.h>
#include <cuda_bf16.h>

namespace {
thread_local std::unordered_map<int, cusolverDnHandle_t> g_cusolver_by_dev;
thread_local cusolverDnHandle_t g_cusolver = nullptr;   // the calling thread's handle for the current device
thread_local cublasHandle_t g_cublas_cur = nullptr;

__global__ void calib_columns_kernel(const float* __restrict__ evec, const float* __restrict__ w, int D, int r,
                                     void* U_out, int bf16, float* eig_out) {
  const int j = blockIdx.x;                 // output column: eigenvector of the j-th largest eigenvalue
  const float* col = evec + (size_t)(D - 1 - j) * D;
  __shared__ float s_v[32];
  __shared__ int s_i[32];
  float best = -1.f;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    const float a = fabsf(col[i]);
    if (a > best || (a == best && i < bi)) { best = a; bi = i; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { s_v[warp] = best; s_i[warp] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (s_v[k] > s_v[0] || (s_v[k] == s_v[0] && s_i[k] < s_i[0])) { s_v[0] = s_v[k]; s_i[0] = s_i[k]; }
  }
  if (eig_out)   // all D eigenvalues, descending (block j writes j, j + r, ...)
    for (int i = j + (int)threadIdx.x * (int)gridDim.x; i < D; i += (int)(blockDim.x * gridDim.x)) eig_out[i] = w[D - 1 - i];
  __syncthreads();
  const float sgn = col[s_i[0]] < 0.f ? -1.f : 1.f;
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    const float v = sgn * col[i];
    if (bf16) reinterpret_cast<__nv_bfloat16*>(U_out)[(size_t)i * r + j] = __float2bfloat16_rn(v);
    else reinterpret_cast<float*>(U_out)[(size_t)i * r + j] = v;
  }
}

bool calib_handles(cudaStream_t st) {
  g_cublas_cur = cublas_handle();
  if (!g_cublas_cur) { g_prefill_err = "cublasCreate failed"; return false; }
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { g_prefill_err = "cudaGetDevice failed"; return false; }
  auto it = g_cusolver_by_dev.find(dev);
  if (it == g_cusolver_by_dev.end()) {
    cusolverDnHandle_t h = nullptr;
    if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS) {
      g_prefill_err = "cusolverDnCreate failed";
      return false;
    }
    it = g_cusolver_by_dev.emplace(dev, h).first;
  }
  g_cusolver = it->second;
  cublasSetStream(g_cublas_cur, st);
  cusolverDnSetStream(g_cusolver, st);
  return true;
}

size_t align256(size_t v) { return (v + 255) / 256 * 256; }
}  // namespace

extern "C" size_t sals_calibrate_ws_impl(int D) {
  if (!calib_handles(0)) return 0;
  int lwork = 0;
  if (cusolverDnSsyevd_bufferSize(g_cusolver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, D, nullptr, D,
                                  nullptr, &lwork) != CUSOLVER_STATUS_SUCCESS)
    return 0;
  return align256((size_t)D * D * 4) + align256((size_t)D * 4) + align256(4) + align256((size_t)lwork * 4);
}

extern "C" int sals_calibrate_impl(const sals_config* cfg, const void* K, int64_t n_rows, void* U_out,
                                   float* eig_out, void* workspace, size_t ws_bytes, void* stream) {
  const int D = cfg->num_kv_heads * cfg->head_dim, r = cfg->rank;
  const bool bf16 = cfg->dtype == SALS_BF16;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!calib_handles(st)) return 1;
  int lwork = 0;
  if (cusolverDnSsyevd_bufferSize(g_cusolver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, D, nullptr, D,
                                  nullptr, &lwork) != CUSOLVER_STATUS_SUCCESS) {
    g_prefill_err = "syevd buffer size query failed";
    return 1;
  }
  char* ws = reinterpret_cast<char*>(workspace);
  float* C = reinterpret_cast<float*>(ws);
  float* W = reinterpret_cast<float*>(ws + align256((size_t)D * D * 4));
  int* info = reinterpret_cast<int*>(ws + align256((size_t)D * D * 4) + align256((size_t)D * 4));
  float* work = reinterpret_cast<float*>(ws + align256((size_t)D * D * 4) + align256((size_t)D * 4) + align256(4));
  if (ws_bytes < align256((size_t)D * D * 4) + align256((size_t)D * 4) + align256(4) + align256((size_t)lwork * 4)) {
    g_prefill_err = "calibration workspace too small";
    return 3;
  }
  // C (col-major D x D) = K_cm (D x N, ld D) * K_cm^T
  const float one = 1.f, zero = 0.f;
  const cudaDataType_t t = bf16 ? CUDA_R_16BF : CUDA_R_32F;
  if (cublasGemmEx(g_cublas_cur, CUBLAS_OP_N, CUBLAS_OP_T, D, D, (int)n_rows, &one, K, t, D, K, t, D, &zero, C,
                   CUDA_R_32F, D, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT) != CUBLAS_STATUS_SUCCESS) {
    g_prefill_err = "Gram matrix GEMM failed";
    return 1;
  }
  if (cusolverDnSsyevd(g_cusolver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, D, C, D, W, work, lwork,
                       info) != CUSOLVER_STATUS_SUCCESS) {
    g_prefill_err = "syevd failed";
    return 1;
  }
  calib_columns_kernel<<<r, 256, 0, st>>>(C, W, D, r, U_out, bf16 ? 1 : 0, eig_out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { g_prefill_err = cudaGetErrorString(e); return 1; }
  return 0;
}
