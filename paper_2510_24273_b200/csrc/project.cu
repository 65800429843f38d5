// K1 / K2: skinny projections onto the latent basis.
//   append (Alg. 1 lines 2-3; Eq. 1):  k~ = U^T k_new  -> latent_cache[b, pos_b]
//   qproj  (Alg. 1 line 2):           q~ = U[:, :r*]^T q_bar   (fp32)
// plus (qproj launch only) RoPE of the query at position s_b - 1 (Alg. 1 line 7).
//
// Design: U [D, r] is read exactly once.  A thread-block cluster of CS CTAs
// splits the D rows (the contraction axis); each CTA owns 64 output columns
// (32 lanes x 2) and 4 warps that stride over its rows.  Partial sums are
// reduced warp -> CTA in shared memory and CTA -> cluster through DSMEM in a
// fixed order, so the result is deterministic and no global workspace or
// atomic is needed.
#include "common.cuh"
#include "kernels.h"

namespace sals {

constexpr int kProjThreads = 128;
constexpr int kProjCols = 64;     // columns per CTA
constexpr int kProjBT = 8;        // requests per pass
constexpr int kProjMaxRows = 256; // rows per CTA (D / CS)

template <typename T> __device__ __forceinline__ void load2(const T* p, float& a, float& b);
template <> __device__ __forceinline__ void load2<float>(const float* p, float& a, float& b) {
  float2 v = __ldg(reinterpret_cast<const float2*>(p)); a = v.x; b = v.y;
}
template <> __device__ __forceinline__ void load2<__nv_bfloat16>(const __nv_bfloat16* p, float& a, float& b) {
  uint32_t v = __ldg(reinterpret_cast<const unsigned int*>(p));
  a = __uint_as_float(v << 16); b = __uint_as_float(v & 0xffff0000u);
}

template <typename T, bool POOL>
__global__ void __launch_bounds__(kProjThreads)
project_kernel(ProjectArgs a) {
  __shared__ float xs[kProjBT][kProjMaxRows];
  __shared__ float wred[4][kProjBT][kProjCols];
  __shared__ float cred[kProjBT][kProjCols];
  const int CS = (int)cluster_nctarank();
  const int rank = (int)cluster_ctarank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const T* U = reinterpret_cast<const T*>(a.U);
  const T* x = reinterpret_cast<const T*>(a.x);

  pdl_wait();

  if (POOL && blockIdx.y == gridDim.y - 1) {
    // ---- role 2: RoPE of the query heads at position s_b - 1 (fp32 out) ----
    const int half = a.rope.half, d = 2 * half;
    const int nq = a.n_q;
    for (int b = rank; b < a.B; b += CS) {
      const int64_t pos = (int64_t)a.seq_len[b] - 1;
      for (int t = tid; t < half * nq; t += kProjThreads) {
        const int p = t % half, h = t / half;
        int lo, hi; rope_pair(p, half, a.rope.style, lo, hi);
        float c, s; rope_cs(a.rope.theta[p], pos, c, s);
        const float xl = Elem<T>::to_f(x[(size_t)b * a.x_stride + h * d + lo]);
        const float xh = Elem<T>::to_f(x[(size_t)b * a.x_stride + h * d + hi]);
        a.qrope[((size_t)b * nq + h) * d + lo] = xl * c - xh * s;
        a.qrope[((size_t)b * nq + h) * d + hi] = xl * s + xh * c;
      }
    }
    pdl_launch_dependents();
    return;
  }

  if (!POOL && a.v_new != nullptr) {
    // ---- append: copy v_new[b] -> v_cache[b, pos_b] (16-byte vectors) ----
    const int nvec = a.D * (int)sizeof(T) / 16;
    const int ncta = CS * gridDim.y;
    const int cta = blockIdx.y * CS + rank;
    for (int i = cta * kProjThreads + tid; i < a.B * nvec; i += ncta * kProjThreads) {
      const int b = i / nvec, v = i % nvec;
      const uint4 val = ld_v4(reinterpret_cast<const char*>(a.v_new) + ((size_t)b * a.D) * sizeof(T) + v * 16);
      *reinterpret_cast<uint4*>(reinterpret_cast<char*>(a.v_cache) +
                                (((size_t)b * a.cap + a.pos[b]) * a.D) * sizeof(T) + v * 16) = val;
    }
  }

  const int rows_per = a.rows_per_cta;
  const int row0 = rank * rows_per;
  const int row1 = min(a.D, row0 + rows_per);
  const int col = blockIdx.y * kProjCols + 2 * lane;
  const bool col_ok = col < a.ncols;

  for (int b0 = 0; b0 < a.B; b0 += kProjBT) {
    const int nb = min(kProjBT, a.B - b0);
    // stage x (pooled over the query heads of each KV group for qproj)
    for (int i = tid; i < kProjBT * rows_per; i += kProjThreads) {
      const int bb = i / rows_per, c = row0 + i % rows_per;
      float v = 0.f;
      if (bb < nb && c < row1) {
        const T* xb = x + (size_t)(b0 + bb) * a.x_stride;
        if (POOL) {
          const int g = c / a.head_dim, j = c % a.head_dim;
          for (int hh = 0; hh < a.group; ++hh) v += Elem<T>::to_f(xb[(g * a.group + hh) * a.head_dim + j]);
        } else {
          v = Elem<T>::to_f(xb[c]);
        }
      }
      xs[bb][i % rows_per] = v;
    }
    __syncthreads();

    float acc[kProjBT][2];
#pragma unroll
    for (int bb = 0; bb < kProjBT; ++bb) acc[bb][0] = acc[bb][1] = 0.f;
    if (col_ok) {
      int c = row0 + warp;
#pragma unroll 1
      for (; c + 12 < row1; c += 16) {
        float u[4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q) load2<T>(U + (size_t)(c + 4 * q) * a.r + col, u[q][0], u[q][1]);
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int bb = 0; bb < kProjBT; ++bb) {
            const float xv = xs[bb][c + 4 * q - row0];
            acc[bb][0] = fmaf(u[q][0], xv, acc[bb][0]);
            acc[bb][1] = fmaf(u[q][1], xv, acc[bb][1]);
          }
      }
      for (; c < row1; c += 4) {
        float u0, u1; load2<T>(U + (size_t)c * a.r + col, u0, u1);
#pragma unroll
        for (int bb = 0; bb < kProjBT; ++bb) {
          const float xv = xs[bb][c - row0];
          acc[bb][0] = fmaf(u0, xv, acc[bb][0]);
          acc[bb][1] = fmaf(u1, xv, acc[bb][1]);
        }
      }
    }
#pragma unroll
    for (int bb = 0; bb < kProjBT; ++bb) {
      wred[warp][bb][2 * lane] = acc[bb][0];
      wred[warp][bb][2 * lane + 1] = acc[bb][1];
    }
    __syncthreads();
    for (int i = tid; i < kProjBT * kProjCols; i += kProjThreads) {
      const int bb = i / kProjCols, j = i % kProjCols;
      cred[bb][j] = ((wred[0][bb][j] + wred[1][bb][j]) + wred[2][bb][j]) + wred[3][bb][j];
    }
    cluster_sync_all();
    // each rank reduces a 1/CS share of the outputs over ranks 0..CS-1 (fixed order)
    const int nout = nb * kProjCols;
    const int share = (nout + CS - 1) / CS;
    const uint32_t cred_addr = smem_u32(&cred[0][0]);
    for (int o = rank * share + tid; o < min(nout, (rank + 1) * share); o += kProjThreads) {
      const int bb = o / kProjCols, j = o % kProjCols;
      const int cj = blockIdx.y * kProjCols + j;
      float sum = 0.f;
      for (int c = 0; c < CS; ++c) sum += ld_dsmem_f32(mapa_shared(cred_addr + o * 4, c));
      if (cj < a.ncols) {
        const int b = b0 + bb;
        if (POOL) {
          a.out_f32[(size_t)b * a.ncols + cj] = sum;
        } else {
          T* lat = reinterpret_cast<T*>(a.latent);
          lat[((size_t)b * a.cap + a.pos[b]) * a.r + cj] = Elem<T>::from_f(sum);
        }
      }
    }
    cluster_sync_all();
  }
  pdl_launch_dependents();
}

template __global__ void project_kernel<float, false>(ProjectArgs);
template __global__ void project_kernel<float, true>(ProjectArgs);
template __global__ void project_kernel<__nv_bfloat16, false>(ProjectArgs);
template __global__ void project_kernel<__nv_bfloat16, true>(ProjectArgs);

}  // namespace sals
