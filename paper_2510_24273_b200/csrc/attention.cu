// SIMT kernels of the reconstruction / attention stages (path S) and of the
// dense comparator:
//   recon_rope_simt_kernel  K_C = K~_C U^T then K^R_C = RoPE_j(K_C)   (Alg. 1 lines 6-7)
//   flash_decode_kernel     split-K online-softmax attention over a token list
//                           (Alg. 1 lines 8-9 / Eq. 6; also the dense flash decode)
//   merge_kernel            log-sum-exp merge of the split partials -> y
//   dense_append_kernel     post-RoPE dense cache write (comparator)
#include "common.cuh"
#include "kernels.h"

namespace sals {

// ---------------------------------------------------------------------------
// Reconstruct + RoPE, one (32-row tile, KV head) per CTA.  fp32 FMA GEMM with
// shared-memory tiles; the rows of A are gathered latent rows.
// ---------------------------------------------------------------------------
constexpr int kRcRows = 32, kRcK = 32, kRcThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kRcThreads)
recon_rope_simt_kernel(ReconArgs a) {
  extern __shared__ float rc_smem[];
  const int DH = a.head_dim;
  float* As = rc_smem;                          // [32][33]
  float* Bs = As + kRcRows * (kRcK + 1);        // [DH][33]
  float* Ks = Bs + DH * (kRcK + 1);             // [32][DH]
  __shared__ int rows[kRcRows];
  __shared__ float2 sth[128];   // per-lane indexed: keep the angle table out of param space
  const int b = blockIdx.z, g = blockIdx.y, t0 = blockIdx.x * kRcRows;
  const int tid = threadIdx.x;
  const T* lat = reinterpret_cast<const T*>(a.latent);
  const T* U = reinterpret_cast<const T*>(a.U);
  for (int i = tid; i < a.head_dim / 2; i += kRcThreads) sth[i] = make_float2(a.rope.th_hi[i], a.rope.th_lo[i]);
  __syncthreads();

  pdl_wait();
  const int cnt = a.count[b];
  if (t0 >= cnt) { pdl_launch_dependents(); return; }
  if (tid < kRcRows) rows[tid] = (t0 + tid < cnt) ? a.sel[(size_t)b * a.k_stride + t0 + tid] : -1;
  __syncthreads();

  const int nout = kRcRows * DH / kRcThreads;   // outputs per thread (DH >= 8)
  float acc[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) acc[j] = 0.f;

  for (int k0 = 0; k0 < a.r; k0 += kRcK) {
    for (int i = tid; i < kRcRows * kRcK; i += kRcThreads) {
      const int rr = i / kRcK, kk = i % kRcK;
      const int row = rows[rr];
      As[rr * (kRcK + 1) + kk] = (row >= 0 && k0 + kk < a.r)
          ? Elem<T>::to_f(lat[((size_t)b * a.cap + row) * a.r + k0 + kk]) : 0.f;
    }
    for (int i = tid; i < DH * kRcK; i += kRcThreads) {
      const int nn = i / kRcK, kk = i % kRcK;
      Bs[nn * (kRcK + 1) + kk] = (k0 + kk < a.r) ? Elem<T>::to_f(U[(size_t)(g * DH + nn) * a.r + k0 + kk]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (j < nout) {
        const int o = tid + j * kRcThreads, rr = o / DH, nn = o % DH;
        float s = acc[j];
#pragma unroll 8
        for (int kk = 0; kk < kRcK; ++kk) s = fmaf(As[rr * (kRcK + 1) + kk], Bs[nn * (kRcK + 1) + kk], s);
        acc[j] = s;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < 32; ++j)
    if (j < nout) Ks[tid + j * kRcThreads] = acc[j];
  __syncthreads();
  // RoPE at the original position of each row, then store K^R_C
  const int half = DH / 2;
  T* kr = reinterpret_cast<T*>(a.kr);
  for (int i = tid; i < kRcRows * half; i += kRcThreads) {
    const int rr = i / half, p = i % half;
    const int row = rows[rr];
    if (row < 0) continue;
    int lo, hi; rope_pair(p, half, a.rope.style, lo, hi);
    float c, s; rope_cs_fast(sth[p].x, sth[p].y, (int)(a.pos_base + row), c, s);
    const float xl = Ks[rr * DH + lo], xh = Ks[rr * DH + hi];
    T* dst = kr + ((size_t)b * a.k_stride + t0 + rr) * a.D + g * DH;
    dst[lo] = Elem<T>::from_f(xl * c - xh * s);
    dst[hi] = Elem<T>::from_f(xl * s + xh * c);
  }
  pdl_launch_dependents();
}

template __global__ void recon_rope_simt_kernel<float>(ReconArgs);
template __global__ void recon_rope_simt_kernel<__nv_bfloat16>(ReconArgs);

// ---------------------------------------------------------------------------
// Flash decode over a token list.  One warp per (request, KV head, split);
// the warps of a CTA are CONSECUTIVE KV heads of one split (blockDim = 32 x heads
// per CTA), so together they stream whole contiguous K / V row segments (up to 8
// heads = 2 KB per token at d = 128) instead of 256-byte slivers of rows 2-8 KB
// apart (with the software pipelining below: 0.56 / 0.42 / 0.39 -> 0.62 / 0.46 / 0.41 of
// the measured HBM peak at c2 / c3 / c4).
// LPT lanes cover one token row of one head with 16-byte loads, TPW tokens per
// warp step.  Each lane holds the rotated query of all G heads of the group
// for its EPL dims (so a K/V row load serves G query heads, GQA-aware).
// Logits are in the log2 domain (q pre-scaled by scale * log2 e).
// ---------------------------------------------------------------------------
constexpr int kFdWarps = 8;   // max warps (= KV heads) per CTA

template <typename T, int DH, int G, bool DENSE>
__global__ void __launch_bounds__(kFdWarps * 32, G >= 8 ? 1 : 2)   // G <= 4: <= 128 registers, two CTAs per SM
flash_decode_kernel(FlashArgs a) {
  constexpr int EPL = Elem<T>::kPer16;
  constexpr int LPT = DH / EPL;            // lanes per token row
  static_assert(LPT >= 1 && LPT <= 32, "head row must fit one warp");
  constexpr int TPW = 32 / LPT;            // tokens per warp step
  constexpr int UNR = G <= 2 ? 4 : 2;   // K/V rows per lane-group per step (x2 in flight: pipelined)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / LPT, li = lane % LPT;
  const int hpc = blockDim.x >> 5;                 // KV heads per CTA
  const int b = blockIdx.z, g = blockIdx.y * hpc + warp;
  const int split = blockIdx.x;

  pdl_wait();
  if (split >= a.nsplit) return;
  const int cnt = a.count[b];
  const int t0 = split * a.chunk;
  const int t1 = min(cnt, t0 + a.chunk);

  float q[G][EPL];
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int e = 0; e < EPL; ++e)
      q[h][e] = a.qrope[((size_t)b * a.n_q + g * G + h) * DH + li * EPL + e] * a.scale_log2;
  float m[G], l[G], o[G][EPL];
#pragma unroll
  for (int h = 0; h < G; ++h) {
    m[h] = -INFINITY; l[h] = 0.f;
#pragma unroll
    for (int e = 0; e < EPL; ++e) o[h][e] = 0.f;
  }
  const char* kb = reinterpret_cast<const char*>(a.kbase);
  const char* vb = reinterpret_cast<const char*>(a.v_cache);
  const size_t rowb = (size_t)a.D * sizeof(T);
  const size_t headoff = (size_t)g * DH * sizeof(T) + li * 16;

  // software-pipelined: the K / V rows of step i+1 are in flight while step i is reduced
  auto load_step = [&](int tb, uint4* kr, uint4* vr, bool* ok) {
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int t = tb + u * TPW + sub;
      ok[u] = t < t1;
      if (ok[u]) {
        size_t krow, vrow;
        if (DENSE) {
          krow = vrow = (size_t)b * a.cap + t;
        } else {
          krow = (size_t)b * a.k_stride + t;
          vrow = (size_t)b * a.cap + a.sel[(size_t)b * a.k_stride + t];
        }
        kr[u] = ld_nc_v4(kb + krow * rowb + headoff);
        vr[u] = ld_nc_v4(vb + vrow * rowb + headoff);
      } else {
        kr[u] = vr[u] = make_uint4(0, 0, 0, 0);
      }
    }
  };
  uint4 kr[UNR], vr[UNR];
  bool ok[UNR];
  load_step(t0, kr, vr, ok);
  for (int tb = t0; tb < t1; tb += TPW * UNR) {
    uint4 kn[UNR], vn[UNR];
    bool okn[UNR];
    load_step(tb + TPW * UNR, kn, vn, okn);   // (all !ok past t1: no loads)
    // logits of the UNR tokens first, then ONE online-softmax update per head
    // (a single max / rescale per step instead of a serial chain per token)
    float sc[UNR][G];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      float kf[EPL];
      Elem<T>::unpack(kr[u], kf);
#pragma unroll
      for (int h = 0; h < G; ++h) {
        float s = 0.f;
#pragma unroll
        for (int e = 0; e < EPL; ++e) s = fmaf(q[h][e], kf[e], s);
#pragma unroll
        for (int off = LPT / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        sc[u][h] = ok[u] ? s : -INFINITY;
      }
    }
#pragma unroll
    for (int h = 0; h < G; ++h) {
      float mx = m[h];
#pragma unroll
      for (int u = 0; u < UNR; ++u) mx = fmaxf(mx, sc[u][h]);
      if (mx == -INFINITY) continue;               // nothing valid yet for this lane group
      const float corr = exp2f(m[h] - mx);         // m = -inf -> 0
      l[h] *= corr;
#pragma unroll
      for (int e = 0; e < EPL; ++e) o[h][e] *= corr;
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const float p = exp2f(sc[u][h] - mx);      // -inf (invalid token) -> 0
        float vf[EPL];
        Elem<T>::unpack(vr[u], vf);
        l[h] += p;
#pragma unroll
        for (int e = 0; e < EPL; ++e) o[h][e] = fmaf(p, vf[e], o[h][e]);
      }
      m[h] = mx;
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) { kr[u] = kn[u]; vr[u] = vn[u]; ok[u] = okn[u]; }
  }
  // merge the TPW token groups of the warp
#pragma unroll
  for (int off = LPT; off < 32; off <<= 1) {
#pragma unroll
    for (int h = 0; h < G; ++h) {
      const float mo = __shfl_xor_sync(0xffffffffu, m[h], off);
      const float lo = __shfl_xor_sync(0xffffffffu, l[h], off);
      const float mn = fmaxf(m[h], mo);
      const float c1 = (m[h] == -INFINITY) ? 0.f : exp2f(m[h] - mn);
      const float c2 = (mo == -INFINITY) ? 0.f : exp2f(mo - mn);
      l[h] = l[h] * c1 + lo * c2;
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        const float oo = __shfl_xor_sync(0xffffffffu, o[h][e], off);
        o[h][e] = o[h][e] * c1 + oo * c2;
      }
      m[h] = mn;
    }
  }
  if (sub == 0) {
#pragma unroll
    for (int h = 0; h < G; ++h) {
      float* dst = a.partials + (((size_t)b * a.n_q + g * G + h) * a.nsplit + split) * (DH + 2);
      if (li == 0) { dst[0] = m[h]; dst[1] = l[h]; }
#pragma unroll
      for (int e = 0; e < EPL; ++e) dst[2 + li * EPL + e] = o[h][e];
    }
  }
  pdl_launch_dependents();
}

#define SALS_FD_INST(T, DH)                                                  \
  template __global__ void flash_decode_kernel<T, DH, 1, false>(FlashArgs);  \
  template __global__ void flash_decode_kernel<T, DH, 2, false>(FlashArgs);  \
  template __global__ void flash_decode_kernel<T, DH, 4, false>(FlashArgs);  \
  template __global__ void flash_decode_kernel<T, DH, 8, false>(FlashArgs);  \
  template __global__ void flash_decode_kernel<T, DH, 1, true>(FlashArgs);   \
  template __global__ void flash_decode_kernel<T, DH, 2, true>(FlashArgs);   \
  template __global__ void flash_decode_kernel<T, DH, 4, true>(FlashArgs);   \
  template __global__ void flash_decode_kernel<T, DH, 8, true>(FlashArgs);
SALS_FD_INST(float, 16)
SALS_FD_INST(float, 32)
SALS_FD_INST(float, 64)
SALS_FD_INST(float, 128)
SALS_FD_INST(__nv_bfloat16, 16)
SALS_FD_INST(__nv_bfloat16, 32)
SALS_FD_INST(__nv_bfloat16, 64)
SALS_FD_INST(__nv_bfloat16, 128)
SALS_FD_INST(__nv_bfloat16, 256)

// ---------------------------------------------------------------------------
// LSE merge: y_h = sum_s o_s 2^(m_s - M) / sum_s l_s 2^(m_s - M)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void merge_kernel(MergeArgs a) {
  const int bh = blockIdx.x;
  const int b = bh / a.n_q, h = bh % a.n_q;
  pdl_wait();
  pdl_launch_dependents();   // the next kernels' pre-wait prologues only read weights / their own inputs
  const float* base = a.partials + (size_t)bh * a.bh_stride;
  constexpr int kMaxS = 512;
  __shared__ float sw[kMaxS], sl[kMaxS];
  __shared__ float s_M, s_L;
  if (a.nsplit <= kMaxS) {
    // (1) all (m, l) in one round of loads, (2) max and weights by warp 0,
    // (3) y = sum_s w_s o_s with independent loads -- two dependent L2 round trips
    for (int s = threadIdx.x; s < a.nsplit; s += blockDim.x) {
      sw[s] = base[(size_t)s * a.s_stride];
      sl[s] = base[(size_t)s * a.s_stride + 1];
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      float M = -INFINITY;
      for (int s = threadIdx.x; s < a.nsplit; s += 32) M = fmaxf(M, sw[s]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
      float L = 0.f;
      for (int s = threadIdx.x; s < a.nsplit; s += 32) {
        const float ms = sw[s];
        const float w = ms == -INFINITY ? 0.f : exp2f(ms - M);
        sw[s] = w;
        L = fmaf(sl[s], w, L);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
      if (threadIdx.x == 0) { s_M = M; s_L = L; }
    }
    __syncthreads();
    const float M = s_M, L = s_L;
    // blockDim = head_dim x SG: thread (sg, i) sums the splits sg, sg + SG, ... of dim i
    // (SG independent load streams per dim, launch_merge picks SG from nsplit); the SG
    // partial sums meet in shared memory, summed in sg order (deterministic)
    const int SG = max(1, (int)blockDim.x / a.head_dim);
    const int sg = threadIdx.x / a.head_dim;
    const int i = threadIdx.x - sg * a.head_dim;
    __shared__ float s_part[7][256];
    float acc = 0.f;
    if (sg < SG) {
      const float* po = base + 2 + i;
      int s = sg;
      for (; s + 7 * SG < a.nsplit; s += 8 * SG) {
        float ov[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) ov[j] = po[(size_t)(s + j * SG) * a.s_stride];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc = fmaf(sw[s + j * SG], ov[j], acc);
      }
      for (; s < a.nsplit; s += SG) acc = fmaf(sw[s], po[(size_t)s * a.s_stride], acc);
      if (sg > 0) s_part[sg - 1][i] = acc;
    }
    __syncthreads();
    if (sg == 0) {
      for (int k = 0; k < SG - 1; ++k) acc += s_part[k][i];
      if (a.normalize) {
        T* out = reinterpret_cast<T*>(a.out) + ((size_t)b * a.n_q + h) * a.head_dim;
        out[i] = Elem<T>::from_f(L > 0.f ? acc / L : 0.f);
      } else {   // un-normalised partial (M, L, O) for the cross-rank merge
        float* out = reinterpret_cast<float*>(a.out) + (size_t)bh * (a.head_dim + 2);
        out[2 + i] = acc;
        if (i == 0) { out[0] = M; out[1] = L; }
      }
    }
    pdl_launch_dependents();
    return;
  }
  for (int i = threadIdx.x; i < a.head_dim; i += blockDim.x) {
    // many splits: one pass with a running max
    float M = -INFINITY, L = 0.f, acc = 0.f;
#pragma unroll 4
    for (int s = 0; s < a.nsplit; ++s) {
      const float* ps = base + (size_t)s * a.s_stride;
      const float ms = ps[0], ls = ps[1], os = ps[2 + i];
      if (ms == -INFINITY) continue;
      const float Mn = fmaxf(M, ms);
      const float c0 = exp2f(M - Mn), c1 = exp2f(ms - Mn);
      L = L * c0 + ls * c1;
      acc = acc * c0 + os * c1;
      M = Mn;
    }
    if (a.normalize) {
      T* out = reinterpret_cast<T*>(a.out) + ((size_t)b * a.n_q + h) * a.head_dim;
      out[i] = Elem<T>::from_f(L > 0.f ? acc / L : 0.f);
    } else {
      float* out = reinterpret_cast<float*>(a.out) + (size_t)bh * (a.head_dim + 2);
      out[2 + i] = acc;
      if (i == 0) { out[0] = M; out[1] = L; }
    }
  }
  pdl_launch_dependents();
}
template __global__ void merge_kernel<float>(MergeArgs);
template __global__ void merge_kernel<__nv_bfloat16>(MergeArgs);

// ---------------------------------------------------------------------------
// Dense comparator cache write: k_cache[b, pos] = RoPE_pos(k_new[b]), v copy.
// ---------------------------------------------------------------------------
// One CTA per (KV head, request), one thread per rotation pair: every load of the
// head is issued before any store (no store -> load ordering chain), the value row
// is copied with 16-byte vectors.
template <typename T>
__global__ void dense_append_kernel(DenseAppendArgs a) {
  const int g = blockIdx.x, b = blockIdx.y, p = threadIdx.x;
  const int half = a.head_dim / 2;
  const float2 th = p < half ? make_float2(a.rope.th_hi[p], a.rope.th_lo[p]) : make_float2(0.f, 0.f);
  pdl_wait();
  const int64_t pos = a.pos[b];
  const T* __restrict__ k = reinterpret_cast<const T*>(a.k_new) + (size_t)b * a.D + (size_t)g * a.head_dim;
  const T* __restrict__ v = reinterpret_cast<const T*>(a.v_new) + (size_t)b * a.D + (size_t)g * a.head_dim;
  T* __restrict__ kc = reinterpret_cast<T*>(a.k_cache) + ((size_t)b * a.cap + pos) * a.D + (size_t)g * a.head_dim;
  T* __restrict__ vc = reinterpret_cast<T*>(a.v_cache) + ((size_t)b * a.cap + pos) * a.D + (size_t)g * a.head_dim;
  constexpr int EPV = 16 / sizeof(T);
  const int nvec = a.head_dim / EPV;
  uint4 vv = make_uint4(0, 0, 0, 0);
  if (p < nvec) vv = *reinterpret_cast<const uint4*>(v + p * EPV);
  if (p < half) {
    int lo, hi; rope_pair(p, half, a.rope.style, lo, hi);
    const float xl = Elem<T>::to_f(k[lo]), xh = Elem<T>::to_f(k[hi]);
    float c, sn; rope_cs_fast(th.x, th.y, (int)pos, c, sn);
    kc[lo] = Elem<T>::from_f(xl * c - xh * sn);
    kc[hi] = Elem<T>::from_f(xl * sn + xh * c);
  }
  if (p < nvec) *reinterpret_cast<uint4*>(vc + p * EPV) = vv;
  pdl_launch_dependents();
}

// Query RoPE of the dense comparator: qrope[b, h] = RoPE_{s_b - 1}(q[b, h]) (fp32),
// one CTA per (query head, request), one thread per rotation pair.
template <typename T>
__global__ void dense_qrope_kernel(DenseAppendArgs a, const int* seq_len, float* qrope, int n_q) {
  const int h = blockIdx.x, b = blockIdx.y, p = threadIdx.x;
  const int half = a.head_dim / 2;
  const float2 th = p < half ? make_float2(a.rope.th_hi[p], a.rope.th_lo[p]) : make_float2(0.f, 0.f);
  pdl_wait();
  if (p < half) {
    const int pos = seq_len[b] - 1;
    const T* q = reinterpret_cast<const T*>(a.k_new) + ((size_t)b * n_q + h) * a.head_dim;
    float* o = qrope + ((size_t)b * n_q + h) * a.head_dim;
    int lo, hi; rope_pair(p, half, a.rope.style, lo, hi);
    const float xl = Elem<T>::to_f(q[lo]), xh = Elem<T>::to_f(q[hi]);
    float c, sn; rope_cs_fast(th.x, th.y, pos, c, sn);
    o[lo] = xl * c - xh * sn;
    o[hi] = xl * sn + xh * c;
  }
  pdl_launch_dependents();
}
template __global__ void dense_qrope_kernel<float>(DenseAppendArgs, const int*, float*, int);
template __global__ void dense_qrope_kernel<__nv_bfloat16>(DenseAppendArgs, const int*, float*, int);
template __global__ void dense_append_kernel<float>(DenseAppendArgs);
template __global__ void dense_append_kernel<__nv_bfloat16>(DenseAppendArgs);

// ---------------------------------------------------------------------------
// Sharded: the rows this rank attends to = owned sinks, owned global picks,
// owned recents (three ascending, disjoint, ordered ranges).  One CTA / request.
}  // namespace sals
