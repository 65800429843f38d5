// K1 / K2: skinny projections onto the latent basis.
//   append (Alg. 1 lines 2-3; Eq. 1):  k~ = U^T k_new  -> latent_cache[b, pos_b]
//   qproj  (Alg. 1 line 2):           q~ = U[:, :r*]^T q_bar   (fp32)
// plus (qproj launch only) RoPE of the query at position s_b - 1 (Alg. 1 line 7).
//
// Design: U [D, r] is read exactly once and the kernel is latency-bound (a few
// MiB), so the goal is bytes in flight.  A thread-block cluster of CS CTAs
// splits the D rows (the contraction axis); each CTA owns 8*EPC output columns
// (8 lanes x one 16-byte vector) and its 8 warps stride over its rows four at a
// time (lane / 8 = row slot), every lane keeping all its row loads in flight
// before the FMAs.  Partials are reduced row-slot -> warp (shuffles) -> CTA
// (shared memory, fixed warp order) -> cluster (DSMEM, fixed rank order), so
// the result is deterministic and needs no global workspace or atomics.
#include "common.cuh"
#include "kernels.h"
#include "quant.cuh"

namespace sals {

#ifdef SALS_TC_TRACE
__device__ unsigned long long g_proj_trace[16];
#define PJ_STAMP(i) do { if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) g_proj_trace[(i)] = clock64(); } while (0)
#else
#define PJ_STAMP(i) do {} while (0)
#endif

constexpr int kProjBT = 8;        // requests per pass
constexpr int kProjMaxRows = 512; // rows per CTA (D / CS)
constexpr int kProjUnroll = 8;    // row loads in flight per lane

#ifndef SALS_PROJ_MINB
#define SALS_PROJ_MINB 1   // measured: an uncapped register budget (no spills) beats co-residence
#endif
// MODE 0: append (k~ = U^T k_new -> latent row, v row copy); 1: query projection
// (+ query RoPE role, histogram zeroing); 2: both in one launch (sals_append_decode):
// blockIdx.y < n_append_blocks are append column blocks, the rest the query role.
// NT threads: 512 when a CTA owns 512 rows of U (D = 4096), else 256 (measured)
// Slot of request b's new token in the cache this call appends to, or -1 when this call
// does not append it (a sequence shard that does not hold position seq_len[b] - 1).
__device__ __forceinline__ int append_slot(const ProjectArgs& a, int b) {
  if (a.pos) return a.pos[b];
  const int slot = a.seq_len[b] - 1 - (int)a.append_base;
  if (a.append_len && (slot < 0 || slot != a.append_len[b] - 1)) return -1;
  return slot;
}

template <typename T, int MODE, int NT>
__global__ void __launch_bounds__(NT, SALS_PROJ_MINB)   // 2: <= 128 registers, co-resident with the next kernel
project_kernel(ProjectArgs a) {
  const bool pool = MODE == 1 || (MODE == 2 && (int)blockIdx.y >= a.n_append_blocks);
  const int yb = (MODE == 2 && pool) ? (int)blockIdx.y - a.n_append_blocks : (int)blockIdx.y;   // block within the role
  const int ncols = (MODE == 2 && !pool) ? a.ncols_a : a.ncols;
  const int x_stride = (MODE == 2 && !pool) ? a.D : a.x_stride;
  constexpr int EPC = Elem<T>::kPer16;       // columns per lane
  constexpr int CPB = 8 * EPC;               // columns per CTA
  __shared__ float xs[kProjBT][kProjMaxRows];

  __shared__ float cred[kProjBT][CPB];
  __shared__ float incoming[kProjBT * CPB];   // [source rank][owned output] partials pushed by peers
  const int CS = (int)cluster_nctarank();
  const int rank = (int)cluster_ctarank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const T* U = reinterpret_cast<const T*>(a.U);
  const T* x = reinterpret_cast<const T*>((MODE == 2 && !pool) ? a.xa : a.x);

  const int rows_per = a.rows_per_cta;
  const int row0 = rank * rows_per;
  const int row1 = min(a.D, row0 + rows_per);
  const int slot = lane >> 3;                       // row slot 0..3 within a warp step
  const int cl = lane & 7;                          // column vector within the CTA's block
  const int col = yb * CPB + cl * EPC;
  const bool col_ok = col < ncols;
  const char* Ub = reinterpret_cast<const char*>(U);
  const size_t row_bytes = (size_t)a.r * sizeof(T);
  const bool rope_role = pool && blockIdx.y == gridDim.y - 1;
  // U is a weight no upstream kernel writes: the CTA's whole U slice
  // (rows [row0, row1) x its CPB columns, 128 B per row) is copied into shared
  // memory by cp.async BEFORE waiting on the upstream grid, so no U load is left
  // on the critical path after the wait, whatever the rows per CTA.
  extern __shared__ __align__(16) uint8_t sU[];   // [rows_per][128 B], then wred
  // per-warp partial outputs [NT / 32][kProjBT][CPB] (dynamic: 32 KB at 16 warps)
  float (*wred)[kProjBT][CPB] = reinterpret_cast<float (*)[kProjBT][CPB]>(sU + (size_t)a.rows_per_cta * 128);
  const int base0 = row0 + 4 * warp + slot;
  PJ_STAMP(0);
  if (!rope_role) {
    const int nvec = (row1 - row0) * 8;
    const uint32_t su = smem_u32(sU);
    for (int i = tid; i < nvec; i += NT) {
      const int rr = i >> 3, cv = i & 7;
      const int cc = yb * CPB + cv * EPC;
      const bool okc = cc < ncols;
      const char* src = Ub + (size_t)(row0 + rr) * row_bytes + (size_t)(okc ? cc : 0) * sizeof(T);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su + rr * 128 + cv * 16), "l"(src),
                   "r"(okc ? 16 : 0) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  __shared__ float2 sth[128];   // (th_hi, th_lo) per rotation pair: indexed per lane, so not from param space
  if (rope_role)
    for (int i = tid; i < a.rope.half; i += NT) sth[i] = make_float2(a.rope.th_hi[i], a.rope.th_lo[i]);
  __syncthreads();

  PJ_STAMP(1);
  pdl_wait();
  PJ_STAMP(2);
  // Dependents may launch now: their pre-wait sections only read weights (U) and
  // the latent rows of earlier steps / of the sals_append_latent that this
  // grid's griddepcontrol.wait has just seen complete (PDL).
  pdl_launch_dependents();

  if (rope_role) {
    // ---- role 2: RoPE of the query heads at position s_b - 1 (fp32 out) ----
    const int half = a.rope.half, d = 2 * half;
    const int nq = a.n_q;
    if (a.hist0_zero)   // the score kernel accumulates the top-digit histogram into this
      for (int i = rank * NT + tid; i < a.hist0_words; i += CS * NT) a.hist0_zero[i] = 0u;
    // (request, head, pair) tasks split over the CS CTAs of this row; loads of 8
    // tasks are issued before any math so the latency is paid once per batch
    const int per_req = half * nq;
    const int total = a.B * per_req;
    for (int t0 = rank * NT + tid; t0 < total; t0 += CS * NT * 8) {
      float xl[8], xh[8];
      int lo_[8], hi_[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int t = t0 + u * CS * NT;
        xl[u] = xh[u] = 0.f;
        if (t < total) {
          const int b = t / per_req, r = t % per_req, p = r % half, h = r / half;
          rope_pair(p, half, a.rope.style, lo_[u], hi_[u]);
          xl[u] = Elem<T>::to_f(x[(size_t)b * a.x_stride + h * d + lo_[u]]);
          xh[u] = Elem<T>::to_f(x[(size_t)b * a.x_stride + h * d + hi_[u]]);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int t = t0 + u * CS * NT;
        if (t < total) {
          const int b = t / per_req, r = t % per_req, p = r % half, h = r / half;
          float c, s; rope_cs_fast(sth[p].x, sth[p].y, a.seq_len[b] - 1, c, s);
          a.qrope[((size_t)b * nq + h) * d + lo_[u]] = xl[u] * c - xh[u] * s;
          a.qrope[((size_t)b * nq + h) * d + hi_[u]] = xl[u] * s + xh[u] * c;
        }
      }
    }
    pdl_launch_dependents();
    return;
  }

  if (!pool && a.v_new != nullptr) {
    const int ncta = CS * (MODE == 2 ? a.n_append_blocks : (int)gridDim.y);
    const int cta = blockIdx.y * CS + rank;
    if (a.v_bits == 0) {
      // ---- append: copy v_new[b] -> v_cache[b, pos_b] (16-byte vectors) ----
      const int nvec = a.D * (int)sizeof(T) / 16;
      for (int i = cta * NT + tid; i < a.B * nvec; i += ncta * NT) {
        const int b = i / nvec, v = i % nvec;
        const int pb = append_slot(a, b);
        if (pb < 0) continue;
        const uint4 val = ld_v4(reinterpret_cast<const char*>(a.v_new) + ((size_t)b * a.D) * sizeof(T) + v * 16);
        *reinterpret_cast<uint4*>(reinterpret_cast<char*>(a.v_cache) +
                                  (((size_t)b * a.cap + pb) * a.D) * sizeof(T) + v * 16) = val;
      }
    } else {
      // ---- append with channel-wise group quantisation (DESIGN R15; quant.cuh):
      // four lanes per 32-channel group, 8 channels (one 16-byte load) each
      const int bits = a.v_bits;
      const int gph = 128 / 32;                       // groups per head (head_dim 128)
      const int hb = 128 * bits / 8 + gph * 4;        // bytes per head in a row
      const int nitems = a.B * (a.D / 8);             // (request, 8-channel slice); 4 per group, lane-adjacent
      for (int i0 = cta * NT; i0 < nitems; i0 += ncta * NT) {
        const int i = i0 + tid;
        const int b = i < nitems ? i / (a.D / 8) : 0;
        const int pb = i < nitems ? append_slot(a, b) : 0;
        const bool ok = i < nitems && pb >= 0;   // (the quantiser's lane groups stay whole: a request is all in or out)
        const int sl = i < nitems ? i - b * (a.D / 8) : 0;
        const int gi = sl >> 2, q = sl & 3, h = gi / gph, gq = gi - h * gph;
        float f[8];
        if (ok) Elem<__nv_bfloat16>::unpack(ld_v4(reinterpret_cast<const char*>(a.v_new) + ((size_t)b * a.D + sl * 8) * 2), f);
        else for (int e = 0; e < 8; ++e) f[e] = 0.f;
        char* row = reinterpret_cast<char*>(a.v_cache) + ((size_t)b * a.cap + pb) * a.v_row_bytes + (size_t)h * hb;
        char* ring = a.hp_window > 0
                         ? reinterpret_cast<char*>(a.v_cache) + a.hp_ring_off +
                               ((size_t)b * a.hp_window + pb % a.hp_window) * (size_t)(a.D / 128) * 144 + (size_t)h * 144
                         : nullptr;
        quantize_slice(f, ok, bits, row, gq, q, ring);
      }
    }
  }

  for (int b0 = 0; b0 < a.B; b0 += kProjBT) {
    const int nb = min(kProjBT, a.B - b0);
    // stage x (pooled over the query heads of each KV group for qproj): one
    // 16-byte vector per thread per head, all loads issued before the sums
    {
      const int nvec_row = (row1 - row0) / EPC;          // rows_per is a multiple of EPC
      for (int i = tid; i < kProjBT * nvec_row; i += NT) {
        const int bb = i / nvec_row, cv = i - bb * nvec_row;
        const int c = row0 + cv * EPC;
        float v[EPC];
#pragma unroll
        for (int e = 0; e < EPC; ++e) v[e] = 0.f;
        if (bb < nb) {
          const T* xb = x + (size_t)(b0 + bb) * x_stride;
          if (pool) {
            const int g = c / a.head_dim, j = c - g * a.head_dim;   // EPC <= head_dim: one head per vector
            for (int hh = 0; hh < a.group; ++hh) {
              float f[EPC];
              Elem<T>::unpack(ld_v4(xb + (g * a.group + hh) * a.head_dim + j), f);
#pragma unroll
              for (int e = 0; e < EPC; ++e) v[e] += f[e];
            }
          } else {
            Elem<T>::unpack(ld_v4(xb + c), v);
          }
        }
#pragma unroll
        for (int e = 0; e < EPC; ++e) xs[bb][cv * EPC + e] = v[e];
      }
    }
    if (b0 == 0) asm volatile("cp.async.wait_all;" ::: "memory");   // this thread's U copies
    __syncthreads();                                                  // everyone's copies and xs visible
    PJ_STAMP(3);

    float acc[kProjBT][EPC];
#pragma unroll
    for (int bb = 0; bb < kProjBT; ++bb)
#pragma unroll
      for (int e = 0; e < EPC; ++e) acc[bb][e] = 0.f;
    if (col_ok) {
      // rows handled by this lane: base0 + 32 i, from the shared-memory copy of U;
      // packed FFMA2 over column pairs (half the FMA-pipe issue slots)
      auto fma_row = [&](const uint4& raw, int c) {
        float uf[EPC];
        Elem<T>::unpack(raw, uf);
#pragma unroll
        for (int bb = 0; bb < kProjBT; ++bb) {
          const float xv = xs[bb][c - row0];
          const float2 x2 = make_float2(xv, xv);
#pragma unroll
          for (int e = 0; e < EPC; e += 2) {
            const float2 r2 = __ffma2_rn(make_float2(uf[e], uf[e + 1]), x2, make_float2(acc[bb][e], acc[bb][e + 1]));
            acc[bb][e] = r2.x;
            acc[bb][e + 1] = r2.y;
          }
        }
      };
#pragma unroll 4
      for (int c = base0; c < row1; c += 4 * (NT / 32))
        fma_row(*reinterpret_cast<const uint4*>(sU + (c - row0) * 128 + cl * 16), c);
    }
    PJ_STAMP(4);
    // reduce the 4 row slots of the warp (lanes cl, cl+8, cl+16, cl+24), transposed:
    // each exchange halves the values a lane keeps (48 shuffles instead of 128), and
    // every lane ends with 2 requests x EPC columns summed over the 4 slots
    {
      const int s1 = (lane >> 4) & 1, s0 = (lane >> 3) & 1;
      float k1[kProjBT / 2][EPC];
#pragma unroll
      for (int bq = 0; bq < kProjBT / 2; ++bq)
#pragma unroll
        for (int e = 0; e < EPC; ++e) {
          const float lo = acc[bq][e], hi = acc[bq + kProjBT / 2][e];
          k1[bq][e] = (s1 ? hi : lo) + __shfl_xor_sync(0xffffffffu, s1 ? lo : hi, 16);
        }
#pragma unroll
      for (int bq = 0; bq < kProjBT / 4; ++bq)
#pragma unroll
        for (int e = 0; e < EPC; ++e) {
          const float lo = k1[bq][e], hi = k1[bq + kProjBT / 4][e];
          const float v = (s0 ? hi : lo) + __shfl_xor_sync(0xffffffffu, s0 ? lo : hi, 8);
          wred[warp][(kProjBT / 2) * s1 + (kProjBT / 4) * s0 + bq][cl * EPC + e] = v;
        }
    }
    __syncthreads();
    for (int i = tid; i < kProjBT * CPB; i += NT) {
      const int bb = i / CPB, j = i % CPB;
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < (NT / 32); ++w) s += wred[w][bb][j];
      cred[bb][j] = s;
    }
    __syncthreads();
    // push every partial to the rank that owns its output (fire-and-forget DSMEM
    // stores), then each rank sums the CS partials of its outputs in rank order
    const int nout = nb * CPB;
    const int share = (nout + CS - 1) / CS;
    {
      const uint32_t inc_addr = smem_u32(&incoming[0]);
      for (int o = tid; o < nout; o += NT) {
        const int owner = o / share, ol = o - owner * share;
        st_dsmem_u32(mapa_shared(inc_addr + (rank * share + ol) * 4, owner),
                     __float_as_uint(cred[o / CPB][o % CPB]));
      }
    }
    PJ_STAMP(5);
    cluster_sync_all();
    PJ_STAMP(6);
    for (int o = rank * share + tid; o < min(nout, (rank + 1) * share); o += NT) {
      const int bb = o / CPB, j = o % CPB;
      const int cj = yb * CPB + j;
      const int ol = o - rank * share;
      float sum = 0.f;
      for (int c = 0; c < CS; ++c) sum += incoming[c * share + ol];
      if (cj < ncols) {
        const int b = b0 + bb;
        if (pool) {
          a.out_f32[(size_t)b * ncols + cj] = sum;
        } else {
          T* lat = reinterpret_cast<T*>(a.latent);
          const int pb = append_slot(a, b);
          if (pb >= 0) lat[((size_t)b * a.cap + pb) * a.r + cj] = Elem<T>::from_f(sum);
        }
      }
    }
    // (the incoming buffer is reused by the next pass; after the last pass no peer
    // touches this CTA's shared memory any more: sync 1 ordered every DSMEM store)
    if (b0 + kProjBT < a.B) cluster_sync_all();
    PJ_STAMP(7);
  }
  pdl_launch_dependents();
}

}  // namespace sals
extern "C" int sals_debug_proj_trace(unsigned long long* out) {
#ifdef SALS_TC_TRACE
  return (int)cudaMemcpyFromSymbol(out, sals::g_proj_trace, sizeof(sals::g_proj_trace));
#else
  (void)out;
  return -1;
#endif
}
namespace sals {

#define SALS_PROJ_INST(T)                                              \
  template __global__ void project_kernel<T, 0, 256>(ProjectArgs);     \
  template __global__ void project_kernel<T, 1, 256>(ProjectArgs);     \
  template __global__ void project_kernel<T, 2, 256>(ProjectArgs);     \
  template __global__ void project_kernel<T, 0, 512>(ProjectArgs);     \
  template __global__ void project_kernel<T, 1, 512>(ProjectArgs);     \
  template __global__ void project_kernel<T, 2, 512>(ProjectArgs);
SALS_PROJ_INST(float)
SALS_PROJ_INST(__nv_bfloat16)

}  // namespace sals
