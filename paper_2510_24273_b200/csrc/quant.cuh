// Channel-wise group quantisation of value rows (P:503-514,
// DESIGN R15), shared by the single-token append (project.cu) and the bulk
// append (prefill_tc.cu).
//
// One thread holds 8 consecutive channels (one 16-byte bf16 vector); the four
// lane-adjacent threads of a 32-channel group find its min / max with two xor
// shuffles (every lane of the warp must call).  zero = min, scale = (max - min) /
// (2^bits - 1), both rounded to bf16 first; codes from the rounded values in
// exact IEEE fp32 (one rounded subtract, one rounded divide, round half to even,
// clamp), packed low bits first.  Row layout per KV head (d = 128):
// [128 * bits / 8 code bytes][4 x (bf16 scale, bf16 zero)].  The optional 8-bit
// copy (the recent window) uses the same rule with 255 levels into a
// 144-byte head row [128 codes][4 x (scale, zero)].
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

namespace sals {

__device__ __forceinline__ void quantize_slice(const float (&f)[8], bool ok, int bits, char* head_row, int gq, int q,
                                               char* head_ring) {
  float lo = f[0], hi = f[0];
#pragma unroll
  for (int e = 1; e < 8; ++e) { lo = fminf(lo, f[e]); hi = fmaxf(hi, f[e]); }
  lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, 1)); hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, 1));
  lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, 2)); hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, 2));
  if (!ok) return;
  const int qmax = (1 << bits) - 1;
  const __nv_bfloat16 zb = __float2bfloat16_rn(lo);
  const __nv_bfloat16 sb = __float2bfloat16_rn(__fdiv_rn(__fsub_rn(hi, lo), (float)qmax));
  const float zf = __bfloat162float(zb), sf = __bfloat162float(sb);
  uint32_t w = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int c = sf > 0.f ? min(qmax, max(0, __float2int_rn(__fdiv_rn(__fsub_rn(f[e], zf), sf)))) : 0;
    w |= (uint32_t)c << (e * bits);
  }
  if (bits == 4) *reinterpret_cast<uint32_t*>(head_row + gq * 16 + q * 4) = w;
  else *reinterpret_cast<uint16_t*>(head_row + gq * 8 + q * 2) = (uint16_t)w;
  if (q == 0)
    *reinterpret_cast<uint32_t*>(head_row + 128 * bits / 8 + gq * 4) =
        (uint32_t)__bfloat16_as_ushort(sb) | ((uint32_t)__bfloat16_as_ushort(zb) << 16);
  if (head_ring) {
    const __nv_bfloat16 s8 = __float2bfloat16_rn(__fdiv_rn(__fsub_rn(hi, lo), 255.f));
    const float s8f = __bfloat162float(s8);
    uint32_t w8[2] = {0, 0};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int c = s8f > 0.f ? min(255, max(0, __float2int_rn(__fdiv_rn(__fsub_rn(f[e], zf), s8f)))) : 0;
      w8[e >> 2] |= (uint32_t)c << ((e & 3) * 8);
    }
    *reinterpret_cast<uint2*>(head_ring + gq * 32 + q * 8) = make_uint2(w8[0], w8[1]);
    if (q == 0)
      *reinterpret_cast<uint32_t*>(head_ring + 128 + gq * 4) =
          (uint32_t)__bfloat16_as_ushort(s8) | ((uint32_t)__bfloat16_as_ushort(zb) << 16);
  }
}

}  // namespace sals
