// Shared device helpers for the SALS sm_100a kernels: vector loads, bf16
// conversion, RoPE angles, cluster / DSMEM, mbarrier and PDL primitives.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

namespace sals {

constexpr int kMaxHeadDim = 256;
constexpr float kLog2e = 1.4426950408889634f;

// RoPE frequencies theta_p = base^(-2p/d) (Eq. 3), computed once on the host
// in double and passed by value to every kernel that rotates.
struct RopeTable {
  double theta[kMaxHeadDim / 2];
  float th_hi[kMaxHeadDim / 2];   // fp32(theta)
  float th_lo[kMaxHeadDim / 2];   // fp32(theta - th_hi)
  int half;       // d/2
  int style;      // 0 = (i, i+d/2), 1 = (2i, 2i+1)
};

// --------------------------------------------------------------- element io
template <typename T> struct Elem;
template <> struct Elem<float> {
  static constexpr int kPer16 = 4;
  __device__ __forceinline__ static void unpack(const uint4& v, float* o) {
    o[0] = __uint_as_float(v.x); o[1] = __uint_as_float(v.y);
    o[2] = __uint_as_float(v.z); o[3] = __uint_as_float(v.w);
  }
  __device__ __forceinline__ static float to_f(float x) { return x; }
  __device__ __forceinline__ static float from_f(float x) { return x; }
};
template <> struct Elem<__nv_bfloat16> {
  static constexpr int kPer16 = 8;
  __device__ __forceinline__ static void unpack(const uint4& v, float* o) {
    o[0] = __uint_as_float(v.x << 16); o[1] = __uint_as_float(v.x & 0xffff0000u);
    o[2] = __uint_as_float(v.y << 16); o[3] = __uint_as_float(v.y & 0xffff0000u);
    o[4] = __uint_as_float(v.z << 16); o[5] = __uint_as_float(v.z & 0xffff0000u);
    o[6] = __uint_as_float(v.w << 16); o[7] = __uint_as_float(v.w & 0xffff0000u);
  }
  __device__ __forceinline__ static float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  __device__ __forceinline__ static __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
};

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Streaming 16-byte load (read-only path, no L1 allocation).
__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_v4(const void* p) {
  return *reinterpret_cast<const uint4*>(p);
}

// ------------------------------------------------------------------- RoPE
// cos/sin of pos * theta_p with the angle formed and reduced mod 2*pi in
// double (an fp32 product would be off by ~1e-2 rad at pos ~ 1.3e5), then
// evaluated in fp32 on the reduced angle.
__device__ __forceinline__ void rope_cs(double theta, int64_t pos, float& c, float& s) {
  const double two_pi = 6.283185307179586476925286766559;
  const double inv_two_pi = 0.15915494309189533576888376337251;
  double phi = (double)pos * theta;
  double n = rint(phi * inv_two_pi);
  double red = fma(-n, two_pi, phi);
  sincosf((float)red, &s, &c);
}

// Same angle without fp64: pos * theta = pos*th_hi (rounded) + its exact FMA
// error + pos*th_lo, reduced mod 2 pi with a two-term Cody-Waite constant on
// the FMA pipe, then the MUFU sin/cos on |r| <~ pi.  |angle error| ~ 3e-7 rad
// up to pos = 2^24 (vs ~1e-2 rad for a plain fp32 product at pos ~ 1.3e5).
__device__ __forceinline__ void rope_cs_fast(float th_hi, float th_lo, int pos, float& c, float& s) {
  const float p = (float)pos;
  const float a = p * th_hi;
  const float a_err = fmaf(p, th_hi, -a);
  const float n = rintf(a * 0.159154943091895336f);
  float r = fmaf(-n, 6.28318548202514648f, a);
  r = fmaf(-n, -1.7484556025237907e-07f, r);
  r += fmaf(p, th_lo, a_err);
  __sincosf(r, &s, &c);
}

// Index pair (lo, hi) of rotation pair p for head_dim 2*half.
__device__ __forceinline__ void rope_pair(int p, int half, int style, int& lo, int& hi) {
  if (style == 0) { lo = p; hi = p + half; } else { lo = 2 * p; hi = 2 * p + 1; }
}

// ------------------------------------------------------------- cluster / PDL
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
  uint32_t r; asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r)); return r;
}
// Full barrier of every thread of every CTA of the cluster, with release /
// acquire ordering of shared (and DSMEM) accesses.  The leading __syncthreads
// keeps the CTA-local ordering explicit also for kernels launched without a
// cluster attribute (an implicit 1-CTA cluster).
__device__ __forceinline__ void cluster_sync_all() {
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Map a local shared-memory address to the same offset in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa_shared(uint32_t local_addr, uint32_t rank) {
  uint32_t r; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank)); return r;
}
__device__ __forceinline__ float ld_dsmem_f32(uint32_t addr) {
  float v; asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr)); return v;
}
// (no "memory" clobber: callers order these after a cluster barrier, which is
// itself a compiler-level memory fence, and batching independent loads matters)
__device__ __forceinline__ uint32_t ld_dsmem_u32(uint32_t addr) {
  uint32_t v; asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr)); return v;
}
__device__ __forceinline__ void st_dsmem_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Programmatic dependent launch: wait for the upstream grid's memory to be
// visible / allow the downstream grid to start its prologue.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }

// Order-preserving float -> uint32 key (larger float => larger key; -0 == +0).
__device__ __forceinline__ uint32_t float_key(float f) {
  f += 0.0f;  // canonicalise -0.0
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_float(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}

}  // namespace sals
