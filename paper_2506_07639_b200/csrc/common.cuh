// Shared device helpers for the Fast-ECoT B200 engine (sm_100a).
//
// The fp32 "canonical" arithmetic below is the device restatement of the
// model definition in DESIGN.md §3 (dot products with 32 lane partials and a
// fixed xor butterfly, a deterministic exp, explicit roundings).  The whole
// library is compiled with --fmad=false, so every fused multiply-add is an
// explicit __fmaf_rn and results are independent of batch composition,
// launch geometry and KV placement.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#define FE_PAGE 64           // KV page = canonical attention chunk (positions)
#define FE_WARP 32

namespace fe {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__host__ __device__ inline uint64_t splitmix64_h(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__host__ __device__ inline uint64_t tensor_key(uint64_t seed, uint64_t tid) {
  return splitmix64_h(splitmix64_h(seed) ^ tid);
}

// (u24 * 2^-24 - 0.5): exact in fp32
__device__ __forceinline__ float centered(uint64_t key, uint64_t i) {
  float u = (float)(splitmix64(key + i) >> 40);
  return __fsub_rn(__fmul_rn(u, 0x1p-24f), 0.5f);
}

constexpr float kLinearMult = 0x1.1bc77ap-4f;   // 2*sqrt(3)*0.02
constexpr float kVisionMult = 0x1.bb67aep+1f;   // 2*sqrt(3)
constexpr float kNormMult = 0x1.99999ap-3f;     // 0.2

__device__ __forceinline__ float xor_butterfly(float v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}

// Deterministic exp: clamp, 2^n * P7(f) with Horner fmaf.
__device__ __forceinline__ float fe_exp(float x) {
  if (!(x > -87.0f)) return 0.0f;
  if (x > 88.0f) x = 88.0f;
  float y = __fmul_rn(x, 0x1.715476p+0f);
  float n = rintf(y);
  float f = __fsub_rn(y, n);
  float p = 0x1.ffcbfcp-17f;
  p = __fmaf_rn(p, f, 0x1.430912p-13f);
  p = __fmaf_rn(p, f, 0x1.5d87fep-10f);
  p = __fmaf_rn(p, f, 0x1.3b2ab6p-7f);
  p = __fmaf_rn(p, f, 0x1.c6b08ep-5f);
  p = __fmaf_rn(p, f, 0x1.ebfbe0p-3f);
  p = __fmaf_rn(p, f, 0x1.62e430p-1f);
  p = __fmaf_rn(p, f, 1.0f);
  float scale = __int_as_float(((int)n + 127) << 23);
  return __fmul_rn(p, scale);
}

__device__ __forceinline__ float silu_mul(float g, float u) {
  float e = fe_exp(-g);
  float sg = __fdiv_rn(g, __fadd_rn(1.0f, e));
  return __fmul_rn(sg, u);
}

// --- element conversions ---------------------------------------------------
template <typename T> struct Elem;
template <> struct Elem<float> {
  static constexpr int kVec = 4;  // elements per 16-byte vector
  __device__ __forceinline__ static float to_f(float v) { return v; }
  __device__ __forceinline__ static float from_f(float v) { return v; }
};
template <> struct Elem<__nv_bfloat16> {
  static constexpr int kVec = 8;
  __device__ __forceinline__ static float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
  __device__ __forceinline__ static __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
};

// 16-byte vector <-> floats
__device__ __forceinline__ void unpack(const uint4& v, float (&f)[4]) {
  f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
  f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
}
__device__ __forceinline__ void unpack(const uint4& v, float (&f)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; i++) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// ordered key for argmax: larger value wins, lower index wins ties
__device__ __forceinline__ unsigned long long argmax_key(float v, int idx) {
  uint32_t b = __float_as_uint(v);
  uint32_t ord = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return ((unsigned long long)ord << 32) | (unsigned long long)(0xffffffffu - (uint32_t)idx);
}
__device__ __forceinline__ int argmax_index(unsigned long long key) {
  return (int)(0xffffffffu - (uint32_t)(key & 0xffffffffull));
}

// Programmatic dependent launch: kernels of the decode chain are launched
// with cudaLaunchAttributeProgrammaticStreamSerialization, may start while the
// previous kernel drains, and must call pdl_wait() before touching anything the
// previous kernel writes (or reads).  Both are no-ops for normal launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

}  // namespace fe
