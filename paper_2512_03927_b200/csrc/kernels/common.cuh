// Device helpers shared by the OD-MoE sm_100a kernels (product code; independent of oracle/).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace odmoe {

constexpr int kMaxE = 64;  // router limit (ABI: E <= 64)
constexpr int kMaxK = 8;

// ---------------------------------------------------------------- element types
// Weight element types the GEMV family streams: bf16, fp32, int8 (row-scaled).
template <typename T> struct WTraits;
template <> struct WTraits<__nv_bfloat16> { static constexpr int kPer16B = 8; };
template <> struct WTraits<float> { static constexpr int kPer16B = 4; };
template <> struct WTraits<int8_t> { static constexpr int kPer16B = 16; };

__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

// Streaming 16-byte global load that bypasses L1 (weights are touched exactly once).
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Same, with an explicit L2 cache policy (createpolicy): evict_first keeps streamed weights from
// displacing other L2 lines (e.g. dirty lines just written by the H2D copy engine).
__device__ __forceinline__ uint4 ld_stream_pol(const void* p, uint64_t pol) {
  uint4 r;
#ifdef FG_NOPF
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
#else
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
#endif
  return r;
}
__device__ __forceinline__ uint64_t l2_policy(bool evict_first) {
  uint64_t pol;
  if (evict_first) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// int8 -> fp32 without I2F: place (q ^ 0x80) in the low mantissa byte of 2^23 and subtract
// 2^23 + 128. Exact for every int8 value.
__device__ __forceinline__ float i8_to_f32(uint32_t biased_word, int byte_sel) {
  return __uint_as_float(__byte_perm(biased_word, 0x4B000000u, 0x7540 | byte_sel)) - 8388736.0f;
}

// Dot product of one 16-byte weight chunk with fp32 activations x[0 .. kPer16B).
template <typename T> __device__ __forceinline__ float dot16(const uint4& w, const float* x);

template <> __device__ __forceinline__ float dot16<__nv_bfloat16>(const uint4& w, const float* x) {
  const float4 x0 = *reinterpret_cast<const float4*>(x);
  const float4 x1 = *reinterpret_cast<const float4*>(x + 4);
  float s = bf16_lo(w.x) * x0.x;
  s = fmaf(bf16_hi(w.x), x0.y, s);
  s = fmaf(bf16_lo(w.y), x0.z, s);
  s = fmaf(bf16_hi(w.y), x0.w, s);
  s = fmaf(bf16_lo(w.z), x1.x, s);
  s = fmaf(bf16_hi(w.z), x1.y, s);
  s = fmaf(bf16_lo(w.w), x1.z, s);
  s = fmaf(bf16_hi(w.w), x1.w, s);
  return s;
}

template <> __device__ __forceinline__ float dot16<float>(const uint4& w, const float* x) {
  const float4 x0 = *reinterpret_cast<const float4*>(x);
  float s = __uint_as_float(w.x) * x0.x;
  s = fmaf(__uint_as_float(w.y), x0.y, s);
  s = fmaf(__uint_as_float(w.z), x0.z, s);
  s = fmaf(__uint_as_float(w.w), x0.w, s);
  return s;
}

__device__ __forceinline__ float dot_i8_word(uint32_t word, const float4& x, float s) {
  const uint32_t b = word ^ 0x80808080u;
  s = fmaf(i8_to_f32(b, 0), x.x, s);
  s = fmaf(i8_to_f32(b, 1), x.y, s);
  s = fmaf(i8_to_f32(b, 2), x.z, s);
  s = fmaf(i8_to_f32(b, 3), x.w, s);
  return s;
}

template <> __device__ __forceinline__ float dot16<int8_t>(const uint4& w, const float* x) {
  const float4* xv = reinterpret_cast<const float4*>(x);
  float s = 0.f;
  s = dot_i8_word(w.x, xv[0], s);
  s = dot_i8_word(w.y, xv[1], s);
  s = dot_i8_word(w.z, xv[2], s);
  s = dot_i8_word(w.w, xv[3], s);
  return s;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Load activations of dtype (0 bf16, 1 fp32) into fp32 shared memory.
__device__ __forceinline__ void load_act_to_smem(float* xs, const void* x, int n, int x_is_f32) {
  if (x_is_f32) {
    const float4* src = reinterpret_cast<const float4*>(x);
    for (int i = threadIdx.x; i < n / 4; i += blockDim.x) reinterpret_cast<float4*>(xs)[i] = src[i];
  } else {
    const uint4* src = reinterpret_cast<const uint4*>(x);
    for (int i = threadIdx.x; i < n / 8; i += blockDim.x) {
      const uint4 v = src[i];
      float4 a = make_float4(bf16_lo(v.x), bf16_hi(v.x), bf16_lo(v.y), bf16_hi(v.y));
      float4 b = make_float4(bf16_lo(v.z), bf16_hi(v.z), bf16_lo(v.w), bf16_hi(v.w));
      reinterpret_cast<float4*>(xs)[2 * i] = a;
      reinterpret_cast<float4*>(xs)[2 * i + 1] = b;
    }
  }
}

// Balanced contiguous partition of n items over parts: [begin, end) of part p.
__device__ __forceinline__ void split_range(long long n, int parts, int p, long long& b, long long& e) {
  b = n * p / parts;
  e = n * (p + 1) / parts;
}

__device__ __forceinline__ float silu_mul(float g, float v) { return g / (1.0f + expf(-g)) * v; }

}  // namespace odmoe
