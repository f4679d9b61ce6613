// Synthetic-weight generator and the INT8-row shadow quantiser (product side).
//
// The generator is the counter-based recipe of DESIGN.md §3, implemented here independently of
// inputs/fixture.py (tests check both give identical bytes). It is setup, not the hot path: the
// engine uses it to fill the pinned host expert pool and the resident non-expert weights.
//
// The quantiser is the shadow's INT8 format (P:86, P:164 name INT8 without a format; reading Q9):
// per output row, m = max|w|, q = clamp(RNE((w*127)/m), -127, 127) with the product and quotient
// in fp64 (so exact half-ties are resolved by RNE), s = fl32(m/127); zero rows -> q=0, s=1.
#include "common.cuh"
#include "kernels.h"

#include <cuda_fp8.h>

namespace odmoe {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += kGolden;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static uint64_t stream_base(uint64_t seed, uint64_t tid) { return splitmix64(splitmix64(seed) ^ tid); }
static uint64_t tensor_id(int kind, int layer, int expert) {
  return ((uint64_t)kind << 40) | ((uint64_t)layer << 20) | (uint64_t)expert;
}
static float fan_in_scale(int64_t fan_in) { return (float)(1.0 / sqrt((double)fan_in)); }

__device__ __forceinline__ float gen_value(uint64_t base, uint64_t i, float scale) {
  const uint64_t x = splitmix64(base + i);
  const int32_t u24 = (int32_t)(x >> 40);
  const float v = (float)(2 * u24 - 16777215) * 5.9604644775390625e-08f;  // exact: odd / 2^24
  return __fmul_rn(v, scale);
}

template <typename T> __device__ __forceinline__ T to_t(float v);
template <> __device__ __forceinline__ __nv_bfloat16 to_t<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
template <> __device__ __forceinline__ float to_t<float>(float v) { return v; }

template <typename T>
__global__ void gen_plain_kernel(T* __restrict__ out, uint64_t base, long long n, float scale) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = to_t<T>(gen_value(base, (uint64_t)i, scale));
}

// Expert blob: W13 [F][2][d] interleaved (row 2f = W1 row f, 2f+1 = W3 row f), then W2 [d][F].
template <typename T>
__global__ void gen_blob_kernel(T* __restrict__ out, uint64_t b1, uint64_t b3, uint64_t b2, int d,
                                int F, float s_d, float s_f) {
  const long long n13 = 2LL * F * d, n = 3LL * F * d;
  for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < n; o += (long long)gridDim.x * blockDim.x) {
    float v;
    if (o < n13) {
      const long long row = o / d, j = o - row * d;
      const long long f = row >> 1;
      v = gen_value((row & 1) ? b3 : b1, (uint64_t)(f * d + j), s_d);
    } else {
      v = gen_value(b2, (uint64_t)(o - n13), s_f);
    }
    out[o] = to_t<T>(v);
  }
}

cudaError_t launch_gen(void* out, int kind, int layer, int expert, int64_t rows, int64_t cols,
                       int64_t fan_in, int d, int F, uint64_t seed, WType wt, cudaStream_t s) {
  const int grid = num_sms() * 8, block = 256;
  if (kind == 0) {
    const uint64_t b1 = stream_base(seed, tensor_id(3, layer, expert));
    const uint64_t b3 = stream_base(seed, tensor_id(4, layer, expert));
    const uint64_t b2 = stream_base(seed, tensor_id(5, layer, expert));
    const float sd = fan_in_scale(d), sf = fan_in_scale(F);
    if (wt == W_BF16) gen_blob_kernel<__nv_bfloat16><<<grid, block, 0, s>>>((__nv_bfloat16*)out, b1, b3, b2, d, F, sd, sf);
    else if (wt == W_F32) gen_blob_kernel<float><<<grid, block, 0, s>>>((float*)out, b1, b3, b2, d, F, sd, sf);
    else return cudaErrorInvalidValue;
  } else {
    const uint64_t b = stream_base(seed, tensor_id(kind, layer, expert));
    const float sc = fan_in_scale(fan_in);
    if (wt == W_BF16) gen_plain_kernel<__nv_bfloat16><<<grid, block, 0, s>>>((__nv_bfloat16*)out, b, rows * cols, sc);
    else if (wt == W_F32) gen_plain_kernel<float><<<grid, block, 0, s>>>((float*)out, b, rows * cols, sc);
    else return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- BF16 shadow of an FP32 model
__global__ void f32_to_bf16_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn(in[i]);
}

cudaError_t launch_f32_to_bf16(const float* in, void* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  f32_to_bf16_kernel<<<num_sms() * 8, 256, 0, s>>>(in, reinterpret_cast<__nv_bfloat16*>(out), n);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- INT8-row quantiser
template <typename T> __device__ __forceinline__ float ld_f(const T* p, long long i);
template <> __device__ __forceinline__ float ld_f<__nv_bfloat16>(const __nv_bfloat16* p, long long i) { return __bfloat162float(p[i]); }
template <> __device__ __forceinline__ float ld_f<float>(const float* p, long long i) { return p[i]; }

template <typename T, bool BIASED = false>
__global__ void __launch_bounds__(256) quantize_rows_kernel(const T* __restrict__ w, long long C,
                                                            int8_t* __restrict__ q, float* __restrict__ sc) {
  __shared__ float red[8];
  const long long r = blockIdx.x;
  const T* wr = w + r * C;
  float m = 0.f;
  for (long long j = threadIdx.x; j < C; j += blockDim.x) m = fmaxf(m, fabsf(ld_f<T>(wr, j)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = fmaxf(t, red[i]);
    red[0] = t;
  }
  __syncthreads();
  m = red[0];
  if (threadIdx.x == 0) sc[r] = m > 0.f ? __double2float_rn((double)m / 127.0) : 1.0f;
  const double md = (double)m;
  for (long long j = threadIdx.x; j < C; j += blockDim.x) {
    int8_t code = 0;
    if (m > 0.f) {
      int qi = __double2int_rn(((double)ld_f<T>(wr, j) * 127.0) / md);
      qi = qi > 127 ? 127 : (qi < -127 ? -127 : qi);
      code = (int8_t)qi;
    }
    q[r * C + j] = BIASED ? (int8_t)(uint8_t)(code + 128) : code;
  }
}

cudaError_t launch_quantize(const void* w, int64_t R, int64_t C, WType wt, int8_t* q, float* sc,
                            cudaStream_t s, bool biased) {
  if (R <= 0) return cudaSuccess;
  if (wt == W_BF16 && !biased) quantize_rows_kernel<__nv_bfloat16><<<(unsigned)R, 256, 0, s>>>((const __nv_bfloat16*)w, C, q, sc);
  else if (wt == W_BF16) quantize_rows_kernel<__nv_bfloat16, true><<<(unsigned)R, 256, 0, s>>>((const __nv_bfloat16*)w, C, q, sc);
  else if (wt == W_F32 && !biased) quantize_rows_kernel<float><<<(unsigned)R, 256, 0, s>>>((const float*)w, C, q, sc);
  else if (wt == W_F32) quantize_rows_kernel<float, true><<<(unsigned)R, 256, 0, s>>>((const float*)w, C, q, sc);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- NF4 blockwise quantiser
// Reading Q27 (QLoRA NF4, blocks of 64 along a row, fp32 absmax): one warp per block, two weights
// per lane; x = w / absmax in fp64 and the nearest code by |x - c_i| in fp64 (lower index on an
// exact tie), so the decision is the oracle's bit for bit. Zero block -> code 7 (0.0).
__constant__ float kNF4Q[16] = {
    -1.0f, -0.6961928009986877f, -0.5250730514526367f, -0.39491748809814453f,
    -0.28444138169288635f, -0.18477343022823334f, -0.09105003625154495f, 0.0f,
    0.07958029955625534f, 0.16093020141124725f, 0.24611230194568634f, 0.33791524171829224f,
    0.44070982933044434f, 0.5626170039176941f, 0.7229568362236023f, 1.0f};

__device__ __forceinline__ uint32_t nf4_code(double x) {
  uint32_t best = 0;
  double bd = fabs(x - (double)kNF4Q[0]);
#pragma unroll
  for (int i = 1; i < 16; ++i) {
    const double di = fabs(x - (double)kNF4Q[i]);
    if (di < bd) { bd = di; best = (uint32_t)i; }
  }
  return best;
}

template <typename T>
__global__ void __launch_bounds__(256) quantize_nf4_kernel(const T* __restrict__ w, long long R, long long C,
                                                           uint8_t* __restrict__ q, float* __restrict__ absmax) {
  const long long nb = R * (C / 64);
  const int lane = threadIdx.x & 31;
  for (long long blk = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; blk < nb;
       blk += ((long long)gridDim.x * blockDim.x) >> 5) {
    const long long r = blk / (C / 64), cb = blk - r * (C / 64);
    const long long o = r * C + cb * 64 + 2 * lane;
    const float v0 = ld_f<T>(w, o), v1 = ld_f<T>(w, o + 1);
    float m = fmaxf(fabsf(v0), fabsf(v1));
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, s));
    uint32_t c0 = 7, c1 = 7;
    if (m > 0.f) {
      c0 = nf4_code((double)v0 / (double)m);
      c1 = nf4_code((double)v1 / (double)m);
    }
    q[o >> 1] = (uint8_t)(c0 | (c1 << 4));
    if (lane == 0) absmax[blk] = m;
  }
}

cudaError_t launch_quantize_nf4(const void* w, int64_t R, int64_t C, WType wt, uint8_t* q, float* absmax,
                                cudaStream_t s) {
  if (R <= 0) return cudaSuccess;
  if (C % 64) return cudaErrorInvalidValue;
  const int grid = num_sms() * 8;
  if (wt == W_BF16) quantize_nf4_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>((const __nv_bfloat16*)w, R, C, q, absmax);
  else if (wt == W_F32) quantize_nf4_kernel<float><<<grid, 256, 0, s>>>((const float*)w, R, C, q, absmax);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- FP8 (E4M3) row quantiser
// Reading Q28: s = fl32(max|w| / 448) (fp64 quotient), x = fl32(w / s) (fp64 quotient), code =
// E4M3 RNE with saturation (the hardware conversion); zero row -> codes 0, s = 1.
template <typename T>
__global__ void __launch_bounds__(256) quantize_fp8_kernel(const T* __restrict__ w, long long C,
                                                           uint8_t* __restrict__ q, float* __restrict__ sc) {
  __shared__ float red[8];
  const long long r = blockIdx.x;
  const T* wr = w + r * C;
  float m = 0.f;
  for (long long j = threadIdx.x; j < C; j += blockDim.x) m = fmaxf(m, fabsf(ld_f<T>(wr, j)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = fmaxf(t, red[i]);
    red[0] = t;
  }
  __syncthreads();
  m = red[0];
  const float s = m > 0.f ? __double2float_rn((double)m / 448.0) : 1.0f;
  if (threadIdx.x == 0) sc[r] = s;
  for (long long j = threadIdx.x; j < C; j += blockDim.x) {
    uint8_t code = 0;
    if (m > 0.f) {
      const float x = __double2float_rn((double)ld_f<T>(wr, j) / (double)s);
      code = (uint8_t)__nv_cvt_float_to_fp8(x, __NV_SATFINITE, __NV_E4M3);
    }
    q[r * C + j] = code;
  }
}

cudaError_t launch_quantize_fp8(const void* w, int64_t R, int64_t C, WType wt, uint8_t* q, float* s, cudaStream_t st) {
  if (R <= 0) return cudaSuccess;
  if (wt == W_BF16) quantize_fp8_kernel<__nv_bfloat16><<<(unsigned)R, 256, 0, st>>>((const __nv_bfloat16*)w, C, q, s);
  else if (wt == W_F32) quantize_fp8_kernel<float><<<(unsigned)R, 256, 0, st>>>((const float*)w, C, q, s);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace odmoe
