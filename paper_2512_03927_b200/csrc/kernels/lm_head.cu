// Final RMSNorm + LM-head GEMV + greedy argmax, and the token
// embedding gather (a1). The LM head is HBM-bound (262 MB bf16 at the Mixtral shape): one CTA
// per SM streams a balanced contiguous row range with 16-byte loads; each CTA normalises h
// itself (16 KB from L2) so no extra launch is needed; the argmax is a deterministic two-level
// max over (logit, -id) keys: per-CTA partial keys, then the last CTA to finish (ticket)
// reduces them. Lowest id wins ties.
#include "common.cuh"
#include "kernels.h"

#include <cstdlib>

namespace odmoe {

constexpr int kLmWarps = 8;
constexpr int kLmThreads = kLmWarps * 32;

// Orderable 64-bit key: high word = monotone image of the float, low word = ~id (lower id wins).
__device__ __forceinline__ unsigned long long argmax_key(float v, int id) {
  uint32_t b = __float_as_uint(v);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return ((unsigned long long)b << 32) | (unsigned long long)(~(uint32_t)id);
}

template <typename WT, int U>
__global__ void __launch_bounds__(kLmThreads, 1)
lm_head_kernel(const float* __restrict__ h, const WT* __restrict__ W, const float* __restrict__ sc, int V, int d,
               float eps, float* __restrict__ logits, unsigned long long* __restrict__ partial,
               unsigned int* __restrict__ ticket, int32_t* __restrict__ token_out) {
  extern __shared__ __align__(16) float us[];
  __shared__ float red[kLmWarps];
  __shared__ unsigned long long kbest[kLmWarps];
  __shared__ bool is_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float ss = 0.f;
  for (int j = tid * 4; j < d; j += kLmThreads * 4) {
    const float4 hv = *reinterpret_cast<const float4*>(h + j);
    *reinterpret_cast<float4*>(us + j) = hv;
    ss = fmaf(hv.x, hv.x, ss); ss = fmaf(hv.y, hv.y, ss);
    ss = fmaf(hv.z, hv.z, ss); ss = fmaf(hv.w, hv.w, ss);
  }
  ss = warp_sum(ss);
  if (lane == 0) red[warp] = ss;
  __syncthreads();
  if (warp == 0) {
    float t = lane < kLmWarps ? red[lane] : 0.f;
    t = warp_sum(t);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  const float rstd = 1.0f / sqrtf(red[0] / (float)d + eps);
  constexpr bool kF32 = std::is_same<WT, float>::value;
  for (int j = tid; j < d; j += kLmThreads) {
    const float v = us[j] * rstd;
    us[j] = kF32 ? v : __bfloat162float(__float2bfloat16_rn(v));
  }
  __syncthreads();

  constexpr int N = WTraits<WT>::kPer16B;
  const int C = d / N;
  long long rb, re;
  split_range(V, gridDim.x, blockIdx.x, rb, re);
  unsigned long long best = 0ull;
  for (long long r = rb + warp; r < re; r += kLmWarps) {
    const uint4* wr = reinterpret_cast<const uint4*>(W + (size_t)r * d);
    float acc = 0.f;
    for (int c0 = 0; c0 < C; c0 += 32 * U) {
      uint4 x[U];
#pragma unroll
      for (int i = 0; i < U; ++i) {
        const int c = c0 + i * 32 + lane;
        if (c < C) x[i] = ld_stream(wr + c);
      }
#pragma unroll
      for (int i = 0; i < U; ++i) {
        const int c = c0 + i * 32 + lane;
        if (c < C) acc += dot16<WT>(x[i], us + c * N);
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) {
      if (sc) acc *= sc[r];
      if (logits) logits[r] = acc;
      const unsigned long long key = argmax_key(acc, (int)r);
      best = key > best ? key : best;
    }
  }
  if (lane == 0) kbest[warp] = best;
  __syncthreads();
  if (tid == 0) {
    unsigned long long b = kbest[0];
    for (int w = 1; w < kLmWarps; ++w) b = kbest[w] > b ? kbest[w] : b;
    partial[blockIdx.x] = b;
    __threadfence();
    const unsigned int t = atomicAdd(ticket, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (is_last && tid == 0) {
    __threadfence();
    unsigned long long b = 0ull;
    for (unsigned int i = 0; i < gridDim.x; ++i) {
      const unsigned long long p = *((volatile unsigned long long*)partial + i);
      b = p > b ? p : b;
    }
    *token_out = (int32_t)(~(uint32_t)(b & 0xffffffffull));
    *ticket = 0u;
  }
}

template <typename WT>
static cudaError_t lm_impl(const float* h, const void* W, const float* sc, int V, int d, float eps,
                           int32_t* token_out, float* logits, void* scratch, cudaStream_t s) {
  constexpr int U = 16;
  const int sms = num_sms();
  const int grid = V / 8 < sms ? (V / 8 > 0 ? V / 8 : 1) : sms;
  unsigned long long* partial = reinterpret_cast<unsigned long long*>(scratch);
  unsigned int* ticket = reinterpret_cast<unsigned int*>(partial + 1024);
  const size_t smem = (size_t)d * sizeof(float);
  auto kern = lm_head_kernel<WT, U>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<grid, kLmThreads, smem, s>>>(h, (const WT*)W, sc, V, d, eps, logits, partial, ticket, token_out);
  return cudaGetLastError();
}

cudaError_t launch_lm_head(const float* h, const void* W, WType wt, int V, int d, float eps,
                           int32_t* token_out, float* logits, void* scratch, cudaStream_t s, bool pdl,
                           const float* scales) {
  if (stream_ok(wt, d)) {
    if (gemv_engine() == 2 || wt == W_I8)
      return launch_lm_head_flat(h, W, wt, V, d, eps, token_out, logits, scratch, s, pdl, scales);
  }
  switch (wt) {
    case W_BF16: return lm_impl<__nv_bfloat16>(h, W, nullptr, V, d, eps, token_out, logits, scratch, s);
    case W_F32: return lm_impl<float>(h, W, nullptr, V, d, eps, token_out, logits, scratch, s);
    case W_I8: return lm_impl<int8_t>(h, W, scales, V, d, eps, token_out, logits, scratch, s);
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------- a1 embedding gather
template <typename WT>
__global__ void embed_kernel(const WT* __restrict__ emb, const float* __restrict__ sc,
                             const int32_t* __restrict__ token, int d, float* __restrict__ h) {
  const long long t = *token;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < d; j += gridDim.x * blockDim.x) {
    float v;
    if constexpr (std::is_same<WT, __nv_bfloat16>::value) v = __bfloat162float(emb[t * d + j]);
    else if constexpr (std::is_same<WT, float>::value) v = emb[t * d + j];
    else v = sc[t] * (float)emb[t * d + j];
    h[j] = v;
  }
}

// Batched embedding gather for prefill: h[t] = Emb[tokens[t]].
template <typename WT>
__global__ void embed_rows_kernel(const WT* __restrict__ emb, const int32_t* __restrict__ tokens, int d,
                                  float* __restrict__ h) {
  const long long t = tokens[blockIdx.x];
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    float v;
    if constexpr (std::is_same<WT, __nv_bfloat16>::value) v = __bfloat162float(emb[t * d + j]);
    else v = emb[t * d + j];
    h[(size_t)blockIdx.x * d + j] = v;
  }
}

cudaError_t launch_embed_rows(const void* emb, WType wt, const int32_t* tokens, int T, int d, float* h,
                              cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  if (wt == W_BF16) embed_rows_kernel<__nv_bfloat16><<<T, 256, 0, s>>>((const __nv_bfloat16*)emb, tokens, d, h);
  else if (wt == W_F32) embed_rows_kernel<float><<<T, 256, 0, s>>>((const float*)emb, tokens, d, h);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_embed(const void* emb, const float* emb_scale, WType wt, const int32_t* token,
                         int d, float* h, cudaStream_t s) {
  const int grid = (d + 255) / 256 < 16 ? (d + 255) / 256 : 16;
  switch (wt) {
    case W_BF16: embed_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>((const __nv_bfloat16*)emb, nullptr, token, d, h); break;
    case W_F32: embed_kernel<float><<<grid, 256, 0, s>>>((const float*)emb, nullptr, token, d, h); break;
    case W_I8: embed_kernel<int8_t><<<grid, 256, 0, s>>>((const int8_t*)emb, emb_scale, token, d, h); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace odmoe
