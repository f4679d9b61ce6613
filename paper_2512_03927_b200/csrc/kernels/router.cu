// Fused residual-combine + RMSNorm + router GEMV + softmax/top-k + renormalisation
// (SURVEY §8(a) a2+a3; readings Q2, Q3, Q6, Q7).
//
// One CTA per token row. For decode (m = 1) this is a latency-bound single-CTA kernel:
// it reads the fp32 residual (16 KB at d=4096), the k partial expert outputs and the
// E x d gate matrix (64 KB bf16), all with 16-byte loads; reductions are warp shuffles.
#include "common.cuh"
#include "kernels.h"

namespace odmoe {

constexpr int kRouterThreads = 256;
constexpr int kRouterWarps = kRouterThreads / 32;

template <typename WT>
__global__ void __launch_bounds__(kRouterThreads) router_kernel(
    float* __restrict__ h, const float* const* __restrict__ y_add, int n_add,
    const WT* __restrict__ gamma, const WT* __restrict__ wg, const float* __restrict__ wg_scale,
    int E, int d, int k, float eps, void* __restrict__ u_out, int32_t* __restrict__ ids,
    float* __restrict__ w, float* __restrict__ logits, int32_t* __restrict__ flag) {
  extern __shared__ __align__(16) float us[];  // d floats: the rounded normalised input
  __shared__ float red[kRouterWarps];
  __shared__ float lg[kMaxE];
  const int row = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* hr = h + (size_t)row * d;

  // Pass 1: h = h + (y_0 + y_1 + ...), partials summed first in the given order so that a
  // pre-reduced sum (NCCL reduce at N > 1) gives the same bits as the 1-GPU combine.
  float ss = 0.f;
  for (int j = tid * 4; j < d; j += kRouterThreads * 4) {
    float4 hv = *reinterpret_cast<const float4*>(hr + j);
    if (n_add > 0) {
      float4 s = *reinterpret_cast<const float4*>(y_add[0] + (size_t)row * d + j);
      for (int a = 1; a < n_add; ++a) {
        const float4 t = *reinterpret_cast<const float4*>(y_add[a] + (size_t)row * d + j);
        s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;
      }
      hv.x += s.x; hv.y += s.y; hv.z += s.z; hv.w += s.w;
      *reinterpret_cast<float4*>(hr + j) = hv;
    }
    *reinterpret_cast<float4*>(us + j) = hv;
    ss = fmaf(hv.x, hv.x, ss); ss = fmaf(hv.y, hv.y, ss);
    ss = fmaf(hv.z, hv.z, ss); ss = fmaf(hv.w, hv.w, ss);
  }
  ss = warp_sum(ss);
  if (lane == 0) red[warp] = ss;
  __syncthreads();
  if (warp == 0) {
    float t = lane < kRouterWarps ? red[lane] : 0.f;
    t = warp_sum(t);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  const float rstd = 1.0f / sqrtf(red[0] / (float)d + eps);

  // Pass 2: u = h * rstd * gamma, rounded to the activation dtype (bf16 unless fp32 weights).
  constexpr bool kF32 = std::is_same<WT, float>::value;
  for (int j = tid; j < d; j += kRouterThreads) {
    float g = 1.f;
    if (gamma != nullptr) {
      if constexpr (kF32) g = gamma[j];
      else if constexpr (std::is_same<WT, __nv_bfloat16>::value) g = __bfloat162float(gamma[j]);
    }
    const float v = us[j] * rstd * g;
    if constexpr (kF32) {
      reinterpret_cast<float*>(u_out)[(size_t)row * d + j] = v;
      us[j] = v;
    } else {
      const __nv_bfloat16 b = __float2bfloat16_rn(v);
      reinterpret_cast<__nv_bfloat16*>(u_out)[(size_t)row * d + j] = b;
      us[j] = __bfloat162float(b);
    }
  }
  __syncthreads();

  // Router GEMV: warp per expert row, 16-byte chunks, shuffle reduction.
  constexpr int N = WTraits<WT>::kPer16B;
  const int C = d / N;
  for (int e = warp; e < E; e += kRouterWarps) {
    const uint4* wr = reinterpret_cast<const uint4*>(wg + (size_t)e * d);
    float acc = 0.f;
    for (int c = lane; c < C; c += 32) acc += dot16<WT>(wr[c], us + c * N);
    acc = warp_sum(acc);
    if (lane == 0) lg[e] = wg_scale ? acc * wg_scale[e] : acc;
  }
  __syncthreads();

  // Top-k (logit descending, lower index on ties) + softmax over the selected logits.
  if (tid == 0) {
    int sel[kMaxK];
    bool bad = false;
    unsigned long long taken = 0ull;
    for (int e = 0; e < E; ++e) bad |= !isfinite(lg[e]);
    for (int i = 0; i < k; ++i) {
      int bi = -1;
      float bv = 0.f;
      for (int e = 0; e < E; ++e) {
        if (taken >> e & 1ull) continue;
        if (bi < 0 || lg[e] > bv) { bi = e; bv = lg[e]; }
      }
      sel[i] = bi;
      taken |= 1ull << bi;
    }
    const float m = lg[sel[0]];
    float ex[kMaxK], sum = 0.f;
    for (int i = 0; i < k; ++i) { ex[i] = expf(lg[sel[i]] - m); sum += ex[i]; }
    for (int i = 0; i < k; ++i) {
      ids[(size_t)row * k + i] = sel[i];
      w[(size_t)row * k + i] = ex[i] / sum;
    }
    if (logits) for (int e = 0; e < E; ++e) logits[(size_t)row * E + e] = lg[e];
    if (bad && flag) *flag = 1;
  }
}

// Residual combine only (after the last layer): h += (y_0 + y_1 + ...), same order as the router.
__global__ void combine_kernel(float* __restrict__ h, const float* const* __restrict__ y_add, int n_add, int d) {
  for (int j = (blockIdx.x * blockDim.x + threadIdx.x) * 4; j < d; j += gridDim.x * blockDim.x * 4) {
    float4 hv = *reinterpret_cast<const float4*>(h + j);
    float4 s = *reinterpret_cast<const float4*>(y_add[0] + j);
    for (int a = 1; a < n_add; ++a) {
      const float4 t = *reinterpret_cast<const float4*>(y_add[a] + j);
      s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;
    }
    hv.x += s.x; hv.y += s.y; hv.z += s.z; hv.w += s.w;
    *reinterpret_cast<float4*>(h + j) = hv;
  }
}

cudaError_t launch_combine(float* h, const float* const* y_add, int n_add, int d, cudaStream_t s) {
  if (n_add <= 0) return cudaSuccess;
  const int grid = (d / 4 + 255) / 256 < 8 ? (d / 4 + 255) / 256 : 8;
  combine_kernel<<<grid > 0 ? grid : 1, 256, 0, s>>>(h, y_add, n_add, d);
  return cudaGetLastError();
}

cudaError_t launch_router(float* h, const float* const* y_add, int n_add, const void* gamma,
                          const void* w_gate, const float* wg_scale, WType wt, int m, int E, int d,
                          int k, float eps, void* u_out, int32_t* ids, float* w, float* logits,
                          int32_t* flag, cudaStream_t s) {
  const size_t smem = (size_t)d * sizeof(float);
  dim3 grid(m), block(kRouterThreads);
  switch (wt) {
    case W_BF16:
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(router_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      router_kernel<__nv_bfloat16><<<grid, block, smem, s>>>(
          h, y_add, n_add, (const __nv_bfloat16*)gamma, (const __nv_bfloat16*)w_gate, nullptr, E, d,
          k, eps, u_out, ids, w, logits, flag);
      break;
    case W_F32:
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(router_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      router_kernel<float><<<grid, block, smem, s>>>(h, y_add, n_add, (const float*)gamma,
                                                     (const float*)w_gate, nullptr, E, d, k, eps,
                                                     u_out, ids, w, logits, flag);
      break;
    case W_I8:
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(router_kernel<int8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      router_kernel<int8_t><<<grid, block, smem, s>>>(h, y_add, n_add, nullptr,
                                                      (const int8_t*)w_gate, wg_scale, E, d, k, eps,
                                                      u_out, ids, w, logits, flag);
      break;
  }
  return cudaGetLastError();
}

}  // namespace odmoe
