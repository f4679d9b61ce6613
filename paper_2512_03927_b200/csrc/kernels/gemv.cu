// Batch-1 expert SwiGLU FFN as two HBM-streaming GEMV kernels (
// readings Q1, Q8). Also the shadow's INT8-row variant (a4; Q9).
//
// Roofline: both kernels are HBM-bound (arithmetic intensity 1 FMA per weight element).
// Design for B200 (148 SMs, HBM3e):
//  * one CTA per SM, each CTA owns a CONTIGUOUS, balanced range of rows, so every SM streams
//    the same number of bytes (no wave-quantisation tail) with DRAM-page-friendly addresses;
//  * 16-byte ld.global.nc.L1::no_allocate loads, U chunks per lane issued back to back
//    (>= 64 KB in flight per SM, above the Little's-law need of ~35 KB);
//  * activations staged once per CTA in shared memory as fp32;
//  * W13 rows are gate/up interleaved so one warp produces a_f = silu(g_f) * v_f directly;
//  * W2 rows are split along K across the CTA's warps (split-K inside the CTA) and reduced
//    through shared memory in a fixed order: deterministic, no atomics.
#include "common.cuh"
#include "kernels.h"

#include <cstdlib>

namespace odmoe {

constexpr int kGemvWarps = 8;
constexpr int kGemvThreads = kGemvWarps * 32;

// Resolve an ExpertRef on the device. Direct mode: `blob`/`scales` point at the matrix itself.
// Indirect mode: table entries point at the whole expert blob; `second` selects W2 (offset
// 2*F*d elements, scales offset 2F).
template <typename WT>
__device__ __forceinline__ void resolve(const ExpertRef& ex, bool second, int d, int F,
                                        const WT*& w, const float*& sc, int& pick) {
  pick = ex.sel;
  if (ex.tbl == nullptr) {
    w = reinterpret_cast<const WT*>(ex.blob);
    sc = ex.scales;
    return;
  }
  if (ex.sorted) {
    for (int j = 0; j < ex.k; ++j) {
      int rank = 0;
      for (int i = 0; i < ex.k; ++i) rank += ex.ids[i] < ex.ids[j];
      if (rank == ex.sel) pick = j;
    }
  }
  const int id = ex.base + ex.ids[pick];
  w = reinterpret_cast<const WT*>(ex.tbl[id]) + (second ? 2LL * F * d : 0LL);
  sc = ex.stbl ? ex.stbl[id] + (second ? 2 * F : 0) : nullptr;
}

template <typename WT, int U>
__global__ void __launch_bounds__(kGemvThreads, 1)
w13_swiglu_kernel(const ExpertRef ex, const void* __restrict__ u, int u_f32, float* __restrict__ a,
                  int d, int F) {
  extern __shared__ __align__(16) float xs[];
  const WT* w13;
  const float* s13;
  int pick;
  resolve<WT>(ex, false, d, F, w13, s13, pick);
  load_act_to_smem(xs, u, d, u_f32);
  __syncthreads();
  constexpr int N = WTraits<WT>::kPer16B;
  const int C = d / N;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long pb, pe;
  split_range(F, gridDim.x, blockIdx.x, pb, pe);
  for (long long p = pb + warp; p < pe; p += kGemvWarps) {
    const uint4* r0 = reinterpret_cast<const uint4*>(w13 + (size_t)(2 * p) * d);
    const uint4* r1 = r0 + C;
    float g = 0.f, v = 0.f;
    for (int c0 = 0; c0 < C; c0 += 32 * U) {
      uint4 x0[U], x1[U];
#pragma unroll
      for (int i = 0; i < U; ++i) {
        const int c = c0 + i * 32 + lane;
        if (c < C) { x0[i] = ld_stream(r0 + c); x1[i] = ld_stream(r1 + c); }
      }
#pragma unroll
      for (int i = 0; i < U; ++i) {
        const int c = c0 + i * 32 + lane;
        if (c < C) {
          g += dot16<WT>(x0[i], xs + c * N);
          v += dot16<WT>(x1[i], xs + c * N);
        }
      }
    }
    g = warp_sum(g);
    v = warp_sum(v);
    if (lane == 0) {
      if (s13 != nullptr) { g *= s13[2 * p]; v *= s13[2 * p + 1]; }
      a[p] = silu_mul(g, v);
    }
  }
}

template <typename WT, int RU, int UK>
__global__ void __launch_bounds__(kGemvThreads, 1)
w2_gemv_kernel(const ExpertRef ex, const float* __restrict__ a, const float* __restrict__ gate_w,
               float* __restrict__ y, int d, int F, int rows_cap) {
  extern __shared__ __align__(16) float sm[];
  const WT* w2;
  const float* s2;
  int gate_idx;
  resolve<WT>(ex, true, d, F, w2, s2, gate_idx);
  float* xs = sm;                     // F floats
  float* part = sm + F;               // [kGemvWarps][rows_cap]
  load_act_to_smem(xs, a, F, 1);
  __syncthreads();
  constexpr int N = WTraits<WT>::kPer16B;
  const int C = F / N;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long rb, re;
  split_range(d, gridDim.x, blockIdx.x, rb, re);
  const int nrows = (int)(re - rb);
  for (int r0 = 0; r0 < nrows; r0 += RU) {
    float acc[RU];
#pragma unroll
    for (int rr = 0; rr < RU; ++rr) acc[rr] = 0.f;
    for (int c0 = warp * 32 + lane; c0 < C; c0 += kGemvWarps * 32 * UK) {
      uint4 wv[RU][UK];
#pragma unroll
      for (int rr = 0; rr < RU; ++rr)
#pragma unroll
        for (int i = 0; i < UK; ++i) {
          const int c = c0 + i * kGemvWarps * 32;
          if (r0 + rr < nrows && c < C)
            wv[rr][i] = ld_stream(reinterpret_cast<const uint4*>(w2 + (size_t)(rb + r0 + rr) * F) + c);
        }
#pragma unroll
      for (int rr = 0; rr < RU; ++rr)
#pragma unroll
        for (int i = 0; i < UK; ++i) {
          const int c = c0 + i * kGemvWarps * 32;
          if (r0 + rr < nrows && c < C) acc[rr] += dot16<WT>(wv[rr][i], xs + c * N);
        }
    }
#pragma unroll
    for (int rr = 0; rr < RU; ++rr) {
      const float t = warp_sum(acc[rr]);
      if (lane == 0 && r0 + rr < nrows) part[warp * rows_cap + r0 + rr] = t;
    }
  }
  __syncthreads();
  const float gw = gate_w ? gate_w[gate_idx] : 1.f;
  for (int r = threadIdx.x; r < nrows; r += kGemvThreads) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < kGemvWarps; ++w) s += part[w * rows_cap + r];
    if (s2 != nullptr) s *= s2[rb + r];
    y[rb + r] = gw * s;
  }
}

static int gemv_grid(long long units) {
  const int sms = num_sms();
  return (int)(units < sms ? (units > 0 ? units : 1) : sms);
}

template <typename WT>
static cudaError_t w13_impl(const ExpertRef& ex, const void* u, int u_f32, float* a, int d, int F,
                            cudaStream_t s) {
  constexpr int U = sizeof(WT) == 4 ? 16 : (sizeof(WT) == 2 ? 16 : 8);
  const size_t smem = (size_t)d * sizeof(float);
  auto kern = w13_swiglu_kernel<WT, U>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = gemv_grid(F / 8 > 0 ? F / 8 : 1);
  kern<<<grid, kGemvThreads, smem, s>>>(ex, u, u_f32, a, d, F);
  return cudaGetLastError();
}

template <typename WT>
static cudaError_t w2_impl(const ExpertRef& ex, const float* a, const float* gate_w, float* y, int d,
                           int F, cudaStream_t s) {
  constexpr int RU = 2;
  constexpr int UK = sizeof(WT) == 1 ? 4 : 8;
  const int grid = gemv_grid(d / 4 > 0 ? d / 4 : 1);
  const int rows_cap = (d + grid - 1) / grid + 1;
  const size_t smem = ((size_t)F + (size_t)kGemvWarps * rows_cap) * sizeof(float);
  auto kern = w2_gemv_kernel<WT, RU, UK>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<grid, kGemvThreads, smem, s>>>(ex, a, gate_w, y, d, F, rows_cap);
  return cudaGetLastError();
}

// GEMV engine selection: flat (default) | tma | ldg (ODMOE_GEMV env var, for A/B measurements).
int gemv_engine() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ODMOE_GEMV");
    v = (e && e[0] == 'l') ? 0 : 2;
  }
  return v;
}

// Whether the flat engine handles a [R, C] matrix of type wt (rows must be whole 512-byte groups;
// activations must fit in shared memory).
bool stream_ok(WType wt, int C) {
  if (wt == W_NF4) return C % 1024 == 0 && (long long)C * 4 <= 64 * 1024;  // flat engine only
  const int esz = wt == W_F32 ? 4 : (wt == W_BF16 ? 2 : 1);
  return ((long long)C * esz) % 512 == 0 && (long long)C * 4 <= 64 * 1024;
}

cudaError_t launch_w13(ExpertRef ex, WType wt, const void* u, int u_f32, float* a, int d, int F,
                       cudaStream_t s, bool pdl) {
  if (wt == W_I8P) return launch_mma_shadow(1, &ex, 0, u, nullptr, a, d, F, s, pdl);
  if (wt == W_U8)  // flat engine only (the engine picks W_U8 only where it applies)
    return stream_ok(wt, d) ? launch_w13_flat(ex, wt, u, u_f32, a, d, F, s, pdl) : cudaErrorInvalidValue;
  if (wt == W_NF4 || wt == W_F8)
    return stream_ok(wt, d) ? launch_w13_flat(ex, wt, u, u_f32, a, d, F, s, pdl)
                            : launch_lowbit_small(ex, wt, 0, u, u_f32, d, F, nullptr, a, s);
  if (stream_ok(wt, d)) {
    if (gemv_engine() == 2) return launch_w13_flat(ex, wt, u, u_f32, a, d, F, s, pdl);
  }
  switch (wt) {
    case W_BF16: return w13_impl<__nv_bfloat16>(ex, u, u_f32, a, d, F, s);
    case W_F32: return w13_impl<float>(ex, u, u_f32, a, d, F, s);
    case W_I8: return w13_impl<int8_t>(ex, u, u_f32, a, d, F, s);
    default: break;
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_w2(ExpertRef ex, WType wt, const float* a, const float* gate_w, float* y, int d,
                      int F, cudaStream_t s, bool pdl) {
  if (wt == W_I8P) return launch_mma_shadow(1, &ex, 1, a, gate_w, y, d, F, s, pdl);
  if (wt == W_U8)
    return stream_ok(wt, F) ? launch_w2_flat(ex, wt, a, gate_w, y, d, F, s, pdl) : cudaErrorInvalidValue;
  if (wt == W_NF4 || wt == W_F8)
    return stream_ok(wt, F) ? launch_w2_flat(ex, wt, a, gate_w, y, d, F, s, pdl)
                            : launch_lowbit_small(ex, wt, 1, a, 1, d, F, gate_w, y, s);
  if (stream_ok(wt, F)) {
    if (gemv_engine() == 2) return launch_w2_flat(ex, wt, a, gate_w, y, d, F, s, pdl);
  }
  switch (wt) {
    case W_BF16: return w2_impl<__nv_bfloat16>(ex, a, gate_w, y, d, F, s);
    case W_F32: return w2_impl<float>(ex, a, gate_w, y, d, F, s);
    case W_I8: return w2_impl<int8_t>(ex, a, gate_w, y, d, F, s);
    default: break;
  }
  return cudaErrorInvalidValue;
}

bool use_fused_expert() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ODMOE_FUSED");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1 && gemv_engine() == 2;
}

// SMs a one-CTA-per-SM streaming grid may count on (flat engine). At N > 1 the engine reserves one:
// the prediction communicator's broadcasts (one CTA, maxCTAs = 1) spin on the shadow stream, and a
// grid of all 148 CTAs would leave one CTA waiting for that SM until the broadcast completes.
static int g_sm_reserve[64] = {0};
void set_stream_sm_reserve(int n) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64) g_sm_reserve[dev] = n < 0 ? 0 : n;
}
int stream_grid_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  const int r = (dev >= 0 && dev < 64) ? g_sm_reserve[dev] : 0;
  const int n = num_sms() - r;
  return n > 0 ? n : 1;
}

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cached[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}

}  // namespace odmoe
