// Prefill token permutation around the grouped expert GEMM ("embeddings
// are grouped by their desired experts"; S:330 coverage: every (token, expert) pair exactly once).
//
//  * route_group_kernel: stable counting sort of the T*k (token, slot) pairs by expert id in ONE
//    CTA (one warp per expert, ballot + popc prefix => stable in pair order), writing expert
//    offsets, the source pair of every grouped row, its gate weight and the inverse map.
//  * gather_rows_kernel: X_perm[r] = u[src_pair[r] / k] (16-byte copies).
//  * scatter_combine_kernel: h[t] += (y[inv[t,0]] + ... + y[inv[t,k-1]]) in router rank order,
//    the same arithmetic as the decode router's residual pass (bitwise-consistent combine).
#include "common.cuh"
#include "kernels.h"

namespace odmoe {

__global__ void route_group_kernel(const int32_t* __restrict__ ids, const float* __restrict__ w, int n_pairs,
                                   int E, int32_t* __restrict__ offsets, int32_t* __restrict__ src_pair,
                                   int32_t* __restrict__ inv, float* __restrict__ gate_perm) {
  extern __shared__ int32_t cnt[];  // [E + 1]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int e = warp; e < E; e += nw) {
    int c = 0;
    for (int p0 = 0; p0 < n_pairs; p0 += 32) {
      const int p = p0 + lane;
      const bool m = p < n_pairs && ids[p] == e;
      c += __popc(__ballot_sync(0xffffffffu, m));
    }
    if (lane == 0) cnt[e] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int e = 0; e < E; ++e) { const int c = cnt[e]; cnt[e] = s; offsets[e] = s; s += c; }
    cnt[E] = s;
    offsets[E] = s;
  }
  __syncthreads();
  for (int e = warp; e < E; e += nw) {
    int base = cnt[e];
    for (int p0 = 0; p0 < n_pairs; p0 += 32) {
      const int p = p0 + lane;
      const bool m = p < n_pairs && ids[p] == e;
      const unsigned b = __ballot_sync(0xffffffffu, m);
      if (m) {
        const int r = base + __popc(b & ((1u << lane) - 1u));
        src_pair[r] = p;
        inv[p] = r;
        gate_perm[r] = w[p];
      }
      base += __popc(b);
    }
  }
}

__global__ void gather_rows_kernel(const uint4* __restrict__ u, const int32_t* __restrict__ src_pair, int k,
                                   int row_vecs, uint4* __restrict__ out) {
  const int r = blockIdx.x;
  const int t = src_pair[r] / k;
  for (int i = threadIdx.x; i < row_vecs; i += blockDim.x) out[(size_t)r * row_vecs + i] = u[(size_t)t * row_vecs + i];
}

__global__ void scatter_combine_kernel(float* __restrict__ h, const float* __restrict__ y,
                                       const int32_t* __restrict__ inv, int k, int d, int partial) {
  const int t = blockIdx.x;
  for (int j = threadIdx.x * 4; j < d; j += blockDim.x * 4) {
    float4 s = *reinterpret_cast<const float4*>(y + (size_t)inv[t * k] * d + j);
    for (int a = 1; a < k; ++a) {
      const float4 v = *reinterpret_cast<const float4*>(y + (size_t)inv[t * k + a] * d + j);
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    if (partial) {  // N > 1: this rank's share of the combine, reduced across ranks later
      *reinterpret_cast<float4*>(h + (size_t)t * d + j) = s;
      continue;
    }
    float4 hv = *reinterpret_cast<float4*>(h + (size_t)t * d + j);
    hv.x += s.x; hv.y += s.y; hv.z += s.z; hv.w += s.w;
    *reinterpret_cast<float4*>(h + (size_t)t * d + j) = hv;
  }
}

__global__ void add_rows_kernel(float* __restrict__ h, const float* __restrict__ y, long long n) {
  for (long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 4; i < n; i += (long long)gridDim.x * blockDim.x * 4) {
    float4 a = *reinterpret_cast<float4*>(h + i);
    const float4 b = *reinterpret_cast<const float4*>(y + i);
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    *reinterpret_cast<float4*>(h + i) = a;
  }
}

cudaError_t launch_route_group(const int32_t* ids, const float* w, int n_pairs, int E, int32_t* offsets,
                               int32_t* src_pair, int32_t* inv, float* gate_perm, cudaStream_t s) {
  const int threads = 32 * (E < 32 ? E : 32);
  route_group_kernel<<<1, threads, (E + 1) * sizeof(int32_t), s>>>(ids, w, n_pairs, E, offsets, src_pair, inv, gate_perm);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const void* u, const int32_t* src_pair, int k, int M, int d, void* out,
                               cudaStream_t s) {
  if (M == 0) return cudaSuccess;
  gather_rows_kernel<<<M, 128, 0, s>>>((const uint4*)u, src_pair, k, d * 2 / 16, (uint4*)out);
  return cudaGetLastError();
}

cudaError_t launch_scatter_combine(float* h, const float* y, const int32_t* inv, int T, int k, int d,
                                   int partial, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  scatter_combine_kernel<<<T, 256, 0, s>>>(h, y, inv, k, d, partial);
  return cudaGetLastError();
}

cudaError_t launch_add_rows(float* h, const float* y, long long n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  add_rows_kernel<<<num_sms() * 2, 256, 0, s>>>(h, y, n);
  return cudaGetLastError();
}

}  // namespace odmoe
