// Fused residual-combine + RMSNorm + router GEMV + softmax/top-k + renormalisation
// (SURVEY §8(a) a2+a3; readings Q2, Q3, Q6, Q7).
//
// One CTA per token row. For decode (m = 1) this is a latency-bound single-CTA kernel:
// it reads the fp32 residual (16 KB at d=4096), the k partial expert outputs and the
// E x d gate matrix (64 KB bf16), all with 16-byte loads; reductions are warp shuffles.
#include "common.cuh"
#include "kernels.h"

#include <cooperative_groups.h>

namespace odmoe {

namespace cg = cooperative_groups;

constexpr int kRouterThreads = 256;
constexpr int kRouterWarps = kRouterThreads / 32;

constexpr int kRouterPrefetchMax = 128 * 1024;  // W_g bytes staged in smem by one bulk copy

__device__ __forceinline__ uint32_t r_smem(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// Launch latency hiding (programmatic dependent launch): everything before pdl_wait() may run
// while the previous kernel on the stream is still finishing; pdl_trigger() lets the next kernel
// be scheduled early. Both are no-ops for launches without the PDL attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename WT>
__global__ void __launch_bounds__(kRouterThreads) router_kernel(
    float* __restrict__ h, const float* const* __restrict__ y_add, int n_add,
    const WT* __restrict__ gamma, const WT* __restrict__ wg, const float* __restrict__ wg_scale,
    int E, int d, int k, float eps, void* __restrict__ u_out, int32_t* __restrict__ ids,
    float* __restrict__ w, float* __restrict__ logits, int32_t* __restrict__ flag, int prefetch) {
  extern __shared__ __align__(128) uint8_t rsm[];
  float* us = reinterpret_cast<float*>(rsm);                      // d floats: rounded normalised input
  uint8_t* wsm = rsm + (((size_t)d * sizeof(float) + 127) & ~(size_t)127);  // W_g copy (prefetch)
  __shared__ uint64_t wbar;
  __shared__ float red[kRouterWarps];
  __shared__ float lg[kMaxE];
  const int row = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* hr = h + (size_t)row * d;
  const uint32_t wbytes = (uint32_t)((size_t)E * d * sizeof(WT));

  // W_g does not depend on the previous kernel: start its bulk copy before the dependency wait.
  if (prefetch) {
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(r_smem(&wbar)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(r_smem(&wbar)), "r"(wbytes) : "memory");
      for (uint32_t off = 0; off < wbytes; off += 32768) {
        const uint32_t n = wbytes - off < 32768 ? wbytes - off : 32768;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         r_smem(wsm + off)),
                     "l"(reinterpret_cast<const char*>(wg) + off), "r"(n), "r"(r_smem(&wbar))
                     : "memory");
      }
    }
  }
  pdl_wait();
  pdl_trigger();

  // Pass 1: h = h + (y_0 + y_1 + ...), partials summed first in the given order so that a
  // pre-reduced sum (NCCL reduce at N > 1) gives the same bits as the 1-GPU combine. All loads of
  // a thread are issued before any is used.
  constexpr int kV = 4;  // float4 per thread per batch (covers d = 4096 in one batch)
  float ss = 0.f;
  for (int j0 = tid * 4; j0 < d; j0 += kRouterThreads * 4 * kV) {
    float4 hv[kV], s[kV];
#pragma unroll
    for (int i = 0; i < kV; ++i) {
      const int j = j0 + i * kRouterThreads * 4;
      if (j < d) {
        hv[i] = *reinterpret_cast<const float4*>(hr + j);
        if (n_add > 0) s[i] = *reinterpret_cast<const float4*>(y_add[0] + (size_t)row * d + j);
      }
    }
    for (int a = 1; a < n_add; ++a) {
#pragma unroll
      for (int i = 0; i < kV; ++i) {
        const int j = j0 + i * kRouterThreads * 4;
        if (j < d) {
          const float4 t = *reinterpret_cast<const float4*>(y_add[a] + (size_t)row * d + j);
          s[i].x += t.x; s[i].y += t.y; s[i].z += t.z; s[i].w += t.w;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kV; ++i) {
      const int j = j0 + i * kRouterThreads * 4;
      if (j < d) {
        if (n_add > 0) {
          hv[i].x += s[i].x; hv[i].y += s[i].y; hv[i].z += s[i].z; hv[i].w += s[i].w;
          *reinterpret_cast<float4*>(hr + j) = hv[i];
        }
        *reinterpret_cast<float4*>(us + j) = hv[i];
        ss = fmaf(hv[i].x, hv[i].x, ss); ss = fmaf(hv[i].y, hv[i].y, ss);
        ss = fmaf(hv[i].z, hv[i].z, ss); ss = fmaf(hv[i].w, hv[i].w, ss);
      }
    }
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

  // Router GEMV: warp per expert row, 16-byte chunks from smem (prefetched) or global, shuffle sum.
  constexpr int N = WTraits<WT>::kPer16B;
  const int C = d / N;
  if (prefetch) {
    asm volatile(
        "{\n .reg .pred p;\n RW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra RW_%=;\n}\n" ::"r"(
            r_smem(&wbar))
        : "memory");
  }
  const uint4* wbase = prefetch ? reinterpret_cast<const uint4*>(wsm) : reinterpret_cast<const uint4*>(wg);
  for (int e = warp; e < E; e += kRouterWarps) {
    const uint4* wr = wbase + (size_t)e * C;
    float acc0 = 0.f, acc1 = 0.f;
    int c = lane;
    for (; c + 32 < C; c += 64) {
      acc0 += dot16<WT>(wr[c], us + c * N);
      acc1 += dot16<WT>(wr[c + 32], us + (c + 32) * N);
    }
    if (c < C) acc0 += dot16<WT>(wr[c], us + c * N);
    const float acc = warp_sum(acc0 + acc1);
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

// ---------------------------------------------------------------- decode router on a CTA cluster
// m = 1 (the decode step's router: <= 5 us): the d columns are split over a
// cluster of kRC CTAs; each CTA adds the partial outputs to its slice of h, contributes a partial
// sum of squares and E partial logits through distributed shared memory, and CTA 0 picks the top-k
// with warp shuffles (keys (logit, -index): lowest index on ties). Every CTA reads the kRC partial
// sums of squares in the same order, so all slices are normalised with identical bits. Each CTA
// issues its W_g slice loads (E x d/kRC) before the dependency wait. The exchanges are st.async
// stores into the receivers' shared memory that complete on the receiver's mbarrier (transaction
// bytes), so no cluster-wide barrier sits on the critical path: the one cluster barrier (mbarrier
// initialisation visible cluster-wide) runs before the dependency wait, under the previous kernel.
constexpr int kRC = 8;             // CTAs per cluster
constexpr int kRCThreads = 128;
constexpr int kRCWarps = kRCThreads / 32;

__device__ __forceinline__ unsigned long long topk_key(float v, int id) {
  uint32_t b = __float_as_uint(v);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return ((unsigned long long)b << 32) | (unsigned long long)(~(uint32_t)id);
}

template <typename WT>
__global__ void __cluster_dims__(kRC, 1, 1) __launch_bounds__(kRCThreads, 1) router_cluster_kernel(
    float* __restrict__ h, const float* const* __restrict__ y_add, int n_add, const WT* __restrict__ gamma,
    const WT* __restrict__ wg, const float* __restrict__ wg_scale, int E, int d, int k, float eps,
    void* __restrict__ u_out, int32_t* __restrict__ ids, float* __restrict__ w, float* __restrict__ logits,
    int32_t* __restrict__ flag) {
  constexpr int N = WTraits<WT>::kPer16B;   // weights per 16-byte chunk
  cg::cluster_group cluster = cg::this_cluster();
  const int c = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cols = d / kRC, j0 = c * cols;  // this CTA's column slice
  const int chunks = cols / N;              // 16-byte chunks of one W_g row slice
  __shared__ __align__(16) float us[4096 / kRC * 4];  // slice of u (fp32 copy), d <= 16384
  __shared__ float ss_part[kRC];
  __shared__ float lg_part[kRC][kMaxE];
  __shared__ float red[kRCWarps];
  __shared__ __align__(8) uint64_t bar_ss;  // this CTA: the kRC partial sums of squares have landed
  __shared__ __align__(8) uint64_t bar_lg;  // CTA 0: the kRC x E partial logits have landed
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(r_smem(&bar_ss)));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(r_smem(&bar_ss)), "r"(kRC * 4)
                 : "memory");
    if (c == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(r_smem(&bar_lg)));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(r_smem(&bar_lg)), "r"(kRC * E * 4)
                   : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // remote st.async only after every CTA's barriers exist (before the dependency wait: off the path)
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  // st.async of one fp32 into CTA `dst`'s copy of `slot`, completing on its copy of `bar`
  auto st_async = [&](float* slot, uint64_t* bar, int dst, float v) {
    uint32_t ra, rb;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(r_smem(slot)), "r"(dst));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(r_smem(bar)), "r"(dst));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(ra),
                 "r"(__float_as_uint(v)), "r"(rb)
                 : "memory");
  };
  auto wait_bar = [&](uint64_t* bar) {
    asm volatile("{\n .reg .pred p;\n RW_%=:\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], 0;\n"
                 " @!p bra RW_%=;\n}\n" ::"r"(r_smem(bar))
                 : "memory");
  };

  // W_g slice: expert e's chunks [e][j0 .. j0 + cols), lane i takes chunks i, i + 32, ... of the
  // experts of its warp (e = warp, warp + kRCWarps, ...); loaded before the dependency wait
  // (2 experts x 2 chunks per lane covers E = 8, d = 4096 bf16; larger shapes load the rest later)
  uint4 wv00 = make_uint4(0, 0, 0, 0), wv01 = wv00, wv10 = wv00, wv11 = wv00;
  {
    const int e0 = warp, e1 = warp + kRCWarps, q0 = lane, q1 = lane + 32;
    if (e0 < E && q0 < chunks) wv00 = *reinterpret_cast<const uint4*>(wg + (size_t)e0 * d + j0 + (size_t)q0 * N);
    if (e0 < E && q1 < chunks) wv01 = *reinterpret_cast<const uint4*>(wg + (size_t)e0 * d + j0 + (size_t)q1 * N);
    if (e1 < E && q0 < chunks) wv10 = *reinterpret_cast<const uint4*>(wg + (size_t)e1 * d + j0 + (size_t)q0 * N);
    if (e1 < E && q1 < chunks) wv11 = *reinterpret_cast<const uint4*>(wg + (size_t)e1 * d + j0 + (size_t)q1 * N);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // pass 1: h += y_0 + y_1 + ... on the slice (partials summed first, as router_kernel)
  float ss = 0.f;
  for (int j = tid * 4; j < cols; j += kRCThreads * 4) {
    float4 hv = *reinterpret_cast<const float4*>(h + j0 + j);
    if (n_add > 0) {
      float4 s = *reinterpret_cast<const float4*>(y_add[0] + j0 + j);
      for (int a = 1; a < n_add; ++a) {
        const float4 t = *reinterpret_cast<const float4*>(y_add[a] + j0 + j);
        s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;
      }
      hv.x += s.x; hv.y += s.y; hv.z += s.z; hv.w += s.w;
      *reinterpret_cast<float4*>(h + j0 + j) = hv;
    }
    *reinterpret_cast<float4*>(us + j) = hv;
    ss = fmaf(hv.x, hv.x, ss); ss = fmaf(hv.y, hv.y, ss);
    ss = fmaf(hv.z, hv.z, ss); ss = fmaf(hv.w, hv.w, ss);
  }
  ss = warp_sum(ss);
  if (lane == 0) red[warp] = ss;
  __syncthreads();
  if (tid < kRC) {  // this slice's sum of squares into slot c of every CTA (thread r -> CTA r)
    float t = 0.f;
    for (int i = 0; i < kRCWarps; ++i) t += red[i];
    st_async(&ss_part[c], &bar_ss, tid, t);
  }
  wait_bar(&bar_ss);
  float tot = 0.f;
  for (int r = 0; r < kRC; ++r) tot += ss_part[r];  // same order everywhere: identical rstd
  const float rstd = 1.0f / sqrtf(tot / (float)d + eps);

  // pass 2: u = h * rstd * gamma, rounded to the activation dtype
  constexpr bool kF32 = std::is_same<WT, float>::value;
  for (int j = tid; j < cols; j += kRCThreads) {
    float gm = 1.f;
    if (gamma != nullptr) {
      if constexpr (kF32) gm = gamma[j0 + j];
      else if constexpr (std::is_same<WT, __nv_bfloat16>::value) gm = __bfloat162float(gamma[j0 + j]);
    }
    const float v = us[j] * rstd * gm;
    if constexpr (kF32) {
      reinterpret_cast<float*>(u_out)[j0 + j] = v;
      us[j] = v;
    } else {
      const __nv_bfloat16 b = __float2bfloat16_rn(v);
      reinterpret_cast<__nv_bfloat16*>(u_out)[j0 + j] = b;
      us[j] = __bfloat162float(b);
    }
  }
  __syncthreads();

  // partial logits of this slice: warp per expert, the prefetched chunks first
  for (int e = warp, i = 0; e < E; e += kRCWarps, ++i) {
    float acc = 0.f;
    for (int q = lane, j = 0; q < chunks; q += 32, ++j) {
      uint4 wq;
      if (i < 2 && j < 2) wq = i == 0 ? (j == 0 ? wv00 : wv01) : (j == 0 ? wv10 : wv11);
      else wq = *reinterpret_cast<const uint4*>(wg + (size_t)e * d + j0 + (size_t)q * N);
      acc += dot16<WT>(wq, us + q * N);
    }
    acc = warp_sum(acc);
    if (lane == 0) st_async(&lg_part[c][e], &bar_lg, 0, acc);
  }
  if (c != 0 || warp != 0) return;
  wait_bar(&bar_lg);

  // CTA 0, warp 0: logits (slices summed in CTA order), top-k by warp argmax, softmax
  float lv = 0.f;
  if (lane < E) {
    for (int r = 0; r < kRC; ++r) lv += lg_part[r][lane];
    if (wg_scale) lv *= wg_scale[lane];
  }
  float lv2 = 0.f;  // experts 32..63
  if (lane + 32 < E) {
    for (int r = 0; r < kRC; ++r) lv2 += lg_part[r][lane + 32];
    if (wg_scale) lv2 *= wg_scale[lane + 32];
  }
  const bool bad = __any_sync(0xffffffffu, (lane < E && !isfinite(lv)) || (lane + 32 < E && !isfinite(lv2)));
  unsigned long long k1 = lane < E ? topk_key(lv, lane) : 0ull;
  unsigned long long k2 = lane + 32 < E ? topk_key(lv2, lane + 32) : 0ull;
  // k rounds of a warp argmax; lane i keeps the i-th pick (id, logit)
  int my_id = 0;
  float my_v = 0.f, m = 0.f;
#pragma unroll
  for (int i = 0; i < kMaxK; ++i) {
    if (i < k) {
      unsigned long long best = k1 > k2 ? k1 : k2;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
        best = other > best ? other : best;
      }
      const int id = (int)(~(uint32_t)(best & 0xffffffffull));
      const float v = __shfl_sync(0xffffffffu, id < 32 ? lv : lv2, id & 31);
      if (i == 0) m = v;
      if (lane == i) { my_id = id; my_v = v; }
      if (id == lane) k1 = 0ull;
      if (id == lane + 32) k2 = 0ull;
    }
  }
  // softmax over the k selected logits (summed in pick order by lane 0, as router_kernel)
  const float ex = lane < k ? expf(my_v - m) : 0.f;
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < kMaxK; ++i) sum += i < k ? __shfl_sync(0xffffffffu, ex, i) : 0.f;
  if (lane < k) {
    ids[lane] = my_id;
    w[lane] = ex / sum;
  }
  if (lane == 0 && bad && flag) *flag = 1;
  if (logits) {
    if (lane < E) logits[lane] = lv;
    if (lane + 32 < E) logits[lane + 32] = lv2;
  }
}

// Residual combine only (after the last layer): h += (y_0 + y_1 + ...), same order as the router.
__global__ void combine_kernel(float* __restrict__ h, const float* const* __restrict__ y_add, int n_add, int d) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the next kernel may prefetch its weights
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

template <typename K, typename... Args>
static cudaError_t launch_ex(K kern, dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

static bool router_cluster_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ODMOE_ROUTER_CLUSTER");  // ODMOE_ROUTER_CLUSTER=0: the one-CTA kernel (A/B)
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <typename WT>
static cudaError_t router_impl(float* h, const float* const* y_add, int n_add, const void* gamma,
                               const void* w_gate, const float* wg_scale, int m, int E, int d, int k,
                               float eps, void* u_out, int32_t* ids, float* w, float* logits, int32_t* flag,
                               cudaStream_t s, bool pdl) {
  constexpr int N = WTraits<WT>::kPer16B;
  if (m == 1 && router_cluster_on() && d % (kRC * N) == 0 && d % (kRC * 4) == 0 && d / kRC <= 4096 / kRC * 4) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(kRC);
    cfg.blockDim = dim3(kRCThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, router_cluster_kernel<WT>, h, y_add, n_add, (const WT*)gamma, (const WT*)w_gate,
                              wg_scale, E, d, k, eps, u_out, ids, w, logits, flag);
  }
  const size_t wbytes = (size_t)E * d * sizeof(WT);
  const int prefetch = (wbytes <= (size_t)kRouterPrefetchMax && wbytes % 16 == 0) ? 1 : 0;
  const size_t smem = (((size_t)d * sizeof(float) + 127) & ~(size_t)127) + (prefetch ? wbytes : 0);
  auto kern = router_kernel<WT>;
  if (smem > 40 * 1024) {  // static smem (~0.4 KB) + dynamic must fit: opt in early
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  return launch_ex(kern, dim3(m), dim3(kRouterThreads), smem, s, pdl, h, y_add, n_add, (const WT*)gamma,
                   (const WT*)w_gate, wg_scale, E, d, k, eps, u_out, ids, w, logits, flag, prefetch);
}

cudaError_t launch_router(float* h, const float* const* y_add, int n_add, const void* gamma,
                          const void* w_gate, const float* wg_scale, WType wt, int m, int E, int d,
                          int k, float eps, void* u_out, int32_t* ids, float* w, float* logits,
                          int32_t* flag, cudaStream_t s, bool pdl) {
  switch (wt) {
    case W_BF16:
      return router_impl<__nv_bfloat16>(h, y_add, n_add, gamma, w_gate, nullptr, m, E, d, k, eps, u_out, ids, w,
                                        logits, flag, s, pdl);
    case W_F32:
      return router_impl<float>(h, y_add, n_add, gamma, w_gate, nullptr, m, E, d, k, eps, u_out, ids, w, logits,
                                flag, s, pdl);
    case W_I8:
      return router_impl<int8_t>(h, y_add, n_add, nullptr, w_gate, wg_scale, m, E, d, k, eps, u_out, ids, w,
                                 logits, flag, s, pdl);
    default: break;
  }
  return cudaErrorInvalidValue;
}

}  // namespace odmoe
