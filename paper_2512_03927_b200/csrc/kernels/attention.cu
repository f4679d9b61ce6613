// Attention block of the main node (reading Q29: Mixtral's GQA with rotary
// embedding). The projections run on the flat GEMV (decode) / tcgen05 grouped GEMM (prefill);
// this file holds what sits between them:
//   rope_kv   : rotate q and k of the current position(s) (rotate-half form, theta = 1e6), store k, v
//               (bf16) into the KV cache rows (or a caller buffer), q stays fp32;
//   attn_split: flash-decoding over the cached positions: CTA = (kv head g, position split s), one
//               warp per query head of the group; per split a running max, sum and un-normalised
//               output; scores q.k / sqrt(hd) in fp32 with k, v read as bf16;
//   attn_merge: merges the splits with their log-sum-exp weights into o (fp32 or bf16).
// Decode reads at most pos+1 rows per KV head: the work is tiny next to the weight GEMVs and is
// latency-bound; splits of 32 positions spread it over Hkv * ceil((pos+1)/32) CTAs.
#include "common.cuh"
#include "kernels.h"

namespace odmoe {

constexpr int kAttnSplit = 32;  // positions per split (one per lane in the scoring pass)

// Programmatic dependent launch for the small kernels of the block: each waits for its predecessor
// (griddepcontrol.wait) and lets its successor's launch start right away (launch_dependents), so the
// chain QKV -> RoPE -> split -> merge -> W_o pays one launch latency instead of five.
template <typename K, typename... Args>
static cudaError_t pdl_launch(K kern, dim3 grid, dim3 block, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}
constexpr int kMaxHd = 128;

__device__ __forceinline__ float bf16_to_f(uint16_t b) { return __uint_as_float((uint32_t)b << 16); }
// KV-cache element: bf16 for the bf16 model, fp32 for the fp32 model (P:260's 8 KB fp32 per token)
__device__ __forceinline__ float kv_ld(const uint16_t* p) { return bf16_to_f(*p); }
__device__ __forceinline__ float kv_ld(const float* p) { return *p; }
__device__ __forceinline__ void kv_st(uint16_t* p, float v) {
  const __nv_bfloat16 b = __float2bfloat16_rn(v);
  *p = *reinterpret_cast<const uint16_t*>(&b);
}
__device__ __forceinline__ void kv_st(float* p, float v) { *p = v; }

// grid = (T tokens, H + Hkv heads), block = hd/2 threads: one rotation pair per thread.
template <typename KT>
__global__ void rope_kv_kernel(float* __restrict__ qkv, int qkv_stride, int H, int Hkv, int hd, int pos0,
                               KT* __restrict__ kc, KT* __restrict__ vc, int kv_stride, float log2_theta) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int t = blockIdx.x, head = blockIdx.y, i = threadIdx.x, half = hd / 2;
  const int pos = pos0 + t;
  float* row = qkv + (size_t)t * qkv_stride;
  // angle = pos * theta^(-2i/hd), in fp64 so the rotation is exact to fp32 output precision
  const double ang = (double)pos * exp2(-(double)log2_theta * (2.0 * i) / hd);
  double sd, cd;
  sincos(ang, &sd, &cd);
  const float c = (float)cd, s = (float)sd;
  if (head < H) {
    float* q = row + head * hd;
    const float x1 = q[i], x2 = q[i + half];
    __syncthreads();
    q[i] = x1 * c - x2 * s;
    q[i + half] = x2 * c + x1 * s;
  } else {
    const int g = head - H;
    const float* k = row + H * hd + g * hd;
    const float* v = row + (H + Hkv) * hd + g * hd;
    const float x1 = k[i], x2 = k[i + half];
    KT* kd = kc + (size_t)t * kv_stride + g * hd;
    KT* vd = vc + (size_t)t * kv_stride + g * hd;
    kv_st(kd + i, x1 * c - x2 * s);
    kv_st(kd + i + half, x2 * c + x1 * s);
    kv_st(vd + i, v[i]);
    kv_st(vd + i + half, v[i + half]);
  }
}

cudaError_t launch_rope_kv(float* qkv, int qkv_stride, int T, int H, int Hkv, int hd, int pos0, void* kc, void* vc,
                           int kv_stride, int kv_f32, cudaStream_t s) {
  if (hd % 2 || hd > kMaxHd || T < 1) return cudaErrorInvalidValue;
  const float lt = (float)19.931568569324174;  // log2(1e6)
  if (kv_f32)
    return pdl_launch(rope_kv_kernel<float>, dim3(T, H + Hkv), dim3(hd / 2), s, qkv, qkv_stride, H, Hkv, hd, pos0,
                      (float*)kc, (float*)vc, kv_stride, lt);
  return pdl_launch(rope_kv_kernel<uint16_t>, dim3(T, H + Hkv), dim3(hd / 2), s, qkv, qkv_stride, H, Hkv, hd, pos0,
                    (uint16_t*)kc, (uint16_t*)vc, kv_stride, lt);
}

// Partials: part[((t * H + head) * nsplit + s) * (hd + 2)] = {o[0..hd), m, l}.
// Query t (of T) sits at position pos0 + t and attends to positions [0, pos0 + t] (causal).
// K rows for positions < pos0 come from kc_past (the cache); rows >= pos0 from kc_cur
// (the rows written by rope_kv for these queries: the cache itself for the main model, a private
// buffer for the shadow, which reads the main model's cache for the past: KV alignment).
// q . k over HD (q pre-scaled; both operands in shared memory)
template <typename KT, int HD>
__device__ __forceinline__ float dot_row(const float* __restrict__ q, const KT* __restrict__ k) {
  float s0 = 0.f, s1 = 0.f;
  if constexpr (std::is_same<KT, uint16_t>::value) {
    const uint4* k4 = reinterpret_cast<const uint4*>(k);
    uint4 w[HD / 8];
#pragma unroll
    for (int c = 0; c < HD / 8; ++c) w[c] = k4[c];
#pragma unroll
    for (int c = 0; c < HD / 8; ++c) {
      const float* qc = q + 8 * c;
      s0 = fmaf(qc[0], bf16_lo(w[c].x), s0); s1 = fmaf(qc[1], bf16_hi(w[c].x), s1);
      s0 = fmaf(qc[2], bf16_lo(w[c].y), s0); s1 = fmaf(qc[3], bf16_hi(w[c].y), s1);
      s0 = fmaf(qc[4], bf16_lo(w[c].z), s0); s1 = fmaf(qc[5], bf16_hi(w[c].z), s1);
      s0 = fmaf(qc[6], bf16_lo(w[c].w), s0); s1 = fmaf(qc[7], bf16_hi(w[c].w), s1);
    }
  } else {
    const float4* k4 = reinterpret_cast<const float4*>(k);
    float4 w[HD / 4];
#pragma unroll
    for (int c = 0; c < HD / 4; ++c) w[c] = k4[c];
#pragma unroll
    for (int c = 0; c < HD / 4; ++c) {
      const float* qc = q + 4 * c;
      s0 = fmaf(qc[0], w[c].x, s0); s1 = fmaf(qc[1], w[c].y, s1);
      s0 = fmaf(qc[2], w[c].z, s0); s1 = fmaf(qc[3], w[c].w, s1);
    }
  }
  return s0 + s1;
}

// HD/32 consecutive elements of a value row owned by one lane
template <typename KT, int PER>
__device__ __forceinline__ void ld_vals(const KT* p, float (&v)[PER]) {
  if constexpr (std::is_same<KT, float>::value) {
#pragma unroll
    for (int j = 0; j < PER; ++j) v[j] = p[j];
  } else if constexpr (PER == 4) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    v[0] = bf16_lo(u.x); v[1] = bf16_hi(u.x); v[2] = bf16_lo(u.y); v[3] = bf16_hi(u.y);
  } else if constexpr (PER == 2) {
    const uint32_t u = *reinterpret_cast<const uint32_t*>(p);
    v[0] = bf16_lo(u); v[1] = bf16_hi(u);
  } else {
    v[0] = bf16_to_f(*p);
  }
}

// CTA = (kv head g, split of kAttnSplit positions, query t); one warp per query head of the group.
// The split's key and value rows of head g (32 x HD each) are staged into shared memory with
// cp.async first -- every load in flight at once, shared by the group's query heads -- then
// (1) each lane scores one position, (2) softmax statistics by warp reductions, (3) lanes own HD/32
// dimensions and accumulate p_t v_t from shared memory. Rows are padded by 16 B so a warp reading
// 32 different rows at the same offset hits distinct banks.
template <typename KT, int HD>
__global__ void __launch_bounds__(32 * 8) attn_split_kernel(const float* __restrict__ q, int q_stride, int H, int Hkv,
                                                           int pos0, const KT* __restrict__ kc_past,
                                                           const KT* __restrict__ vc_past,
                                                           const KT* __restrict__ kc_cur,
                                                           const KT* __restrict__ vc_cur, int kv_stride,
                                                           int nsplit, float* __restrict__ part) {
  constexpr int PER = HD / 32;
  constexpr int ROWB = HD * (int)sizeof(KT) + 16;      // padded row bytes in shared memory
  constexpr int CH = HD * (int)sizeof(KT) / 16;        // 16-byte chunks per row
  __shared__ float qs[8][HD];
  __shared__ float ps[8][kAttnSplit];
  __shared__ __align__(16) uint8_t ks[kAttnSplit * ROWB];
  __shared__ __align__(16) uint8_t vs[kAttnSplit * ROWB];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int t = blockIdx.z, g = blockIdx.x, sp = blockIdx.y;
  const int rep = H / Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pos = pos0 + t;
  const int p_begin = sp * kAttnSplit;
  const int n = max(0, min(pos + 1, p_begin + kAttnSplit) - p_begin);
  auto row = [&](const KT* past, const KT* cur, int p) -> const KT* {
    return (p < pos0 ? past + (size_t)p * kv_stride : cur + (size_t)(p - pos0) * kv_stride) + g * HD;
  };
  // stage K and V rows of this split (all threads of the CTA)
  for (int i = threadIdx.x; i < n * CH; i += blockDim.x) {
    const int r = i / CH, c = i - r * CH;
    const uint32_t dk = (uint32_t)__cvta_generic_to_shared(ks + r * ROWB + c * 16);
    const uint32_t dv = (uint32_t)__cvta_generic_to_shared(vs + r * ROWB + c * 16);
    const char* sk = reinterpret_cast<const char*>(row(kc_past, kc_cur, p_begin + r)) + c * 16;
    const char* sv = reinterpret_cast<const char*>(row(vc_past, vc_cur, p_begin + r)) + c * 16;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dk), "l"(sk) : "memory");
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dv), "l"(sv) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  const bool active = warp < rep;
  const int head = g * rep + (active ? warp : 0);
  const float scale = rsqrtf((float)HD);
  if (active) {
    const float* qh = q + (size_t)t * q_stride + head * HD;
    for (int j = lane; j < HD; j += 32) qs[warp][j] = qh[j] * scale;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if (!active) return;
  float* out = part + ((size_t)(t * H + head) * nsplit + sp) * (HD + 2);
  float m = -INFINITY, sdot = -INFINITY;
  if (lane < n) {
    sdot = dot_row<KT, HD>(qs[warp], reinterpret_cast<const KT*>(ks + lane * ROWB));
    m = sdot;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  const float w = lane < n ? __expf(sdot - m) : 0.f;
  ps[warp][lane] = w;
  const float l = warp_sum(w);
  __syncwarp();
  float acc[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) acc[j] = 0.f;
  for (int u = 0; u < n; ++u) {
    const float pw = ps[warp][u];
    float v[PER];
    ld_vals<KT, PER>(reinterpret_cast<const KT*>(vs + u * ROWB) + lane * PER, v);
#pragma unroll
    for (int j = 0; j < PER; ++j) acc[j] = fmaf(pw, v[j], acc[j]);
  }
#pragma unroll
  for (int j = 0; j < PER; ++j) out[lane * PER + j] = acc[j];
  if (lane == 0) {
    out[HD] = n > 0 ? m : -INFINITY;
    out[HD + 1] = l;
  }
}

// o[t][head*hd + i] = sum_s e^{m_s - M} acc_s[i] / sum_s e^{m_s - M} l_s; grid (T, H), block hd.
__global__ void attn_merge_kernel(const float* __restrict__ part, int H, int hd, int nsplit, int pos0,
                                  float* __restrict__ o_f32, uint16_t* __restrict__ o_bf16, int o_stride) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int t = blockIdx.x, head = blockIdx.y, i = threadIdx.x;
  const int used = (pos0 + t) / kAttnSplit + 1;  // splits that saw at least one position
  const float* p0 = part + (size_t)(t * H + head) * nsplit * (hd + 2);
  float M = -INFINITY;
  for (int s = 0; s < used; ++s) M = fmaxf(M, p0[s * (hd + 2) + hd]);
  float num = 0.f, den = 0.f;
  for (int s = 0; s < used; ++s) {
    const float w = __expf(p0[s * (hd + 2) + hd] - M);
    num = fmaf(w, p0[s * (hd + 2) + i], num);
    den = fmaf(w, p0[s * (hd + 2) + hd + 1], den);
  }
  const float v = num / den;
  if (o_f32) o_f32[(size_t)t * o_stride + head * hd + i] = v;
  if (o_bf16) {
    const __nv_bfloat16 b = __float2bfloat16_rn(v);
    o_bf16[(size_t)t * o_stride + head * hd + i] = *reinterpret_cast<const uint16_t*>(&b);
  }
}

int attn_splits(int max_pos) { return max_pos / kAttnSplit + 1; }

// x[t] = bf16(RMSNorm(h[t])) for T rows (prefill: the A operand of the QKV GEMM); block per row.
__global__ void __launch_bounds__(256) rmsnorm_rows_kernel(const float* __restrict__ h, int d, float eps,
                                                           uint16_t* __restrict__ x) {
  __shared__ float red[9];
  const int t = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* hr = h + (size_t)t * d;
  float ss = 0.f;
  for (int j = tid; j < d; j += blockDim.x) ss = fmaf(hr[j], hr[j], ss);
  ss = warp_sum(ss);
  if (lane == 0) red[warp] = ss;
  __syncthreads();
  if (tid == 0) {
    float s = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    red[8] = s;
  }
  __syncthreads();
  const float rstd = 1.0f / sqrtf(red[8] / (float)d + eps);
  for (int j = tid; j < d; j += blockDim.x) {
    const __nv_bfloat16 b = __float2bfloat16_rn(hr[j] * rstd);
    x[(size_t)t * d + j] = *reinterpret_cast<const uint16_t*>(&b);
  }
}

cudaError_t launch_rmsnorm_rows(const float* h, int T, int d, float eps, void* x_bf16, cudaStream_t s) {
  rmsnorm_rows_kernel<<<T, 256, 0, s>>>(h, d, eps, (uint16_t*)x_bf16);
  return cudaGetLastError();
}

cudaError_t launch_attention(const float* q, int q_stride, int T, int H, int Hkv, int hd, int pos0, const void* kc_past,
                             const void* vc_past, const void* kc_cur, const void* vc_cur, int kv_stride, int kv_f32,
                             float* part, float* o_f32, void* o_bf16, int o_stride, cudaStream_t s) {
  if (hd % 32 || hd > kMaxHd || H % Hkv || H / Hkv > 8 || T < 1) return cudaErrorInvalidValue;
  const int nsplit = attn_splits(pos0 + T - 1);
  const dim3 grid(Hkv, nsplit, T);
  const int threads = 32 * (H / Hkv);
  cudaError_t e = cudaSuccess;
#define ODMOE_ATTN_LAUNCH(KT, HD)                                                                         \
  e = pdl_launch(attn_split_kernel<KT, HD>, grid, dim3(threads), s, q, q_stride, H, Hkv, pos0, (const KT*)kc_past, \
                 (const KT*)vc_past, (const KT*)kc_cur, (const KT*)vc_cur, kv_stride, nsplit, part)
  if (kv_f32) {
    if (hd == 32) ODMOE_ATTN_LAUNCH(float, 32);
    else if (hd == 64) ODMOE_ATTN_LAUNCH(float, 64);
    else ODMOE_ATTN_LAUNCH(float, 128);
  } else {
    if (hd == 32) ODMOE_ATTN_LAUNCH(uint16_t, 32);
    else if (hd == 64) ODMOE_ATTN_LAUNCH(uint16_t, 64);
    else ODMOE_ATTN_LAUNCH(uint16_t, 128);
  }
#undef ODMOE_ATTN_LAUNCH
  if (e != cudaSuccess) return e;
  return pdl_launch(attn_merge_kernel, dim3(T, H), dim3(hd), s, (const float*)part, H, hd, nsplit, pos0, o_f32,
                    (uint16_t*)o_bf16, o_stride);
}

}  // namespace odmoe
