// ARCHIVED A/B CODE (round 2): not compiled into libodmoe.so. The TMA bulk-ring GEMV engine measured
// in round 1 (profiles/kbench_r01_gemv_tma.json: 114 us per expert vs the flat engine's 73 -> 65.6 us);
// kept for reference next to DESIGN.md section 6. It no longer builds against kernels.h as is.
// HBM-streaming GEMV engine with TMA bulk copies (the expert SwiGLU FFN at batch 1, a8; the INT8
// shadow experts, a4; the LM head, a10). y = W x for a row-major W whose rows are consumed exactly
// once, so the kernel is a pure HBM stream and the whole design is about keeping enough bytes in
// flight on every SM:
//
//  * one CTA per SM owns a CONTIGUOUS, balanced row range; its bytes form one linear stream;
//  * a producer warp streams it with cp.async.bulk (1-D TMA, L2 evict-first hint) into an 8-stage
//    x 16 KB shared-memory ring guarded by mbarriers (128 KB in flight per SM, independent of
//    registers and of the row length; Little's law needs ~35 KB at 6.5 TB/s);
//  * 8 consumer warps take 512-byte groups round-robin (a group never straddles a row because
//    row bytes are a multiple of 512), dot them with the activations (staged once in smem), keep a
//    running sum per row and flush it with a warp shuffle when the row changes;
//  * per-warp row partials are reduced in a fixed warp order at the end: deterministic, no atomics.
//
// Epilogues: MODE 0 = W13 gate/up pairs -> a_f = silu(g_f) v_f; MODE 1 = W2 -> y = gate * row;
// MODE 2 = LM head -> logits + deterministic argmax (ticket: last CTA reduces the CTA keys).
#include "common.cuh"
#include "kernels.h"

namespace odmoe {

constexpr int kSG_CONSUMERS = 8;
constexpr int kSG_THREADS = (kSG_CONSUMERS + 1) * 32;
constexpr int kSG_STAGES = 8;
constexpr int kSG_STAGE_BYTES = 16384;

__device__ __forceinline__ uint32_t sg_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void sg_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sg_smem(bar)), "r"(count));
}
__device__ __forceinline__ void sg_mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "SGW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra SGW_%=;\n"
      "}\n" ::"r"(sg_smem(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void sg_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sg_smem(bar)) : "memory");
}
__device__ __forceinline__ void sg_bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                             uint64_t policy) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sg_smem(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          sg_smem(dst)),
      "l"(src), "r"(bytes), "r"(sg_smem(bar)), "l"(policy)
      : "memory");
}

// ------------------------------------------------ dot of one 16-byte weight granule with x (smem)
// XT = activation storage type in shared memory (bf16 bits as uint16 or fp32).
template <typename WT, typename XT> struct Dot;

template <> struct Dot<__nv_bfloat16, float> {
  static constexpr int kN = 8;
  __device__ __forceinline__ static float run(const uint4& w, const float* x) { return dot16<__nv_bfloat16>(w, x); }
};
template <> struct Dot<float, float> {
  static constexpr int kN = 4;
  __device__ __forceinline__ static float run(const uint4& w, const float* x) { return dot16<float>(w, x); }
};
template <> struct Dot<int8_t, float> {
  static constexpr int kN = 16;
  __device__ __forceinline__ static float run(const uint4& w, const float* x) { return dot16<int8_t>(w, x); }
};
__device__ __forceinline__ float bf2_dot(uint32_t w, uint32_t x, float s) {
  s = fmaf(bf16_lo(w), bf16_lo(x), s);
  return fmaf(bf16_hi(w), bf16_hi(x), s);
}
template <> struct Dot<__nv_bfloat16, uint16_t> {
  static constexpr int kN = 8;
  __device__ __forceinline__ static float run(const uint4& w, const uint16_t* x) {
    const uint4 xv = *reinterpret_cast<const uint4*>(x);
    float s = bf16_lo(w.x) * bf16_lo(xv.x);
    s = fmaf(bf16_hi(w.x), bf16_hi(xv.x), s);
    s = bf2_dot(w.y, xv.y, s);
    s = bf2_dot(w.z, xv.z, s);
    return bf2_dot(w.w, xv.w, s);
  }
};
__device__ __forceinline__ float i8x4_bf(uint32_t word, uint32_t x01, uint32_t x23, float s) {
  const uint32_t b = word ^ 0x80808080u;
  s = fmaf(i8_to_f32(b, 0), bf16_lo(x01), s);
  s = fmaf(i8_to_f32(b, 1), bf16_hi(x01), s);
  s = fmaf(i8_to_f32(b, 2), bf16_lo(x23), s);
  return fmaf(i8_to_f32(b, 3), bf16_hi(x23), s);
}
template <> struct Dot<int8_t, uint16_t> {
  static constexpr int kN = 16;
  __device__ __forceinline__ static float run(const uint4& w, const uint16_t* x) {
    const uint4 x0 = *reinterpret_cast<const uint4*>(x);
    const uint4 x1 = *reinterpret_cast<const uint4*>(x + 8);
    float s = 0.f;
    s = i8x4_bf(w.x, x0.x, x0.y, s);
    s = i8x4_bf(w.y, x0.z, x0.w, s);
    s = i8x4_bf(w.z, x1.x, x1.y, s);
    return i8x4_bf(w.w, x1.z, x1.w, s);
  }
};

__device__ __forceinline__ unsigned long long sg_argmax_key(float v, int id) {
  uint32_t b = __float_as_uint(v);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return ((unsigned long long)b << 32) | (unsigned long long)(~(uint32_t)id);
}

struct StreamArgs {
  ExpertRef ex;          // weights (W13 / W2 selection like the LDG kernels) or plain matrix
  int second;            // 1: the W2 part of an indirect blob
  const void* x;         // activations: bf16 [C] (x_bf16 = 1) or fp32 [C]
  int x_bf16;
  int R, C;              // rows, elements per row
  const float* gate_w;   // MODE 1
  float* out;            // MODE 0: a [R/2]; MODE 1: y [R]; MODE 2: logits [R] or NULL
  // MODE 2
  const float* h;        // un-normalised residual (MODE 2 normalises it)
  float eps;
  unsigned long long* partial;
  unsigned int* ticket;
  int32_t* token_out;
  int rows_cap;
  int d_full, F_full;    // blob geometry for indirect W2 resolution
};

template <typename WT, typename XT, int MODE>
__global__ void __launch_bounds__(kSG_THREADS, 1) stream_gemv_kernel(const StreamArgs a) {
  constexpr int N = Dot<WT, XT>::kN;                   // elements per 16-byte granule
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t* ring = sm;                                   // kSG_STAGES x kSG_STAGE_BYTES
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kSG_STAGES * kSG_STAGE_BYTES);
  uint64_t* empty = full + kSG_STAGES;
  float* part = reinterpret_cast<float*>(empty + kSG_STAGES);   // [consumers][rows_cap]
  XT* xs = reinterpret_cast<XT*>(part + kSG_CONSUMERS * a.rows_cap);
  __shared__ float red[kSG_CONSUMERS + 1];
  __shared__ unsigned long long kbest[kSG_CONSUMERS + 1];
  __shared__ bool is_last;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // resolve the weight matrix (direct, or indirect through the expert table)
  const WT* W;
  const float* sc;
  int gate_idx;
  {
    const ExpertRef& ex = a.ex;
    gate_idx = ex.sel;
    if (ex.tbl == nullptr) {
      W = reinterpret_cast<const WT*>(ex.blob);
      sc = ex.scales;
    } else {
      if (ex.sorted) {
        for (int j = 0; j < ex.k; ++j) {
          int rank = 0;
          for (int i = 0; i < ex.k; ++i) rank += ex.ids[i] < ex.ids[j];
          if (rank == ex.sel) gate_idx = j;
        }
      }
      const int id = ex.base + ex.ids[gate_idx];
      W = reinterpret_cast<const WT*>(ex.tbl[id]) + (a.second ? 2LL * a.F_full * a.d_full : 0LL);
      sc = ex.stbl ? ex.stbl[id] + (a.second ? 2 * a.F_full : 0) : nullptr;
    }
  }
  // row range of this CTA (MODE 0 partitions gate/up PAIRS)
  long long rb, re;
  if (MODE == 0) {
    split_range(a.R / 2, gridDim.x, blockIdx.x, rb, re);
    rb *= 2; re *= 2;
  } else {
    split_range(a.R, gridDim.x, blockIdx.x, rb, re);
  }
  const int nrows = (int)(re - rb);
  const long long row_bytes = (long long)a.C * sizeof(WT);
  const long long total = (long long)nrows * row_bytes;
  const int n_stages = (int)((total + kSG_STAGE_BYTES - 1) / kSG_STAGE_BYTES);
  const char* src = reinterpret_cast<const char*>(W) + rb * row_bytes;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kSG_STAGES; ++s) { sg_mbar_init(&full[s], 1); sg_mbar_init(&empty[s], kSG_CONSUMERS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kSG_CONSUMERS) {
    // ---------------- producer: stream this CTA's rows through the ring
    if (lane == 0) {
      uint64_t policy;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
      for (int s = 0; s < n_stages; ++s) {
        const int slot = s % kSG_STAGES;
        const uint32_t ph = (uint32_t)(s / kSG_STAGES) & 1u;
        sg_mbar_wait(&empty[slot], ph ^ 1u);
        const long long off = (long long)s * kSG_STAGE_BYTES;
        const uint32_t bytes = (uint32_t)(total - off < kSG_STAGE_BYTES ? total - off : kSG_STAGE_BYTES);
        sg_bulk_load(ring + slot * kSG_STAGE_BYTES, src + off, bytes, &full[slot], policy);
      }
    }
  } else {
    // ---------------- consumers
    // stage activations (and for MODE 2 normalise h first)
    const int tid = threadIdx.x, nthr = kSG_CONSUMERS * 32;
    if (MODE == 2) {
      float ss = 0.f;
      for (int j = tid; j < a.C; j += nthr) { const float v = a.h[j]; ss = fmaf(v, v, ss); }
      ss = warp_sum(ss);
      if (lane == 0) red[warp] = ss;
      asm volatile("bar.sync 1, %0;" ::"r"(nthr));
      if (tid == 0) {
        float t = 0.f;
        for (int w = 0; w < kSG_CONSUMERS; ++w) t += red[w];
        red[kSG_CONSUMERS] = t;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(nthr));
      const float rstd = 1.0f / sqrtf(red[kSG_CONSUMERS] / (float)a.C + a.eps);
      for (int j = tid; j < a.C; j += nthr) {
        const float v = a.h[j] * rstd;
        if constexpr (std::is_same<XT, uint16_t>::value) {
          const __nv_bfloat16 b = __float2bfloat16_rn(v);
          xs[j] = *reinterpret_cast<const uint16_t*>(&b);
        } else {
          xs[j] = v;
        }
      }
    } else if constexpr (std::is_same<XT, uint16_t>::value) {
      const uint4* s4 = reinterpret_cast<const uint4*>(a.x);  // bf16 activations copied verbatim
      for (int i = tid; i < a.C / 8; i += nthr) reinterpret_cast<uint4*>(xs)[i] = s4[i];
    } else {
      if (a.x_bf16) {
        const uint16_t* s16 = reinterpret_cast<const uint16_t*>(a.x);
        for (int i = tid; i < a.C; i += nthr) xs[i] = __uint_as_float((uint32_t)s16[i] << 16);
      } else {
        const float4* s4 = reinterpret_cast<const float4*>(a.x);
        for (int i = tid; i < a.C / 4; i += nthr) reinterpret_cast<float4*>(xs)[i] = s4[i];
      }
    }
    for (int i = tid; i < kSG_CONSUMERS * a.rows_cap; i += nthr) part[i] = 0.f;
    asm volatile("bar.sync 1, %0;" ::"r"(nthr));

    // Warp w consumes the CTA stream's 512-byte groups w, w+8, w+16, ... (32 groups per 16 KB
    // stage), so its (row, column) position advances by 8 groups = 256 granules per step: tracked
    // incrementally, no division in the loop.
    const int Cg = a.C / N;  // granules per row (multiple of 32)
    int row = 0, col = warp * 32;
    while (col >= Cg) { col -= Cg; ++row; }
    int cur = -1;
    float acc = 0.f;
    for (int s = 0; s < n_stages; ++s) {
      const int slot = s % kSG_STAGES;
      const uint32_t ph = (uint32_t)(s / kSG_STAGES) & 1u;
      sg_mbar_wait(&full[slot], ph);
      const long long off = (long long)s * kSG_STAGE_BYTES;
      const int groups = (int)((total - off < kSG_STAGE_BYTES ? total - off : kSG_STAGE_BYTES) / 512);
      const uint4* stage = reinterpret_cast<const uint4*>(ring + slot * kSG_STAGE_BYTES);
#pragma unroll 2
      for (int gi = warp; gi < groups; gi += kSG_CONSUMERS) {
        const uint4 wv = stage[gi * 32 + lane];
        const float p = Dot<WT, XT>::run(wv, xs + (size_t)(col + lane) * N);
        if (row != cur) {
          if (cur >= 0) {
            const float t = warp_sum(acc);
            if (lane == 0) part[warp * a.rows_cap + cur] += t;
          }
          cur = row;
          acc = 0.f;
        }
        acc += p;
        col += kSG_CONSUMERS * 32;
        while (col >= Cg) { col -= Cg; ++row; }
      }
      __syncwarp();
      if (lane == 0) sg_mbar_arrive(&empty[slot]);
    }
    if (cur >= 0) {
      const float t = warp_sum(acc);
      if (lane == 0) part[warp * a.rows_cap + cur] += t;
    }
  }
  __syncthreads();

  // ---------------- epilogue: fixed-order reduction over consumer warps
  if (MODE == 0) {
    for (int p = threadIdx.x; p < nrows / 2; p += kSG_THREADS) {
      float g = 0.f, v = 0.f;
#pragma unroll
      for (int w = 0; w < kSG_CONSUMERS; ++w) {
        g += part[w * a.rows_cap + 2 * p];
        v += part[w * a.rows_cap + 2 * p + 1];
      }
      if (sc != nullptr) { g *= sc[rb + 2 * p]; v *= sc[rb + 2 * p + 1]; }
      a.out[rb / 2 + p] = silu_mul(g, v);
    }
  } else if (MODE == 1) {
    const float gw = a.gate_w ? a.gate_w[gate_idx] : 1.f;
    for (int r = threadIdx.x; r < nrows; r += kSG_THREADS) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < kSG_CONSUMERS; ++w) s += part[w * a.rows_cap + r];
      if (sc != nullptr) s *= sc[rb + r];
      a.out[rb + r] = gw * s;
    }
  } else {
    unsigned long long best = 0ull;
    for (int r = threadIdx.x; r < nrows; r += kSG_THREADS) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < kSG_CONSUMERS; ++w) s += part[w * a.rows_cap + r];
      if (a.out) a.out[rb + r] = s;
      const unsigned long long key = sg_argmax_key(s, (int)(rb + r));
      best = key > best ? key : best;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
      best = other > best ? other : best;
    }
    if (lane == 0) kbest[warp] = best;  // all 9 warps took part in the strided row loop
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long b = kbest[0];
      for (int w = 1; w <= kSG_CONSUMERS; ++w) b = kbest[w] > b ? kbest[w] : b;
      a.partial[blockIdx.x] = b;
      __threadfence();
      const unsigned int t = atomicAdd(a.ticket, 1u);
      is_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (is_last && threadIdx.x == 0) {
      __threadfence();
      unsigned long long b = 0ull;
      for (unsigned int i = 0; i < gridDim.x; ++i) {
        const unsigned long long p = *((volatile unsigned long long*)a.partial + i);
        b = p > b ? p : b;
      }
      *a.token_out = (int32_t)(~(uint32_t)(b & 0xffffffffull));
      *a.ticket = 0u;
    }
  }
}

template <typename WT, typename XT, int MODE>
static cudaError_t sg_launch(StreamArgs a, cudaStream_t s) {
  const int sms = num_sms();
  const long long units = MODE == 0 ? a.R / 2 : a.R;
  const int grid = (int)(units < sms ? (units > 0 ? units : 1) : sms);
  a.rows_cap = (int)((units + grid - 1) / grid) * (MODE == 0 ? 2 : 1) + 2;
  const size_t smem = (size_t)kSG_STAGES * kSG_STAGE_BYTES + 2 * kSG_STAGES * sizeof(uint64_t) +
                      (size_t)kSG_CONSUMERS * a.rows_cap * sizeof(float) + (size_t)a.C * sizeof(XT) + 16;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  auto kern = stream_gemv_kernel<WT, XT, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kSG_THREADS, smem, s>>>(a);
  return cudaGetLastError();
}

// Whether the streaming engine handles a [R, C] matrix of type wt (rows must be whole 512-byte
// groups; activations must fit in shared memory next to the ring).
bool stream_ok(WType wt, int C) {
  if (wt == W_NF4) return C % 1024 == 0 && (long long)C * 4 <= 64 * 1024;  // flat engine only
  const int esz = wt == W_F32 ? 4 : (wt == W_BF16 ? 2 : 1);
  return ((long long)C * esz) % 512 == 0 && (long long)C * 4 <= 64 * 1024;
}

cudaError_t launch_w13_stream(ExpertRef ex, WType wt, const void* u, int u_f32, float* a_out, int d, int F,
                              cudaStream_t s) {
  StreamArgs a{};
  a.ex = ex; a.second = 0; a.x = u; a.x_bf16 = !u_f32; a.R = 2 * F; a.C = d; a.out = a_out;
  a.d_full = d; a.F_full = F;
  switch (wt) {
    case W_BF16: return sg_launch<__nv_bfloat16, uint16_t, 0>(a, s);
    case W_F32: return sg_launch<float, float, 0>(a, s);
    case W_I8: return sg_launch<int8_t, uint16_t, 0>(a, s);
    default: break;
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_w2_stream(ExpertRef ex, WType wt, const float* act, const float* gate_w, float* y, int d,
                             int F, cudaStream_t s) {
  StreamArgs a{};
  a.ex = ex; a.second = 1; a.x = act; a.x_bf16 = 0; a.R = d; a.C = F; a.gate_w = gate_w; a.out = y;
  a.d_full = d; a.F_full = F;
  switch (wt) {
    case W_BF16: return sg_launch<__nv_bfloat16, float, 1>(a, s);
    case W_F32: return sg_launch<float, float, 1>(a, s);
    case W_I8: return sg_launch<int8_t, float, 1>(a, s);
    default: break;
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_lm_head_stream(const float* h, const void* W, WType wt, int V, int d, float eps,
                                  int32_t* token_out, float* logits, void* scratch, cudaStream_t s) {
  StreamArgs a{};
  a.ex = direct_ref(W, nullptr, 0); a.second = 0; a.R = V; a.C = d; a.out = logits; a.h = h; a.eps = eps;
  a.partial = reinterpret_cast<unsigned long long*>(scratch);
  a.ticket = reinterpret_cast<unsigned int*>(a.partial + 1024);
  a.token_out = token_out;
  switch (wt) {
    case W_BF16: return sg_launch<__nv_bfloat16, uint16_t, 2>(a, s);
    case W_F32: return sg_launch<float, float, 2>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace odmoe
