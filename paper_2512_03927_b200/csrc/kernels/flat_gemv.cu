// Flat-stream GEMV (expert W13+SwiGLU, W2+gate, INT8 shadow, LM head + argmax): the third and
// fastest design measured on B200 (profiles/kbench_r01_*.json). Each CTA (one per SM, kFG_WARPS =
// 24 warps) owns a contiguous, balanced row range; that range is ONE byte stream which is cut into
// kFG_WARPS contiguous per-warp slices of 512-byte groups. A warp issues UNROLL (4) groups (one
// 16-byte ld.global.nc.L1::no_allocate per lane each) per register batch and keeps two batches in
// flight, so every SM has 24 x 2 x 4 x 512 B = 96 KB of weights in flight, and walks its slice with
// a running (row, column) position: rows are whole groups, so a row boundary is detected with one
// compare and the row's partial is flushed with a warp shuffle only then. Per-warp row partials are
// reduced in a fixed warp order at the end (deterministic, no atomics).
#include "common.cuh"
#include "kernels.h"

#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include <cstdlib>
#include <map>
#include <mutex>

namespace odmoe {

#ifndef FG_WARPS
#define FG_WARPS 24  // 24 warps x 4-granule batches (profiles/kb_r01_warps_ab.json): every type faster
#endif            // than 16 x 8 (bf16 66.4 -> 65.6 us, INT8 53.2 -> 49.2, NF4 79.9 -> 68.6 per expert)
constexpr int kFG_WARPS = FG_WARPS;
#ifndef FG_NO_F32X2
#define FG_F32X2 1  // packed fp32x2 FMA/ADD (sm_100 FFMA2/FADD2) in the bf16-x and INT8 dot products
#endif
#ifndef FG_SLOW
#define FG_FAST 1  // branch-free consume of whole batches (at most one row boundary per batch)
#else
#define FG_FAST 0
#endif
#ifndef FG_PIPE
#define FG_PIPE 0  // register pipeline variant (0: 2 batches, load-then-consume; 1: 2 batches
                   // prefetched before the wait; 2: 3 batches of UNROLL 6), see profiles/kbench_r01_*
#endif
#if defined(FG_UNROLL)
constexpr int kFG_UNROLL = FG_UNROLL;
#elif FG_PIPE == 2
constexpr int kFG_UNROLL = 6;
#else
constexpr int kFG_UNROLL = 4;
#endif
constexpr int kFG_THREADS = kFG_WARPS * 32;

// FDot<WT, XT>::run(w, xp): one 16-byte weight granule (kN weights) . its kN activations.
// Activations live in shared memory in a lane-interleaved ("swizzled") order: a granule's kN
// activations are Q = kN*sizeof(XT)/16 uint4 words, and word q of lane L for granule column g
// sits at uint4 index (g*Q + q)*32 + L. A warp's q-th loads are then 512 contiguous bytes (no bank
// conflicts) for every weight/activation type; xp = word 0 of this lane, word q at xp[32*q].
template <typename WT, typename XT> struct FDot;
// Packed fp32x2 arithmetic (sm_100 FFMA2 / FADD2): one instruction per element PAIR.
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2_pack(float lo, float hi) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ f2_t f2_fma(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f2_t f2_add(f2_t a, f2_t b) {
  f2_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float f2_sum(f2_t a) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a));
  return lo + hi;
}
__device__ __forceinline__ f2_t bf2_unpack(uint32_t v) { return f2_pack(bf16_lo(v), bf16_hi(v)); }
__device__ __forceinline__ f2_t f2_of(uint32_t lo, uint32_t hi) { return f2_pack(__uint_as_float(lo), __uint_as_float(hi)); }

template <> struct FDot<__nv_bfloat16, float> {
  static constexpr int kN = 8;
  __device__ __forceinline__ static float run(const uint4& w, const uint4* xp) {
    const uint4 x0 = xp[0], x1 = xp[32];
    f2_t s = f2_fma(bf2_unpack(w.x), f2_of(x0.x, x0.y), 0ull);
    s = f2_fma(bf2_unpack(w.y), f2_of(x0.z, x0.w), s);
    s = f2_fma(bf2_unpack(w.z), f2_of(x1.x, x1.y), s);
    s = f2_fma(bf2_unpack(w.w), f2_of(x1.z, x1.w), s);
    return f2_sum(s);
  }
};
template <> struct FDot<float, float> {
  static constexpr int kN = 4;
  __device__ __forceinline__ static float run(const uint4& w, const uint4* xp) {
    const uint4 x0 = xp[0];
    f2_t s = f2_fma(f2_of(w.x, w.y), f2_of(x0.x, x0.y), 0ull);
    s = f2_fma(f2_of(w.z, w.w), f2_of(x0.z, x0.w), s);
    return f2_sum(s);
  }
};
// 4 int8 of one word -> two exact fp32 pairs (byte into the mantissa of 2^23, one FADD2 per pair)
__device__ __forceinline__ void i8x4_unpack(uint32_t word, f2_t& q01, f2_t& q23) {
  const uint32_t b = word ^ 0x80808080u;
  const f2_t m = f2_pack(-8388736.0f, -8388736.0f);
  q01 = f2_add(f2_pack(__uint_as_float(__byte_perm(b, 0x4B000000u, 0x7540)),
                       __uint_as_float(__byte_perm(b, 0x4B000000u, 0x7541))), m);
  q23 = f2_add(f2_pack(__uint_as_float(__byte_perm(b, 0x4B000000u, 0x7542)),
                       __uint_as_float(__byte_perm(b, 0x4B000000u, 0x7543))), m);
}
template <> struct FDot<int8_t, float> {
  static constexpr int kN = 16;
  __device__ __forceinline__ static float run(const uint4& w, const uint4* xp) {
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    f2_t s = 0ull;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 xq = xp[32 * q];
      f2_t q01, q23;
      i8x4_unpack(ws[q], q01, q23);
      s = f2_fma(q01, f2_of(xq.x, xq.y), s);
      s = f2_fma(q23, f2_of(xq.z, xq.w), s);
    }
    return f2_sum(s);
  }
};


// ---------------------------------------------------------------- NF4 (shadow, reading Q27)
// Two NF4 codes per byte (low nibble = even column); one fp32 absmax per 64 weights of a row,
// stored row-major [R][C/64]. A 16-byte granule (32 weights) lies inside one block, and since C/32
// is even the block of granule n of the matrix is n/2: the scale address needs no division.
struct nf4x2 { uint8_t v; };
template <typename WT> struct FTraits { static constexpr int bits = 8 * (int)sizeof(WT); static constexpr bool nf4 = false; };
template <> struct FTraits<nf4x2> { static constexpr int bits = 4; static constexpr bool nf4 = true; };
template <> struct FDot<nf4x2, uint16_t> { static constexpr int kN = 32; };
struct fp8e4 { uint8_t v; };  // E4M3 code (FP8 shadow, reading Q28); row scales like int8
struct u8b { uint8_t v; };    // INT8-row code stored as q + 128 (W_U8)
// bf16 weights (row-major, the W_BF16 blob) consumed by the tensor cores: mma.sync m16n8k16, fp32
// accumulate (flat_phase's kMMA branch). Activations are staged as bf16 hi + lo (x = hi + lo to
// 2^-16 relative) in B columns 0 and 1, so the fp32 W2 input keeps ~fp32 accuracy.
struct bf16m { uint16_t v; };
template <> struct FDot<bf16m, float> { static constexpr int kN = 8; };
__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
#ifndef FG_MMA_KU
#define FG_MMA_KU 2  // (16-row tile, 32-column block) units per register batch; two batches in flight
#endif
template <> struct FDot<nf4x2, float> { static constexpr int kN = 32; };

// QLoRA's published NF4 codebook (Dettmers et al. 2023)
__constant__ float kNF4Code[16] = {
    -1.0f, -0.6961928009986877f, -0.5250730514526367f, -0.39491748809814453f,
    -0.28444138169288635f, -0.18477343022823334f, -0.09105003625154495f, 0.0f,
    0.07958029955625534f, 0.16093020141124725f, 0.24611230194568634f, 0.33791524171829224f,
    0.44070982933044434f, 0.5626170039176941f, 0.7229568362236023f, 1.0f};
constexpr int kNF4LutWords = 256 * 32;  // byte -> f16x2(code lo, code hi), one copy per lane (no bank conflicts)

__device__ __forceinline__ f2_t h2_unpack(uint32_t v) {
  float lo, hi;
  asm("{.reg .f16 l, h;\n mov.b32 {l, h}, %2;\n cvt.f32.f16 %0, l;\n cvt.f32.f16 %1, h;}"
      : "=f"(lo), "=f"(hi) : "r"(v));
  return f2_pack(lo, hi);
}
__device__ __forceinline__ void nf4_build_lut(uint32_t* lut, int tid, int nthreads) {
  for (int i = tid; i < kNF4LutWords; i += nthreads) {
    const int b = i >> 5;
    const __half2 h = __floats2half2_rn(kNF4Code[b & 15], kNF4Code[b >> 4]);
    lut[i] = *reinterpret_cast<const uint32_t*>(&h);
  }
}
// 32 weights (one granule) . 32 activations; `lut` already offset by the lane.
__device__ __forceinline__ float nf4_dot(const uint4& w, const uint4* xp, const uint32_t* lut, uint16_t) {
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
  f2_t s = 0ull;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint4 xq = xp[32 * k];
    const uint32_t xw[4] = {xq.x, xq.y, xq.z, xq.w};
#pragma unroll
    for (int b = 0; b < 4; ++b)
      s = f2_fma(h2_unpack(lut[((ws[k] >> (8 * b)) & 0xFFu) * 32]), bf2_unpack(xw[b]), s);
  }
  return f2_sum(s);
}
__device__ __forceinline__ float nf4_dot(const uint4& w, const uint4* xp, const uint32_t* lut, float) {
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
  f2_t s = 0ull;
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint4 xq = xp[32 * (2 * k + h)];  // activations 8k+4h .. 8k+4h+3
      s = f2_fma(h2_unpack(lut[((ws[k] >> (16 * h)) & 0xFFu) * 32]), f2_of(xq.x, xq.y), s);
      s = f2_fma(h2_unpack(lut[((ws[k] >> (16 * h + 8)) & 0xFFu) * 32]), f2_of(xq.z, xq.w), s);
    }
  return f2_sum(s);
}

// ---------------------------------------------------------------- FP8 E4M3 (shadow, reading Q28)
__device__ __forceinline__ uint32_t e4m3x2_to_h2(uint32_t v16) {
  uint32_t r;
  asm("{.reg .b16 t;\n cvt.u16.u32 t, %1;\n cvt.rn.f16x2.e4m3x2 %0, t;}" : "=r"(r) : "r"(v16));
  return r;
}
template <> struct FDot<fp8e4, uint16_t> {
  static constexpr int kN = 16;
  __device__ __forceinline__ static float run(const uint4& w, const uint4* xp) {
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    const uint4 x0 = xp[0], x1 = xp[32];
    const uint32_t xw[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
    f2_t s = 0ull;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      s = f2_fma(h2_unpack(e4m3x2_to_h2(ws[k] & 0xFFFFu)), bf2_unpack(xw[2 * k]), s);
      s = f2_fma(h2_unpack(e4m3x2_to_h2(ws[k] >> 16)), bf2_unpack(xw[2 * k + 1]), s);
    }
    return f2_sum(s);
  }
};
template <> struct FDot<fp8e4, float> {
  static constexpr int kN = 16;
  __device__ __forceinline__ static float run(const uint4& w, const uint4* xp) {
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    f2_t s = 0ull;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint4 xq = xp[32 * k];
      s = f2_fma(h2_unpack(e4m3x2_to_h2(ws[k] & 0xFFFFu)), f2_of(xq.x, xq.y), s);
      s = f2_fma(h2_unpack(e4m3x2_to_h2(ws[k] >> 16)), f2_of(xq.z, xq.w), s);
    }
    return f2_sum(s);
  }
};

__device__ __forceinline__ float fbf2(uint32_t w, uint32_t x, float s) {
  s = fmaf(bf16_lo(w), bf16_lo(x), s);
  return fmaf(bf16_hi(w), bf16_hi(x), s);
}
template <> struct FDot<__nv_bfloat16, uint16_t> {
  static constexpr int kN = 8;
  __device__ __forceinline__ static float run(const uint4& w, const uint4* xp) {
    const uint4 xv = xp[0];
#ifdef FG_F32X2
    f2_t s = f2_fma(bf2_unpack(w.x), bf2_unpack(xv.x), 0ull);
    s = f2_fma(bf2_unpack(w.y), bf2_unpack(xv.y), s);
    s = f2_fma(bf2_unpack(w.z), bf2_unpack(xv.z), s);
    s = f2_fma(bf2_unpack(w.w), bf2_unpack(xv.w), s);
    return f2_sum(s);
#endif
    // two independent chains (even/odd words) for ILP
    float s0 = bf16_lo(w.x) * bf16_lo(xv.x);
    float s1 = bf16_lo(w.y) * bf16_lo(xv.y);
    s0 = fmaf(bf16_hi(w.x), bf16_hi(xv.x), s0);
    s1 = fmaf(bf16_hi(w.y), bf16_hi(xv.y), s1);
    s0 = fbf2(w.z, xv.z, s0);
    s1 = fbf2(w.w, xv.w, s1);
    return s0 + s1;
  }
};
__device__ __forceinline__ float fi8(uint32_t word, uint32_t x01, uint32_t x23, float s) {
  const uint32_t b = word ^ 0x80808080u;
  s = fmaf(i8_to_f32(b, 0), bf16_lo(x01), s);
  s = fmaf(i8_to_f32(b, 1), bf16_hi(x01), s);
  s = fmaf(i8_to_f32(b, 2), bf16_lo(x23), s);
  return fmaf(i8_to_f32(b, 3), bf16_hi(x23), s);
}
#ifdef FG_F32X2
// 4 int8 of one word -> two fp32 pairs (exact: byte into the mantissa of 2^23, one FADD2 per pair)
__device__ __forceinline__ f2_t i8x4_dot2(uint32_t word, uint32_t x01, uint32_t x23, f2_t s) {
  const uint32_t b = word ^ 0x80808080u;
  const f2_t m = f2_pack(-8388736.0f, -8388736.0f);
  const f2_t q01 = f2_add(f2_pack(__uint_as_float(__byte_perm(b, 0x4B000000u, 0x7540)),
                                  __uint_as_float(__byte_perm(b, 0x4B000000u, 0x7541))), m);
  const f2_t q23 = f2_add(f2_pack(__uint_as_float(__byte_perm(b, 0x4B000000u, 0x7542)),
                                  __uint_as_float(__byte_perm(b, 0x4B000000u, 0x7543))), m);
  s = f2_fma(q01, bf2_unpack(x01), s);
  return f2_fma(q23, bf2_unpack(x23), s);
}
#endif
// W_U8: the byte already is q + 128, so it goes into the mantissa of 2^23 without the sign flip
__device__ __forceinline__ f2_t u8x4_dot2(uint32_t b, uint32_t x01, uint32_t x23, f2_t s) {
  const f2_t m = f2_pack(-8388736.0f, -8388736.0f);
  const f2_t q01 = f2_add(f2_pack(__uint_as_float(__byte_perm(b, 0x4B000000u, 0x7540)),
                                  __uint_as_float(__byte_perm(b, 0x4B000000u, 0x7541))), m);
  const f2_t q23 = f2_add(f2_pack(__uint_as_float(__byte_perm(b, 0x4B000000u, 0x7542)),
                                  __uint_as_float(__byte_perm(b, 0x4B000000u, 0x7543))), m);
  s = f2_fma(q01, bf2_unpack(x01), s);
  return f2_fma(q23, bf2_unpack(x23), s);
}
template <> struct FDot<u8b, float> {
  static constexpr int kN = 16;
  __device__ __forceinline__ static float run(const uint4& w, const uint4* xp) {
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    const f2_t m = f2_pack(-8388736.0f, -8388736.0f);
    f2_t s = 0ull;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 xq = xp[32 * q];
      const uint32_t b = ws[q];
      const f2_t q01 = f2_add(f2_pack(__uint_as_float(__byte_perm(b, 0x4B000000u, 0x7540)),
                                      __uint_as_float(__byte_perm(b, 0x4B000000u, 0x7541))), m);
      const f2_t q23 = f2_add(f2_pack(__uint_as_float(__byte_perm(b, 0x4B000000u, 0x7542)),
                                      __uint_as_float(__byte_perm(b, 0x4B000000u, 0x7543))), m);
      s = f2_fma(q01, f2_of(xq.x, xq.y), s);
      s = f2_fma(q23, f2_of(xq.z, xq.w), s);
    }
    return f2_sum(s);
  }
};
template <> struct FDot<u8b, uint16_t> {
  static constexpr int kN = 16;
  __device__ __forceinline__ static float run(const uint4& w, const uint4* xp) {
    const uint4 x0 = xp[0];
    const uint4 x1 = xp[32];
    f2_t s = u8x4_dot2(w.x, x0.x, x0.y, 0ull);
    s = u8x4_dot2(w.y, x0.z, x0.w, s);
    s = u8x4_dot2(w.z, x1.x, x1.y, s);
    s = u8x4_dot2(w.w, x1.z, x1.w, s);
    return f2_sum(s);
  }
};
template <> struct FDot<int8_t, uint16_t> {
  static constexpr int kN = 16;
  __device__ __forceinline__ static float run(const uint4& w, const uint4* xp) {
    const uint4 x0 = xp[0];
    const uint4 x1 = xp[32];
#ifdef FG_F32X2
    f2_t s = i8x4_dot2(w.x, x0.x, x0.y, 0ull);
    s = i8x4_dot2(w.y, x0.z, x0.w, s);
    s = i8x4_dot2(w.z, x1.x, x1.y, s);
    s = i8x4_dot2(w.w, x1.z, x1.w, s);
    return f2_sum(s);
#endif
    float s0 = fi8(w.x, x0.x, x0.y, 0.f);
    float s1 = fi8(w.y, x0.z, x0.w, 0.f);
    s0 = fi8(w.z, x1.x, x1.y, s0);
    s1 = fi8(w.w, x1.z, x1.w, s1);
    return s0 + s1;
  }
};

__device__ __forceinline__ unsigned long long fg_argmax_key(float v, int id) {
  uint32_t b = __float_as_uint(v);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return ((unsigned long long)b << 32) | (unsigned long long)(~(uint32_t)id);
}

struct FlatArgs {
  ExpertRef ex;
  int second;
  const void* x;
  int x_bf16;
  int R, C;
  const float* gate_w;
  float* out;
  const float* h;
  float eps;
  unsigned long long* partial;
  unsigned int* ticket;
  int32_t* token_out;
  int rows_cap;
  int d_full, F_full;
  int evict_first;       // L2 policy of the weight stream
  int accumulate;        // MODE 1/3: out[r] += result instead of out[r] = result
  P2PSend send;          // MODE 1: send.dst != NULL -> the fused P2P combine (kernels.h)
};

struct PdlWait {
  __device__ __forceinline__ void operator()() const { asm volatile("griddepcontrol.wait;" ::: "memory"); }
};

// One streaming pass (see the file comment). `wait_dep` is called once the data this pass consumes
// from earlier work may be read: griddepcontrol.wait (PDL) for a stand-alone launch, a grid-wide
// barrier for the W2 phase of the fused expert kernel. Weights are prefetched before it.
template <typename WT, typename XT, int MODE, int UNROLL, typename WaitFn>
__device__ __forceinline__ void flat_phase(const FlatArgs& a, uint8_t* sm, const WaitFn& wait_dep,
                                           bool ids_ready = false, long long rb_ovr = -1, long long re_ovr = -1) {
  constexpr int N = FDot<WT, XT>::kN;
  constexpr int Q = N * (int)sizeof(XT) / 16;       // uint4 activation words per granule
  constexpr int EPU = 16 / (int)sizeof(XT);         // activations per uint4
  static_assert(Q >= 1 && (Q & (Q - 1)) == 0, "Q must be a power of two");
  // natural uint4 index o of the activation vector -> its swizzled slot (see FDot)
  auto swz4 = [](int o) { const int q = o & (Q - 1), t = o / Q; return ((t >> 5) * Q + q) * 32 + (t & 31); };
  auto swz = [&](int e) { return swz4(e / EPU) * EPU + (e & (EPU - 1)); };
  constexpr bool kNF4 = FTraits<WT>::nf4;
  constexpr bool kMMA = std::is_same<WT, bf16m>::value;
  static_assert(!kMMA || MODE == 0 || MODE == 1, "tensor-core path: expert phases only");
  static_assert(!kNF4 || FG_PIPE == 0, "NF4 is implemented for the default pipeline");
  float* part = reinterpret_cast<float*>(sm);                          // [warps][rows_cap]
  XT* xs = reinterpret_cast<XT*>(part + kFG_WARPS * a.rows_cap);       // [C]
  uint32_t* lut = reinterpret_cast<uint32_t*>(xs + a.C);               // NF4 only: [256][32]
  __shared__ float red[kFG_WARPS + 1];
  __shared__ unsigned long long kbest[kFG_WARPS];
  __shared__ bool is_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;

  // Indirect experts are chosen by the PREVIOUS kernel's router output: wait for it (PDL) before
  // reading the ids. Direct weights do not depend on it and are prefetched first (below).
  const bool indirect = a.ex.tbl != nullptr;
  const bool early = indirect && !ids_ready;  // the expert ids come from the previous kernel
  if (early) wait_dep();
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
      W = reinterpret_cast<const WT*>(reinterpret_cast<const char*>(ex.tbl[id]) +
                                      (a.second ? 2LL * a.F_full * a.d_full * FTraits<WT>::bits / 8 : 0LL));
      sc = ex.stbl ? ex.stbl[id] + (a.second ? (kNF4 ? 2LL * a.F_full * a.d_full / 64 : 2LL * a.F_full) : 0LL)
                   : nullptr;
    }
  }
  long long rb, re;
  if (rb_ovr >= 0) {  // the caller assigns this CTA's rows (multi-expert kernel)
    rb = rb_ovr; re = re_ovr;
  } else if (MODE == 0) {
    split_range(a.R / 2, gridDim.x, blockIdx.x, rb, re);
    rb *= 2; re *= 2;
  } else {
    split_range(a.R, gridDim.x, blockIdx.x, rb, re);
  }
  const int nrows = (int)(re - rb);
  if constexpr (!kMMA) {
  const int Cg = a.C / N;                 // 16-byte granules per row (multiple of 32)
  const int Gr = Cg / 32;                 // 512-byte groups per row
  const long long G = (long long)nrows * Gr;
  // this warp's slice of groups
#if FG_PIPE == 3
  // interleaved: warp w takes batches w, w + 16, ... of UNROLL groups -> one sequential stream per SM
  const long long g_begin = (long long)warp * UNROLL, g_end = G;
#else
  const long long g_begin = G * warp / kFG_WARPS, g_end = G * (warp + 1) / kFG_WARPS;
#endif
  const uint4* base = reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(W) +
                                                     rb * (long long)a.C * FTraits<WT>::bits / 8);
  const float* scb = kNF4 ? sc + ((rb * Cg) >> 1) : nullptr;  // block absmax of this CTA's first row

  // The weights do not depend on the previous kernel: issue this warp's first batch before the
  // programmatic-dependent-launch wait (no-op without PDL), then stage the activations.
  const uint64_t pol = l2_policy(a.evict_first != 0);
  uint4 wa[UNROLL], wb[UNROLL];
  float sa[UNROLL], sb[UNROLL];  // NF4 block scales of the batch (unused otherwise)
#if FG_PIPE == 2
  uint4 wc[UNROLL];
#endif
#pragma unroll
  for (int i = 0; i < UNROLL; ++i)
    if (g_begin + i < g_end) {
      wa[i] = ld_stream_pol(base + (g_begin + i) * 32 + lane, pol);
      if constexpr (kNF4) sa[i] = __ldg(scb + (((g_begin + i) * 32 + lane) >> 1));
    }
#if FG_PIPE >= 1
#pragma unroll
  for (int i = 0; i < UNROLL; ++i)
    if (g_begin + UNROLL + i < g_end) wb[i] = ld_stream_pol(base + (g_begin + UNROLL + i) * 32 + lane, pol);
#endif
#if FG_PIPE == 2
#pragma unroll
  for (int i = 0; i < UNROLL; ++i)
    if (g_begin + 2 * UNROLL + i < g_end) wc[i] = ld_stream_pol(base + (g_begin + 2 * UNROLL + i) * 32 + lane, pol);
#endif
  if (!early) wait_dep();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // stage activations (MODE 2: RMSNorm of h first) and zero the partials
  if (MODE == 2 || MODE == 3) {
    float ss = 0.f;
    for (int j = tid; j < a.C; j += kFG_THREADS) { const float v = a.h[j]; ss = fmaf(v, v, ss); }
    ss = warp_sum(ss);
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    if (tid == 0) {
      float t = 0.f;
      for (int w = 0; w < kFG_WARPS; ++w) t += red[w];
      red[kFG_WARPS] = t;
    }
    __syncthreads();
    const float rstd = 1.0f / sqrtf(red[kFG_WARPS] / (float)a.C + a.eps);
    for (int j = tid; j < a.C; j += kFG_THREADS) {
      const float v = a.h[j] * rstd;
      if constexpr (std::is_same<XT, uint16_t>::value) {
        const __nv_bfloat16 b = __float2bfloat16_rn(v);
        xs[swz(j)] = *reinterpret_cast<const uint16_t*>(&b);
      } else {
        xs[swz(j)] = v;
      }
    }
  } else if constexpr (std::is_same<XT, uint16_t>::value) {
    const uint4* s4 = reinterpret_cast<const uint4*>(a.x);
    for (int i = tid; i < a.C / 8; i += kFG_THREADS) reinterpret_cast<uint4*>(xs)[swz4(i)] = s4[i];
  } else {
    if (a.x_bf16) {
      const uint16_t* s16 = reinterpret_cast<const uint16_t*>(a.x);
      for (int i = tid; i < a.C; i += kFG_THREADS) xs[swz(i)] = __uint_as_float((uint32_t)s16[i] << 16);
    } else {
      // all loads of a thread first (latency-bound otherwise: 57 KB per CTA for W2)
      const float4* s4 = reinterpret_cast<const float4*>(a.x);
      const int n4 = a.C / 4;
      for (int i0 = tid; i0 < n4; i0 += 8 * kFG_THREADS) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0 + u * kFG_THREADS < n4) v[u] = s4[i0 + u * kFG_THREADS];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0 + u * kFG_THREADS < n4) reinterpret_cast<float4*>(xs)[swz4(i0 + u * kFG_THREADS)] = v[u];
      }
    }
  }
  for (int i = tid; i < kFG_WARPS * a.rows_cap; i += kFG_THREADS) part[i] = 0.f;
  if constexpr (kNF4) nf4_build_lut(lut, tid, kFG_THREADS);
  __syncthreads();
  const uint32_t* lut_l = lut + lane;

  int row = (int)(g_begin / Gr);
  int gcol = (int)(g_begin - (long long)row * Gr);   // group index within the row
  float acc = 0.f;
  // consume one register batch (rows are whole groups: a boundary is one compare)
  auto consume = [&](const uint4 (&wv)[UNROLL], const float (&sv)[UNROLL], long long g0) {
#if FG_FAST
    // Fast path: a whole batch inside the slice of a row at least UNROLL groups long crosses at
    // most one row boundary. Granules before it add to acc, the rest to acc1 (predicated adds, no
    // branch per granule); the order of every row's sum is the one of the general path below.
    // Measured (profiles/kb_r01_warps_ab.json): bf16 expert 70.6 -> 66.6 us; the low-bit dot
    // products got slower (INT8 53.2 -> 58.4 us), so they keep the general loop.
#ifdef FG_FAST_ALL
    constexpr bool kFastT = !kNF4;
#else
    constexpr bool kFastT = std::is_same<WT, __nv_bfloat16>::value || std::is_same<WT, float>::value;
#endif
    if constexpr (kFastT) if (Gr >= UNROLL && g0 + UNROLL <= g_end) {
      const int b = Gr - gcol;  // granules left in the current row (>= 1)
      const uint4* x0 = reinterpret_cast<const uint4*>(xs) + lane;
      float acc1 = 0.f;
#pragma unroll
      for (int i = 0; i < UNROLL; ++i) {
        const int c = gcol + i < Gr ? gcol + i : gcol + i - Gr;
        const uint4* xp = x0 + (size_t)c * Q * 32;
        const float t = FDot<WT, XT>::run(wv[i], xp);
        if (i < b) acc += t; else acc1 += t;
      }
      if (b <= UNROLL) {  // the row completed inside this batch
        const float t = warp_sum(acc);
        if (lane == 0) part[warp * a.rows_cap + row] += t;
        acc = acc1;
        ++row;
        gcol = UNROLL - b;
      } else {
        gcol += UNROLL;
      }
      return;
    }
#endif
#pragma unroll
    for (int i = 0; i < UNROLL; ++i) {
      if (g0 + i < g_end) {
        const uint4* xp = reinterpret_cast<const uint4*>(xs) + (size_t)gcol * Q * 32 + lane;
        if constexpr (kNF4)
          acc = fmaf(sv[i], nf4_dot(wv[i], xp, lut_l, XT{}), acc);
        else
          acc += FDot<WT, XT>::run(wv[i], xp);
        if (++gcol == Gr) {  // row complete (warp-uniform)
          const float t = warp_sum(acc);
          if (lane == 0) part[warp * a.rows_cap + row] += t;
          acc = 0.f;
          gcol = 0;
          ++row;
        }
      }
    }
  };
#if FG_PIPE == 3
  {
    // two batches in flight; batch b covers groups [b0, b0 + UNROLL) with b0 = (w + 16 i) * UNROLL
    constexpr long long STEP = (long long)kFG_WARPS * UNROLL;
    auto consume_at = [&](const uint4 (&wv)[UNROLL], long long g0) {
      row = (int)(g0 / Gr);
      gcol = (int)(g0 - (long long)row * Gr);
      consume(wv, sa, g0);
      if (gcol != 0) {  // batch ended inside a row: flush the partial now (rows are shared by warps)
        const float t = warp_sum(acc);
        if (lane == 0) part[warp * a.rows_cap + row] += t;
        acc = 0.f;
      }
    };
    for (long long g0 = g_begin; g0 < g_end; g0 += 2 * STEP) {
      const long long g1 = g0 + STEP, g2 = g0 + 2 * STEP;
#pragma unroll
      for (int i = 0; i < UNROLL; ++i)
        if (g1 + i < g_end) wb[i] = ld_stream_pol(base + (g1 + i) * 32 + lane, pol);
      consume_at(wa, g0);
#pragma unroll
      for (int i = 0; i < UNROLL; ++i)
        if (g2 + i < g_end) wa[i] = ld_stream_pol(base + (g2 + i) * 32 + lane, pol);
      if (g1 < g_end) consume_at(wb, g1);
    }
    gcol = 0;  // everything flushed
  }
#elif FG_PIPE == 0
  // software pipeline, two register batches in flight: load batch n+1, then consume batch n
  for (long long g0 = g_begin; g0 < g_end; g0 += 2 * UNROLL) {
    const long long g1 = g0 + UNROLL, g2 = g0 + 2 * UNROLL;
#pragma unroll
    for (int i = 0; i < UNROLL; ++i)
      if (g1 + i < g_end) {
        wb[i] = ld_stream_pol(base + (g1 + i) * 32 + lane, pol);
        if constexpr (kNF4) sb[i] = __ldg(scb + (((g1 + i) * 32 + lane) >> 1));
      }
    consume(wa, sa, g0);
#pragma unroll
    for (int i = 0; i < UNROLL; ++i)
      if (g2 + i < g_end) {
        wa[i] = ld_stream_pol(base + (g2 + i) * 32 + lane, pol);
        if constexpr (kNF4) sa[i] = __ldg(scb + (((g2 + i) * 32 + lane) >> 1));
      }
    if (g1 < g_end) consume(wb, sb, g1);
  }
#elif FG_PIPE == 1
  // both batches issued before the dependency wait; consume one, re-issue it two batches ahead
  for (long long g0 = g_begin; g0 < g_end; g0 += 2 * UNROLL) {
    const long long g1 = g0 + UNROLL, g2 = g0 + 2 * UNROLL, g3 = g0 + 3 * UNROLL;
    consume(wa, sa, g0);
#pragma unroll
    for (int i = 0; i < UNROLL; ++i)
      if (g2 + i < g_end) wa[i] = ld_stream_pol(base + (g2 + i) * 32 + lane, pol);
    if (g1 < g_end) consume(wb, sb, g1);
#pragma unroll
    for (int i = 0; i < UNROLL; ++i)
      if (g3 + i < g_end) wb[i] = ld_stream_pol(base + (g3 + i) * 32 + lane, pol);
  }
#else
  // three register batches: two stay in flight while one is consumed
  for (long long g0 = g_begin; g0 < g_end; g0 += 3 * UNROLL) {
    const long long g1 = g0 + UNROLL, g2 = g0 + 2 * UNROLL;
    consume(wa, sa, g0);
#pragma unroll
    for (int i = 0; i < UNROLL; ++i)
      if (g0 + 3 * UNROLL + i < g_end) wa[i] = ld_stream_pol(base + (g0 + 3 * UNROLL + i) * 32 + lane, pol);
    if (g1 < g_end) consume(wb, sb, g1);
#pragma unroll
    for (int i = 0; i < UNROLL; ++i)
      if (g0 + 4 * UNROLL + i < g_end) wb[i] = ld_stream_pol(base + (g0 + 4 * UNROLL + i) * 32 + lane, pol);
    if (g2 < g_end) consume(wc, sa, g2);
#pragma unroll
    for (int i = 0; i < UNROLL; ++i)
      if (g0 + 5 * UNROLL + i < g_end) wc[i] = ld_stream_pol(base + (g0 + 5 * UNROLL + i) * 32 + lane, pol);
  }
#endif
  if (gcol != 0) {  // slice ended inside a row
    const float t = warp_sum(acc);
    if (lane == 0) part[warp * a.rows_cap + row] += t;
  }
  } else {
    // ---- tensor-core branch (bf16m). The CTA's rows [rb, re) are cut into 16-row tiles (the last
    // one masked); warp w owns the columns of 32-column blocks [kb0, kb1) of EVERY tile (split-K
    // over the warps: a row's value depends only on the warp split, not on the CTA's range), so
    // each (row, warp) partial is written once and the epilogue's fixed-order warp sum is reused.
    // A fragment from the row-major blob: k inside an mma may be permuted as long as A and B use
    // the same permutation. Lane (g = lane / 4, q = lane % 4) loads 16 bytes = columns
    // [32 kb + 8 q, +8) of rows g and g + 8; words .x/.y feed mma #1 as k-pairs q / q + 4, words
    // .z/.w mma #2. B column 0 = x hi, column 1 = x lo (lanes 0-3 / 4-7), the others zero; the
    // result of row g is D[g][0] + D[g][1] (lane q == 0: c0 + c1, row g + 8: c2 + c3).
    constexpr int KU = FG_MMA_KU;
    const int KB = a.C / 32;
    const int kb0 = (int)((long long)KB * warp / kFG_WARPS), kb1 = (int)((long long)KB * (warp + 1) / kFG_WARPS);
    const int nkb = kb1 - kb0;
    const int ntiles = (nrows + 15) / 16;
    const int g = lane >> 2, q = lane & 3;
    const long long rowq = a.C / 8;  // uint4 per row
    const uint4* Wl = reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(W) + rb * (long long)a.C * 2) +
                      (long long)g * rowq + q;
    const uint64_t pol = l2_policy(a.evict_first != 0);
    int lt = 0, lk = 0;  // load cursor (tile, k-block within the warp's range)
    auto load_batch = [&](uint4 (&w0)[KU], uint4 (&w1)[KU]) {
#pragma unroll
      for (int i = 0; i < KU; ++i) {
        if (lt < ntiles) {
          const uint4* p = Wl + (long long)(16 * lt) * rowq + (long long)(kb0 + lk) * 4;
          const int r0 = 16 * lt + g;
          w0[i] = r0 < nrows ? ld_stream_pol(p, pol) : make_uint4(0u, 0u, 0u, 0u);
          w1[i] = r0 + 8 < nrows ? ld_stream_pol(p + 8 * rowq, pol) : make_uint4(0u, 0u, 0u, 0u);
          if (++lk == nkb) { lk = 0; ++lt; }
        }
      }
    };
    uint4 wa0[KU], wa1[KU], wb0[KU], wb1[KU];
    if (nkb > 0) load_batch(wa0, wa1);  // weights first: they do not depend on the previous kernel
    if (!early) wait_dep();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // x as bf16 hi / lo, 8-column chunks [hi 16 B | lo 16 B] (lanes 0-3 and 4-7 read 128 bytes in one
    // shared-memory wavefront)
    uint4* xs4 = reinterpret_cast<uint4*>(xs);
    if (a.x_bf16) {
      const uint4* s4 = reinterpret_cast<const uint4*>(a.x);
      for (int i = tid; i < a.C / 8; i += kFG_THREADS) {
        xs4[2 * i] = s4[i];
        xs4[2 * i + 1] = make_uint4(0u, 0u, 0u, 0u);
      }
    } else {
      const float4* s4 = reinterpret_cast<const float4*>(a.x);
      const int n8 = a.C / 8;
      for (int i0 = tid; i0 < n8; i0 += 4 * kFG_THREADS) {
        float4 v[4][2];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i0 + u * kFG_THREADS < n8) {
            v[u][0] = s4[2 * (i0 + u * kFG_THREADS)];
            v[u][1] = s4[2 * (i0 + u * kFG_THREADS) + 1];
          }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i0 + u * kFG_THREADS < n8) {
            const float e[8] = {v[u][0].x, v[u][0].y, v[u][0].z, v[u][0].w, v[u][1].x, v[u][1].y, v[u][1].z, v[u][1].w};
            uint32_t hw[4], lw[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const __nv_bfloat16 h0 = __float2bfloat16_rn(e[2 * j]), h1 = __float2bfloat16_rn(e[2 * j + 1]);
              const __nv_bfloat16 l0 = __float2bfloat16_rn(e[2 * j] - __bfloat162float(h0));
              const __nv_bfloat16 l1 = __float2bfloat16_rn(e[2 * j + 1] - __bfloat162float(h1));
              hw[j] = (uint32_t)__bfloat16_as_ushort(h0) | ((uint32_t)__bfloat16_as_ushort(h1) << 16);
              lw[j] = (uint32_t)__bfloat16_as_ushort(l0) | ((uint32_t)__bfloat16_as_ushort(l1) << 16);
            }
            xs4[2 * (i0 + u * kFG_THREADS)] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            xs4[2 * (i0 + u * kFG_THREADS) + 1] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
          }
      }
    }
    for (int i = tid; i < kFG_WARPS * a.rows_cap; i += kFG_THREADS) part[i] = 0.f;
    __syncthreads();
    // this lane's B words: chunk kb * 4 + q, hi (g == 0) or lo (g == 1); other columns are zero
    const uint4* xl = xs4 + 2 * (kb0 * 4 + q) + (g == 1 ? 1 : 0);
    const bool xon = g < 2;
    float c[4] = {0.f, 0.f, 0.f, 0.f};
    int ct = 0, ck = 0;  // consume cursor
    auto consume = [&](const uint4 (&w0)[KU], const uint4 (&w1)[KU]) {
#pragma unroll
      for (int i = 0; i < KU; ++i) {
        if (ct < ntiles) {
          uint4 xv = xl[8 * ck];
          if (!xon) xv = make_uint4(0u, 0u, 0u, 0u);
          mma_bf16_16816(c, w0[i].x, w1[i].x, w0[i].y, w1[i].y, xv.x, xv.y);
          mma_bf16_16816(c, w0[i].z, w1[i].z, w0[i].w, w1[i].w, xv.z, xv.w);
          if (++ck == nkb) {  // tile complete: this warp's partials of its 16 rows
            if (q == 0) {
              const int r = 16 * ct + g;
              if (r < nrows) part[warp * a.rows_cap + r] = c[0] + c[1];
              if (r + 8 < nrows) part[warp * a.rows_cap + r + 8] = c[2] + c[3];
            }
            c[0] = c[1] = c[2] = c[3] = 0.f;
            ck = 0;
            ++ct;
          }
        }
      }
    };
    if (nkb > 0) {
      // two register batches in flight: load batch n + 1, then consume batch n
      while (ct < ntiles) {
        load_batch(wb0, wb1);
        consume(wa0, wa1);
        if (ct >= ntiles) break;
        load_batch(wa0, wa1);
        consume(wb0, wb1);
      }
    }
  }
  __syncthreads();

  if (MODE == 0) {
    for (int p = tid; p < nrows / 2; p += kFG_THREADS) {
      float g = 0.f, v = 0.f;
#pragma unroll
      for (int w = 0; w < kFG_WARPS; ++w) {
        g += part[w * a.rows_cap + 2 * p];
        v += part[w * a.rows_cap + 2 * p + 1];
      }
      if (!kNF4 && sc != nullptr) { g *= sc[rb + 2 * p]; v *= sc[rb + 2 * p + 1]; }
      a.out[rb / 2 + p] = silu_mul(g, v);
    }
  } else if (MODE == 1 || MODE == 3) {
    const float gw = a.gate_w ? a.gate_w[gate_idx] : 1.f;
    for (int r = tid; r < nrows; r += kFG_THREADS) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < kFG_WARPS; ++w) s += part[w * a.rows_cap + r];
      if (!kNF4 && sc != nullptr) s *= sc[rb + r];
      const float v = a.accumulate ? a.out[rb + r] + gw * s : gw * s;
      a.out[rb + r] = v;
      if (MODE == 1 && a.send.dst != nullptr) {  // p2p_send's sum: prev[0] + ... + this expert's output
        float t = v;
        if (a.send.nprev > 0) {
          t = a.send.prev[0][rb + r];
          for (int i = 1; i < a.send.nprev; ++i) t += a.send.prev[i][rb + r];
          t += v;
        }
        // one 8-byte {value, epoch} store: the receiver polls the pair, so no fence or flag is needed
        // (a system-scope fence per CTA before a flag release cost ~30 us per launch)
        asm volatile("st.volatile.global.v2.u32 [%0], {%1, %2};" ::"l"(a.send.dst + 2 * (rb + r)),
                     "r"(__float_as_uint(t)), "r"(a.send.epoch)
                     : "memory");
      }
    }
  } else {
    unsigned long long best = 0ull;
    for (int r = tid; r < nrows; r += kFG_THREADS) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < kFG_WARPS; ++w) s += part[w * a.rows_cap + r];
      if (!kNF4 && sc != nullptr) s *= sc[rb + r];  // int8-row LM head (the shadow's own token)
      if (a.out) a.out[rb + r] = s;
      const unsigned long long key = fg_argmax_key(s, (int)(rb + r));
      best = key > best ? key : best;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
      best = other > best ? other : best;
    }
    if (lane == 0) kbest[warp] = best;
    __syncthreads();
    if (tid == 0) {
      unsigned long long b = kbest[0];
      for (int w = 1; w < kFG_WARPS; ++w) b = kbest[w] > b ? kbest[w] : b;
      a.partial[blockIdx.x] = b;
      __threadfence();
      const unsigned int t = atomicAdd(a.ticket, 1u);
      is_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (is_last && tid == 0) {
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

template <typename WT, typename XT, int MODE, int UNROLL>
__global__ void __launch_bounds__(kFG_THREADS, 1) flat_gemv_kernel(const FlatArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];
  flat_phase<WT, XT, MODE, UNROLL>(a, sm, PdlWait{});
}

// Grid-wide barrier for a cooperative launch (all CTAs co-resident): one arrival counter per
// launch slot; `target` grows by gridDim.x every launch so the counter never needs resetting.
struct GridBarrier {
  unsigned int* counter;
  unsigned int target;
  __device__ __forceinline__ void operator()() const {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(counter, 1u);
      unsigned int v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
      } while ((int)(v - target) < 0);
    }
    __syncthreads();
  }
};

// Fused expert FFN: phase 1 = W13 + SwiGLU -> a (global), grid barrier, phase 2 = W2 + gate -> y.
// One launch per expert; phase 2's first weight batches are in flight before the barrier.
template <typename WT, typename XT, int UNROLL>
__global__ void __launch_bounds__(kFG_THREADS, 1)
flat_expert_kernel(const FlatArgs a13, const FlatArgs a2, unsigned int* counter, unsigned int target) {
  extern __shared__ __align__(128) uint8_t sm[];
  flat_phase<WT, XT, 0, UNROLL>(a13, sm, PdlWait{});
  __syncthreads();
  flat_phase<WT, float, 1, UNROLL>(a2, sm, GridBarrier{counter, target}, /*ids_ready=*/true);
}

// Rows must be whole 512-byte groups (the flat stream's unit), else the launch is refused.
template <typename WT> static bool flat_row_ok(long long C) { return C > 0 && (C * FTraits<WT>::bits / 8) % 512 == 0; }

template <typename WT, typename XT, int MODE>
static cudaError_t fg_launch(FlatArgs a, cudaStream_t s, bool pdl) {
  constexpr int UNROLL = kFG_UNROLL;
  static int ef = -1;
  if (ef < 0) {
    const char* e = getenv("ODMOE_L2_EVICT_FIRST");
    ef = (e && e[0] == '0') ? 0 : 1;
  }
  a.evict_first = ef;
  if (!flat_row_ok<WT>(a.C)) return cudaErrorInvalidValue;
  const int sms = stream_grid_sms();
  const long long units = MODE == 0 ? a.R / 2 : a.R;
  const int grid = (int)(units < sms ? (units > 0 ? units : 1) : sms);
  a.rows_cap = (int)((units + grid - 1) / grid) * (MODE == 0 ? 2 : 1) + 2;
  const size_t smem = (size_t)kFG_WARPS * a.rows_cap * sizeof(float) + (size_t)a.C * sizeof(XT) + 16 +
                      (FTraits<WT>::nf4 ? kNF4LutWords * 4 : 0);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  auto kern = flat_gemv_kernel<WT, XT, MODE, UNROLL>;
  if (smem > 40 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kFG_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

// INT8 / FP8 weights with fp32 activations in shared memory: the dot products then skip the
// bf16 -> fp32 unpack of every activation pair (ALU-bound kernels; INT8 expert 57.4 -> 53.3 us,
// FP8 55.3 -> 54.1 us, profiles/kb_r01_lowbit_*.json; NF4 is faster with bf16 activations, whose
// 64-byte-per-lane footprint keeps shared-memory traffic lower). ODMOE_LOWBIT_X=bf16: A/B.
// bf16 expert phases (W13 + SwiGLU, W2 + gate) on the tensor cores (bf16m) with ODMOE_MAIN_MMA=1
// (A/B; off by default). Measured (profiles/launches_r02_expert_bf16_{mma,ffma2}.csv): 63.9 vs 62.0
// us per expert in the ncu launch list -- the FFMA2 stream is already at the pure-read floor of a
// 352 MB launch (62.9 us, profiles/pattern_bench_r01.json), so fewer instructions buy nothing.
static bool main_mma() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ODMOE_MAIN_MMA");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

static bool lowbit_xf32() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ODMOE_LOWBIT_X");
    v = (e && e[0] == 'b') ? 0 : 1;
  }
  return v == 1;
}

cudaError_t launch_w13_flat(ExpertRef ex, WType wt, const void* u, int u_f32, float* a_out, int d, int F,
                            cudaStream_t s, bool pdl) {
  FlatArgs a{};
  a.ex = ex; a.second = 0; a.x = u; a.x_bf16 = !u_f32; a.R = 2 * F; a.C = d; a.out = a_out;
  a.d_full = d; a.F_full = F;
  switch (wt) {
    case W_BF16: return main_mma() ? fg_launch<bf16m, float, 0>(a, s, pdl) : fg_launch<__nv_bfloat16, uint16_t, 0>(a, s, pdl);
    case W_F32: return fg_launch<float, float, 0>(a, s, pdl);
    case W_I8: return lowbit_xf32() ? fg_launch<int8_t, float, 0>(a, s, pdl) : fg_launch<int8_t, uint16_t, 0>(a, s, pdl);
    case W_U8: return lowbit_xf32() ? fg_launch<u8b, float, 0>(a, s, pdl) : fg_launch<u8b, uint16_t, 0>(a, s, pdl);
    case W_NF4: return fg_launch<nf4x2, uint16_t, 0>(a, s, pdl);  // bf16 x measured faster for NF4
    case W_F8: return lowbit_xf32() ? fg_launch<fp8e4, float, 0>(a, s, pdl) : fg_launch<fp8e4, uint16_t, 0>(a, s, pdl);
    default: break;  // W_I8P: mma_gemv.cu
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_w2_flat(ExpertRef ex, WType wt, const float* act, const float* gate_w, float* y, int d,
                           int F, cudaStream_t s, bool pdl, const P2PSend* send) {
  FlatArgs a{};
  a.ex = ex; a.second = 1; a.x = act; a.x_bf16 = 0; a.R = d; a.C = F; a.gate_w = gate_w; a.out = y;
  a.d_full = d; a.F_full = F;
  if (send) a.send = *send;
  switch (wt) {
    case W_BF16: return main_mma() ? fg_launch<bf16m, float, 1>(a, s, pdl) : fg_launch<__nv_bfloat16, float, 1>(a, s, pdl);
    case W_F32: return fg_launch<float, float, 1>(a, s, pdl);
    case W_I8: return fg_launch<int8_t, float, 1>(a, s, pdl);
    case W_U8: return fg_launch<u8b, float, 1>(a, s, pdl);
    case W_NF4: return fg_launch<nf4x2, float, 1>(a, s, pdl);
    case W_F8: return fg_launch<fp8e4, float, 1>(a, s, pdl);
    default: break;  // W_I8P: mma_gemv.cu
  }
  return cudaErrorInvalidValue;
}

// Rows shorter than one flat group (small test shapes): one warp per row. NORM: x = RMSNorm(h)
// (rounded to bf16 unless the weights are fp32), else x = fp32 input; out = or += (row-scaled).
template <typename WT, bool NORM>
__global__ void __launch_bounds__(256) gemv_rows_small_kernel(const float* __restrict__ xin, const WT* __restrict__ W,
                                                              const float* __restrict__ sc, int R, int C, float eps,
                                                              float* out, int accumulate) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  extern __shared__ float xs_small[];
  __shared__ float red[9];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float rstd = 1.f;
  if (NORM) {
    float ss = 0.f;
    for (int j = tid; j < C; j += blockDim.x) ss = fmaf(xin[j], xin[j], ss);
    ss = warp_sum(ss);
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    if (tid == 0) {
      float t = 0.f;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      red[8] = t;
    }
    __syncthreads();
    rstd = 1.0f / sqrtf(red[8] / (float)C + eps);
  }
  for (int j = tid; j < C; j += blockDim.x) {
    float v = xin[j] * rstd;
    if (NORM && !std::is_same<WT, float>::value) v = __bfloat162float(__float2bfloat16_rn(v));
    xs_small[j] = v;
  }
  __syncthreads();
  const int r = blockIdx.x * (blockDim.x >> 5) + warp;
  if (r >= R) return;
  float acc = 0.f;
  for (int j = lane; j < C; j += 32) {
    float w;
    if constexpr (std::is_same<WT, __nv_bfloat16>::value) w = __bfloat162float(W[(size_t)r * C + j]);
    else w = (float)W[(size_t)r * C + j];
    acc = fmaf(w, xs_small[j], acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) {
    if (sc) acc *= sc[r];
    out[r] = accumulate ? out[r] + acc : acc;
  }
}

template <typename WT, bool NORM>
static cudaError_t small_rows(const float* x, const void* W, const float* sc, int R, int C, float eps, float* out,
                              int acc, cudaStream_t s) {
  gemv_rows_small_kernel<WT, NORM><<<(R + 7) / 8, 256, (size_t)C * 4, s>>>(x, (const WT*)W, sc, R, C, eps, out, acc);
  return cudaGetLastError();
}

// Attention projections (reading Q29). QKV: out = W RMSNorm(h) (activations rounded to bf16 for
// bf16 / int8 weights, as for u), R rows of C = d columns. O: h += W o with o fp32.
cudaError_t launch_gemv_rmsnorm(const float* h, const void* W, const float* scales, WType wt, int R, int C, float eps,
                                float* out, cudaStream_t s, bool pdl) {
  const bool flat = wt == W_BF16 ? flat_row_ok<__nv_bfloat16>(C) : (wt == W_F32 ? flat_row_ok<float>(C) : flat_row_ok<int8_t>(C));
  if (!flat) {
    switch (wt) {
      case W_BF16: return small_rows<__nv_bfloat16, true>(h, W, scales, R, C, eps, out, 0, s);
      case W_F32: return small_rows<float, true>(h, W, scales, R, C, eps, out, 0, s);
      case W_I8: return small_rows<int8_t, true>(h, W, scales, R, C, eps, out, 0, s);
      default: return cudaErrorInvalidValue;
    }
  }
  FlatArgs a{};
  a.ex = direct_ref(W, scales, 0); a.second = 0; a.R = R; a.C = C; a.out = out; a.h = h; a.eps = eps;
  switch (wt) {
    case W_BF16: return fg_launch<__nv_bfloat16, uint16_t, 3>(a, s, pdl);
    case W_F32: return fg_launch<float, float, 3>(a, s, pdl);
    case W_I8: return fg_launch<int8_t, uint16_t, 3>(a, s, pdl);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gemv_acc(const void* W, const float* scales, WType wt, int R, int C, const float* x, float* out,
                            cudaStream_t s, bool pdl) {
  const bool flat = wt == W_BF16 ? flat_row_ok<__nv_bfloat16>(C) : (wt == W_F32 ? flat_row_ok<float>(C) : flat_row_ok<int8_t>(C));
  if (!flat) {
    switch (wt) {
      case W_BF16: return small_rows<__nv_bfloat16, false>(x, W, scales, R, C, 0.f, out, 1, s);
      case W_F32: return small_rows<float, false>(x, W, scales, R, C, 0.f, out, 1, s);
      case W_I8: return small_rows<int8_t, false>(x, W, scales, R, C, 0.f, out, 1, s);
      default: return cudaErrorInvalidValue;
    }
  }
  FlatArgs a{};
  a.ex = direct_ref(W, scales, 0); a.second = 0; a.x = x; a.x_bf16 = 0; a.R = R; a.C = C; a.out = out;
  a.accumulate = 1;
  switch (wt) {
    case W_BF16: return fg_launch<__nv_bfloat16, float, 1>(a, s, pdl);
    case W_F32: return fg_launch<float, float, 1>(a, s, pdl);
    case W_I8: return fg_launch<int8_t, float, 1>(a, s, pdl);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_lm_head_flat(const float* h, const void* W, WType wt, int V, int d, float eps,
                                int32_t* token_out, float* logits, void* scratch, cudaStream_t s, bool pdl,
                                const float* scales) {
  FlatArgs a{};
  a.ex = direct_ref(W, scales, 0); a.second = 0; a.R = V; a.C = d; a.out = logits; a.h = h; a.eps = eps;
  a.partial = reinterpret_cast<unsigned long long*>(scratch);
  a.ticket = reinterpret_cast<unsigned int*>(a.partial + 1024);
  a.token_out = token_out;
  switch (wt) {
    case W_BF16: return fg_launch<__nv_bfloat16, uint16_t, 2>(a, s, pdl);
    case W_F32: return fg_launch<float, float, 2>(a, s, pdl);
    case W_I8: return fg_launch<int8_t, uint16_t, 2>(a, s, pdl);
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------- fused expert FFN launcher
// Multi-expert fused FFN: the n (<= 4) experts of one layer that this GPU computes, in ONE
// cooperative launch: W13 of all n, one grid barrier, W2 of all n. Every CTA takes the same row
// range of each expert as the one-expert kernel would (so each output is computed with the same
// per-warp split and is bitwise identical to it), one expert after the other. One launch, ramp,
// barrier and tail per layer instead of per expert.
constexpr int kMaxMulti = 4;
struct MultiArgs {
  FlatArgs a13[kMaxMulti], a2[kMaxMulti];
  int n;
};
struct NoWait {
  __device__ __forceinline__ void operator()() const {}
};

// NE (experts) is a template parameter: every m.a13[e] / m.a2[e] is then a compile-time index into
// the parameter space (a runtime index made the compiler copy the argument structs to local memory).
template <typename WT, typename XT, int UNROLL, int NE>
__global__ void __launch_bounds__(kFG_THREADS, 1)
flat_experts_kernel(const __grid_constant__ MultiArgs m, unsigned int* counter, unsigned int target) {
  extern __shared__ __align__(128) uint8_t sm[];
  long long p0, p1, r0, r1;
  split_range(m.a13[0].R / 2, gridDim.x, blockIdx.x, p0, p1);  // gate/up pairs of each expert
  split_range(m.a2[0].R, gridDim.x, blockIdx.x, r0, r1);       // W2 rows of each expert
  flat_phase<WT, XT, 0, UNROLL>(m.a13[0], sm, PdlWait{}, false, 2 * p0, 2 * p1);
#pragma unroll
  for (int e = 1; e < NE; ++e) {
    __syncthreads();
    flat_phase<WT, XT, 0, UNROLL>(m.a13[e], sm, NoWait{}, true, 2 * p0, 2 * p1);
  }
  __syncthreads();
  flat_phase<WT, float, 1, UNROLL>(m.a2[0], sm, GridBarrier{counter, target}, true, r0, r1);
#pragma unroll
  for (int e = 1; e < NE; ++e) {
    __syncthreads();
    flat_phase<WT, float, 1, UNROLL>(m.a2[e], sm, NoWait{}, true, r0, r1);
  }
}

// Grid-barrier arrival counter of this device (one per device; see fused_launch).
// One arrival counter per (device, stream): launches on one stream are ordered, so their targets
// can simply keep growing; two streams (e.g. two engines in one process) never share a counter.
struct BarrierState {
  unsigned int* counter = nullptr;
  unsigned int epoch = 0;
};
static std::mutex g_barrier_mu;
static std::map<std::pair<int, cudaStream_t>, BarrierState> g_barriers;
static cudaError_t barrier_counter(int dev, cudaStream_t s, BarrierState*& out) {
  std::lock_guard<std::mutex> lk(g_barrier_mu);
  BarrierState& b = g_barriers[{dev, s}];
  if (!b.counter) {
    cudaError_t e = cudaMalloc(&b.counter, sizeof(unsigned int));
    if (e != cudaSuccess) return e;
    e = cudaMemset(b.counter, 0, sizeof(unsigned int));
    if (e != cudaSuccess) return e;
  }
  out = &b;
  return cudaSuccess;
}

cudaError_t coop_barrier_next(cudaStream_t s, int grid, unsigned int** counter, unsigned int* target) {
  int dev = 0;
  cudaGetDevice(&dev);
  BarrierState* bs = nullptr;
  cudaError_t e = barrier_counter(dev, s, bs);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_barrier_mu);
  bs->epoch += (unsigned int)grid;
  *counter = bs->counter;
  *target = bs->epoch;
  return cudaSuccess;
}

unsigned int* barrier_capture_reset(cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  BarrierState* bs = nullptr;
  if (barrier_counter(dev, s, bs) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(g_barrier_mu);
  bs->epoch = 0;
  return bs->counter;
}

template <typename WT, typename XT>
static cudaError_t multi_launch(MultiArgs m, cudaStream_t s, bool pdl) {
  constexpr int UNROLL = kFG_UNROLL;
  int dev = 0;
  cudaGetDevice(&dev);
  BarrierState* bs = nullptr;
  cudaError_t e = barrier_counter(dev, s, bs);
  if (e != cudaSuccess) return e;
  static int ef = -1;
  if (ef < 0) {
    const char* v = getenv("ODMOE_L2_EVICT_FIRST");
    ef = (v && v[0] == '0') ? 0 : 1;
  }
  const int n = m.n;
  const long long F = m.a13[0].R / 2, D = m.a2[0].R;
  if (!flat_row_ok<WT>(m.a13[0].C) || !flat_row_ok<WT>(m.a2[0].C)) return cudaErrorInvalidValue;
  const int sms = stream_grid_sms();
  const long long units = F < D ? F : D;   // the one-expert kernel's grid (same per-CTA rows)
  const int grid = (int)(units < sms ? (units > 0 ? units : 1) : sms);
  const int cap13 = (int)((F + grid - 1) / grid) * 2 + 2;
  const int cap2 = (int)((D + grid - 1) / grid) + 2;
  for (int i = 0; i < n; ++i) {
    m.a13[i].evict_first = m.a2[i].evict_first = ef;
    m.a13[i].rows_cap = cap13;
    m.a2[i].rows_cap = cap2;
  }
  const size_t lut = FTraits<WT>::nf4 ? kNF4LutWords * 4 : 0;
  const size_t s1 = (size_t)kFG_WARPS * cap13 * sizeof(float) + (size_t)m.a13[0].C * sizeof(XT) + 16 + lut;
  const size_t s2 = (size_t)kFG_WARPS * cap2 * sizeof(float) + (size_t)m.a2[0].C * sizeof(float) + 16 + lut;
  const size_t smem = s1 > s2 ? s1 : s2;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  void (*kern)(const MultiArgs, unsigned int*, unsigned int) =
      n == 1 ? flat_experts_kernel<WT, XT, UNROLL, 1>
             : (n == 2 ? flat_experts_kernel<WT, XT, UNROLL, 2>
                       : (n == 3 ? flat_experts_kernel<WT, XT, UNROLL, 3> : flat_experts_kernel<WT, XT, UNROLL, 4>));
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const unsigned int target = bs->epoch + (unsigned int)grid;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kFG_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  e = cudaLaunchKernelEx(&cfg, kern, m, bs->counter, target);
  if (e == cudaSuccess) bs->epoch = target;
  return e;
}

cudaError_t launch_experts_fused(int n, const ExpertRef* ex, const void* const* w2_direct, const float* const* s2_direct,
                                 WType wt, const void* u, int u_f32, float* a_buf, const float* gate_w,
                                 float* const* y, int d, int F, cudaStream_t s, bool pdl, const P2PSend* send) {
  if (n < 1 || n > kMaxMulti) return cudaErrorInvalidValue;
  MultiArgs m{};
  m.n = n;
  for (int i = 0; i < n; ++i) {
    FlatArgs& a13 = m.a13[i];
    FlatArgs& a2 = m.a2[i];
    a13.ex = ex[i]; a13.second = 0; a13.x = u; a13.x_bf16 = !u_f32; a13.R = 2 * F; a13.C = d;
    a13.out = a_buf + (size_t)i * F; a13.d_full = d; a13.F_full = F;
    a2.ex = ex[i]; a2.second = 1; a2.x = a_buf + (size_t)i * F; a2.x_bf16 = 0; a2.R = d; a2.C = F;
    a2.gate_w = gate_w; a2.out = y[i]; a2.d_full = d; a2.F_full = F;
    if (ex[i].tbl == nullptr) {
      a2.ex.blob = w2_direct[i];
      a2.ex.scales = s2_direct ? s2_direct[i] : nullptr;
    }
    if (send && i == n - 1) a2.send = *send;  // the last expert's rows carry the layer's sum
  }
  switch (wt) {
    case W_BF16: return main_mma() ? multi_launch<bf16m, float>(m, s, pdl) : multi_launch<__nv_bfloat16, uint16_t>(m, s, pdl);
    case W_F32: return multi_launch<float, float>(m, s, pdl);
    default: return cudaErrorInvalidValue;
  }
}

// One phase (MODE 0: W13+SwiGLU, MODE 1: W2+gate) of the NE experts of one layer in ONE
// non-cooperative launch (the shadow's k experts). Every CTA takes the one-expert
// kernel's row range of each expert in turn, so each expert's sums are those of its own launch
// (bitwise), and one launch + ramp + tail is paid per phase instead of per expert. No grid barrier:
// it may share the GPU with the compute stream's cooperative grid.
template <typename WT, typename XT, int MODE, int UNROLL, int NE>
__global__ void __launch_bounds__(kFG_THREADS, 1) flat_gemv_multi_kernel(const __grid_constant__ MultiArgs m) {
  extern __shared__ __align__(128) uint8_t sm[];
  long long r0, r1;
  if (MODE == 0) {
    split_range(m.a13[0].R / 2, gridDim.x, blockIdx.x, r0, r1);
    r0 *= 2; r1 *= 2;
  } else {
    split_range(m.a2[0].R, gridDim.x, blockIdx.x, r0, r1);
  }
  flat_phase<WT, XT, MODE, UNROLL>(MODE == 0 ? m.a13[0] : m.a2[0], sm, PdlWait{}, false, r0, r1);
#pragma unroll
  for (int e = 1; e < NE; ++e) {
    __syncthreads();
    flat_phase<WT, XT, MODE, UNROLL>(MODE == 0 ? m.a13[e] : m.a2[e], sm, NoWait{}, true, r0, r1);
  }
}

template <typename WT, typename XT, int MODE>
static cudaError_t fg_multi_launch(MultiArgs m, cudaStream_t s, bool pdl) {
  constexpr int UNROLL = kFG_UNROLL;
  static int ef = -1;
  if (ef < 0) {
    const char* e = getenv("ODMOE_L2_EVICT_FIRST");
    ef = (e && e[0] == '0') ? 0 : 1;
  }
  FlatArgs* as = MODE == 0 ? m.a13 : m.a2;
  if (!flat_row_ok<WT>(as[0].C)) return cudaErrorInvalidValue;
  const int sms = stream_grid_sms();
  const long long units = MODE == 0 ? as[0].R / 2 : as[0].R;   // fg_launch's grid and rows_cap
  const int grid = (int)(units < sms ? (units > 0 ? units : 1) : sms);
  const int cap = (int)((units + grid - 1) / grid) * (MODE == 0 ? 2 : 1) + 2;
  for (int i = 0; i < m.n; ++i) {
    as[i].evict_first = ef;
    as[i].rows_cap = cap;
  }
  const size_t smem = (size_t)kFG_WARPS * cap * sizeof(float) + (size_t)as[0].C * sizeof(XT) + 16 +
                      (FTraits<WT>::nf4 ? kNF4LutWords * 4 : 0);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  void (*kern)(const MultiArgs) =
      m.n == 1 ? flat_gemv_multi_kernel<WT, XT, MODE, UNROLL, 1>
               : (m.n == 2 ? flat_gemv_multi_kernel<WT, XT, MODE, UNROLL, 2>
                           : (m.n == 3 ? flat_gemv_multi_kernel<WT, XT, MODE, UNROLL, 3>
                                       : flat_gemv_multi_kernel<WT, XT, MODE, UNROLL, 4>));
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kFG_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, m);
}

// the shapes on which launch_w13 / launch_w2 take the flat engine (same decision, same kernels)
bool multi_flat_ok(int n, WType wt, int d, int F) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("ODMOE_MULTI");  // ODMOE_MULTI=0: one launch per expert (A/B)
    on = (e && e[0] == '0') ? 0 : 1;
  }
  if (wt == W_I8P) return on && n >= 1 && n <= kMaxMulti && mma_shadow_ok(d, F);
  return on && n >= 1 && n <= kMaxMulti && gemv_engine() == 2 && stream_ok(wt, d) && stream_ok(wt, F);
}

cudaError_t launch_w13_multi(int n, const ExpertRef* ex, WType wt, const void* u, int u_f32, float* a_buf, int d,
                             int F, cudaStream_t s, bool pdl) {
  if (!multi_flat_ok(n, wt, d, F)) {  // small shapes / other engines: one launch per expert
    for (int i = 0; i < n; ++i) {
      const cudaError_t e = launch_w13(ex[i], wt, u, u_f32, a_buf + (size_t)i * F, d, F, s, pdl);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  if (wt == W_I8P) return launch_mma_shadow(n, ex, 0, u, nullptr, a_buf, d, F, s, pdl);
  MultiArgs m{};
  m.n = n;
  for (int i = 0; i < n; ++i) {
    FlatArgs& a = m.a13[i];
    a.ex = ex[i]; a.second = 0; a.x = u; a.x_bf16 = !u_f32; a.R = 2 * F; a.C = d; a.out = a_buf + (size_t)i * F;
    a.d_full = d; a.F_full = F;
  }
  switch (wt) {
    case W_BF16: return main_mma() ? fg_multi_launch<bf16m, float, 0>(m, s, pdl) : fg_multi_launch<__nv_bfloat16, uint16_t, 0>(m, s, pdl);
    case W_F32: return fg_multi_launch<float, float, 0>(m, s, pdl);
    case W_I8: return lowbit_xf32() ? fg_multi_launch<int8_t, float, 0>(m, s, pdl) : fg_multi_launch<int8_t, uint16_t, 0>(m, s, pdl);
    case W_U8: return lowbit_xf32() ? fg_multi_launch<u8b, float, 0>(m, s, pdl) : fg_multi_launch<u8b, uint16_t, 0>(m, s, pdl);
    case W_NF4: return fg_multi_launch<nf4x2, uint16_t, 0>(m, s, pdl);
    case W_F8: return lowbit_xf32() ? fg_multi_launch<fp8e4, float, 0>(m, s, pdl) : fg_multi_launch<fp8e4, uint16_t, 0>(m, s, pdl);
    default: break;  // W_I8P: mma_gemv.cu
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_w2_multi(int n, const ExpertRef* ex, WType wt, const float* a_buf, const float* gate_w, float* y_buf,
                            int d, int F, cudaStream_t s, bool pdl) {
  if (!multi_flat_ok(n, wt, d, F)) {
    for (int i = 0; i < n; ++i) {
      const cudaError_t e = launch_w2(ex[i], wt, a_buf + (size_t)i * F, gate_w, y_buf + (size_t)i * d, d, F, s, pdl);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  if (wt == W_I8P) return launch_mma_shadow(n, ex, 1, a_buf, gate_w, y_buf, d, F, s, pdl);
  MultiArgs m{};
  m.n = n;
  for (int i = 0; i < n; ++i) {
    FlatArgs& a = m.a2[i];
    a.ex = ex[i]; a.second = 1; a.x = a_buf + (size_t)i * F; a.x_bf16 = 0; a.R = d; a.C = F; a.gate_w = gate_w;
    a.out = y_buf + (size_t)i * d; a.d_full = d; a.F_full = F;
  }
  switch (wt) {
    case W_BF16: return main_mma() ? fg_multi_launch<bf16m, float, 1>(m, s, pdl) : fg_multi_launch<__nv_bfloat16, float, 1>(m, s, pdl);
    case W_F32: return fg_multi_launch<float, float, 1>(m, s, pdl);
    case W_I8: return fg_multi_launch<int8_t, float, 1>(m, s, pdl);
    case W_U8: return fg_multi_launch<u8b, float, 1>(m, s, pdl);
    case W_NF4: return fg_multi_launch<nf4x2, float, 1>(m, s, pdl);
    case W_F8: return fg_multi_launch<fp8e4, float, 1>(m, s, pdl);
    default: break;  // W_I8P: mma_gemv.cu
  }
  return cudaErrorInvalidValue;
}

template <typename WT, typename XT>
static cudaError_t fused_launch(FlatArgs a13, FlatArgs a2, cudaStream_t s, bool pdl) {
  constexpr int UNROLL = kFG_UNROLL;
  int dev = 0;
  cudaGetDevice(&dev);
  BarrierState* bs = nullptr;
  {
    cudaError_t e = barrier_counter(dev, s, bs);
    if (e != cudaSuccess) return e;
  }
  static int ef = -1;
  if (ef < 0) {
    const char* e = getenv("ODMOE_L2_EVICT_FIRST");
    ef = (e && e[0] == '0') ? 0 : 1;
  }
  a13.evict_first = a2.evict_first = ef;
  if (!flat_row_ok<WT>(a13.C) || !flat_row_ok<WT>(a2.C)) return cudaErrorInvalidValue;
  const int sms = stream_grid_sms();
  long long units = a13.R / 2 < a2.R ? a13.R / 2 : a2.R;
  const int grid = (int)(units < sms ? (units > 0 ? units : 1) : sms);
  a13.rows_cap = (int)((a13.R / 2 + grid - 1) / grid) * 2 + 2;
  a2.rows_cap = (int)((a2.R + grid - 1) / grid) + 2;
  const size_t lut = FTraits<WT>::nf4 ? kNF4LutWords * 4 : 0;
  const size_t s1 = (size_t)kFG_WARPS * a13.rows_cap * sizeof(float) + (size_t)a13.C * sizeof(XT) + 16 + lut;
  const size_t s2 = (size_t)kFG_WARPS * a2.rows_cap * sizeof(float) + (size_t)a2.C * sizeof(float) + 16 + lut;
  const size_t smem = s1 > s2 ? s1 : s2;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  auto kern = flat_expert_kernel<WT, XT, UNROLL>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // Stream-ordered launches use increasing barrier targets on their stream's own counter; a
  // cooperative grid becomes resident only as a whole, so grids of two streams serialise instead
  // of holding each other's SMs.
  const unsigned int target = bs->epoch + (unsigned int)grid;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kFG_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  e = cudaLaunchKernelEx(&cfg, kern, a13, a2, bs->counter, target);
  if (e == cudaSuccess) bs->epoch = target;
  return e;
}

cudaError_t launch_expert_fused(ExpertRef ex, const void* w2_direct, const float* s2_direct, WType wt,
                                const void* u, int u_f32, float* a_buf, const float* gate_w, float* y, int d,
                                int F, cudaStream_t s, bool pdl, const P2PSend* send) {
  FlatArgs a13{}, a2{};
  a13.ex = ex; a13.second = 0; a13.x = u; a13.x_bf16 = !u_f32; a13.R = 2 * F; a13.C = d; a13.out = a_buf;
  a13.d_full = d; a13.F_full = F;
  a2.ex = ex; a2.second = 1; a2.x = a_buf; a2.x_bf16 = 0; a2.R = d; a2.C = F; a2.gate_w = gate_w; a2.out = y;
  a2.d_full = d; a2.F_full = F;
  if (ex.tbl == nullptr) {  // direct: W2 has its own pointer
    a2.ex.blob = w2_direct;
    a2.ex.scales = s2_direct;
  }
  if (send) a2.send = *send;
  switch (wt) {
    case W_BF16: return main_mma() ? fused_launch<bf16m, float>(a13, a2, s, pdl) : fused_launch<__nv_bfloat16, uint16_t>(a13, a2, s, pdl);
    case W_F32: return fused_launch<float, float>(a13, a2, s, pdl);
    case W_I8: return lowbit_xf32() ? fused_launch<int8_t, float>(a13, a2, s, pdl) : fused_launch<int8_t, uint16_t>(a13, a2, s, pdl);
    case W_U8: return lowbit_xf32() ? fused_launch<u8b, float>(a13, a2, s, pdl) : fused_launch<u8b, uint16_t>(a13, a2, s, pdl);
    case W_NF4: return fused_launch<nf4x2, uint16_t>(a13, a2, s, pdl);
    case W_F8: return lowbit_xf32() ? fused_launch<fp8e4, float>(a13, a2, s, pdl) : fused_launch<fp8e4, uint16_t>(a13, a2, s, pdl);
    default: break;  // W_I8P: mma_gemv.cu
  }
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------- NF4 / FP8, small shapes
// Rows shorter than one 512-byte group cannot use the flat stream: one warp per output unit (a
// W1/W3 row pair, or a W2 row). Test sizes and odd shapes only; Mixtral shapes take the flat
// kernel above. FMT 0 = NF4 (block absmax), 1 = FP8 E4M3 (row scale).
template <int MODE, int FMT>
__global__ void __launch_bounds__(256) lowbit_rowwarp_kernel(ExpertRef ex, int second, const void* x, int x_f32,
                                                            int R, int C, int d_full, int F_full,
                                                            const float* gate_w, float* out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int unit = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const uint8_t* Wb;
  const float* sc;
  int gate_idx = ex.sel;
  if (ex.tbl == nullptr) {
    Wb = reinterpret_cast<const uint8_t*>(ex.blob);
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
    Wb = reinterpret_cast<const uint8_t*>(ex.tbl[id]) +
         (second ? (size_t)2 * F_full * d_full / (FMT == 0 ? 2 : 1) : 0);
    sc = ex.stbl[id] + (second ? (FMT == 0 ? (size_t)2 * F_full * d_full / 64 : (size_t)2 * F_full) : 0);
  }
  const int nunits = MODE == 0 ? R / 2 : R;
  if (unit >= nunits) return;
  auto xv = [&](int j) -> float {
    return x_f32 ? reinterpret_cast<const float*>(x)[j]
                 : __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(x)[j] << 16);
  };
  float acc[2] = {0.f, 0.f};
  for (int q = 0; q < (MODE == 0 ? 2 : 1); ++q) {
    const int r = MODE == 0 ? 2 * unit + q : unit;
    float t = 0.f;
    if (FMT == 0) {
      for (int jb = lane; jb < C / 2; jb += 32) {
        const uint8_t b = Wb[(size_t)r * (C / 2) + jb];
        const float a = sc[(size_t)r * (C / 64) + (2 * jb) / 64];
        t = fmaf(a, kNF4Code[b & 15] * xv(2 * jb) + kNF4Code[b >> 4] * xv(2 * jb + 1), t);
      }
    } else {
      for (int j = lane; j < C; j += 32) {
        __nv_fp8_e4m3 f;
        f.__x = Wb[(size_t)r * C + j];
        t = fmaf(float(f), xv(j), t);
      }
      t *= sc[r];
    }
    acc[q] = warp_sum(t);
  }
  if (lane == 0) {
    if (MODE == 0) out[unit] = silu_mul(acc[0], acc[1]);
    else out[unit] = (gate_w ? gate_w[gate_idx] : 1.f) * acc[0];
  }
}

cudaError_t launch_lowbit_small(ExpertRef ex, WType wt, int second, const void* x, int x_f32, int d, int F,
                                const float* gate_w, float* out, cudaStream_t s) {
  const int R = second ? d : 2 * F, C = second ? F : d;
  if (wt == W_NF4 && C % 64) return cudaErrorInvalidValue;
  const int units = second ? R : R / 2;
  const int grid = (units + 7) / 8;
  if (wt == W_NF4) {
    if (second) lowbit_rowwarp_kernel<1, 0><<<grid, 256, 0, s>>>(ex, 1, x, 1, R, C, d, F, gate_w, out);
    else lowbit_rowwarp_kernel<0, 0><<<grid, 256, 0, s>>>(ex, 0, x, x_f32, R, C, d, F, gate_w, out);
  } else if (wt == W_F8) {
    if (second) lowbit_rowwarp_kernel<1, 1><<<grid, 256, 0, s>>>(ex, 1, x, 1, R, C, d, F, gate_w, out);
    else lowbit_rowwarp_kernel<0, 1><<<grid, 256, 0, s>>>(ex, 0, x, x_f32, R, C, d, F, gate_w, out);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace odmoe
