// INT8 shadow expert GEMV on the tensor cores' warp-level path (mma.sync m16n8k16, f16 inputs, fp32
// accumulate): the SEP shadow's expert phases (reading Q9).
//
// Why: the flat CUDA-core engine (flat_gemv.cu) spends ~3 instructions per INT8 weight on widening
// (byte -> fp32 via the 2^23 mantissa trick, 2 FADD2 + 4 PRMT per word), activation unpacking and
// FFMA2; at batch 1 that made the shadow instruction/latency-bound at 0.48-0.61 of HBM
// (profiles/ncu_r01_shadow_multi_insitu.json). Here one PRMT turns two biased codes (q + 128) into
// the f16 pair 1152 + q (byte into the low mantissa byte of 1024), one HSUB2 removes 1152 exactly,
// and one HMMA consumes 16 rows x 16 columns: ~0.05 warp instructions per weight byte instead of
// ~0.11, so the stream stays memory-bound.
//
// Exactness: q (|q| <= 127) is exact in f16; the activation x (bf16 u or fp32 a) is split into
// x = hi + lo with hi = f16(x), lo = f16(x - hi) (22 of x's 24 significand bits; exact for bf16 u in
// f16's normal range); the MMA's B operand carries hi in columns 0-3 and lo in columns 4-7, so ONE
// HMMA per k-block gives A.hi and A.lo, and hi + lo is summed in fp32 after the k loop. Products are
// exact; the fp32 accumulation order differs from the oracle's (fp32 rounding only).
//
// Layout ("fragment-packed", written once at shadow build by pack_i8_frag_kernel): a matrix of R rows
// x C columns is cut into 16-row tiles and 32-column blocks; block (t, cb) is 512 contiguous bytes,
// 16 per lane, lane (g = lane / 4, tq = lane % 4) holding exactly its A fragments of k-blocks 2cb and
// 2cb + 1: A[g][2tq..+1], A[g+8][2tq..+1], A[g][2tq+8..+9], A[g+8][2tq+8..+9]. For W13 tile row g is
// the gate row and tile row g + 8 the up row of gate/up pair 8t + g, so one lane ends with both
// halves of its SwiGLU unit. Row scales stay in natural order.
//
// Work split: the units (t, cb) of a matrix form one stream, cut into balanced contiguous ranges
// per CTA (one per SM) and per warp (24 warps); a warp keeps 2 x 4 units (8 x 16 B per lane) in
// flight. Tiles cut by a range boundary are reduced across CTAs deterministically: each CTA writes
// its warp-ordered partial to a slot, the last arrival (ticket) sums the slots in CTA order.
#include "common.cuh"
#include "kernels.h"

#include <map>
#include <mutex>

namespace odmoe {

#ifndef MG_WARPS
#define MG_WARPS 16
#endif
#ifndef MG_UNROLL
#define MG_UNROLL 8
#endif
#ifndef MG_PF
#define MG_PF 0     // L2 bulk prefetch of the units MG_PF batches beyond the two in registers (0 = off)
#endif
constexpr int kMG_WARPS = MG_WARPS;     // 16 warps x 2 batches x 8 units x 512 B = 128 KB in flight per SM
constexpr int kMG_THREADS = kMG_WARPS * 32;
constexpr int kMG_UNROLL = MG_UNROLL;
constexpr int kMG_MAXSPLIT = 4;   // CTAs sharing one tile (grid sizing keeps it <= 3)
constexpr int kMG_MAXE = 4;       // experts per launch

struct MgArgs {
  // expert e: direct (w[e], sc[e]) or indirect (tbl[base + ids[pick]] + off, stbl[...] + soff)
  const uint8_t* w[kMG_MAXE];
  const float* sc[kMG_MAXE];
  const void* const* tbl;
  const float* const* stbl;
  const int32_t* ids;
  int base, k, sel[kMG_MAXE];
  long long off, soff;      // byte offset of this matrix in a blob / float offset of its scales
  float* out[kMG_MAXE];     // mode 0: a [R/2] in B-fragment form (4 B per element); mode 1: y [R] fp32
  const void* x;            // mode 0: bf16 u [C] (shared); mode 1: the phase-1 activations in B-fragment
                            // form (store_frag), expert e at x + e * C * 4 bytes
  const float* gate_w;      // mode 1: y = gate_w[pick] * (W2 a) (NULL = 1)
  int n, R, C;
  float* gpart;             // [n * tiles][kMG_MAXSPLIT][16] (global tile = expert * tiles + tile)
  unsigned int* ticket;     // [n * tiles]
  int tiles_cap;            // tiles per CTA (smem partials)
};

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
// two biased codes (bytes i, i+1 of w: q + 128) -> f16x2 (q_i, q_{i+1}), exact
__device__ __forceinline__ uint32_t u8x2_to_h2(uint32_t w, uint32_t sel) {
  const uint32_t h = prmt(w, 0x64646464u, sel);   // f16 bits 0x64bb = 1024 + bb = 1152 + q
  uint32_t r;
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(h), "r"(0x64806480u));  // 1152.0 = 0x6480
  return r;
}
__device__ __forceinline__ void hmma16816(float& c0, float& c1, float& c2, float& c3, uint32_t a0, uint32_t a1,
                                          uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c0), "+f"(c1), "+f"(c2), "+f"(c3)
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t h2_bits(float lo, float hi) {
  const __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// CTA whose split_range(U, grid) range contains unit u
__device__ __forceinline__ int cta_of(long long u, long long U, int grid) {
  int p = (int)((u * grid) / U);
  while (p + 1 < grid && U * (p + 1) / grid <= u) ++p;
  while (p > 0 && U * p / grid > u) --p;
  return p;
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// The activation handed from phase 1 to phase 2 in the B-fragment format (4 B per element, the size of
// the fp32 vector it replaces): element c of k-block kb is f16 hi at uint2 [kb*8 + tq], lo at
// [kb*8 + 4 + tq], word (c >= 8), half (c & 1), tq = (c & 7) >> 1.
__device__ __forceinline__ void store_frag(uint32_t* frag, int p, float v) {
  const int kb = p >> 4, c = p & 15, tq = (c & 7) >> 1;
  const int w = (c >> 3) & 1, hf = c & 1;
  const __half hi = __float2half_rn(v);
  const __half lo = __float2half_rn(v - __half2float(hi));
  __half* h = reinterpret_cast<__half*>(frag);
  h[((kb * 8 + tq) * 2 + w) * 2 + hf] = hi;
  h[((kb * 8 + 4 + tq) * 2 + w) * 2 + hf] = lo;
}

struct MgPdlWait {
  __device__ __forceinline__ void operator()() const { asm volatile("griddepcontrol.wait;" ::: "memory"); }
};
// grid-wide barrier of a cooperative launch (arrival counter with monotonically growing targets)
struct MgGridBarrier {
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

// One phase: MODE 0 = W13 + SwiGLU, MODE 1 = W2 + gate, for NE experts. `wait_dep` runs once the
// data this phase consumes from earlier work may be read (PDL wait for a stand-alone launch, the grid
// barrier in the fused layer kernel); this phase's first weight batches are issued before it.
template <int MODE, int NE, typename WaitFn>
__device__ __forceinline__ void mma_phase(const MgArgs& a, uint8_t* sm, const WaitFn& wait_dep, bool ids_ready = false) {
  // The NE experts' units form ONE stream (expert-major): a CTA's range and a warp's slice may cross
  // from one expert into the next, so pipeline fill, staging and tail are paid once per launch.
  const int nkb = a.C / 16;
  constexpr int NX = MODE == 0 ? 1 : NE;                             // activation vectors staged
  uint2* xs = reinterpret_cast<uint2*>(sm);                          // [NX][C/16][8]: hi tq0..3, lo tq0..3
  float* part = reinterpret_cast<float*>(sm + (size_t)NX * nkb * 64);  // [warps][tiles_cap][16]
  __shared__ const uint4* sW[NE];   // expert e's packed matrix, pre-offset by -e*U units
  __shared__ const float* sS[NE];
  __shared__ float sG[NE];
  __shared__ __align__(8) uint64_t xbar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int g = lane >> 2, tq = lane & 3;
  const int tiles = a.R / 16, CB = a.C / 32;
  const int U = tiles * CB, UT = U * NE;
  const int u0 = (int)((long long)UT * blockIdx.x / gridDim.x), u1 = (int)((long long)UT * (blockIdx.x + 1) / gridDim.x);
  const int t_first = u0 / CB;                                       // global tile = e * tiles + t
  const int t_last = u1 > u0 ? (u1 - 1) / CB : t_first - 1;
  const int wb = u0 + (int)((long long)(u1 - u0) * warp / kMG_WARPS);
  const int we = u0 + (int)((long long)(u1 - u0) * (warp + 1) / kMG_WARPS);
  const uint64_t pol = l2_policy(true);
  const bool indirect = a.tbl != nullptr;
  const bool early = indirect && !ids_ready;
  if (early) wait_dep();  // the expert ids come from the router
  if (tid < NE) {
    const int e = tid;
    const int pick = a.sel[e];
    const uint8_t* W;
    if (indirect) {
      const int id = a.base + a.ids[pick];
      W = reinterpret_cast<const uint8_t*>(a.tbl[id]) + a.off;
      sS[e] = a.stbl[id] + a.soff;
    } else {
      W = a.w[e];
      sS[e] = a.sc[e];
    }
    sW[e] = reinterpret_cast<const uint4*>(W) - (size_t)e * U * 32;
    sG[e] = MODE == 1 ? (a.gate_w ? a.gate_w[pick] : 1.f) : 1.f;
  }
  if (MODE == 1 && tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&xbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // unit v of the stream -> its 16 B for this lane
  const uint4* adj[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) adj[e] = sW[e] + lane;
  auto ld_unit = [&](int v) -> uint4 {
    const uint4* b = adj[0];
#pragma unroll
    for (int e = 1; e < NE; ++e) b = v >= e * U ? adj[e] : b;
    return ld_stream_pol(b + (size_t)v * 32, pol);
  };
  uint4 wa[kMG_UNROLL], wc[kMG_UNROLL];
#pragma unroll
  for (int i = 0; i < kMG_UNROLL; ++i)
    if (wb + i < we) wa[i] = ld_unit(wb + i);
  if (!early) wait_dep();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (MODE == 0) {  // u (bf16) -> f16 hi/lo B fragments
    for (int i = tid; i < nkb * 4; i += kMG_THREADS) {
      const int kb = i >> 2, q = i & 3;
      const uint16_t* u = reinterpret_cast<const uint16_t*>(a.x) + kb * 16 + 2 * q;
      float v[4] = {__uint_as_float((uint32_t)u[0] << 16), __uint_as_float((uint32_t)u[1] << 16),
                    __uint_as_float((uint32_t)u[8] << 16), __uint_as_float((uint32_t)u[9] << 16)};
      float hi[4], lo[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        hi[j] = __half2float(__float2half_rn(v[j]));
        lo[j] = v[j] - hi[j];
      }
      xs[kb * 8 + q] = make_uint2(h2_bits(hi[0], hi[1]), h2_bits(hi[2], hi[3]));
      xs[kb * 8 + 4 + q] = make_uint2(h2_bits(lo[0], lo[1]), h2_bits(lo[2], lo[3]));
    }
  } else if (tid == 0) {  // phase 1 left the activations in fragment form: one bulk copy per 32 KB
    const uint32_t bytes = (uint32_t)NX * nkb * 64;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&xbar)), "r"(bytes) : "memory");
    for (uint32_t off = 0; off < bytes; off += 32768) {
      const uint32_t nb = bytes - off < 32768 ? bytes - off : 32768;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_addr(sm + off)),
                   "l"(reinterpret_cast<const char*>(a.x) + off), "r"(nb), "r"(smem_addr(&xbar))
                   : "memory");
    }
  }
  const int ntl = t_last - t_first + 1;
  for (int i = tid; i < kMG_WARPS * a.tiles_cap * 16; i += kMG_THREADS) part[i] = 0.f;
  __syncthreads();
  if (MODE == 1)
    asm volatile("{\n .reg .pred p;\n XW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra XW_%=;\n}\n" ::"r"(
                     smem_addr(&xbar))
                 : "memory");

  float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
  // running (global tile, column block) of the next unit; xk = this lane's B fragments of k-block 2cb
  int tcur = wb / CB, cb = wb - tcur * CB;
  const uint2* xlane = xs + (g >= 4 ? 4 : 0) + tq;
  const uint2* xk = xlane + (size_t)(MODE == 0 ? 0 : tcur / tiles) * nkb * 8 + (size_t)cb * 16;
  float* pw = part + (size_t)warp * a.tiles_cap * 16 + (tq == 0 ? g : 0);
  auto flush = [&]() {
    // columns 0-3 hold A.hi, 4-7 A.lo: lane (g, 0) adds lane (g, 2)'s value
    const float h0 = c0 + __shfl_down_sync(0xffffffffu, c0, 2);
    const float h2 = c2 + __shfl_down_sync(0xffffffffu, c2, 2);
    if (tq == 0) {
      float* p = pw + (tcur - t_first) * 16;
      p[0] = h0;
      p[8] = h2;
    }
    c0 = c1 = c2 = c3 = 0.f;
  };
  auto unit = [&](const uint4& w) {
    const uint2 b0 = xk[0];
    const uint2 b1 = xk[8];
    hmma16816(c0, c1, c2, c3, u8x2_to_h2(w.x, 0x4140u), u8x2_to_h2(w.x, 0x4342u), u8x2_to_h2(w.y, 0x4140u),
              u8x2_to_h2(w.y, 0x4342u), b0.x, b0.y);
    hmma16816(c0, c1, c2, c3, u8x2_to_h2(w.z, 0x4140u), u8x2_to_h2(w.z, 0x4342u), u8x2_to_h2(w.w, 0x4140u),
              u8x2_to_h2(w.w, 0x4342u), b1.x, b1.y);
    xk += 16;
    if (++cb == CB) {  // tile complete (warp-uniform)
      flush();
      ++tcur;
      cb = 0;
      xk = xlane + (size_t)(MODE == 0 ? 0 : tcur / tiles) * nkb * 8;
    }
  };
  for (int ub = wb; ub < we; ub += 2 * kMG_UNROLL) {
#if MG_PF > 0
    if (lane == 0) {  // the 2 batches after the register pipeline, into L2 (no registers held)
      const int p0 = ub + 2 * kMG_UNROLL * MG_PF;
      const int p1 = min(p0 + 2 * kMG_UNROLL, we);
      for (int pv = p0; pv < p1;) {  // one bulk prefetch per contiguous run (an expert boundary splits it)
        int e = 0;
#pragma unroll
        for (int j = 1; j < NE; ++j) e += pv >= j * U;
        const int run_end = min(p1, (e + 1) * U);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(sW[e] + (size_t)pv * 32),
                     "r"((uint32_t)(run_end - pv) * 512u) : "memory");
        pv = run_end;
      }
    }
#endif
#pragma unroll
    for (int i = 0; i < kMG_UNROLL; ++i)
      if (ub + kMG_UNROLL + i < we) wc[i] = ld_unit(ub + kMG_UNROLL + i);
    if (ub + kMG_UNROLL <= we) {
#pragma unroll
      for (int i = 0; i < kMG_UNROLL; ++i) unit(wa[i]);
    } else {
#pragma unroll
      for (int i = 0; i < kMG_UNROLL; ++i)
        if (ub + i < we) unit(wa[i]);
    }
#pragma unroll
    for (int i = 0; i < kMG_UNROLL; ++i)
      if (ub + 2 * kMG_UNROLL + i < we) wa[i] = ld_unit(ub + 2 * kMG_UNROLL + i);
    if (ub + 2 * kMG_UNROLL <= we) {
#pragma unroll
      for (int i = 0; i < kMG_UNROLL; ++i) unit(wc[i]);
    } else {
#pragma unroll
      for (int i = 0; i < kMG_UNROLL; ++i)
        if (ub + kMG_UNROLL + i < we) unit(wc[i]);
    }
  }
  if (cb != 0) flush();  // the slice ended inside a tile
  __syncthreads();

  // per global tile of this CTA: warps summed in a fixed order; whole tiles finalise here, cut tiles
  // go through the cross-CTA slots (the last arrival sums the slots in CTA order)
  for (int tl = warp; tl < ntl; tl += kMG_WARPS) {
    const int tg = t_first + tl;
    const int e = tg / tiles, t = tg - e * tiles;
    float v = 0.f;
    if (lane < 16)
      for (int w = 0; w < kMG_WARPS; ++w) v += part[((size_t)w * a.tiles_cap + tl) * 16 + lane];
    const int tb = tg * CB, te = tb + CB;
    const bool whole = tb >= u0 && te <= u1;
    if (!whole) {
      const int c_first = cta_of(tb, UT, gridDim.x), c_last = cta_of(te - 1, UT, gridDim.x);
      const int slot = blockIdx.x - c_first;
      if (lane < 16) a.gpart[((size_t)tg * kMG_MAXSPLIT + slot) * 16 + lane] = v;
      __threadfence();
      __syncwarp();
      unsigned int prev = 0;
      if (lane == 0) prev = atomicAdd(a.ticket + tg, 1u);
      prev = __shfl_sync(0xffffffffu, prev, 0);
      if (prev != (unsigned)(c_last - c_first)) continue;  // not the last arrival
      __threadfence();
      v = 0.f;
      if (lane < 16)
        for (int s2 = 0; s2 <= c_last - c_first; ++s2) v += __ldcg(a.gpart + ((size_t)tg * kMG_MAXSPLIT + s2) * 16 + lane);
      if (lane == 0) a.ticket[tg] = 0u;
    }
    const float* S = sS[e];
    float* out = e == 0 ? a.out[0] : (e == 1 ? a.out[NE > 1 ? 1 : 0] : (e == 2 ? a.out[NE > 2 ? 2 : 0] : a.out[NE > 3 ? 3 : 0]));
    if (MODE == 0) {
      // lane g < 8: gate of pair 8t + g in v (row g), its up in row g + 8 (lane g + 8); the result goes
      // to phase 2 in B-fragment form
      const float up = __shfl_down_sync(0xffffffffu, v, 8);
      if (lane < 8) {
        const int p = 8 * t + lane;
        store_frag(reinterpret_cast<uint32_t*>(out), p, silu_mul(v * S[2 * p], up * S[2 * p + 1]));
      }
    } else if (lane < 16) {
      const int r = 16 * t + lane;
      out[r] = sG[e] * (v * S[r]);
    }
  }
}

template <int MODE, int NE>
__global__ void __launch_bounds__(kMG_THREADS, 1) mma_gemv_kernel(const __grid_constant__ MgArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];
  mma_phase<MODE, NE>(a, sm, MgPdlWait{});
}

// The shadow's whole expert layer in ONE cooperative launch: W13 + SwiGLU of the NE experts, a grid
// barrier, W2 + gate (one launch, ramp and tail per layer instead of two). Phase 2's first weight
// batches are in flight before the barrier.
template <int NE>
__global__ void __launch_bounds__(kMG_THREADS, 1)
mma_layer_kernel(const __grid_constant__ MgArgs a13, const __grid_constant__ MgArgs a2, unsigned int* counter,
                 unsigned int target) {
  extern __shared__ __align__(128) uint8_t sm[];
  mma_phase<0, NE>(a13, sm, MgPdlWait{});
  __syncthreads();
  mma_phase<1, NE>(a2, sm, MgGridBarrier{counter, target}, /*ids_ready=*/true);
}

// ---------------------------------------------------------------- packing (shadow build)
// q [R][C] biased codes (q + 128, row-major) -> the fragment-packed layout above. pair_rows: W13
// (tile row g = row 2(8t + g), tile row g + 8 = row 2(8t + g) + 1); else tile row r = row 16t + r.
__global__ void pack_i8_frag_kernel(const uint8_t* __restrict__ q, uint8_t* __restrict__ out, int R, int C,
                                    int pair_rows, uint32_t flip) {
  const long long n_units = (long long)(R / 16) * (C / 32);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_units * 32;
       i += (long long)gridDim.x * blockDim.x) {
    const long long unit = i >> 5;
    const int lane = (int)(i & 31), g = lane >> 2, tq = lane & 3;
    const int CB = C / 32;
    const int t = (int)(unit / CB), cb = (int)(unit % CB);
    const int rg = pair_rows ? 2 * (8 * t + g) : 16 * t + g;       // tile row g
    const int rh = pair_rows ? 2 * (8 * t + g) + 1 : 16 * t + g + 8;  // tile row g + 8
    uint8_t b[16];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k0 = (2 * cb + h) * 16 + 2 * tq;
      b[8 * h + 0] = q[(size_t)rg * C + k0];
      b[8 * h + 1] = q[(size_t)rg * C + k0 + 1];
      b[8 * h + 2] = q[(size_t)rh * C + k0];
      b[8 * h + 3] = q[(size_t)rh * C + k0 + 1];
      b[8 * h + 4] = q[(size_t)rg * C + k0 + 8];
      b[8 * h + 5] = q[(size_t)rg * C + k0 + 9];
      b[8 * h + 6] = q[(size_t)rh * C + k0 + 8];
      b[8 * h + 7] = q[(size_t)rh * C + k0 + 9];
    }
    uint4 v;
    v.x = b[0] | (b[1] << 8) | (b[2] << 16) | ((uint32_t)b[3] << 24);
    v.y = b[4] | (b[5] << 8) | (b[6] << 16) | ((uint32_t)b[7] << 24);
    v.z = b[8] | (b[9] << 8) | (b[10] << 16) | ((uint32_t)b[11] << 24);
    v.w = b[12] | (b[13] << 8) | (b[14] << 16) | ((uint32_t)b[15] << 24);
    v.x ^= flip; v.y ^= flip; v.z ^= flip; v.w ^= flip;  // signed q -> q + 128
    reinterpret_cast<uint4*>(out)[i] = v;
  }
}

bool mma_shadow_ok(int d, int F) { return d % 32 == 0 && F % 32 == 0 && d >= 32 && F >= 32; }

cudaError_t launch_pack_i8_frag(const uint8_t* q_biased, uint8_t* out, int R, int C, int pair_rows, cudaStream_t s,
                                bool signed_codes) {
  if (R % 16 || C % 32) return cudaErrorInvalidValue;
  const long long n = (long long)(R / 16) * (C / 32) * 32;
  const int grid = (int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
  pack_i8_frag_kernel<<<grid > 0 ? grid : 1, 256, 0, s>>>(q_biased, out, R, C, pair_rows,
                                                          signed_codes ? 0x80808080u : 0u);
  return cudaGetLastError();
}

// Cross-CTA scratch per (device, stream): partial slots + tickets (tickets start at 0 and are reset by
// the last arrival of every cut tile).
struct MgScratch {
  float* gpart = nullptr;
  unsigned int* ticket = nullptr;
  long long tiles = 0;
};
static std::mutex g_mg_mu;
static std::map<std::pair<int, cudaStream_t>, MgScratch> g_mg;

static cudaError_t mg_scratch(cudaStream_t s, long long tiles, MgScratch*& out) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mg_mu);
  MgScratch& m = g_mg[{dev, s}];
  if (m.tiles < tiles) {
    if (m.gpart) {
      cudaStreamSynchronize(s);
      cudaFree(m.gpart);
      cudaFree(m.ticket);
    }
    cudaError_t e = cudaMalloc(&m.gpart, (size_t)tiles * kMG_MAXSPLIT * 16 * sizeof(float));
    if (e != cudaSuccess) return e;
    e = cudaMalloc(&m.ticket, (size_t)tiles * sizeof(unsigned int));
    if (e != cudaSuccess) return e;
    e = cudaMemset(m.ticket, 0, (size_t)tiles * sizeof(unsigned int));
    if (e != cudaSuccess) return e;
    m.tiles = tiles;
  }
  out = &m;
  return cudaSuccess;
}

// One phase of n experts on the packed INT8 layout. mode 0: R = 2F, C = d (W13 + SwiGLU -> a [F]);
// mode 1: R = d, C = F (W2 + gate -> y [d]). ex: as for launch_w13_multi (second = mode).
cudaError_t launch_mma_shadow(int n, const ExpertRef* ex, int mode, const void* x, const float* gate_w,
                              float* out, int d, int F, cudaStream_t s, bool pdl) {
  if (n < 1 || n > kMG_MAXE || !mma_shadow_ok(d, F)) return cudaErrorInvalidValue;
  MgArgs a{};
  a.n = n;
  a.R = mode == 0 ? 2 * F : d;
  a.C = mode == 0 ? d : F;
  a.x = x;
  a.gate_w = gate_w;
  const bool ind = ex[0].tbl != nullptr;
  a.tbl = ind ? ex[0].tbl : nullptr;
  a.stbl = ind ? ex[0].stbl : nullptr;
  a.ids = ind ? ex[0].ids : nullptr;
  a.base = ex[0].base;
  a.k = ex[0].k;
  a.off = mode == 0 ? 0 : 2LL * F * d;
  a.soff = mode == 0 ? 0 : 2LL * F;
  for (int i = 0; i < n; ++i) {
    if ((ex[i].tbl != nullptr) != ind || (ind && (ex[i].tbl != a.tbl || ex[i].ids != a.ids || ex[i].base != a.base)))
      return cudaErrorInvalidValue;
    a.sel[i] = ex[i].sel;
    a.w[i] = ind ? nullptr : reinterpret_cast<const uint8_t*>(ex[i].blob);
    a.sc[i] = ind ? nullptr : ex[i].scales;
    a.out[i] = out + (size_t)i * (mode == 0 ? F : d);
  }
  const int tiles = a.R / 16, CB = a.C / 32;
  const long long UT = (long long)tiles * CB * n;   // the n experts' units, one stream
  const int sms = stream_grid_sms();
  long long gmax = UT / ((CB + 1) / 2);         // a CTA's range >= half a tile: <= 3 CTAs share one
  if (gmax < 1) gmax = 1;
  const int grid = (int)(gmax < sms ? gmax : sms);
  a.tiles_cap = (int)((UT + grid - 1) / grid / CB) + 2;
  MgScratch* sc = nullptr;
  cudaError_t e = mg_scratch(s, (long long)tiles * kMG_MAXE, sc);
  if (e != cudaSuccess) return e;
  a.gpart = sc->gpart;
  a.ticket = sc->ticket;
  const int nx = mode == 0 ? 1 : n;             // activation vectors staged (W2: one per expert)
  const size_t smem = (size_t)nx * a.C / 16 * 64 + (size_t)kMG_WARPS * a.tiles_cap * 16 * sizeof(float);
  if (smem > 227 * 1024) {  // W2 of many wide experts: one launch per expert
    if (n == 1) return cudaErrorInvalidValue;
    for (int i = 0; i < n; ++i) {
      e = launch_mma_shadow(1, ex + i, mode, mode == 0 ? x : (const void*)((const uint32_t*)x + (size_t)i * F), gate_w,
                            out + (size_t)i * (mode == 0 ? F : d), d, F, s, pdl);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  void (*kern)(const MgArgs);
  if (mode == 0) kern = n == 1 ? mma_gemv_kernel<0, 1> : n == 2 ? mma_gemv_kernel<0, 2> : n == 3 ? mma_gemv_kernel<0, 3> : mma_gemv_kernel<0, 4>;
  else kern = n == 1 ? mma_gemv_kernel<1, 1> : n == 2 ? mma_gemv_kernel<1, 2> : n == 3 ? mma_gemv_kernel<1, 3> : mma_gemv_kernel<1, 4>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kMG_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

// The shadow's expert layer (both phases, n experts) in one cooperative launch; grid barrier
// counter from the flat engine's per-stream state (coop_barrier_next).
cudaError_t launch_mma_shadow_layer(int n, const ExpertRef* ex, const void* u, float* a_buf, const float* gate_w,
                                    float* y_buf, int d, int F, cudaStream_t s, bool pdl) {
  if (n < 1 || n > kMG_MAXE || !mma_shadow_ok(d, F)) return cudaErrorInvalidValue;
  MgArgs a[2];
  // one SM stays free: a one-warp kernel (the compute stream's warm wait) may hold it, and a cooperative
  // grid only starts once all its CTAs fit
  int grid = stream_grid_sms() < num_sms() - 1 ? stream_grid_sms() : num_sms() - 1;
  size_t smem = 0;
  for (int mode = 0; mode < 2; ++mode) {
    MgArgs& g = a[mode];
    g = MgArgs{};
    g.n = n;
    g.R = mode == 0 ? 2 * F : d;
    g.C = mode == 0 ? d : F;
    g.x = mode == 0 ? u : (const void*)a_buf;
    g.gate_w = mode == 1 ? gate_w : nullptr;
    const bool ind = ex[0].tbl != nullptr;
    g.tbl = ind ? ex[0].tbl : nullptr;
    g.stbl = ind ? ex[0].stbl : nullptr;
    g.ids = ind ? ex[0].ids : nullptr;
    g.base = ex[0].base;
    g.k = ex[0].k;
    g.off = mode == 0 ? 0 : 2LL * F * d;
    g.soff = mode == 0 ? 0 : 2LL * F;
    for (int i = 0; i < n; ++i) {
      if ((ex[i].tbl != nullptr) != ind || ex[i].tbl != nullptr) {  // direct refs only through launch_mma_shadow
        if (!ind || ex[i].tbl != g.tbl || ex[i].ids != g.ids || ex[i].base != g.base) return cudaErrorInvalidValue;
      }
      g.sel[i] = ex[i].sel;
      g.w[i] = ind ? nullptr : reinterpret_cast<const uint8_t*>(ex[i].blob);
      g.sc[i] = ind ? nullptr : ex[i].scales;
      g.out[i] = (mode == 0 ? a_buf : y_buf) + (size_t)i * (mode == 0 ? F : d);
    }
    const int tiles = g.R / 16, CB = g.C / 32;
    const long long UT = (long long)tiles * CB * n;
    long long gmax = UT / ((CB + 1) / 2);
    if (gmax < grid) grid = (int)(gmax > 0 ? gmax : 1);
  }
  if (ex[0].tbl == nullptr) return cudaErrorInvalidValue;  // the engine passes indirect (device-chosen) experts
  MgScratch* sc = nullptr;
  cudaError_t e = mg_scratch(s, (long long)(2 * F / 16) * kMG_MAXE, sc);
  if (e != cudaSuccess) return e;
  for (int mode = 0; mode < 2; ++mode) {
    MgArgs& g = a[mode];
    const int tiles = g.R / 16, CB = g.C / 32;
    const long long UT = (long long)tiles * CB * n;
    g.tiles_cap = (int)((UT + grid - 1) / grid / CB) + 2;
    g.gpart = sc->gpart;
    g.ticket = sc->ticket;
    const int nx = mode == 0 ? 1 : n;
    const size_t sm = (size_t)nx * g.C / 16 * 64 + (size_t)kMG_WARPS * g.tiles_cap * 16 * sizeof(float);
    smem = sm > smem ? sm : smem;
  }
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  void (*kern)(const MgArgs, const MgArgs, unsigned int*, unsigned int) =
      n == 1 ? mma_layer_kernel<1> : n == 2 ? mma_layer_kernel<2> : n == 3 ? mma_layer_kernel<3> : mma_layer_kernel<4>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  unsigned int* counter = nullptr;
  unsigned int target = 0;
  e = coop_barrier_next(s, grid, &counter, &target);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kMG_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, a[0], a[1], counter, target);
}

}  // namespace odmoe
