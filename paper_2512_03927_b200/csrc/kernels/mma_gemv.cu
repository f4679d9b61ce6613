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

constexpr int kMG_WARPS = 24;
constexpr int kMG_THREADS = kMG_WARPS * 32;
constexpr int kMG_UNROLL = 4;
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
  float* out[kMG_MAXE];     // mode 0: a [R/2]; mode 1: y [R]
  const void* x;            // mode 0: bf16 u [C] (shared); mode 1: fp32 a, expert e at x + e * C
  const float* gate_w;      // mode 1: y = gate_w[pick] * (W2 a) (NULL = 1)
  int n, R, C;
  float* gpart;             // [n][tiles][kMG_MAXSPLIT][16]
  unsigned int* ticket;     // [n][tiles]
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

template <int MODE, int NE>
__global__ void __launch_bounds__(kMG_THREADS, 1) mma_gemv_kernel(const __grid_constant__ MgArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint2* xs = reinterpret_cast<uint2*>(sm);                      // [C/16 k-blocks][8]: hi tq0..3, lo tq0..3
  float* part = reinterpret_cast<float*>(sm + (size_t)a.C / 16 * 64);  // [warps][tiles_cap][16]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int g = lane >> 2, tq = lane & 3;
  const int tiles = a.R / 16, CB = a.C / 32;
  const long long U = (long long)tiles * CB;
  long long u0, u1;
  split_range(U, gridDim.x, blockIdx.x, u0, u1);
  const int t_first = (int)(u0 / CB);
  const int t_last = u1 > u0 ? (int)((u1 - 1) / CB) : t_first - 1;
  const long long wb = u0 + (u1 - u0) * warp / kMG_WARPS, we = u0 + (u1 - u0) * (warp + 1) / kMG_WARPS;
  const uint64_t pol = l2_policy(true);
  const bool indirect = a.tbl != nullptr;
  if (indirect) asm volatile("griddepcontrol.wait;" ::: "memory");

#pragma unroll
  for (int e = 0; e < NE; ++e) {  // unrolled: every a.w[e] / a.out[e] is a compile-time parameter offset
    int pick = a.sel[e];
    const uint8_t* W;
    const float* S;
    if (indirect) {
      const int id = a.base + a.ids[pick];
      W = reinterpret_cast<const uint8_t*>(a.tbl[id]) + a.off;
      S = a.stbl[id] + a.soff;
    } else {
      W = a.w[e];
      S = a.sc[e];
    }
    const uint4* base = reinterpret_cast<const uint4*>(W);
    uint4 wa[kMG_UNROLL], wc[kMG_UNROLL];
#pragma unroll
    for (int i = 0; i < kMG_UNROLL; ++i)
      if (wb + i < we) wa[i] = ld_stream_pol(base + (wb + i) * 32 + lane, pol);
    if (!indirect && e == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (e == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    // stage the activations as f16 hi/lo B fragments (mode 0 once; mode 1 per expert)
    if (e == 0 || MODE == 1) {
      if (e > 0) __syncthreads();
      const int nkb = a.C / 16;
      for (int i = tid; i < nkb * 4; i += kMG_THREADS) {
        const int kb = i >> 2, q = i & 3;
        float v[4];
        const int cols[4] = {kb * 16 + 2 * q, kb * 16 + 2 * q + 1, kb * 16 + 2 * q + 8, kb * 16 + 2 * q + 9};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (MODE == 0) v[j] = __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(a.x)[cols[j]] << 16);
          else v[j] = reinterpret_cast<const float*>(a.x)[(size_t)e * a.C + cols[j]];
        }
        float hi[4], lo[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          hi[j] = __half2float(__float2half_rn(v[j]));
          lo[j] = v[j] - hi[j];
        }
        xs[kb * 8 + q] = make_uint2(h2_bits(hi[0], hi[1]), h2_bits(hi[2], hi[3]));
        xs[kb * 8 + 4 + q] = make_uint2(h2_bits(lo[0], lo[1]), h2_bits(lo[2], lo[3]));
      }
    }
    const int ntl = t_last - t_first + 1;
    for (int i = tid; i < kMG_WARPS * a.tiles_cap * 16; i += kMG_THREADS) part[i] = 0.f;
    __syncthreads();

    float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
    // running (tile, column block) of the next unit: the slice is consumed in order
    int tcur = (int)(wb / CB), cb = (int)(wb - (long long)tcur * CB);
    const uint2* xl = xs + (g >= 4 ? 4 : 0) + tq;
    auto flush = [&](int t) {
      // columns 0-3 hold A.hi, 4-7 A.lo: lane (g, 0) adds lane (g, 2)'s value
      const float h0 = c0 + __shfl_down_sync(0xffffffffu, c0, 2);
      const float h2 = c2 + __shfl_down_sync(0xffffffffu, c2, 2);
      if (tq == 0) {
        float* p = part + ((size_t)warp * a.tiles_cap + (t - t_first)) * 16;
        p[g] = h0;
        p[g + 8] = h2;
      }
      c0 = c1 = c2 = c3 = 0.f;
    };
    auto consume = [&](const uint4 (&wv)[kMG_UNROLL], long long ub) {
#pragma unroll
      for (int i = 0; i < kMG_UNROLL; ++i) {
        if (ub + i < we) {
          const uint2 b0 = xl[(2 * cb) * 8];
          const uint2 b1 = xl[(2 * cb + 1) * 8];
          hmma16816(c0, c1, c2, c3, u8x2_to_h2(wv[i].x, 0x4140u), u8x2_to_h2(wv[i].x, 0x4342u),
                    u8x2_to_h2(wv[i].y, 0x4140u), u8x2_to_h2(wv[i].y, 0x4342u), b0.x, b0.y);
          hmma16816(c0, c1, c2, c3, u8x2_to_h2(wv[i].z, 0x4140u), u8x2_to_h2(wv[i].z, 0x4342u),
                    u8x2_to_h2(wv[i].w, 0x4140u), u8x2_to_h2(wv[i].w, 0x4342u), b1.x, b1.y);
          if (++cb == CB) {  // tile complete (warp-uniform)
            flush(tcur);
            ++tcur;
            cb = 0;
          }
        }
      }
    };
    for (long long ub = wb; ub < we; ub += 2 * kMG_UNROLL) {
#pragma unroll
      for (int i = 0; i < kMG_UNROLL; ++i)
        if (ub + kMG_UNROLL + i < we) wc[i] = ld_stream_pol(base + (ub + kMG_UNROLL + i) * 32 + lane, pol);
      consume(wa, ub);
#pragma unroll
      for (int i = 0; i < kMG_UNROLL; ++i)
        if (ub + 2 * kMG_UNROLL + i < we) wa[i] = ld_stream_pol(base + (ub + 2 * kMG_UNROLL + i) * 32 + lane, pol);
      if (ub + kMG_UNROLL < we) consume(wc, ub + kMG_UNROLL);
    }
    if (cb != 0) flush(tcur);  // the slice ended inside a tile
    __syncthreads();

    // per tile of this CTA: warps summed in a fixed order; whole tiles finalise here, cut tiles go
    // through the cross-CTA slots (the last arrival sums the slots in CTA order)
    float* gp = a.gpart + (size_t)e * tiles * kMG_MAXSPLIT * 16;
    unsigned int* tk = a.ticket + (size_t)e * tiles;
    const float gw = MODE == 1 ? (a.gate_w ? a.gate_w[pick] : 1.f) : 1.f;
    for (int tl = warp; tl < ntl; tl += kMG_WARPS) {
      const int t = t_first + tl;
      float v = 0.f;
      if (lane < 16)
        for (int w = 0; w < kMG_WARPS; ++w) v += part[((size_t)w * a.tiles_cap + tl) * 16 + lane];
      const long long tb = (long long)t * CB, te = tb + CB;
      const bool whole = tb >= u0 && te <= u1;
      if (!whole) {
        const int c_first = cta_of(tb, U, gridDim.x), c_last = cta_of(te - 1, U, gridDim.x);
        const int slot = blockIdx.x - c_first;
        if (lane < 16) gp[((size_t)t * kMG_MAXSPLIT + slot) * 16 + lane] = v;
        __threadfence();
        __syncwarp();
        unsigned int prev = 0;
        if (lane == 0) prev = atomicAdd(tk + t, 1u);
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev != (unsigned)(c_last - c_first)) continue;  // not the last arrival
        __threadfence();
        v = 0.f;
        if (lane < 16)
          for (int s2 = 0; s2 <= c_last - c_first; ++s2) v += __ldcg(gp + ((size_t)t * kMG_MAXSPLIT + s2) * 16 + lane);
        if (lane == 0) tk[t] = 0u;
      }
      if (MODE == 0) {
        // lane g < 8: gate of pair 8t + g in v (row g), its up in row g + 8 (lane g + 8)
        const float up = __shfl_down_sync(0xffffffffu, v, 8);
        if (lane < 8) {
          const int p = 8 * t + lane;
          a.out[e][p] = silu_mul(v * S[2 * p], up * S[2 * p + 1]);
        }
      } else if (lane < 16) {
        const int r = 16 * t + lane;
        a.out[e][r] = gw * (v * S[r]);
      }
    }
    if (e + 1 < NE) __syncthreads();
  }
}

// ---------------------------------------------------------------- packing (shadow build)
// q [R][C] biased codes (q + 128, row-major) -> the fragment-packed layout above. pair_rows: W13
// (tile row g = row 2(8t + g), tile row g + 8 = row 2(8t + g) + 1); else tile row r = row 16t + r.
__global__ void pack_i8_frag_kernel(const uint8_t* __restrict__ q, uint8_t* __restrict__ out, int R, int C,
                                    int pair_rows) {
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
    reinterpret_cast<uint4*>(out)[i] = v;
  }
}

bool mma_shadow_ok(int d, int F) { return d % 32 == 0 && F % 32 == 0 && d >= 32 && F >= 32; }

cudaError_t launch_pack_i8_frag(const uint8_t* q_biased, uint8_t* out, int R, int C, int pair_rows, cudaStream_t s) {
  if (R % 16 || C % 32) return cudaErrorInvalidValue;
  const long long n = (long long)(R / 16) * (C / 32) * 32;
  const int grid = (int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
  pack_i8_frag_kernel<<<grid > 0 ? grid : 1, 256, 0, s>>>(q_biased, out, R, C, pair_rows);
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
    cudaError_t e = cudaMalloc(&m.gpart, (size_t)kMG_MAXE * tiles * kMG_MAXSPLIT * 16 * sizeof(float));
    if (e != cudaSuccess) return e;
    e = cudaMalloc(&m.ticket, (size_t)kMG_MAXE * tiles * sizeof(unsigned int));
    if (e != cudaSuccess) return e;
    e = cudaMemset(m.ticket, 0, (size_t)kMG_MAXE * tiles * sizeof(unsigned int));
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
  const long long U = (long long)tiles * CB;
  const int sms = stream_grid_sms();
  long long gmax = U / ((CB + 1) / 2);          // a CTA's range >= half a tile: <= 3 CTAs share one
  if (gmax < 1) gmax = 1;
  const int grid = (int)(gmax < sms ? gmax : sms);
  a.tiles_cap = (int)((U + grid - 1) / grid / CB) + 2;
  MgScratch* sc = nullptr;
  cudaError_t e = mg_scratch(s, tiles, sc);
  if (e != cudaSuccess) return e;
  a.gpart = sc->gpart;
  a.ticket = sc->ticket;
  const size_t smem = (size_t)a.C / 16 * 64 + (size_t)kMG_WARPS * a.tiles_cap * 16 * sizeof(float);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
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

}  // namespace odmoe
