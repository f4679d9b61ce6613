// Prefill grouped expert GEMM on the 5th-generation tensor cores (P:214
// "token embeddings routed to the same expert can be grouped and computed via a larger matrix
// multiplication"). This is the one place on the path where the work is a real dense contraction
// (m_e ~ T*k/E = 128 rows per expert at T = 512), so it runs on tcgen05:
//
//   C_e[m_e x N] = A[rows of expert e] (K-major bf16) . B_e[N x K]^T (K-major bf16), fp32 in TMEM
//
// GEMM1: A = X_perm [M, d], B_e = W13_e [2F, d] (gate/up interleaved) -> SwiGLU epilogue ->
//        A2 [M, F] bf16 (reading Q8: the prefill intermediate is bf16, the tensor-core input type).
// GEMM2: A = A2 [M, F], B_e = W2_e [d, F] -> gate-scale epilogue -> Y_perm [M, d] fp32.
//
// Kernel anatomy (one (up to) 256 x BN output tile per CTA, 6 warps). An expert's rows (m_e ~ 128
// at T = 512, often a little more) are covered by ONE CTA column with two M=128 accumulators in
// TMEM, so every weight (B) stage fetched by TMA feeds both halves and the expert's weights stream
// from HBM exactly once (a 128-row tiling would re-read them for every expert with m_e > 128):
//   warp 0   : TMA producer, ring of {A 2x128x64, B BNx64} bf16 tiles (128B swizzle); the second
//              A half is skipped when the tile has <= 128 rows
//   warp 1   : TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16 per MMA, one
//              or two accumulators), tcgen05.commit -> stage "empty" barriers / accumulator ready
//   warps 2-5: epilogue, tcgen05.ld 32x32b (each warp owns its 32-lane TMEM quadrant), both halves
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.h"

namespace odmoe {

constexpr int kGG_BM = 128;   // rows per accumulator (UMMA M)
constexpr int kGG_MT = 2;     // accumulators per CTA -> up to 256 rows per tile
constexpr int kGG_BK = 64;    // 64 bf16 = 128 bytes = one swizzle row
constexpr int kGG_THREADS = 192;
template <int BN> __host__ __device__ constexpr int gg_stages() { return BN >= 224 ? 3 : 4; }
// TMEM columns of the two accumulators, rounded up to the power of two tcgen05.alloc takes
template <int BN> __host__ __device__ constexpr uint32_t gg_tmem_cols() {
  return kGG_MT * BN <= 128 ? 128u : (kGG_MT * BN <= 256 ? 256u : 512u);
}

struct GGMaps {
  CUtensorMap b[kMaxGGExperts];
  int dyn_stages;  // 1: ring depth per tile (more B stages when the tile has one A half)
};
constexpr int kGG_MAX_ST = 8;  // barrier slots

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// K-major operand, 128-byte swizzle: rows of 128 B, 8-row atoms 1024 B apart (SBO), LBO unused (1),
// descriptor version 1 (sm100), layout type 2 (SWIZZLE_128B).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// kind::f16 instruction descriptor: D fp32, A/B bf16, both K-major, M = 128, N = BN.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// MODE 0: SwiGLU -> bf16 [M, N/2]; MODE 1: gate-scale -> fp32 [M, N]. STAGES: smem ring depth
// (2 with BN = 128 leaves room for two CTAs per SM, whose epilogues then overlap the other's loads).
//
// Persistent (round 2): a CTA walks the tiles blockIdx.x, blockIdx.x + gridDim.x, ...; the producer's
// ring runs across tile boundaries, so the next tile's weight stages stream in while the epilogue
// warps drain the accumulator of the current one (acc_full / acc_empty barriers hand TMEM between the
// MMA issuer and the epilogue), and the prologue (barriers, TMEM allocation, tensor-map prefetch) is
// paid once per CTA instead of once per tile.
template <int BN, int MODE, int STAGES = gg_stages<BN>()>
__global__ void __launch_bounds__(kGG_THREADS, 1)
grouped_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ GGMaps maps_b,
                    const int4* __restrict__ tiles, int n_tiles, int K, int N, void* __restrict__ out,
                    const float* __restrict__ gate) {
  constexpr int A_BYTES = kGG_BM * kGG_BK * 2;          // one 128-row half
  constexpr int B_BYTES = BN * kGG_BK * 2;
  constexpr int STAGE = kGG_MT * A_BYTES + B_BYTES;
  constexpr int RING = STAGES * STAGE;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + RING);
  uint64_t* empty = full + kGG_MAX_ST;
  uint64_t* acc_full = empty + kGG_MAX_ST;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KB = K / kGG_BK;
  auto sA_of = [&](int s, int hh) { return smem + s * STAGE + hh * A_BYTES; };
  auto sB_of = [&](int s) { return smem + s * STAGE + kGG_MT * A_BYTES; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 4);  // one arrival per epilogue warp
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    for (int e = 0; e < kMaxGGExperts; ++e)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps_b.b[e])) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(gg_tmem_cols<BN>()));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0, ph = 0;
      for (int ti = blockIdx.x; ti < n_tiles; ti += gridDim.x) {
        const int4 tile = tiles[ti];  // {expert, row0, rows (<= 256), n0}
        const int halves = tile.z > kGG_BM ? 2 : 1;
        const uint32_t tx = (uint32_t)(halves * A_BYTES + B_BYTES);
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&empty[s], (uint32_t)ph ^ 1u);
          mbar_expect_tx(&full[s], tx);
          for (int hh = 0; hh < halves; ++hh)
            tma_load_2d(sA_of(s, hh), &map_a, &full[s], kb * kGG_BK, tile.y + hh * kGG_BM);
          tma_load_2d(sB_of(s), &maps_b.b[tile.x], &full[s], kb * kGG_BK, tile.w);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(kGG_BM, BN);
      int s = 0, ph = 0, it = 0;
      for (int ti = blockIdx.x; ti < n_tiles; ti += gridDim.x, ++it) {
        const int halves = tiles[ti].z > kGG_BM ? 2 : 1;
        mbar_wait(acc_empty, (uint32_t)(it & 1) ^ 1u);  // the epilogue has drained the previous tile
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full[s], (uint32_t)ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t b0 = smem_u32(sB_of(s));
          for (int hh = 0; hh < halves; ++hh) {
            const uint32_t a0 = smem_u32(sA_of(s, hh));
#pragma unroll
            for (int k = 0; k < kGG_BK / 16; ++k)
              umma_bf16(tmem + (uint32_t)(hh * BN), umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32),
                        idesc, (kb | k) != 0);
          }
          umma_commit(&empty[s]);  // smem slot free once these MMAs have read it
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        umma_commit(acc_full);
      }
    }
  } else {
    // epilogue: warp w owns TMEM lanes [32*(w%4), +32) of each accumulator half
    const int q = warp & 3;
    int it = 0;
    for (int ti = blockIdx.x; ti < n_tiles; ti += gridDim.x, ++it) {
      const int4 tile = tiles[ti];
      const int row0 = tile.y, rows = tile.z, n0 = tile.w;
      const int halves = rows > kGG_BM ? 2 : 1;
      mbar_wait(acc_full, (uint32_t)(it & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int hh = 0; hh < halves; ++hh) {
        const int r = hh * kGG_BM + q * 32 + lane;
        const bool valid = r < rows;
        const long long grow = (long long)row0 + r;
        const float g = (MODE == 1 && valid) ? (gate ? gate[grow] : 1.f) : 0.f;  // no gate: plain GEMM
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
          uint32_t v[16];
          tmem_ld16(tmem + (uint32_t)(hh * BN) + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, v);
          if (!valid) continue;
          if constexpr (MODE == 0) {
            uint32_t packed[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float a0 = silu_mul(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]));
              const float a1 = silu_mul(__uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
              const __nv_bfloat162 b = __floats2bfloat162_rn(a0, a1);
              packed[i] = *reinterpret_cast<const uint32_t*>(&b);
            }
            __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(out) + grow * (N / 2) + (n0 + c0) / 2;
            *reinterpret_cast<uint4*>(o) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
          } else {
            float* o = reinterpret_cast<float*>(out) + grow * N + n0 + c0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
              reinterpret_cast<float4*>(o)[i] =
                  make_float4(g * __uint_as_float(v[4 * i]), g * __uint_as_float(v[4 * i + 1]),
                              g * __uint_as_float(v[4 * i + 2]), g * __uint_as_float(v[4 * i + 3]));
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(acc_empty)) : "memory");
    }
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(gg_tmem_cols<BN>()));
  }
}

// ---------------------------------------------------------------- host side
// ODMOE_GG_2CTA=1: 128-wide tiles with a 2-stage ring (97 KB smem, 256 TMEM columns), two CTAs per SM
static bool gg_two_ctas() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ODMOE_GG_2CTA");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D bf16 row-major [rows, cols] tensor, box = {64 cols, box_rows rows}, 128B swizzle.
static bool make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)kGG_BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, int MODE, int STAGES = gg_stages<BN>()>
static cudaError_t gg_launch(const GroupedGemmArgs& g, cudaStream_t s) {
  CUtensorMap ma;
  GGMaps mb;
  static int dyn = -1;
  if (dyn < 0) {
    const char* e = getenv("ODMOE_GG_DYN");  // ODMOE_GG_DYN=0: the fixed ring (A/B)
    dyn = (e && e[0] == '0') ? 0 : 1;
  }
  mb.dyn_stages = dyn;
  if (!make_map(&ma, g.a, (uint64_t)g.M, (uint64_t)g.K, kGG_BM)) return cudaErrorInvalidValue;
  for (int e = 0; e < g.n_experts; ++e)
    if (g.b[e] && !make_map(&mb.b[e], g.b[e], (uint64_t)g.N, (uint64_t)g.K, BN)) return cudaErrorInvalidValue;
  const size_t smem = 1024 + (size_t)STAGES * (kGG_MT * kGG_BM + BN) * kGG_BK * 2 + 256;
  auto kern = grouped_gemm_kernel<BN, MODE, STAGES>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // persistent: one CTA per SM (two with the 128-wide 2-stage variant), tiles dealt round-robin
  const int per_sm = STAGES <= 2 ? 2 : 1;
  const int grid = g.n_tiles < num_sms() * per_sm ? g.n_tiles : num_sms() * per_sm;
  kern<<<grid, kGG_THREADS, smem, s>>>(ma, mb, g.tiles, g.n_tiles, g.K, g.N, g.out, g.gate);
  return cudaGetLastError();
}

cudaError_t launch_grouped_gemm(const GroupedGemmArgs& g, cudaStream_t s) {
  if (g.n_experts > kMaxGGExperts || g.K % kGG_BK) return cudaErrorInvalidValue;
  if (g.n_tiles == 0) return cudaSuccess;
  if (gg_two_ctas()) {
    if (g.N % 128) return cudaErrorInvalidValue;
    return g.mode == 0 ? gg_launch<128, 0, 2>(g, s) : gg_launch<128, 1, 2>(g, s);
  }
  if (g.mode == 0) {
    if (grouped_gemm_bn(0, g.N) == 224) return gg_launch<224, 0>(g, s);
    if (g.N % 256) return cudaErrorInvalidValue;
    return gg_launch<256, 0>(g, s);
  }
  if (g.N % 128) return cudaErrorInvalidValue;
  return gg_launch<128, 1>(g, s);
}

// GEMM1 tile width. 224 (where it divides N; Mixtral's 2F = 28672 -> 1024 tiles = 6.9 waves of 148
// CTAs instead of 896 = 6.05) was measured no faster than 256 (0.673 vs 0.668 ms for the T = 512
// grouped FFN, profiles/kb_r01_grouped_bn_ab.json): the per-tile prologue / epilogue, not the
// wave tail, sets the gap to the HBM floor. ODMOE_GG_BN=224 keeps it selectable.
int grouped_gemm_bn(int mode, int N) {
  static int use224 = -1;
  if (use224 < 0) {
    const char* e = getenv("ODMOE_GG_BN");
    use224 = (e && e[0] == '2' && e[1] == '2' && e[2] == '4') ? 1 : 0;
  }
  if (mode != 0 || gg_two_ctas()) return 128;
  return (use224 && N % 224 == 0) ? 224 : 256;
}

int grouped_gemm_bm() { return kGG_MT * kGG_BM; }

}  // namespace odmoe
