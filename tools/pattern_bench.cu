// Access-pattern microbenchmark (not part of the library): how fast can 148 SMs stream N bytes
// with (a) the flat GEMV's pattern -- each warp one contiguous slice, 8 x 16 B per lane per batch,
// two batches in flight -- versus (b) a grid-stride pattern where all CTAs sweep the buffer
// front to back together, (c) block-interleaved slices (64 KB blocks dealt round-robin to CTAs).
// (d) dynamic: every warp claims 32 KB chunks from a global atomic counter (the claim for its next
// chunk is issued when it starts the current one), so SMs that get less bandwidth simply take fewer
// chunks (no tail of slow CTAs). No arithmetic beyond an XOR per load. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

constexpr int U = 8, WARPS = 16;

// (a) contiguous per-warp slices of the CTA's contiguous range
__global__ void __launch_bounds__(WARPS * 32, 1) slices(const uint4* __restrict__ p, long long n16, unsigned* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long groups = n16 / 32;
  const long long cb = groups * blockIdx.x / gridDim.x, ce = groups * (blockIdx.x + 1) / gridDim.x;
  const long long wb = cb + (ce - cb) * warp / WARPS, we = cb + (ce - cb) * (warp + 1) / WARPS;
  unsigned acc = 0;
  uint4 a[U], b[U];
  long long g = wb;
#pragma unroll
  for (int i = 0; i < U; ++i) if (g + i < we) a[i] = ldg_stream(p + (g + i) * 32 + lane);
  for (; g < we; g += 2 * U) {
#pragma unroll
    for (int i = 0; i < U; ++i) if (g + U + i < we) b[i] = ldg_stream(p + (g + U + i) * 32 + lane);
#pragma unroll
    for (int i = 0; i < U; ++i) if (g + i < we) acc ^= a[i].x ^ a[i].y ^ a[i].z ^ a[i].w;
#pragma unroll
    for (int i = 0; i < U; ++i) if (g + 2 * U + i < we) a[i] = ldg_stream(p + (g + 2 * U + i) * 32 + lane);
#pragma unroll
    for (int i = 0; i < U; ++i) if (g + U + i < we) acc ^= b[i].x ^ b[i].y ^ b[i].z ^ b[i].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// (b) grid-stride: the CTA's warps take consecutive 512 B groups; CTAs interleave at group level
__global__ void __launch_bounds__(WARPS * 32, 1) gridstride(const uint4* __restrict__ p, long long n16, unsigned* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long groups = n16 / 32;
  const long long stride = (long long)gridDim.x * WARPS;
  unsigned acc = 0;
  for (long long g0 = (long long)blockIdx.x * WARPS + warp; g0 < groups; g0 += stride * U) {
    uint4 a[U];
#pragma unroll
    for (int i = 0; i < U; ++i) if (g0 + i * stride < groups) a[i] = ldg_stream(p + (g0 + i * stride) * 32 + lane);
#pragma unroll
    for (int i = 0; i < U; ++i) if (g0 + i * stride < groups) acc ^= a[i].x ^ a[i].y ^ a[i].z ^ a[i].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// (c) block-interleaved: blocks of BLK groups (64 KB) dealt round-robin to CTAs; inside a CTA's
// block sequence, contiguous per-warp slices as in (a)
constexpr long long BLK = 128;
__global__ void __launch_bounds__(WARPS * 32, 1) blocks(const uint4* __restrict__ p, long long n16, unsigned* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long groups = n16 / 32, nblk = groups / BLK;
  const long long my = (nblk - blockIdx.x + gridDim.x - 1) / gridDim.x;  // blocks of this CTA
  const long long vg = my * BLK;                                       // its virtual groups
  const long long wb = vg * warp / WARPS, we = vg * (warp + 1) / WARPS;
  auto addr = [&](long long v) {
    const long long b = v / BLK, o = v % BLK;
    return p + ((b * gridDim.x + blockIdx.x) * BLK + o) * 32 + lane;
  };
  unsigned acc = 0;
  uint4 a[U], b[U];
  long long g = wb;
#pragma unroll
  for (int i = 0; i < U; ++i) if (g + i < we) a[i] = ldg_stream(addr(g + i));
  for (; g < we; g += 2 * U) {
#pragma unroll
    for (int i = 0; i < U; ++i) if (g + U + i < we) b[i] = ldg_stream(addr(g + U + i));
#pragma unroll
    for (int i = 0; i < U; ++i) if (g + i < we) acc ^= a[i].x ^ a[i].y ^ a[i].z ^ a[i].w;
#pragma unroll
    for (int i = 0; i < U; ++i) if (g + 2 * U + i < we) a[i] = ldg_stream(addr(g + 2 * U + i));
#pragma unroll
    for (int i = 0; i < U; ++i) if (g + U + i < we) acc ^= b[i].x ^ b[i].y ^ b[i].z ^ b[i].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// (d) dynamic chunks of CH groups (CH * 512 B) claimed per warp
constexpr long long CH = 64;
__global__ void __launch_bounds__(WARPS * 32, 1) dynamic(const uint4* __restrict__ p, long long n16, unsigned* out,
                                                         unsigned long long* counter) {
  const int lane = threadIdx.x & 31;
  const long long nch = (n16 / 32) / CH;
  unsigned acc = 0;
  unsigned long long cur = 0;
  if (lane == 0) cur = atomicAdd(counter, 1ull);
  cur = __shfl_sync(0xffffffffu, cur, 0);
  while ((long long)cur < nch) {
    unsigned long long nxt = 0;
    if (lane == 0) nxt = atomicAdd(counter, 1ull);
    const uint4* base = p + (long long)cur * CH * 32 + lane;
    uint4 a[U], b[U];
#pragma unroll
    for (int i = 0; i < U; ++i) a[i] = ldg_stream(base + i * 32);
    for (int g = 0; g < CH; g += 2 * U) {
#pragma unroll
      for (int i = 0; i < U; ++i) b[i] = ldg_stream(base + (g + U + i) * 32);
#pragma unroll
      for (int i = 0; i < U; ++i) acc ^= a[i].x ^ a[i].y ^ a[i].z ^ a[i].w;
      if (g + 2 * U < CH) {
#pragma unroll
        for (int i = 0; i < U; ++i) a[i] = ldg_stream(base + (g + 2 * U + i) * 32);
      }
#pragma unroll
      for (int i = 0; i < U; ++i) acc ^= b[i].x ^ b[i].y ^ b[i].z ^ b[i].w;
    }
    cur = __shfl_sync(0xffffffffu, nxt, 0);
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  const long long sizes[3] = {352321536LL, 704643072LL, 1073741824LL};
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  char* buf;
  cudaMalloc(&buf, sizes[2]);
  cudaMemset(buf, 1, sizes[2]);
  char* flush;
  cudaMalloc(&flush, 256 << 20);
  unsigned* out;
  cudaMalloc(&out, 4);
  unsigned long long* counter;
  cudaMalloc(&counter, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[4] = {"slices", "gridstride", "blocks64K", "dynamic32K"};
  printf("{\n");
  for (int k = 0; k < 4; ++k) {
    for (int si = 0; si < 3; ++si) {
      const long long n16 = sizes[si] / 16;
      float best = 1e9f, sum = 0.f;
      for (int it = 0; it < 12; ++it) {
        cudaMemsetAsync(flush, it, 256 << 20);
        cudaMemsetAsync(counter, 0, 8);
        cudaEventRecord(e0);
        if (k == 0) slices<<<sms, WARPS * 32>>>((const uint4*)buf, n16, out);
        if (k == 1) gridstride<<<sms, WARPS * 32>>>((const uint4*)buf, n16, out);
        if (k == 2) blocks<<<sms, WARPS * 32>>>((const uint4*)buf, n16, out);
        if (k == 3) dynamic<<<sms, WARPS * 32>>>((const uint4*)buf, n16, out, counter);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it >= 2) { best = ms < best ? ms : best; sum += ms; }
      }
      const float med = sum / 10;
      printf(" \"%s_%lldMB\": {\"us_mean\": %.2f, \"us_best\": %.2f, \"GBps_mean\": %.1f},\n", names[k],
             sizes[si] >> 20, med * 1e3, best * 1e3, sizes[si] / (med * 1e-3) / 1e9);
    }
  }
  printf(" \"err\": \"%s\"\n}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
