// Peer-to-peer combine over NVLink (the per-layer "workers -> main node" transfer of P:117 with
// its sum): replaces memset + local sum + ncclReduce with one small kernel per sender and one
// per receiver.
//
// Sender (every GPU that computed expert work for the layer): sums its n gated partials in router
// rank order and stores the result straight into its row of GPU 0's receive buffer (peer memory
// mapped with CUDA IPC, stores travel over NVLink). Every element travels WITH the layer's epoch in
// one 8-byte store {value bits, epoch} (single-copy atomic, the "LL" protocol NCCL uses for small
// messages), so no fence and no separate flag are needed: a value is valid once its epoch word is.
// Receiver (GPU 0, before the next router / the final combine): polls each expected sender's
// {value, epoch} pairs with volatile 16-byte loads until both epochs match, then sums the rows in rank
// order (deterministic; for the paper's placement the rows are whole experts and the sum equals the
// 1-GPU combine bit for bit). A wait longer than ~20 s sets err_flag = 2 and returns (the host
// reports it) instead of hanging. The receive buffer holds 2 words per element.
#include "common.cuh"
#include "kernels.h"

namespace odmoe {

// two {value, epoch} pairs per 16-byte volatile store (each 8-byte half lands atomically)
__device__ __forceinline__ void st_ll2(float* p, float a, float b, uint32_t ep) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(__float_as_uint(a)), "r"(ep),
               "r"(__float_as_uint(b)), "r"(ep)
               : "memory");
}
__device__ __forceinline__ void st_ll4(float* p, const float4& v, uint32_t ep) {
  st_ll2(p, v.x, v.y, ep);
  st_ll2(p + 4, v.z, v.w, ep);
}
__device__ __forceinline__ uint4 ld_volatile4(const float* p) {
  uint4 r;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(256) p2p_send_kernel(const float* const* __restrict__ y, int n, int d,
                                                       float* dst, uint32_t epoch) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int j = threadIdx.x * 4; j < d; j += blockDim.x * 4) {
    float4 s = *reinterpret_cast<const float4*>(y[0] + j);
    for (int a = 1; a < n; ++a) {
      const float4 t = *reinterpret_cast<const float4*>(y[a] + j);
      s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;
    }
    st_ll4(dst + 2 * (size_t)j, s, epoch);
  }
}

__global__ void __launch_bounds__(256) p2p_gather_kernel(const float* part, uint32_t mask, int d, uint32_t epoch,
                                                         float* __restrict__ out, int32_t* err_flag) {
  const uint64_t t0 = globaltimer();
  bool timed_out = false;
  for (int j = threadIdx.x * 4; j < d && !timed_out; j += blockDim.x * 4) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    bool first = true;
    for (int r = 0; r < 32 && !timed_out; ++r) {
      if (!((mask >> r) & 1u)) continue;
      const float* q = part + 2 * ((size_t)r * d + j);
      uint4 a, b;
      for (;;) {  // both 16-byte pieces of this rank's 4 elements carry this layer's epoch
        a = ld_volatile4(q);
        b = ld_volatile4(q + 4);
        if (a.y == epoch && a.w == epoch && b.y == epoch && b.w == epoch) break;
        if (globaltimer() - t0 > 20000000000ull) { timed_out = true; break; }
        __nanosleep(128);  // back off: the sender's NVLink stores land in these lines
      }
      const float4 t = make_float4(__uint_as_float(a.x), __uint_as_float(a.z), __uint_as_float(b.x),
                                   __uint_as_float(b.z));
      if (first) { s = t; first = false; }
      else { s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w; }
    }
    if (!timed_out) *reinterpret_cast<float4*>(out + j) = s;
  }
  if (timed_out) *err_flag = 2;
}

// Warm wait for an expert load (the on-demand path's idle-to-busy ramp): instead of letting the
// compute stream idle on the copy event for milliseconds -- after which the next expert kernel runs
// ~20 % slower (profiles/kb_r02_ramp_*.json: 80.1 us after a 6 ms idle gap, 66.3 us when one CTA
// spins through the gap) -- one warp spins on the slot's flag until the copy stream has written the
// load's epoch. A wait over ~30 s sets err_flag = 3 and returns (reported as a CUDA-side error).
__global__ void __launch_bounds__(32) wait_flag_kernel(const uint32_t* flag, uint32_t epoch, int32_t* err_flag) {
  if (threadIdx.x != 0) return;
  const uint64_t t0 = globaltimer();
  uint32_t v;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if ((int32_t)(v - epoch) >= 0) break;
    if (globaltimer() - t0 > 30000000000ull) {
      *err_flag = 3;
      break;
    }
  }
}

cudaError_t launch_wait_flag(const uint32_t* flag, uint32_t epoch, int32_t* err_flag, cudaStream_t s) {
  wait_flag_kernel<<<1, 32, 0, s>>>(flag, epoch, err_flag);
  return cudaGetLastError();
}

cudaError_t launch_p2p_send(const float* const* y, int n, int d, float* dst, uint32_t epoch, cudaStream_t s) {
  if (d % 4) return cudaErrorInvalidValue;
  p2p_send_kernel<<<1, 256, 0, s>>>(y, n, d, dst, epoch);
  return cudaGetLastError();
}

cudaError_t launch_p2p_gather(const float* part, uint32_t mask, int d, uint32_t epoch, float* out, int32_t* err_flag,
                              cudaStream_t s) {
  if (d % 4) return cudaErrorInvalidValue;
  p2p_gather_kernel<<<1, 256, 0, s>>>(part, mask, d, epoch, out, err_flag);
  return cudaGetLastError();
}

}  // namespace odmoe
