// Peer-to-peer combine over NVLink (the per-layer "workers -> main node" transfer of P:117 with
// its sum): replaces memset + local sum + ncclReduce with one small kernel per sender and one
// per receiver.
//
// Sender (every GPU that computed expert work for the layer): sums its n gated partials in router
// rank order and stores the result straight into its row of GPU 0's receive buffer (peer memory
// mapped with CUDA IPC, stores travel over NVLink), then publishes the layer's epoch in its flag
// with a system-scope release after a system-scope fence.
// Receiver (GPU 0, before the next router / the final combine): waits with acquire loads until every
// expected sender's flag holds the epoch, then sums the rows in rank order (deterministic; for the
// paper's placement the rows are whole experts and the sum equals the 1-GPU combine bit for bit).
// A wait longer than ~20 s sets err_flag = 2 and returns (the host reports it) instead of hanging.
#include "common.cuh"
#include "kernels.h"

namespace odmoe {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(256) p2p_send_kernel(const float* const* __restrict__ y, int n, int d,
                                                       float* dst, uint32_t* flag, uint32_t epoch) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int j = threadIdx.x * 4; j < d; j += blockDim.x * 4) {
    float4 s = *reinterpret_cast<const float4*>(y[0] + j);
    for (int a = 1; a < n; ++a) {
      const float4 t = *reinterpret_cast<const float4*>(y[a] + j);
      s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;
    }
    *reinterpret_cast<float4*>(dst + j) = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(flag, epoch);
  }
}

__global__ void __launch_bounds__(256) p2p_gather_kernel(const float* part, const uint32_t* flags, uint32_t mask,
                                                         int d, uint32_t epoch, float* __restrict__ out,
                                                         int32_t* err_flag) {
  __shared__ int ok;
  if (threadIdx.x < 32) {
    const int r = threadIdx.x;
    bool timed_out = false;
    if ((mask >> r) & 1u) {
      const uint64_t t0 = globaltimer();
      while ((int32_t)(ld_acquire_sys(flags + r) - epoch) < 0) {
        if (globaltimer() - t0 > 20000000000ull) { timed_out = true; break; }
        __nanosleep(200);
      }
    }
    const unsigned bad = __ballot_sync(0xffffffffu, timed_out);
    if (r == 0) {
      ok = bad == 0u;
      if (bad) *err_flag = 2;
    }
  }
  __syncthreads();
  if (!ok) return;
  for (int j = threadIdx.x * 4; j < d; j += blockDim.x * 4) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    bool first = true;
    for (int r = 0; r < 32; ++r) {
      if (!((mask >> r) & 1u)) continue;
      const float4 t = __ldcv(reinterpret_cast<const float4*>(part + (size_t)r * d + j));
      if (first) { s = t; first = false; }
      else { s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w; }
    }
    *reinterpret_cast<float4*>(out + j) = s;
  }
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

cudaError_t launch_p2p_send(const float* const* y, int n, int d, float* dst, uint32_t* flag, uint32_t epoch,
                            cudaStream_t s) {
  if (d % 4) return cudaErrorInvalidValue;
  p2p_send_kernel<<<1, 256, 0, s>>>(y, n, d, dst, flag, epoch);
  return cudaGetLastError();
}

cudaError_t launch_p2p_gather(const float* part, const uint32_t* flags, uint32_t mask, int d, uint32_t epoch,
                              float* out, int32_t* err_flag, cudaStream_t s) {
  if (d % 4) return cudaErrorInvalidValue;
  p2p_gather_kernel<<<1, 256, 0, s>>>(part, flags, mask, d, epoch, out, err_flag);
  return cudaGetLastError();
}

}  // namespace odmoe
