// p2p.cu -- flag kernels of the peer-to-peer exchange (exchange.cpp, mode 1).
//
// Every rank owns a window (CUDA IPC shared with its peers) holding, per
// source rank, the chunk lengths / offsets and the chunk bytes the source
// wrote there with its own encode kernels (NVLink stores), plus two flag
// arrays: data[s] (source s finished writing for this epoch) and ack[d]
// (destination d finished decoding what this rank wrote in its window).  The
// epoch is a device counter bumped once per exchange on every rank, so a
// captured CUDA graph replays with fresh epochs.  Releases are system-scope
// stores after a system fence; acquires are system-scope loads; a waiter gives
// up after ~10 s (a peer that never signals) and raises a device error flag
// instead of hanging the GPU.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void k_bump(uint64_t* ctr) {
  if (threadIdx.x == 0) *ctr += 1;
}

// dst[i] = epoch (+ add), after every earlier write of the stream is visible system-wide
__global__ void k_signal(uint64_t* const* dst, uint32_t n, const uint64_t* ctr) {
  const uint32_t i = threadIdx.x + blockIdx.x * blockDim.x;
  __threadfence_system();
  if (i < n && dst[i]) st_release_sys(dst[i], *ctr);
}

// every flags[i] (i < n, skip[i] == 0) reaches epoch - minus
__global__ void k_wait(const uint64_t* flags, uint32_t n, const uint64_t* ctr, uint64_t minus, uint32_t* timeout) {
  const uint32_t i = threadIdx.x + blockIdx.x * blockDim.x;
  if (i >= n) return;
  const uint64_t e = *ctr;
  const uint64_t target = e > minus ? e - minus : 0;
  if (target == 0) return;
  const long long t0 = clock64();
  uint32_t d = 32;
  while (ld_acquire_sys(flags + i) < target) {
    __nanosleep(d);
    d = d < 1024 ? 2 * d : d;
    if (clock64() - t0 > 20000000000ll) {  // ~10 s at 2 GHz
      atomicOr(timeout, 1u);
      return;
    }
  }
}

}  // namespace

namespace embc_p2p {

cudaError_t bump(uint64_t* ctr, cudaStream_t s) {
  k_bump<<<1, 32, 0, s>>>(ctr);
  return cudaGetLastError();
}

cudaError_t signal(uint64_t* const* d_dst, uint32_t n, const uint64_t* ctr, cudaStream_t s) {
  if (!n) return cudaSuccess;
  k_signal<<<(n + 127) / 128, 128, 0, s>>>(d_dst, n, ctr);
  return cudaGetLastError();
}

cudaError_t wait(const uint64_t* flags, uint32_t n, const uint64_t* ctr, uint64_t minus, uint32_t* timeout,
                 cudaStream_t s) {
  if (!n) return cudaSuccess;
  k_wait<<<(n + 127) / 128, 128, 0, s>>>(flags, n, ctr, minus, timeout);
  return cudaGetLastError();
}

}  // namespace embc_p2p
