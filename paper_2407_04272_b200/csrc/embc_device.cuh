// embc_device.cuh -- device-side building blocks shared by the encode and
// decode kernels: the bit-exact quantizer, varint/zigzag helpers, block scans,
// staged unaligned byte output, and the device error record.
//
// Reference semantics cited as file:line under /root/reference/proj/include/embc/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/embc_cuda.h"

namespace embc_dev {

constexpr int kBlock = 256;           // threads per tile CTA
constexpr uint32_t kHeader = 30;      // CompressedChunk::kHeaderSize (container.hpp:67)
constexpr uint32_t kMetaSize = 25;    // ChunkMetadata::kWireSize (container.hpp:193)
constexpr uint32_t kMaxWindow = 65536;  // VlzConfig::kMaxWindow (vlz.hpp:45)
constexpr uint32_t kHistCap = 1u << 17;   // GPU Huffman alphabet span limit (EMBC_R_RANGE)
constexpr uint32_t kWin = 4096;           // K1 speculative histogram window, codes [-2048, 2048)
constexpr uint32_t kWidePool = 4 * kHistCap;  // histogram entries for wider alphabets per call

// ---------------------------------------------------------------------------
// Device error record.  Each job keeps a 64-bit key (index << 6 | reason); the
// minimum over the grid is the first failure in element order, matching the
// reference's sequential stop-at-first-error loops (quantizer.hpp:87-89).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t err_key(uint64_t index, uint32_t reason) {
  return (index << 6) | reason;
}

// Sticky failure record folded from per-job keys by the last kernel of a call.
struct DevError {
  int32_t status;
  int32_t reason;
  uint32_t job;
  uint32_t valid;
  uint64_t index;
  uint64_t a, b;
  double eb;
};

// ---------------------------------------------------------------------------
// Fast integer division by a runtime constant (row/column of an element).
// ---------------------------------------------------------------------------
struct FastDiv {
  uint32_t d, m, s;  // n / d == __umulhi(n, m) >> s   (for d > 1); m == 0 => d == 1
};

__host__ inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0, 0};
  if (d <= 1) return f;
  uint32_t s = 0;
  while ((1ull << s) < d) ++s;               // s = ceil(log2 d)
  uint64_t m = ((1ull << (32 + s)) + d - 1) / d;  // ceil(2^(32+s) / d)
  f.m = static_cast<uint32_t>(m);              // m - 2^32 fits in 32 bits for s >= 1
  f.s = s;
  return f;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  if (f.d <= 1) return n;
  // m' = m - 2^32;  q = (umulhi(n, m') + n) >> s   computed without overflow
  const uint32_t t = __umulhi(n, f.m);
  return static_cast<uint32_t>((static_cast<uint64_t>(t) + n) >> f.s);
}

// ---------------------------------------------------------------------------
// Quantizer (quantizer.hpp:43-76), bit-exact.
//
// Slow path: the reference's algorithm verbatim in IEEE binary64 with every
// operation separately rounded (__d*_rn intrinsics: no FMA contraction).
//
// Fast path (fp32 inputs): q_f = RN32(x * RN32(1/w)).  When |q_f| <= 1024 and
// q_f is farther than 2^-12 from every half-integer, then
//   (1) |q_f - x/w| <= 2^-13 (two fp32 roundings on |x/w| <= 1025), so
//       llround(RN64(x/w)) == rint(q_f);
//   (2) |x/w - c| <= 1/2 - 2^-13, so |c*w - x| <= eb*(1 - 2^-12), which the
//       reference's within_bound check (with its 2^-52 slack, all binary64
//       roundings <= 2^-41 eb at |c| <= 1025) always accepts;
//   (3) no overflow is possible.
// Everything else (non-finite, large or near-half quotients, subnormal
// reciprocals) takes the exact slow path.  The rounding uses the 1.5*2^23
// magic-number trick so the fast path is four FP32-pipe ops.
// ---------------------------------------------------------------------------
struct QParams {
  double eb;  // ErrorBound::value()
  double w;   // bin_width() = 2*eb (batch.hpp:45), exact
  float rw;   // RN32(RN64(1/w))
  int fast;   // rw is a normal float well inside range
};

static __device__ __noinline__ int32_t quantize_slow(double x, double eb, double w, uint32_t* reason) {
  if (!isfinite(x)) {
    *reason = EMBC_R_NONFINITE;
    return 0;
  }
  const double q = __ddiv_rn(x, w);
  if (fabs(q) > 4294967294.0) {  // 2.0 * INT32_MAX (quantizer.hpp:50)
    *reason = EMBC_R_OVERFLOW;
    return 0;
  }
  // std::llround: half away from zero.  q - trunc(q) is exact.
  const double t = trunc(q);
  long long c = static_cast<long long>(t);
  if (fabs(__dsub_rn(q, t)) >= 0.5) c += (q > 0.0) ? 1 : -1;
  auto within = [&](long long cc) {
    const double recon = __dmul_rn(static_cast<double>(cc), w);
    const double slack = __dmul_rn(fabs(recon), 0x1.0p-52);
    return fabs(__dsub_rn(recon, x)) <= __dadd_rn(eb, slack);
  };
  if (!within(c)) {
    const long long nb = (x > __dmul_rn(static_cast<double>(c), w)) ? c + 1 : c - 1;
    if (!within(nb)) {
      *reason = EMBC_R_EB_TOO_SMALL;
      return 0;
    }
    c = nb;
  }
  if (c > 2147483647LL || c < -2147483647LL) {
    *reason = EMBC_R_OVERFLOW;
    return 0;
  }
  return static_cast<int32_t>(c);
}

__device__ __forceinline__ int32_t quantize_f32(float xf, const QParams& p, uint32_t* reason) {
  if (p.fast) {
    const float q = __fmul_rn(xf, p.rw);
    const float t = __fadd_rn(q, 12582912.0f);  // 1.5 * 2^23
    const float r = __fsub_rn(t, 12582912.0f);
    const float d = fabsf(__fsub_rn(q, r));
    if (fabsf(q) <= 1024.0f && d < 0.499755859375f) return __float_as_int(t) - 0x4B400000;
  }
  return quantize_slow(static_cast<double>(xf), p.eb, p.w, reason);
}

// reconstruct_value (quantizer.hpp:29-31): double(code) * (2*eb)
__device__ __forceinline__ double reconstruct(int32_t c, double w) {
  return __dmul_rn(static_cast<double>(c), w);
}

// ---------------------------------------------------------------------------
// zigzag (bytes.hpp:168-174) and unsigned LEB128 (bytes.hpp:61-67)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t zigzag(int32_t v) {
  return (static_cast<uint32_t>(v) << 1) ^ static_cast<uint32_t>(v >> 31);
}
__device__ __forceinline__ int32_t unzigzag(uint32_t z) {
  return static_cast<int32_t>(z >> 1) ^ -static_cast<int32_t>(z & 1);
}
// bytes in the LEB128 encoding of a u32
__device__ __forceinline__ uint32_t varint_len(uint32_t v) {
  // ceil(bits / 7) for bits = significant bits of v (>= 1): ((bits + 6) * 37) >> 8 is exact for bits <= 32
  const uint32_t bits = 32u - __clz(v | 1u);
  return ((bits + 6u) * 37u) >> 8;
}
__device__ __forceinline__ uint8_t* put_varint(uint8_t* p, uint32_t v) {
  while (v >= 0x80u) {
    *p++ = static_cast<uint8_t>(v | 0x80u);
    v >>= 7;
  }
  *p++ = static_cast<uint8_t>(v);
  return p;
}

// ---------------------------------------------------------------------------
// Block-wide exclusive scan / reduction (any blockDim multiple of 32 <= 1024).
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Exclusive scan across the block; returns the block total in *total.
// `tmp` must hold 33 T in shared memory.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* tmp, T* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) tmp[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    T s = lane < nw ? tmp[lane] : T(0);
    T si = warp_incl_scan(s);
    if (lane < nw) tmp[lane] = si - s;
    if (lane == nw - 1) tmp[32] = si;
  }
  __syncthreads();
  T res = tmp[wid] + inc - v;
  *total = tmp[32];
  __syncthreads();
  return res;
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* tmp) {
  T total;
  (void)block_excl_scan(v, tmp, &total);
  return total;
}

// ---------------------------------------------------------------------------
// Copy a staged byte range to global memory at an arbitrary byte address.
// The stage holds byte k of the output at stage[(dst & 15) + k], so 16-byte
// shared reads line up with 16-byte aligned global stores.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void copy_out_staged(uint8_t* dst, const uint8_t* stage, uint64_t len) {
  if (len == 0) return;
  const uint64_t a0 = reinterpret_cast<uint64_t>(dst);
  const uint32_t mis = static_cast<uint32_t>(a0 & 15);
  const uint64_t first_al = (a0 + 15) & ~uint64_t(15);
  const uint64_t end = a0 + len;
  const uint64_t last_al = end & ~uint64_t(15);
  if (first_al >= last_al) {
    for (uint64_t k = threadIdx.x; k < len; k += blockDim.x) dst[k] = stage[mis + k];
    return;
  }
  const uint64_t head = first_al - a0;
  for (uint64_t k = threadIdx.x; k < head; k += blockDim.x) dst[k] = stage[mis + k];
  const uint64_t nvec = (last_al - first_al) >> 4;
  const uint4* s4 = reinterpret_cast<const uint4*>(stage + mis + head);
  uint4* d4 = reinterpret_cast<uint4*>(first_al);
  for (uint64_t k = threadIdx.x; k < nvec; k += blockDim.x) d4[k] = s4[k];
  const uint64_t tail0 = last_al - a0;
  for (uint64_t k = tail0 + threadIdx.x; k < len; k += blockDim.x) dst[k] = stage[mis + k];
}

// stage[s0 + k] -> dst[k] for k < len, with a 16-B aligned stage and dst at
// any alignment: 16-B stores of words funnel-shifted out of the stage.
__device__ __forceinline__ void copy_out_shifted(uint8_t* dst, const uint8_t* stage, uint32_t s0, uint32_t len) {
  if (len == 0) return;
  const uint32_t mis = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(dst) & 15);
  const uint32_t head = min(len, (16u - mis) & 15u);
  for (uint32_t k = threadIdx.x; k < head; k += blockDim.x) dst[k] = stage[s0 + k];
  // whole 16-B stores whose five source words lie inside the staged bytes
  const uint32_t nvec = len >= head + 20 ? (len - head - 4) / 16 : 0;
  const uint32_t sb = s0 + head, sh = 8 * (sb & 3);
  const uint32_t* sw = reinterpret_cast<const uint32_t*>(stage) + (sb >> 2);
  uint4* d4 = reinterpret_cast<uint4*>(dst + head);
  for (uint32_t v = threadIdx.x; v < nvec; v += blockDim.x) {
    const uint32_t x0 = sw[4 * v], x1 = sw[4 * v + 1], x2 = sw[4 * v + 2], x3 = sw[4 * v + 3], x4 = sw[4 * v + 4];
    uint4 o;
    o.x = __funnelshift_r(x0, x1, sh);
    o.y = __funnelshift_r(x1, x2, sh);
    o.z = __funnelshift_r(x2, x3, sh);
    o.w = __funnelshift_r(x3, x4, sh);
    d4[v] = o;
  }
  for (uint32_t k = head + 16 * nvec + threadIdx.x; k < len; k += blockDim.x) dst[k] = stage[s0 + k];
}

// Little-endian scalar stores into a byte array (header fields).
__device__ __forceinline__ void st_le(uint8_t* p, uint64_t v, int nb) {
  for (int i = 0; i < nb; ++i) p[i] = static_cast<uint8_t>(v >> (8 * i));
}
__device__ __forceinline__ void st_be(uint8_t* p, uint64_t v, int nb) {
  for (int i = 0; i < nb; ++i) p[i] = static_cast<uint8_t>(v >> (8 * (nb - 1 - i)));
}
__device__ __forceinline__ uint64_t ld_le(const uint8_t* p, int nb) {
  uint64_t v = 0;
  for (int i = 0; i < nb; ++i) v |= static_cast<uint64_t>(p[i]) << (8 * i);
  return v;
}
__device__ __forceinline__ uint64_t ld_be(const uint8_t* p, int nb) {
  uint64_t v = 0;
  for (int i = 0; i < nb; ++i) v = (v << 8) | p[i];
  return v;
}

// Ascending bitonic sort of 32*K keys held in registers across one warp:
// element (r, lane) is position r*32 + lane.
template <int K>
__device__ __forceinline__ void warp_sort_regs(uint64_t (&v)[K]) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (uint32_t k = 2; k <= 32u * K; k <<= 1) {
#pragma unroll
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
#pragma unroll
        for (int r = 0; r < K; ++r) {
          const int r2 = r ^ static_cast<int>(j >> 5);
          if (r2 > r) {
            const uint32_t i = static_cast<uint32_t>(r) * 32 + lane;
            const bool up = (i & k) == 0;
            const uint64_t x = v[r], y = v[r2];
            if ((x > y) == up) {
              v[r] = y;
              v[r2] = x;
            }
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < K; ++r) {
          const uint32_t i = static_cast<uint32_t>(r) * 32 + lane;
          const uint64_t o = __shfl_xor_sync(0xffffffffu, v[r], j);
          const bool up = (i & k) == 0;
          const bool lower = (lane & j) == 0;  // this lane holds the smaller index of the pair
          // lower keeps min when ascending, max when descending; the upper the opposite
          const bool keep_min = (lower == up);
          v[r] = keep_min ? (v[r] < o ? v[r] : o) : (v[r] > o ? v[r] : o);
        }
      }
    }
  }
}

// Sort p2 (<= 256) keys of shared memory with one warp, through registers.
__device__ __forceinline__ void warp_sort_smem(uint64_t* key, uint32_t p2) {
  const uint32_t lane = threadIdx.x & 31;
  if (p2 <= 32) {
    uint64_t v[1] = {lane < p2 ? key[lane] : ~0ull};
    warp_sort_regs<1>(v);
    if (lane < p2) key[lane] = v[0];
  } else if (p2 <= 64) {
    uint64_t v[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) v[r] = key[r * 32 + lane];
    warp_sort_regs<2>(v);
#pragma unroll
    for (int r = 0; r < 2; ++r) key[r * 32 + lane] = v[r];
  } else if (p2 <= 128) {
    uint64_t v[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) v[r] = key[r * 32 + lane];
    warp_sort_regs<4>(v);
#pragma unroll
    for (int r = 0; r < 4; ++r) key[r * 32 + lane] = v[r];
  } else {
    uint64_t v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = key[r * 32 + lane];
    warp_sort_regs<8>(v);
#pragma unroll
    for (int r = 0; r < 8; ++r) key[r * 32 + lane] = v[r];
  }
  __syncwarp();
}

}  // namespace embc_dev
