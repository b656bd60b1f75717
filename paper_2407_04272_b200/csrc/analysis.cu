// analysis.cu -- embedding-vector analysis for the table-wise controller:
// distinct value rows and distinct quantization-code rows of a sample
// (detail::count_unique_rows / pattern_counts, policy.hpp:141-173).
//
// Rows are hashed, (hash, row) keys are sorted on the device, and each run of
// equal hashes is resolved by exact row comparison, so the counts are exact.
// Values compare with double operator< semantics (the reference's
// lexicographical_compare), i.e. -0.0 == +0.0.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>

#include "embc_internal.h"

namespace embc_dev {

__global__ void k_pc_quantize_hash(const float* __restrict__ x, uint32_t dim, uint32_t rows,
                                   QParams qp, int32_t* __restrict__ codes,
                                   uint64_t* __restrict__ kv, uint64_t* __restrict__ kc,
                                   unsigned long long* __restrict__ err) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long lerr = ~0ull;
  if (r < rows) {
    uint64_t hv = 0xCBF29CE484222325ull, hc = 0x84222325CBF29CE4ull;
    for (uint32_t j = 0; j < dim; ++j) {
      const uint64_t e = static_cast<uint64_t>(r) * dim + j;
      const float v = x[e];
      uint32_t reason = 0;
      const int32_t c = quantize_f32(v, qp, &reason);
      if (reason) lerr = min(lerr, static_cast<unsigned long long>(err_key(e, reason)));
      codes[e] = c;
      const uint32_t vb = v == 0.0f ? 0u : __float_as_uint(v);  // -0.0 == +0.0
      hv = (hv ^ vb) * 0x100000001B3ull;
      hc = (hc ^ static_cast<uint32_t>(c)) * 0x100000001B3ull;
    }
    hv ^= hv >> 31;
    hc ^= hc >> 31;
    kv[r] = (hv & ~0xFFFFFFull) | r;  // rows < 2^24
    kc[r] = (hc & ~0xFFFFFFull) | r;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long v = __shfl_xor_sync(0xffffffffu, lerr, o);
    lerr = v < lerr ? v : lerr;
  }
  if ((threadIdx.x & 31) == 0 && lerr != ~0ull) atomicMin(err, lerr);
}

__global__ void __launch_bounds__(1024) k_pc_sort(uint64_t* __restrict__ kv, uint64_t* __restrict__ kc,
                                                  uint32_t p2) {
  uint64_t* key = blockIdx.x == 0 ? kv : kc;
  for (uint32_t k = 2; k <= p2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < p2; i += blockDim.x) {
        const uint32_t ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = key[i], b = key[ixj];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            key[i] = b;
            key[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

// A sorted position starts a new class unless an earlier row of its hash run
// has identical content.
__global__ void k_pc_count(const float* __restrict__ x, const int32_t* __restrict__ codes,
                           uint32_t dim, uint32_t rows, const uint64_t* __restrict__ kv,
                           const uint64_t* __restrict__ kc, unsigned long long* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool codes_pass = blockIdx.y == 1;
  const uint64_t* key = codes_pass ? kc : kv;
  bool fresh = false;
  if (i < rows) {
    const uint64_t hi = key[i] >> 24;
    fresh = true;
    if (i > 0 && (key[i - 1] >> 24) == hi) {
      uint32_t j = i;
      while (j > 0 && (key[j - 1] >> 24) == hi) --j;  // run start
      const uint32_t ri = static_cast<uint32_t>(key[i] & 0xFFFFFF);
      for (; j < i && fresh; ++j) {
        const uint32_t rj = static_cast<uint32_t>(key[j] & 0xFFFFFF);
        bool eq = true;
        for (uint32_t d = 0; d < dim && eq; ++d) {
          const uint64_t a = static_cast<uint64_t>(ri) * dim + d, b = static_cast<uint64_t>(rj) * dim + d;
          eq = codes_pass ? codes[a] == codes[b]
                          : static_cast<double>(x[a]) == static_cast<double>(x[b]);
        }
        if (eq) fresh = false;
      }
    }
  }
  const uint32_t n = __popc(__ballot_sync(0xffffffffu, fresh));
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(&out[codes_pass ? 1 : 0], n);
}

}  // namespace embc_dev

namespace embc_host {

using namespace embc_dev;

embc_status pattern_counts(embc_ctx* ctx, const float* d_x, uint32_t dim, uint32_t rows, double eb,
                           uint64_t* h_orig, uint64_t* h_quant, cudaStream_t stream) {
  if (dim == 0)
    return set_error(ctx, EMBC_ERR_VALUE, EMBC_R_DIM0, 0, 0, 0, 0, "embedding batch dim must be >= 1");
  if (rows == 0)
    return set_error(ctx, EMBC_ERR_VALUE, 0, 0, 0, 0, 0, "survival ratio needs a nonempty sample");
  if (!(std::isfinite(eb) && eb > 0.0))
    return set_error(ctx, EMBC_ERR_VALUE, EMBC_R_BAD_EB, 0, 0, 0, 0,
                     "error bound must be finite and > 0, got " + fmt_double(eb));
  if (rows >= (1u << 24))
    return set_error(ctx, EMBC_ERR_UNSUPPORTED, 0, 0, 0, 0, 0, "pattern_counts sample of >= 2^24 rows");
  uint32_t p2 = 1;
  while (p2 < rows) p2 <<= 1;
  const size_t n = static_cast<size_t>(dim) * rows;
  const size_t o_codes = 0;
  const size_t o_kv = (o_codes + 4 * n + 15) & ~size_t(15);
  const size_t o_kc = o_kv + 8 * static_cast<size_t>(p2);
  const size_t o_err = o_kc + 8 * static_cast<size_t>(p2);
  const size_t total = o_err + 32;
  cudaError_t ce = ensure_scratch(ctx, total);
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "pattern_counts scratch");
  uint8_t* d = ctx->d_scratch;
  int32_t* codes = reinterpret_cast<int32_t*>(d + o_codes);
  uint64_t* kv = reinterpret_cast<uint64_t*>(d + o_kv);
  uint64_t* kc = reinterpret_cast<uint64_t*>(d + o_kc);
  unsigned long long* err = reinterpret_cast<unsigned long long*>(d + o_err);
  cudaMemsetAsync(kv, 0xFF, 16 * static_cast<size_t>(p2), stream);
  cudaMemsetAsync(err, 0xFF, 8, stream);
  cudaMemsetAsync(err + 1, 0, 16, stream);
  QParams qp;
  qp.eb = eb;
  qp.w = 2.0 * eb;
  const double rw = 1.0 / qp.w;
  qp.rw = static_cast<float>(rw);
  qp.fast = (rw >= 0x1.0p-100 && rw <= 0x1.0p100) ? 1 : 0;
  k_pc_quantize_hash<<<(rows + 127) / 128, 128, 0, stream>>>(d_x, dim, rows, qp, codes, kv, kc, err);
  k_pc_sort<<<2, 1024, 0, stream>>>(kv, kc, p2);
  k_pc_count<<<dim3((rows + 255) / 256, 2), 256, 0, stream>>>(d_x, codes, dim, rows, kv, kc, err + 1);
  unsigned long long h[3];
  ce = cudaMemcpyAsync(h, err, 24, cudaMemcpyDeviceToHost, stream);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(stream);
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "pattern_counts");
  if (h[0] != ~0ull) {  // quantize() throws first (policy.hpp:170)
    const int reason = static_cast<int>(h[0] & 63);
    return set_error(ctx, EMBC_ERR_VALUE, reason, 0, h[0] >> 6, 0, 0,
                     format_message(reason, h[0] >> 6, 0, 0, eb));
  }
  *h_orig = h[1];
  *h_quant = h[2];
  return EMBC_OK;
}

}  // namespace embc_host
