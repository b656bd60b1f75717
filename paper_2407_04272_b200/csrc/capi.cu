// capi.cu -- extern "C" boundary (include/embc_cuda.h): contexts, scratch,
// the device failure record and its translation into the reference's
// exception text, plus the small elementwise kernels (quantize/dequantize).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "embc_internal.h"

namespace embc_host {

uint64_t encode_bound(const embc_job* jobs, uint32_t njobs, int layout);
embc_status encode(embc_ctx* ctx, const embc_job* hj, uint32_t njobs, int layout, uint8_t* d_out,
                   uint64_t cap, uint64_t* d_offsets, uint64_t* d_lengths, uint8_t* d_meta,
                   uint64_t* d_total, cudaStream_t stream);
embc_status decode(embc_ctx* ctx, const uint8_t* d_in, const embc_chunk_ref* refs, uint32_t n,
                   int out_kind, int payload_only, cudaStream_t stream, const uint64_t* d_len = nullptr,
                   const uint64_t* d_off = nullptr);
embc_status match_stats(embc_ctx* ctx, const int32_t* d_codes, uint32_t dim, uint32_t n,
                        uint32_t window, uint64_t* h_lit, uint64_t* h_ref, cudaStream_t stream);
embc_status pattern_counts(embc_ctx* ctx, const float* d_x, uint32_t dim, uint32_t rows, double eb,
                           uint64_t* h_orig, uint64_t* h_quant, cudaStream_t stream);
cudaError_t encode_set_attributes();
cudaError_t decode_set_attributes();

std::string fmt_double(double v) {  // std::to_string(double) == "%f"
  char buf[512];
  std::snprintf(buf, sizeof(buf), "%f", v);
  return buf;
}

static std::string u(uint64_t v) { return std::to_string(v); }

std::string format_message(int reason, uint64_t index, uint64_t a, uint64_t b, double eb) {
  switch (reason) {
    case EMBC_R_NONFINITE: return "non-finite value at index " + u(index);
    case EMBC_R_OVERFLOW:
      return "quantization code overflow at index " + u(index) +
             ": error bound too small for value magnitude";
    case EMBC_R_EB_TOO_SMALL:
      return "error bound " + fmt_double(eb) + " too small to represent value at index " + u(index);
    case EMBC_R_BAD_WINDOW: return "vlz window must be in [1, 65536], got " + u(b);
    case EMBC_R_TRUNCATED:
      return "truncated input: need " + u(a) + " bytes at offset " + u(b) + ", have " + u(index);
    case EMBC_R_VARINT_LONG: return "varint too long at offset " + u(a);
    case EMBC_R_VLZ_DIM0: return "vlz stream with dim 0";
    case EMBC_R_VLZ_BAD_OFFSET:
      return "vlz reference offset " + u(a) + " invalid at token " + u(index);
    case EMBC_R_VLZ_BAD_TAG: return "vlz unknown token tag " + u(a) + " at token " + u(index);
    case EMBC_R_VLZ_TRAILING:
      return "vlz stream has " + u(a) + " trailing bytes after " + u(b) + " vectors";
    case EMBC_R_HUF_EMPTY: return "huffman encoder requires a nonempty sequence";
    case EMBC_R_HUF_LEN_CAP: return "huffman code length " + u(a) + " exceeds cap 32";
    case EMBC_R_HUF_EMPTY_BOOK: return "empty codebook";
    case EMBC_R_HUF_LEN_RANGE: return "codebook length " + u(a) + " out of range";
    case EMBC_R_HUF_KRAFT: return "codebook violates the Kraft inequality";
    case EMBC_R_HUF_PREFIX: return "codebook lengths do not form a prefix code";
    case EMBC_R_HUF_DUP: return "duplicate symbol in codebook";
    case EMBC_R_HUF_EXHAUSTED: return "bitstream exhausted at bit " + u(a);
    case EMBC_R_HUF_BAD_CODE: return "invalid huffman prefix at symbol " + u(index);
    case EMBC_R_BAD_MAGIC: return "bad chunk magic";
    case EMBC_R_BAD_VERSION: return "unsupported chunk version " + u(a);
    case EMBC_R_BAD_CODEC: return "unknown codec tag " + u(a);
    case EMBC_R_PAYLEN:
      return "chunk payload length " + u(a) + " does not match " + u(b) + " available bytes";
    case EMBC_R_BAD_EB: return "error bound must be finite and > 0, got " + fmt_double(eb);
    case EMBC_R_RAW_SIZE:
      return "raw payload of " + u(a) + " bytes does not hold " + u(b) + " codes";
    case EMBC_R_HUF_COUNT:
      return "huffman payload decoded " + u(a) + " symbols, expected " + u(b);
    case EMBC_R_DIM0: return "embedding batch dim must be >= 1";
    case EMBC_R_PACK_OFFSET:
      return "send buffer offset " + u(a) + " for entry " + u(index) +
             " overlaps or skips bytes (expected " + u(b) + ")";
    case EMBC_R_PACK_OVERRUN: return "send buffer entry " + u(index) + " runs past the end";
    case EMBC_R_PACK_TRAILING: return "send buffer has " + u(a) + " unclaimed trailing bytes";
    case EMBC_R_CAPACITY:
      return "encoded output of " + u(a) + " bytes exceeds the buffer capacity of " + u(b);
    case EMBC_R_META_MISMATCH: return "metadata disagrees with its chunk";
    case EMBC_R_RANGE:
      return "huffman alphabet span " + u(a) + " exceeds the GPU codebook limit of 131072 symbols";
    default: return "embc error";
  }
}

embc_status set_error(embc_ctx* ctx, embc_status st, int reason, uint32_t job, uint64_t index,
                      uint64_t a, uint64_t b, const std::string& msg) {
  embc_error& e = ctx->last;
  e.status = st;
  e.reason = reason;
  e.job = job;
  e.index = index;
  e.a = a;
  e.b = b;
  std::snprintf(e.message, sizeof(e.message), "%s", msg.c_str());
  return st;
}

embc_status cuda_fail(embc_ctx* ctx, cudaError_t e, const char* where) {
  return set_error(ctx, EMBC_ERR_CUDA, 0, 0, 0, static_cast<uint64_t>(e), 0,
                   std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e));
}

cudaError_t ensure_scratch(embc_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->scratch_cap) return cudaSuccess;
  size_t cap = std::max(bytes, ctx->scratch_cap * 2);
  cap = (cap + (1 << 20) - 1) & ~size_t((1 << 20) - 1);
  if (ctx->d_scratch) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return e;
    cudaFree(ctx->d_scratch);
    ctx->d_scratch = nullptr;
    ctx->scratch_cap = 0;
  }
  cudaError_t e = cudaMalloc(&ctx->d_scratch, cap);
  if (e == cudaSuccess) ctx->scratch_cap = cap;
  return e;
}

static bool capturing(cudaStream_t stream) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &st) != cudaSuccess) return false;
  return st != cudaStreamCaptureStatusNone;
}

cudaError_t stage_acquire(embc_ctx* ctx, size_t bytes, cudaStream_t stream, uint8_t** out, int* slot) {
  bytes = (bytes + 255) & ~size_t(255);
  if (capturing(stream)) {  // graph-owned descriptors: never reused until embc_capture_reset
    if (ctx->arena_used + bytes > ctx->arena_cap) return cudaErrorMemoryAllocation;
    *out = ctx->arena + ctx->arena_used;
    ctx->arena_used += bytes;
    *slot = -1;
    return cudaSuccess;
  }
  const int k = ctx->ring_next;
  ctx->ring_next = (k + 1) % embc_ctx::kRing;
  cudaError_t e;
  if (!ctx->ring_evt[k]) {
    e = cudaEventCreateWithFlags(&ctx->ring_evt[k], cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  } else {
    e = cudaEventSynchronize(ctx->ring_evt[k]);  // the previous upload from this slot is done
    if (e != cudaSuccess) return e;
  }
  if (bytes > ctx->ring_cap[k]) {
    if (ctx->ring[k]) cudaFreeHost(ctx->ring[k]);
    ctx->ring[k] = nullptr;
    ctx->ring_cap[k] = 0;
    const size_t cap = std::max<size_t>(bytes, 1 << 16);
    e = cudaMallocHost(&ctx->ring[k], cap);
    if (e != cudaSuccess) return e;
    ctx->ring_cap[k] = cap;
  }
  *out = ctx->ring[k];
  *slot = k;
  return cudaSuccess;
}

cudaError_t stage_commit(embc_ctx* ctx, int slot, cudaStream_t stream) {
  if (slot < 0) return cudaSuccess;
  return cudaEventRecord(ctx->ring_evt[slot], stream);
}

cudaError_t stage_upload(embc_ctx* ctx, void* dst, const uint8_t* hs, size_t bytes, int slot, cudaStream_t stream) {
  if (slot >= 0 || !ctx->darena || hs < ctx->arena || hs >= ctx->arena + ctx->arena_cap) {
    cudaError_t e = cudaMemcpyAsync(dst, hs, bytes, cudaMemcpyHostToDevice, stream);
    return e == cudaSuccess ? stage_commit(ctx, slot, stream) : e;
  }
  // capturing: the bytes go to the device mirror now, outside the graph (a
  // relaxed-mode window for the synchronous side-stream copy); the graph
  // copies device to device
  uint8_t* dm = ctx->darena + (hs - ctx->arena);
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  cudaError_t e = cudaThreadExchangeStreamCaptureMode(&mode);
  if (e != cudaSuccess) return e;
  if (!ctx->side) e = cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dm, hs, bytes, cudaMemcpyHostToDevice, ctx->side);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->side);
  cudaError_t e2 = cudaThreadExchangeStreamCaptureMode(&mode);
  if (e != cudaSuccess) return e;
  if (e2 != cudaSuccess) return e2;
  return cudaMemcpyAsync(dst, dm, bytes, cudaMemcpyDeviceToDevice, stream);
}

static cudaEvent_t pool_event(embc_ctx* ctx) {
  if (!ctx->ev_pool.empty()) {
    cudaEvent_t e = ctx->ev_pool.back();
    ctx->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

void tmark_begin(embc_ctx* ctx, const char* name, cudaStream_t stream) {
  if (!ctx->timing || capturing(stream)) return;
  cudaEvent_t a = pool_event(ctx), b = pool_event(ctx);
  cudaEventRecord(a, stream);
  ctx->tev.push_back({name, {a, b}});
}

void tmark_end(embc_ctx* ctx, cudaStream_t stream) {
  if (!ctx->timing || capturing(stream) || ctx->tev.empty()) return;
  cudaEventRecord(ctx->tev.back().second.second, stream);
}

cudaError_t ensure_hist(embc_ctx* ctx, size_t entries) {
  if (entries <= ctx->hist_cap) return cudaSuccess;
  if (ctx->d_hist) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return e;
    cudaFree(ctx->d_hist);
    ctx->d_hist = nullptr;
    ctx->hist_cap = 0;
  }
  cudaError_t e = cudaMalloc(&ctx->d_hist, entries * sizeof(uint32_t));
  if (e != cudaSuccess) return e;
  e = cudaMemset(ctx->d_hist, 0, entries * sizeof(uint32_t));  // kept zero by its consumers
  if (e == cudaSuccess) ctx->hist_cap = entries;
  return e;
}

}  // namespace embc_host

// ===========================================================================
// elementwise kernels
// ===========================================================================
namespace embc_dev {

__global__ void k_quantize(const void* __restrict__ x, int x_f64, uint64_t n, QParams qp,
                           int32_t* __restrict__ out, unsigned long long* __restrict__ err) {
  unsigned long long lerr = ~0ull;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint32_t reason = 0;
    int32_t c;
    if (x_f64) c = quantize_slow(static_cast<const double*>(x)[i], qp.eb, qp.w, &reason);
    else c = quantize_f32(static_cast<const float*>(x)[i], qp, &reason);
    if (reason) lerr = min(lerr, static_cast<unsigned long long>(err_key(i, reason)));
    out[i] = c;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long v = __shfl_xor_sync(0xffffffffu, lerr, o);
    lerr = v < lerr ? v : lerr;
  }
  if ((threadIdx.x & 31) == 0 && lerr != ~0ull) atomicMin(err, lerr);
}

__global__ void k_dequantize(const int32_t* __restrict__ c, uint64_t n, double w, void* out,
                             int out_f64) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const double v = reconstruct(c[i], w);
    if (out_f64) static_cast<double*>(out)[i] = v;
    else static_cast<float*>(out)[i] = __double2float_rn(v);
  }
}

__global__ void k_fold_key(const unsigned long long* __restrict__ key, DevError* err, double eb,
                           int32_t status) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const unsigned long long k = *key;
  if (k == ~0ull || err->valid) return;
  err->valid = 1;
  err->job = 0;
  err->reason = static_cast<int32_t>(k & 63);
  err->index = k >> 6;
  err->a = err->b = 0;
  err->eb = eb;
  err->status = status;
}

__global__ void k_gather_rows(const float* __restrict__ table, uint32_t dim,
                              const uint32_t* __restrict__ idx, uint32_t batch,
                              float* __restrict__ out) {
  const uint64_t total = static_cast<uint64_t>(dim) * batch;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = i / dim, j = i - r * dim;
    out[i] = table[static_cast<uint64_t>(idx[r]) * dim + j];
  }
}

}  // namespace embc_dev

// ===========================================================================
// extern "C"
// ===========================================================================
using namespace embc_host;
using embc_dev::DevError;
using embc_dev::QParams;

static std::once_flag g_attr_once;
static cudaError_t g_attr_err = cudaSuccess;

static inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

extern "C" {

const char* embc_version(void) { return "embc_cuda 1 sm_100a"; }

embc_status embc_ctx_create(int device, embc_ctx** out) {
  if (!out) return EMBC_ERR_ARGUMENT;
  *out = nullptr;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return EMBC_ERR_CUDA;
  std::call_once(g_attr_once, [] {
    g_attr_err = encode_set_attributes();
    if (g_attr_err == cudaSuccess) g_attr_err = decode_set_attributes();
  });
  if (g_attr_err != cudaSuccess) return EMBC_ERR_CUDA;
  embc_ctx* ctx = new embc_ctx();
  ctx->device = device;
  if (cudaMalloc(&ctx->d_err, sizeof(DevError)) != cudaSuccess ||
      cudaMemset(ctx->d_err, 0, sizeof(DevError)) != cudaSuccess ||
      cudaMallocHost(&ctx->h_err, sizeof(DevError)) != cudaSuccess ||
      cudaMalloc(&ctx->d_diag, 16) != cudaSuccess || cudaMemset(ctx->d_diag, 0, 16) != cudaSuccess) {
    embc_ctx_destroy(ctx);
    return EMBC_ERR_CUDA;
  }
  *out = ctx;
  return EMBC_OK;
}

void embc_ctx_destroy(embc_ctx* ctx) {
  if (!ctx) return;
  cudaDeviceSynchronize();
  if (ctx->d_err) cudaFree(ctx->d_err);
  if (ctx->d_diag) cudaFree(ctx->d_diag);
  if (ctx->h_err) cudaFreeHost(ctx->h_err);
  if (ctx->d_scratch) cudaFree(ctx->d_scratch);
  for (int k = 0; k < embc_ctx::kRing; ++k) {
    if (ctx->ring[k]) cudaFreeHost(ctx->ring[k]);
    if (ctx->ring_evt[k]) cudaEventDestroy(ctx->ring_evt[k]);
  }
  if (ctx->arena) cudaFreeHost(ctx->arena);
  if (ctx->darena) cudaFree(ctx->darena);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  for (auto& t : ctx->tev) {
    cudaEventDestroy(t.second.first);
    cudaEventDestroy(t.second.second);
  }
  for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->d_hist) cudaFree(ctx->d_hist);
  delete ctx;
}

embc_status embc_reserve(embc_ctx* ctx, uint32_t max_jobs, uint64_t max_values,
                         uint64_t max_payload_bytes) {
  if (!ctx) return EMBC_ERR_ARGUMENT;
  // generous bound of the encode carve (descriptors + per-row/per-tile arrays)
  const size_t bytes = static_cast<size_t>(max_jobs) * 512 + static_cast<size_t>(max_values) * 8 +
                       static_cast<size_t>(max_payload_bytes) + (64u << 20);
  cudaError_t e = ensure_scratch(ctx, bytes);
  if (e == cudaSuccess) e = ensure_hist(ctx, std::max<size_t>(embc_dev::kHistCap, static_cast<size_t>(max_jobs) * 8192));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "embc_reserve");
  return EMBC_OK;
}

embc_status embc_sync(embc_ctx* ctx, void* stream) {
  if (!ctx) return EMBC_ERR_ARGUMENT;
  cudaError_t e = cudaStreamSynchronize(S(stream));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "embc_sync");
  e = cudaMemcpy(ctx->h_err, ctx->d_err, sizeof(DevError), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "embc_sync error readback");
  const DevError r = *ctx->h_err;
  if (!r.valid) return EMBC_OK;
  cudaMemset(ctx->d_err, 0, sizeof(DevError));
  return set_error(ctx, static_cast<embc_status>(r.status), r.reason, r.job, r.index, r.a, r.b,
                   format_message(r.reason, r.index, r.a, r.b, r.eb));
}

embc_status embc_get_error(const embc_ctx* ctx, embc_error* out) {
  if (!ctx || !out) return EMBC_ERR_ARGUMENT;
  *out = ctx->last;
  return EMBC_OK;
}

uint64_t embc_encode_bound(const embc_job* h_jobs, uint32_t njobs, int layout) {
  if (!h_jobs && njobs) return 0;
  return encode_bound(h_jobs, njobs, layout);
}

embc_status embc_encode(embc_ctx* ctx, const embc_job* h_jobs, uint32_t njobs, int layout,
                        uint8_t* d_out, uint64_t cap, uint64_t* d_offsets, uint64_t* d_lengths,
                        uint8_t* d_meta, uint64_t* d_total, void* stream) {
  if (!ctx || (!h_jobs && njobs) || (!d_out && cap) || layout < 0 || layout > 2)
    return ctx ? set_error(ctx, EMBC_ERR_ARGUMENT, 0, 0, 0, 0, 0, "invalid embc_encode arguments")
               : EMBC_ERR_ARGUMENT;
  return encode(ctx, h_jobs, njobs, layout, d_out, cap, d_offsets, d_lengths, d_meta, d_total,
                S(stream));
}

embc_status embc_decode(embc_ctx* ctx, const uint8_t* d_in, const embc_chunk_ref* h_refs,
                        uint32_t nrefs, int out_kind, int payload_only, void* stream) {
  if (!ctx || (!h_refs && nrefs) || out_kind < 0 || out_kind > 2)
    return ctx ? set_error(ctx, EMBC_ERR_ARGUMENT, 0, 0, 0, 0, 0, "invalid embc_decode arguments")
               : EMBC_ERR_ARGUMENT;
  return decode(ctx, d_in, h_refs, nrefs, out_kind, payload_only, S(stream));
}

embc_status embc_decode_dev(embc_ctx* ctx, const uint8_t* d_in, const embc_chunk_ref* h_refs, uint32_t nrefs,
                            const uint64_t* d_off, const uint64_t* d_len, int out_kind, int payload_only,
                            void* stream) {
  if (!ctx || (!h_refs && nrefs) || (!d_len && nrefs) || out_kind < 0 || out_kind > 2)
    return ctx ? set_error(ctx, EMBC_ERR_ARGUMENT, 0, 0, 0, 0, 0, "invalid embc_decode_dev arguments")
               : EMBC_ERR_ARGUMENT;
  return decode(ctx, d_in, h_refs, nrefs, out_kind, payload_only, S(stream), d_len, d_off);
}

embc_status embc_quantize(embc_ctx* ctx, const void* d_x, int x_f64, uint64_t n, double eb,
                          int32_t* d_codes, void* stream) {
  if (!ctx || ((!d_x || !d_codes) && n)) return EMBC_ERR_ARGUMENT;
  if (!(std::isfinite(eb) && eb > 0.0))
    return set_error(ctx, EMBC_ERR_VALUE, EMBC_R_BAD_EB, 0, 0, 0, 0,
                     "error bound must be finite and > 0, got " + fmt_double(eb));
  cudaError_t e = ensure_scratch(ctx, 64);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "scratch");
  auto* key = reinterpret_cast<unsigned long long*>(ctx->d_scratch);
  cudaMemsetAsync(key, 0xFF, 8, S(stream));
  QParams qp;
  qp.eb = eb;
  qp.w = 2.0 * eb;
  const double rw = 1.0 / qp.w;
  qp.rw = static_cast<float>(rw);
  qp.fast = (rw >= 0x1.0p-100 && rw <= 0x1.0p100) ? 1 : 0;
  if (n) {
    const uint32_t blocks = static_cast<uint32_t>(std::min<uint64_t>((n + 255) / 256, 148 * 16));
    embc_dev::k_quantize<<<blocks, 256, 0, S(stream)>>>(d_x, x_f64, n, qp, d_codes, key);
  }
  embc_dev::k_fold_key<<<1, 32, 0, S(stream)>>>(key, ctx->d_err, eb, EMBC_ERR_VALUE);
  e = cudaGetLastError();
  return e == cudaSuccess ? EMBC_OK : cuda_fail(ctx, e, "embc_quantize");
}

embc_status embc_dequantize(embc_ctx* ctx, const int32_t* d_codes, uint64_t n, double eb,
                            void* d_out, int out_f64, void* stream) {
  if (!ctx || ((!d_codes || !d_out) && n)) return EMBC_ERR_ARGUMENT;
  if (!(std::isfinite(eb) && eb > 0.0))
    return set_error(ctx, EMBC_ERR_VALUE, EMBC_R_BAD_EB, 0, 0, 0, 0,
                     "error bound must be finite and > 0, got " + fmt_double(eb));
  if (n) {
    const uint32_t blocks = static_cast<uint32_t>(std::min<uint64_t>((n + 255) / 256, 148 * 16));
    embc_dev::k_dequantize<<<blocks, 256, 0, S(stream)>>>(d_codes, n, 2.0 * eb, d_out, out_f64);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? EMBC_OK : cuda_fail(ctx, e, "embc_dequantize");
}

embc_status embc_match_stats(embc_ctx* ctx, const int32_t* d_codes, uint32_t dim, uint32_t n,
                             uint32_t window, uint64_t* h_literals, uint64_t* h_references,
                             void* stream) {
  if (!ctx || !h_literals || !h_references) return EMBC_ERR_ARGUMENT;
  return match_stats(ctx, d_codes, dim, n, window, h_literals, h_references, S(stream));
}

embc_status embc_pattern_counts(embc_ctx* ctx, const float* d_x, uint32_t dim, uint32_t rows,
                                double eb, uint64_t* h_original, uint64_t* h_quantized,
                                void* stream) {
  if (!ctx || !h_original || !h_quantized) return EMBC_ERR_ARGUMENT;
  return pattern_counts(ctx, d_x, dim, rows, eb, h_original, h_quantized, S(stream));
}

embc_status embc_gather_rows(const float* d_table, uint32_t dim, const uint32_t* d_idx,
                             uint32_t batch, float* d_out, void* stream) {
  if ((!d_table || !d_idx || !d_out) && batch) return EMBC_ERR_ARGUMENT;
  const uint64_t total = static_cast<uint64_t>(dim) * batch;
  if (total) {
    const uint32_t blocks = static_cast<uint32_t>(std::min<uint64_t>((total + 255) / 256, 148 * 16));
    embc_dev::k_gather_rows<<<blocks, 256, 0, S(stream)>>>(d_table, dim, d_idx, batch, d_out);
  }
  return cudaGetLastError() == cudaSuccess ? EMBC_OK : EMBC_ERR_CUDA;
}

embc_status embc_reserve_capture(embc_ctx* ctx, uint64_t bytes) {
  if (!ctx) return EMBC_ERR_ARGUMENT;
  if (bytes <= ctx->arena_cap) return EMBC_OK;
  if (ctx->arena) {
    cudaDeviceSynchronize();
    cudaFreeHost(ctx->arena);
    cudaFree(ctx->darena);
    ctx->arena = ctx->darena = nullptr;
    ctx->arena_cap = ctx->arena_used = 0;
  }
  cudaError_t e = cudaMallocHost(&ctx->arena, bytes);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->darena, bytes);
  if (e != cudaSuccess) {
    if (ctx->arena) cudaFreeHost(ctx->arena);
    ctx->arena = nullptr;
    return cuda_fail(ctx, e, "embc_reserve_capture");
  }
  ctx->arena_cap = bytes;
  return EMBC_OK;
}

embc_status embc_decode_fallbacks(embc_ctx* ctx, uint32_t* h_count) {
  if (!ctx || !h_count) return EMBC_ERR_ARGUMENT;
  cudaError_t e = cudaMemcpy(h_count, ctx->d_diag, sizeof(uint32_t), cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? EMBC_OK : cuda_fail(ctx, e, "embc_decode_fallbacks");
}

embc_status embc_capture_reset(embc_ctx* ctx) {
  if (!ctx) return EMBC_ERR_ARGUMENT;
  ctx->arena_used = 0;
  return EMBC_OK;
}

embc_status embc_timing_enable(embc_ctx* ctx, int on) {
  if (!ctx) return EMBC_ERR_ARGUMENT;
  ctx->timing = on != 0;
  return EMBC_OK;
}

int embc_timing_collect(embc_ctx* ctx, void* stream, char* names, size_t names_cap, float* ms,
                        int max_entries) {
  if (!ctx) return -1;
  if (cudaStreamSynchronize(S(stream)) != cudaSuccess) return -1;
  int n = 0;
  size_t used = 0;
  for (auto& t : ctx->tev) {
    float v = 0.f;
    cudaEventElapsedTime(&v, t.second.first, t.second.second);
    if (n < max_entries && names && used + t.first.size() + 1 <= names_cap) {
      std::memcpy(names + used, t.first.c_str(), t.first.size() + 1);
      used += t.first.size() + 1;
      if (ms) ms[n] = v;
      ++n;
    }
    ctx->ev_pool.push_back(t.second.first);
    ctx->ev_pool.push_back(t.second.second);
  }
  ctx->tev.clear();
  return n;
}

}  // extern "C"
