// embc_b200.hpp -- header-only C++20 wrapper over the C ABI (embc_cuda.h) with
// the reference's names, types and exception classes (namespace embc,
// /root/reference/proj/include/embc/).  A reference caller swaps
//
//     #include "embc/embc.hpp"          ->  #include "embc_b200.hpp"
//     embc::encode_chunks(jobs, w)      ->  embc_b200::encode_chunks(ctx, jobs, ...)
//
// and keeps its exception handling: failures surface as embc_b200::ValueError /
// FormatError / ConfigError (subclasses of embc_b200::Error, std::runtime_error)
// carrying the reference's what() text.  Batches live in device memory
// (fp32 values, exactly representable in the reference's double batches).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "embc_cuda.h"

namespace embc_b200 {

// errors.hpp:24-45
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};
class ValueError : public Error {
 public:
  explicit ValueError(const std::string& what) : Error(what) {}
};
class FormatError : public Error {
 public:
  explicit FormatError(const std::string& what) : Error(what) {}
};
class ConfigError : public Error {
 public:
  explicit ConfigError(const std::string& what) : Error(what) {}
};
class UnsupportedError : public Error {
 public:
  explicit UnsupportedError(const std::string& what) : Error(what) {}
};

// container.hpp:32-36
enum class Codec : uint8_t { raw = EMBC_CODEC_RAW, vlz = EMBC_CODEC_VLZ, huffman = EMBC_CODEC_HUFFMAN };

inline constexpr size_t kHeaderSize = 30;    // CompressedChunk::kHeaderSize
inline constexpr size_t kMetadataSize = 25;  // ChunkMetadata::kWireSize

// One embc_ctx per (device, host thread).
class Context {
 public:
  explicit Context(int device = 0) {
    if (embc_ctx_create(device, &ctx_) != EMBC_OK) throw Error("embc_ctx_create failed");
  }
  ~Context() { embc_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  embc_ctx* get() const { return ctx_; }

  // Raises the failure recorded for `st` (or by the device, after a sync).
  void check(embc_status st) const {
    if (st == EMBC_OK) return;
    embc_error e{};
    embc_get_error(ctx_, &e);
    const std::string msg(e.message);
    switch (st) {
      case EMBC_ERR_VALUE: throw ValueError(msg);
      case EMBC_ERR_FORMAT: throw FormatError(msg);
      case EMBC_ERR_CONFIG: throw ConfigError(msg);
      case EMBC_ERR_UNSUPPORTED: throw UnsupportedError(msg);
      default: throw Error(msg.empty() ? "embc error " + std::to_string(st) : msg);
    }
  }
  void sync(cudaStream_t s = nullptr) const { check(embc_sync(ctx_, s)); }

 private:
  embc_ctx* ctx_ = nullptr;
};

// EncodeJob (container.hpp:295-300) over a device batch.
struct EncodeJob {
  const float* d_values = nullptr;  // n * dim fp32, row-major, device
  uint32_t dim = 0;
  uint32_t n = 0;
  double eb = 0.0;
  Codec codec = Codec::raw;
  uint32_t window = 255;  // VlzConfig::window

  embc_job to_c() const {
    embc_job j{};
    j.src = d_values;
    j.dim = dim;
    j.n = n;
    j.eb = eb;
    j.window = window;
    j.codec = static_cast<uint8_t>(codec);
    j.src_kind = EMBC_SRC_F32;
    return j;
  }
};

struct EncodedChunks {
  uint64_t total = 0;                // bytes written to d_out
  std::vector<uint64_t> offsets;     // chunk placement (host copy)
  std::vector<uint64_t> lengths;
};

inline std::vector<embc_job> to_c(std::span<const EncodeJob> jobs) {
  std::vector<embc_job> v;
  v.reserve(jobs.size());
  for (const auto& j : jobs) v.push_back(j.to_c());
  return v;
}

// Worst-case output size of encode_chunks (container bound).
inline uint64_t encode_bound(std::span<const EncodeJob> jobs, bool packed) {
  const auto cj = to_c(jobs);
  return embc_encode_bound(cj.data(), static_cast<uint32_t>(cj.size()),
                           packed ? EMBC_LAYOUT_PACKED : EMBC_LAYOUT_CHUNKS);
}

// encode_chunks(jobs) [+ pack()] (container.hpp:304-311, :242-256) into the
// device buffer d_out; d_meta (optional, 25 * jobs bytes, device) receives the
// serialize_metadata() records.  Synchronises `s` (the byte counts are read back).
inline EncodedChunks encode_chunks(Context& ctx, std::span<const EncodeJob> jobs, uint8_t* d_out,
                                   uint64_t cap, bool packed, uint8_t* d_meta = nullptr,
                                   cudaStream_t s = nullptr) {
  const auto cj = to_c(jobs);
  EncodedChunks r;
  const size_t n = cj.size();
  uint64_t* d = nullptr;
  if (cudaMalloc(&d, sizeof(uint64_t) * (2 * n + 1)) != cudaSuccess) throw Error("cudaMalloc failed");
  const embc_status st = embc_encode(ctx.get(), cj.data(), static_cast<uint32_t>(n),
                                     packed ? EMBC_LAYOUT_PACKED : EMBC_LAYOUT_CHUNKS, d_out, cap, d,
                                     d + n, d_meta, d + 2 * n, s);
  if (st != EMBC_OK) {
    cudaFree(d);
    ctx.check(st);
  }
  const embc_status st2 = embc_sync(ctx.get(), s);
  std::vector<uint64_t> h(2 * n + 1);
  cudaMemcpy(h.data(), d, sizeof(uint64_t) * h.size(), cudaMemcpyDeviceToHost);
  cudaFree(d);
  ctx.check(st2);
  r.offsets.assign(h.begin(), h.begin() + n);
  r.lengths.assign(h.begin() + n, h.begin() + 2 * n);
  r.total = h[2 * n];
  return r;
}

// serialize_chunk(encode_chunk(batch, eb, codec, VlzConfig{window})) as host bytes.
inline std::vector<uint8_t> encode_chunk(Context& ctx, const EncodeJob& job) {
  const EncodeJob jobs[1] = {job};
  const uint64_t cap = encode_bound(jobs, false);
  uint8_t* d_out = nullptr;
  if (cudaMalloc(&d_out, cap ? cap : 1) != cudaSuccess) throw Error("cudaMalloc failed");
  EncodedChunks r;
  try {
    r = encode_chunks(ctx, jobs, d_out, cap, false);
  } catch (...) {
    cudaFree(d_out);
    throw;
  }
  std::vector<uint8_t> bytes(r.total);
  cudaMemcpy(bytes.data(), d_out, r.total, cudaMemcpyDeviceToHost);
  cudaFree(d_out);
  return bytes;
}

// One chunk to decode (shape/codec from ChunkMetadata, container.hpp:186-194).
struct ChunkRef {
  uint64_t offset = 0, length = 0;
  float* d_out = nullptr;  // count * dim fp32
  uint32_t dim = 0, count = 0;
  Codec codec = Codec::raw;
};

// parse_chunk() + decode_chunk() (container.hpp:89-115, :146-181) of every ref
// in the device buffer d_in, into fp32 = float(reference double).  Synchronises.
inline void decode_chunks(Context& ctx, const uint8_t* d_in, std::span<const ChunkRef> refs,
                          cudaStream_t s = nullptr) {
  std::vector<embc_chunk_ref> c(refs.size());
  for (size_t i = 0; i < refs.size(); ++i) {
    c[i].offset = refs[i].offset;
    c[i].length = refs[i].length;
    c[i].out = refs[i].d_out;
    c[i].dim = refs[i].dim;
    c[i].count = refs[i].count;
    c[i].codec = static_cast<uint8_t>(refs[i].codec);
  }
  ctx.check(embc_decode(ctx.get(), d_in, c.data(), static_cast<uint32_t>(c.size()), EMBC_OUT_F32, 0, s));
  ctx.sync(s);
}

// ---- controller arithmetic (policy.hpp) ---------------------------------

enum class TableClass { large = 0, medium = 1, small = 2 };

inline double decay_multiplier(uint64_t iteration, int fn, double start_scale, uint64_t decay_end,
                               uint32_t step_count) {
  double v = 1.0;
  if (embc_decay_multiplier(iteration, fn, start_scale, decay_end, step_count, &v) != EMBC_OK)
    throw ConfigError("invalid decay configuration");
  return v;
}

inline TableClass classify_table(double survival, double global_eb, double alpha, double beta,
                                 double large_thr, double small_thr, double* eb = nullptr) {
  int cls = 1;
  double e = 0.0;
  if (embc_classify_table(survival, global_eb, alpha, beta, large_thr, small_thr, &cls, &e) != EMBC_OK)
    throw ConfigError("invalid policy configuration");
  if (eb) *eb = e;
  return static_cast<TableClass>(cls);
}

inline double estimate_speedup(double ratio, double bandwidth, double comp_bps, double decomp_bps) {
  double v = 0.0;
  if (embc_estimate_speedup(ratio, bandwidth, comp_bps, decomp_bps, &v) != EMBC_OK)
    throw ValueError("estimate_speedup arguments must all be positive");
  return v;
}

}  // namespace embc_b200
