// embc_b200.hpp -- header-only C++20 layer over the C ABI (embc_cuda.h) with
// the reference's names, types and exception classes (namespace embc,
// /root/reference/proj/include/embc/).  A reference caller swaps
//
//     #include "embc/embc.hpp"          ->  #include "embc_b200.hpp"
//     embc::encode_chunks(jobs, w)      ->  embc_b200::encode_chunks(ctx, jobs)
//     Simulator::rank_body's stages     ->  embc_b200::Exchange::fwd / bwd (NCCL)
//     embc::offline_analysis / eb_at    ->  embc_b200::offline_analysis / eb_at
//
// and keeps its exception handling: failures surface as embc_b200::ValueError /
// FormatError / ConfigError (subclasses of embc_b200::Error, std::runtime_error)
// carrying the reference's what() text.  Batches live in device memory
// (fp32 values, exactly representable in the reference's double batches).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
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

inline void throw_for(embc_status st, const embc_error& e) {
  const std::string msg(e.message);
  switch (st) {
    case EMBC_OK: return;
    case EMBC_ERR_VALUE: throw ValueError(msg);
    case EMBC_ERR_FORMAT: throw FormatError(msg);
    case EMBC_ERR_CONFIG: throw ConfigError(msg);
    case EMBC_ERR_UNSUPPORTED: throw UnsupportedError(msg);
    default: throw Error(msg.empty() ? "embc error " + std::to_string(st) : msg);
  }
}

// container.hpp:32-36
enum class Codec : uint8_t { raw = EMBC_CODEC_RAW, vlz = EMBC_CODEC_VLZ, huffman = EMBC_CODEC_HUFFMAN };

inline const char* codec_name(Codec c) {
  switch (c) {
    case Codec::raw: return "raw";
    case Codec::vlz: return "vlz";
    case Codec::huffman: return "huffman";
  }
  return "raw";
}

inline constexpr size_t kHeaderSize = 30;    // CompressedChunk::kHeaderSize
inline constexpr size_t kMetadataSize = 25;  // ChunkMetadata::kWireSize

// One embc_ctx per (device, host thread).  It also keeps a small device block
// for the per-call placement arrays, so the synchronous wrappers below do not
// allocate on every call.
class Context {
 public:
  explicit Context(int device = 0) {
    if (embc_ctx_create(device, &ctx_) != EMBC_OK) throw Error("embc_ctx_create failed");
  }
  ~Context() {
    if (aux_) cudaFree(aux_);
    embc_ctx_destroy(ctx_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  embc_ctx* get() const { return ctx_; }

  // Raises the failure recorded for `st` (or by the device, after a sync).
  void check(embc_status st) const {
    if (st == EMBC_OK) return;
    embc_error e{};
    embc_get_error(ctx_, &e);
    throw_for(st, e);
  }
  void sync(cudaStream_t s = nullptr) const { check(embc_sync(ctx_, s)); }

  // device u64 scratch of at least n entries (grown, never shrunk)
  uint64_t* aux(size_t n) {
    if (n > aux_n_) {
      if (aux_) cudaFree(aux_);
      aux_ = nullptr;
      aux_n_ = 0;
      if (cudaMalloc(&aux_, sizeof(uint64_t) * n) != cudaSuccess) throw Error("cudaMalloc failed");
      aux_n_ = n;
    }
    return aux_;
  }

 private:
  embc_ctx* ctx_ = nullptr;
  uint64_t* aux_ = nullptr;
  size_t aux_n_ = 0;
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
  uint64_t total = 0;             // bytes written to d_out
  std::vector<uint64_t> offsets;  // chunk placement (host copy)
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

// Asynchronous encode_chunks [+ pack] on `s`: no allocation, no host wait.
// Placement arrays, metadata records and the total stay on the device; data
// failures surface at the next ctx.sync(s).
inline void encode_chunks_async(Context& ctx, std::span<const EncodeJob> jobs, uint8_t* d_out, uint64_t cap,
                                bool packed, uint64_t* d_offsets, uint64_t* d_lengths, uint8_t* d_meta,
                                uint64_t* d_total, cudaStream_t s) {
  const auto cj = to_c(jobs);
  ctx.check(embc_encode(ctx.get(), cj.data(), static_cast<uint32_t>(cj.size()),
                        packed ? EMBC_LAYOUT_PACKED : EMBC_LAYOUT_CHUNKS, d_out, cap, d_offsets, d_lengths,
                        d_meta, d_total, s));
}

// encode_chunks(jobs) [+ pack()] (container.hpp:304-311, :242-256) into the
// device buffer d_out; d_meta (optional, 25 * jobs bytes, device) receives the
// serialize_metadata() records.  Synchronises `s` (the byte counts are read back).
inline EncodedChunks encode_chunks(Context& ctx, std::span<const EncodeJob> jobs, uint8_t* d_out,
                                   uint64_t cap, bool packed, uint8_t* d_meta = nullptr,
                                   cudaStream_t s = nullptr) {
  const size_t n = jobs.size();
  uint64_t* d = ctx.aux(2 * n + 1);
  encode_chunks_async(ctx, jobs, d_out, cap, packed, d, d + n, d_meta, d + 2 * n, s);
  const embc_status st = embc_sync(ctx.get(), s);
  std::vector<uint64_t> h(2 * n + 1);
  cudaMemcpy(h.data(), d, sizeof(uint64_t) * h.size(), cudaMemcpyDeviceToHost);
  ctx.check(st);
  EncodedChunks r;
  r.offsets.assign(h.begin(), h.begin() + n);
  r.lengths.assign(h.begin() + n, h.begin() + 2 * n);
  r.total = h[2 * n];
  return r;
}

// The reference's shape: encode_chunks(jobs) -> one serialized chunk per job,
// in job order (container.hpp:304-311 + serialize_chunk), as host bytes.
inline std::vector<std::vector<uint8_t>> encode_chunks(Context& ctx, std::span<const EncodeJob> jobs) {
  const uint64_t cap = encode_bound(jobs, false);
  uint8_t* d_out = nullptr;
  if (cudaMalloc(&d_out, cap ? cap : 1) != cudaSuccess) throw Error("cudaMalloc failed");
  std::vector<std::vector<uint8_t>> out;
  try {
    const EncodedChunks r = encode_chunks(ctx, jobs, d_out, cap, false);
    std::vector<uint8_t> all(r.total);
    cudaMemcpy(all.data(), d_out, r.total, cudaMemcpyDeviceToHost);
    for (size_t j = 0; j < jobs.size(); ++j)
      out.emplace_back(all.begin() + r.offsets[j], all.begin() + r.offsets[j] + r.lengths[j]);
  } catch (...) {
    cudaFree(d_out);
    throw;
  }
  cudaFree(d_out);
  return out;
}

// serialize_chunk(encode_chunk(batch, eb, codec, VlzConfig{window})) as host bytes.
inline std::vector<uint8_t> encode_chunk(Context& ctx, const EncodeJob& job) {
  const EncodeJob jobs[1] = {job};
  return std::move(encode_chunks(ctx, std::span<const EncodeJob>(jobs, 1))[0]);
}

// One chunk to decode (shape/codec from ChunkMetadata, container.hpp:186-194).
struct ChunkRef {
  uint64_t offset = 0, length = 0;
  float* d_out = nullptr;  // count * dim fp32
  uint32_t dim = 0, count = 0;
  Codec codec = Codec::raw;
};

// parse_chunk() + decode_chunk() (container.hpp:89-115, :146-181) of every ref
// in the device buffer d_in, into fp32 = float(reference double).  Asynchronous
// on `s` (failures at the next ctx.sync(s)).
inline void decode_chunks_async(Context& ctx, const uint8_t* d_in, std::span<const ChunkRef> refs, cudaStream_t s) {
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
}

// The same, synchronising `s`.
inline void decode_chunks(Context& ctx, const uint8_t* d_in, std::span<const ChunkRef> refs,
                          cudaStream_t s = nullptr) {
  decode_chunks_async(ctx, d_in, refs, s);
  ctx.sync(s);
}

// unpack() (container.hpp:258-292): the packed send buffer's table, validated;
// returns (offset, length) per entry.  Chunk bodies are parsed on the device
// by decode_chunks.
inline std::vector<std::pair<uint64_t, uint64_t>> unpack(std::span<const uint8_t> buf) {
  const uint32_t cap = static_cast<uint32_t>(buf.size() / 16 + 1);
  std::vector<uint64_t> offs(cap), lens(cap);
  uint32_t n = 0;
  embc_error e{};
  const embc_status st = embc_unpack(buf.data(), buf.size(), offs.data(), lens.data(), cap, &n, &e);
  throw_for(st, e);
  std::vector<std::pair<uint64_t, uint64_t>> out;
  for (uint32_t i = 0; i < n; ++i) out.emplace_back(offs[i], lens[i]);
  return out;
}

// ---- controller (policy.hpp) ---------------------------------------------

enum class TableClass { large = 0, medium = 1, small = 2 };

inline const char* table_class_name(TableClass c) {
  return c == TableClass::large ? "large" : c == TableClass::small ? "small" : "medium";
}

// policy.hpp:58-70
struct DecayConfig {
  enum class Fn { stepwise = 0, linear = 1, logarithmic = 2 };
  Fn function = Fn::stepwise;
  double start_scale = 1.0;
  uint64_t decay_end = 0;
  uint32_t step_count = 4;
};

// policy.hpp:75-103
struct PolicyConfig {
  double global_eb = 0.02;
  double alpha = 5.0 / 3.0;
  double beta = 3.0;
  double large_threshold = 0.70;
  double small_threshold = 0.95;
  DecayConfig decay;

  void validate() const {
    if (!(global_eb > 0.0 && std::isfinite(global_eb))) throw ConfigError("global_eb must be finite and > 0");
    if (!(alpha >= 1.0)) throw ConfigError("alpha must be >= 1");
    if (!(beta >= 1.0)) throw ConfigError("beta must be >= 1");
    if (!(0.0 < large_threshold && large_threshold < small_threshold && small_threshold <= 1.0))
      throw ConfigError("thresholds must satisfy 0 < large < small <= 1");
    if (!(decay.start_scale >= 1.0)) throw ConfigError("decay start_scale must be >= 1");
    if (decay.step_count < 1) throw ConfigError("decay step_count must be >= 1");
  }
  double eb_for(TableClass c) const {
    return c == TableClass::large ? global_eb * alpha : c == TableClass::small ? global_eb / beta : global_eb;
  }
};

// policy.hpp:107-125
struct ThroughputSample {
  Codec codec = Codec::raw;
  double comp_bps = 0.0;
  double decomp_bps = 0.0;
  double ratio = 1.0;
};

struct TableProfile {
  int32_t table_id = 0;
  uint64_t n_original_patterns = 0;
  uint64_t n_quantized_patterns = 0;
  double survival_ratio = 1.0;
  double homo_index = 0.0;
  TableClass cls = TableClass::medium;
  Codec codec = Codec::raw;
  double eb = 0.02;
  std::vector<ThroughputSample> measured;
};

// policy.hpp:127-137
inline double survival_ratio(uint64_t n_original, uint64_t n_quantized) {
  if (n_original == 0) throw ValueError("survival ratio needs a nonempty sample");
  return static_cast<double>(n_quantized) / static_cast<double>(n_original);
}
inline double homo_index(uint64_t n_original, uint64_t n_quantized) {
  return 1.0 - survival_ratio(n_original, n_quantized);
}

inline double decay_multiplier(uint64_t iteration, int fn, double start_scale, uint64_t decay_end,
                               uint32_t step_count) {
  double v = 1.0;
  if (embc_decay_multiplier(iteration, fn, start_scale, decay_end, step_count, &v) != EMBC_OK)
    throw ConfigError("invalid decay configuration");
  return v;
}
// policy.hpp:308-331
inline double decay_multiplier(uint64_t iteration, const DecayConfig& d) {
  if (!(d.start_scale >= 1.0)) throw ConfigError("decay start_scale must be >= 1");
  if (d.step_count < 1) throw ConfigError("decay step_count must be >= 1");
  return decay_multiplier(iteration, static_cast<int>(d.function), d.start_scale, d.decay_end, d.step_count);
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
// policy.hpp:188-193
inline TableClass classify_table(double survival, const PolicyConfig& cfg) {
  cfg.validate();
  return classify_table(survival, cfg.global_eb, cfg.alpha, cfg.beta, cfg.large_threshold, cfg.small_threshold);
}

inline double estimate_speedup(double ratio, double bandwidth, double comp_bps, double decomp_bps) {
  double v = 0.0;
  if (embc_estimate_speedup(ratio, bandwidth, comp_bps, decomp_bps, &v) != EMBC_OK)
    throw ValueError("estimate_speedup arguments must all be positive");
  return v;
}

// eb_at (policy.hpp:336-342): the profile's bound (global_eb without one) x the decay.
inline double eb_at(int32_t table_id, uint64_t iteration, const std::map<int32_t, TableProfile>& profiles,
                    const PolicyConfig& cfg) {
  const auto it = profiles.find(table_id);
  const double base = it != profiles.end() ? it->second.eb : cfg.global_eb;
  const double eb = base * decay_multiplier(iteration, cfg.decay);
  if (!(std::isfinite(eb) && eb > 0.0)) {
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%f", eb);
    throw ValueError(std::string("error bound must be finite and > 0, got ") + buf);
  }
  return eb;
}

// A device sample of one table for offline analysis: [rows, dim] fp32.
struct Sample {
  int32_t table_id = 0;
  const float* d_values = nullptr;
  uint32_t dim = 0;
  uint32_t rows = 0;
};

// select_codec (policy.hpp:239-274) with the GPU codecs: the Eq. 2 argmax
// (ties -> the lower tag), raw when even the best ratio is <= 1.  timed ==
// false prices the candidates by ratio alone (Eq. 2 as the bandwidth -> 0),
// which makes the choice deterministic; timed == true measures the median of
// five GPU runs of each codec, as the reference does with wall clock.
inline Codec select_codec(Context& ctx, const Sample& s, double eb, std::span<const Codec> candidates,
                          double bandwidth, uint32_t window, bool timed, std::vector<ThroughputSample>* measured) {
  if (candidates.empty()) throw ValueError("select_codec needs at least one candidate");
  const double unc = 4.0 * s.rows * s.dim;
  double best = -1.0, best_ratio = 0.0;
  Codec chosen = Codec::raw;
  for (const Codec c : candidates) {
    const EncodeJob job{s.d_values, s.dim, s.rows, eb, c, window};
    const EncodeJob jobs[1] = {job};
    const uint64_t cap = encode_bound(jobs, false);
    uint8_t* d_out = nullptr;
    float* d_dec = nullptr;
    if (cudaMalloc(&d_out, cap ? cap : 1) != cudaSuccess || cudaMalloc(&d_dec, 4ull * s.rows * s.dim + 4) != cudaSuccess)
      throw Error("cudaMalloc failed");
    ThroughputSample m;
    m.codec = c;
    try {
      const EncodedChunks r = encode_chunks(ctx, jobs, d_out, cap, false);
      m.ratio = unc / static_cast<double>(r.total - kHeaderSize);
      if (timed) {
        auto median = [&](auto&& fn) {
          double t[5];
          cudaEvent_t a, b;
          cudaEventCreate(&a);
          cudaEventCreate(&b);
          for (double& x : t) {
            cudaEventRecord(a);
            fn();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, a, b);
            x = std::max(1e-9, ms * 1e-3);
          }
          cudaEventDestroy(a);
          cudaEventDestroy(b);
          std::sort(t, t + 5);
          return t[2];
        };
        const ChunkRef ref{0, r.total, d_dec, s.dim, s.rows, c};
        m.comp_bps = unc / median([&] { encode_chunks_async(ctx, jobs, d_out, cap, false, nullptr, nullptr, nullptr, nullptr, nullptr); });
        m.decomp_bps = unc / median([&] { decode_chunks_async(ctx, d_out, std::span<const ChunkRef>(&ref, 1), nullptr); });
        ctx.sync();
      }
    } catch (...) {
      cudaFree(d_out);
      cudaFree(d_dec);
      throw;
    }
    cudaFree(d_out);
    cudaFree(d_dec);
    const double speedup = timed ? estimate_speedup(m.ratio, bandwidth, m.comp_bps, m.decomp_bps) : m.ratio;
    if (best < 0.0 || speedup > best || (speedup == best && c < chosen)) {
      best = speedup;
      best_ratio = m.ratio;
      chosen = c;
    }
    if (measured) measured->push_back(m);
  }
  return best_ratio <= 1.0 ? Codec::raw : chosen;
}

// offline_analysis (policy.hpp:278-302): pattern counts on the device
// (embc_pattern_counts), class bound, codec by select_codec at that bound.
inline std::map<int32_t, TableProfile> offline_analysis(Context& ctx, std::span<const Sample> samples,
                                                        const PolicyConfig& cfg, double bandwidth,
                                                        uint32_t window = 255, bool timed = false) {
  cfg.validate();
  std::map<int32_t, TableProfile> profiles;
  const Codec candidates[2] = {Codec::vlz, Codec::huffman};
  for (const Sample& s : samples) {
    TableProfile p;
    p.table_id = s.table_id;
    uint64_t o = 0, q = 0;
    ctx.check(embc_pattern_counts(ctx.get(), s.d_values, s.dim, s.rows, cfg.global_eb, &o, &q, nullptr));
    p.n_original_patterns = o;
    p.n_quantized_patterns = q;
    p.survival_ratio = survival_ratio(o, q);
    p.homo_index = homo_index(o, q);
    p.cls = classify_table(p.survival_ratio, cfg);
    p.eb = cfg.eb_for(p.cls);
    p.codec = select_codec(ctx, s, p.eb, candidates, bandwidth, window, timed, &p.measured);
    profiles[p.table_id] = p;
  }
  return profiles;
}

// detail::format_double (csv.hpp:31-37)
inline std::string format_double(double v) {
  char buf[32];
  const auto [ptr, ec] = std::to_chars(buf, buf + sizeof(buf), v);
  if (ec != std::errc()) throw Error("double formatting failed");
  return std::string(buf, ptr);
}

// write_profiles (config.hpp:247-271): the reference's key-value profile file.
inline void write_profiles(const std::string& path, const std::map<int32_t, TableProfile>& profiles) {
  std::string out = "profiles.count = " + std::to_string(profiles.size()) + "\n";
  size_t i = 0;
  for (const auto& [id, p] : profiles) {
    const std::string pre = "profile." + std::to_string(i) + ".";
    out += pre + "table = " + std::to_string(id) + "\n";
    out += pre + "n_original = " + std::to_string(p.n_original_patterns) + "\n";
    out += pre + "n_quantized = " + std::to_string(p.n_quantized_patterns) + "\n";
    out += pre + "survival = " + format_double(p.survival_ratio) + "\n";
    out += pre + "homo = " + format_double(p.homo_index) + "\n";
    out += pre + "class = " + table_class_name(p.cls) + "\n";
    out += pre + "codec = " + codec_name(p.codec) + "\n";
    out += pre + "eb = " + format_double(p.eb) + "\n";
    for (const auto& m : p.measured) {
      const std::string mp = pre + codec_name(m.codec) + ".";
      out += mp + "ratio = " + format_double(m.ratio) + "\n";
      out += mp + "comp_bps = " + format_double(m.comp_bps) + "\n";
      out += mp + "decomp_bps = " + format_double(m.decomp_bps) + "\n";
    }
    ++i;
  }
  std::ofstream f(path);
  if (!f) throw ConfigError("cannot write config file '" + path + "'");
  f << out;
}

// read_profiles (config.hpp:273-303), KeyValueConfig::parse_file semantics (:37-68).
inline std::map<int32_t, TableProfile> read_profiles(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw ConfigError("cannot open config file '" + path + "'");
  std::map<std::string, std::string> kv;
  std::string line;
  size_t lineno = 0;
  auto trim = [](const std::string& s) {
    const auto b = s.find_first_not_of(" \t\r");
    if (b == std::string::npos) return std::string();
    return s.substr(b, s.find_last_not_of(" \t\r") - b + 1);
  };
  while (std::getline(f, line)) {
    ++lineno;
    const std::string t = trim(line);
    if (t.empty() || t[0] == '#') continue;
    const size_t eq = t.find('=');
    if (eq == std::string::npos) throw ConfigError(path + ":" + std::to_string(lineno) + ": expected 'key = value'");
    const std::string k = trim(t.substr(0, eq));
    if (k.empty()) throw ConfigError(path + ":" + std::to_string(lineno) + ": empty key");
    kv[k] = trim(t.substr(eq + 1));
  }
  auto get = [&](const std::string& k) -> const std::string& {
    const auto it = kv.find(k);
    if (it == kv.end()) throw ConfigError("missing config key '" + k + "'");
    return it->second;
  };
  auto u64 = [&](const std::string& k) {
    const std::string& v = get(k);
    uint64_t out = 0;
    const auto [p, ec] = std::from_chars(v.data(), v.data() + v.size(), out);
    if (ec != std::errc() || p != v.data() + v.size())
      throw ConfigError("key '" + k + "' expects a non-negative integer, got '" + v + "'");
    return out;
  };
  auto f64 = [&](const std::string& k) {
    const std::string& v = get(k);
    double out = 0.0;
    const auto [p, ec] = std::from_chars(v.data(), v.data() + v.size(), out);
    if (ec != std::errc() || p != v.data() + v.size())
      throw ConfigError("key '" + k + "' expects a number, got '" + v + "'");
    return out;
  };
  std::map<int32_t, TableProfile> profiles;
  const uint64_t count = u64("profiles.count");
  for (uint64_t i = 0; i < count; ++i) {
    const std::string pre = "profile." + std::to_string(i) + ".";
    TableProfile p;
    p.table_id = static_cast<int32_t>(u64(pre + "table"));
    p.n_original_patterns = u64(pre + "n_original");
    p.n_quantized_patterns = u64(pre + "n_quantized");
    p.survival_ratio = f64(pre + "survival");
    p.homo_index = f64(pre + "homo");
    const std::string cls = get(pre + "class");
    if (cls == "large") p.cls = TableClass::large;
    else if (cls == "medium") p.cls = TableClass::medium;
    else if (cls == "small") p.cls = TableClass::small;
    else throw ConfigError("unknown table class '" + cls + "'");
    const std::string codec = get(pre + "codec");
    if (codec == "raw") p.codec = Codec::raw;
    else if (codec == "vlz") p.codec = Codec::vlz;
    else if (codec == "huffman") p.codec = Codec::huffman;
    else throw ConfigError("unknown codec '" + codec + "'");
    p.eb = f64(pre + "eb");
    for (const Codec c : {Codec::vlz, Codec::huffman}) {
      const std::string mp = pre + codec_name(c) + ".";
      if (!kv.count(mp + "ratio")) continue;
      ThroughputSample m;
      m.codec = c;
      m.ratio = f64(mp + "ratio");
      m.comp_bps = f64(mp + "comp_bps");
      m.decomp_bps = f64(mp + "decomp_bps");
      p.measured.push_back(m);
    }
    profiles[p.table_id] = p;
  }
  return profiles;
}

// ---- the compressed embedding all-to-all (commsim.hpp:286-435, over NCCL) --

using ExchangeStats = embc_exchange_stats;

// One per (process, GPU).  Rank 0 makes the id (unique_id()) and the caller
// shares it with the other ranks (MPI, a TCP store, torch.distributed, ...).
class Exchange {
 public:
  static std::vector<uint8_t> unique_id() {
    std::vector<uint8_t> id(128);
    const embc_status st = embc_exchange_unique_id(id.data());
    if (st != EMBC_OK) throw Error("embc_exchange_unique_id failed with status " + std::to_string(st));
    return id;
  }
  Exchange(int device, int rank, int nranks, std::span<const uint8_t> id, uint32_t groups = 1) {
    if (id.size() != 128) throw ValueError("exchange id must be 128 bytes");
    const embc_status st = embc_exchange_create(device, rank, nranks, id.data(), groups, &ex_);
    if (st != EMBC_OK) throw Error("embc_exchange_create failed with status " + std::to_string(st));
  }
  ~Exchange() { embc_exchange_destroy(ex_); }
  Exchange(const Exchange&) = delete;
  Exchange& operator=(const Exchange&) = delete;

  // Forward: d_lookups[t] = [R*batch, dim] for owned tables; d_outs[t] = [batch, dim] for all.
  ExchangeStats fwd(uint32_t dim, uint32_t batch, std::span<const float* const> d_lookups,
                    std::span<const double> ebs, std::span<const uint8_t> codecs, std::span<float* const> d_outs,
                    cudaStream_t s = nullptr, uint32_t window = 255) {
    ExchangeStats st{};
    check(embc_exchange_fwd(ex_, static_cast<uint32_t>(d_lookups.size()), dim, batch, d_lookups.data(), ebs.data(),
                            codecs.data(), window, d_outs.data(), &st, s));
    return st;
  }
  // Backward: d_grads[t] = [batch, dim] for all tables; d_outs[t] = [R*batch, dim] for owned.
  ExchangeStats bwd(uint32_t dim, uint32_t batch, std::span<const float* const> d_grads,
                    std::span<const double> ebs, std::span<const uint8_t> codecs, std::span<float* const> d_outs,
                    cudaStream_t s = nullptr, uint32_t window = 255) {
    ExchangeStats st{};
    check(embc_exchange_bwd(ex_, static_cast<uint32_t>(d_grads.size()), dim, batch, d_grads.data(), ebs.data(),
                            codecs.data(), window, d_outs.data(), &st, s));
    return st;
  }
  void baseline_fwd(uint32_t dim, uint32_t batch, std::span<const float* const> d_lookups,
                    std::span<float* const> d_outs, cudaStream_t s = nullptr) {
    check(embc_exchange_baseline_fwd(ex_, static_cast<uint32_t>(d_lookups.size()), dim, batch, d_lookups.data(),
                                     d_outs.data(), s));
  }
  void baseline_bwd(uint32_t dim, uint32_t batch, std::span<const float* const> d_grads,
                    std::span<float* const> d_outs, cudaStream_t s = nullptr) {
    check(embc_exchange_baseline_bwd(ex_, static_cast<uint32_t>(d_grads.size()), dim, batch, d_grads.data(),
                                     d_outs.data(), s));
  }

 private:
  void check(embc_status st) const {
    if (st == EMBC_OK) return;
    embc_error e{};
    embc_exchange_get_error(ex_, &e);
    throw_for(st, e);
  }
  embc_exchange* ex_ = nullptr;
};

}  // namespace embc_b200
