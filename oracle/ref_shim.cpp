// ref_shim.cpp -- C entry points over the UNMODIFIED reference headers
// (/root/reference/proj/include, included at build time, never copied).
// Built by oracle/Makefile into oracle/_ref/libembc_ref.so (git-ignored, it
// travels to the GPU box inside the gpurun snapshot).  Test infrastructure
// only: tests/, smoke() and bench.py's cpu_baseline / --impl reference leg.
//
// Status codes: 0 ok, 1 embc::ValueError, 2 embc::FormatError, 3 other embc::Error,
// 4 a std::exception escaping the reference (e.g. vector::reserve on a corrupt count).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <span>
#include <string>
#include <vector>

#include "embc/embc.hpp"

namespace {

int fail(const std::exception& e, int code, char* err, size_t cap) {
  if (err && cap) {
    std::strncpy(err, e.what(), cap - 1);
    err[cap - 1] = 0;
  }
  return code;
}

#define GUARD(...)                                           \
  try {                                                      \
    __VA_ARGS__;                                             \
  } catch (const embc::ValueError& e) {                      \
    return fail(e, 1, err, errcap);                          \
  } catch (const embc::FormatError& e) {                     \
    return fail(e, 2, err, errcap);                          \
  } catch (const embc::Error& e) {                           \
    return fail(e, 3, err, errcap);                          \
  } catch (const std::exception& e) {                        \
    return fail(e, 4, err, errcap);                          \
  }                                                          \
  return 0;

template <typename T>
T* dup(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.size() ? v.size() : 1)));
  if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
  return p;
}

embc::TableSpec make_spec(int32_t id, uint32_t rows, uint32_t dim, int dist, double mu, double sigma,
                          double lo, double hi, double zipf, uint64_t seed) {
  embc::TableSpec s;
  s.table_id = id;
  s.rows = rows;
  s.dim = dim;
  s.dist = dist == 0 ? embc::ValueDist::gaussian : embc::ValueDist::uniform;
  s.mu = mu;
  s.sigma = sigma;
  s.lo = lo;
  s.hi = hi;
  s.zipf_s = zipf;
  s.seed = seed;
  return s;
}

}  // namespace

extern "C" {

void ref_free(void* p) { std::free(p); }

int ref_quantize(const double* x, uint64_t n, uint32_t dim, double eb, int32_t* codes, char* err,
                 size_t errcap) {
  GUARD({
    embc::EmbeddingBatch b{0, dim, std::vector<double>(x, x + n)};
    const embc::QuantizedBatch q = embc::quantize(b, embc::ErrorBound(eb));
    std::memcpy(codes, q.codes.data(), sizeof(int32_t) * n);
  })
}

int ref_dequantize(const int32_t* codes, uint64_t n, uint32_t dim, double eb, double* out,
                   char* err, size_t errcap) {
  GUARD({
    embc::QuantizedBatch q{0, dim, std::vector<int32_t>(codes, codes + n), embc::ErrorBound(eb)};
    const embc::EmbeddingBatch b = embc::dequantize(q);
    std::memcpy(out, b.values.data(), sizeof(double) * n);
  })
}

int ref_encode_chunk(const double* x, uint32_t dim, uint32_t n, double eb, int codec,
                     uint32_t window, uint8_t** out, uint64_t* len, char* err, size_t errcap) {
  GUARD({
    embc::EmbeddingBatch b{0, dim, std::vector<double>(x, x + static_cast<size_t>(dim) * n)};
    const embc::CompressedChunk c = embc::encode_chunk(
        b, embc::ErrorBound(eb), static_cast<embc::Codec>(codec), embc::VlzConfig{window});
    const std::vector<uint8_t> s = embc::serialize_chunk(c);
    *out = dup(s);
    *len = s.size();
  })
}

int ref_decode_chunk(const uint8_t* in, uint64_t len, double** out, uint64_t* nvals, uint32_t* dim,
                     uint32_t* count, char* err, size_t errcap) {
  GUARD({
    const embc::CompressedChunk c = embc::parse_chunk(std::span<const uint8_t>(in, len));
    const embc::EmbeddingBatch b = embc::decode_chunk(c);
    *out = dup(b.values);
    *nvals = b.values.size();
    *dim = c.dim;
    *count = c.vector_count;
  })
}

int ref_vlz_encode(const int32_t* codes, uint32_t dim, uint32_t n, uint32_t window, uint8_t** out,
                   uint64_t* len, char* err, size_t errcap) {
  GUARD({
    embc::QuantizedBatch q{0, dim, std::vector<int32_t>(codes, codes + static_cast<size_t>(dim) * n),
                           embc::ErrorBound(0.01)};
    const embc::VlzStream s = embc::vlz_encode(q, embc::VlzConfig{window});
    *out = dup(s.tokens);
    *len = s.tokens.size();
  })
}

int ref_vlz_decode(const uint8_t* in, uint64_t len, uint32_t dim, uint32_t n, int32_t* out,
                   char* err, size_t errcap) {
  GUARD({
    embc::VlzStream s{dim, n, std::vector<uint8_t>(in, in + len)};
    const embc::QuantizedBatch q = embc::vlz_decode(s, embc::ErrorBound(0.01));
    std::memcpy(out, q.codes.data(), sizeof(int32_t) * q.codes.size());
  })
}

int ref_match_stats(const int32_t* codes, uint32_t dim, uint32_t n, uint32_t window, uint64_t* lit,
                    uint64_t* ref, char* err, size_t errcap) {
  GUARD({
    embc::QuantizedBatch q{0, dim, std::vector<int32_t>(codes, codes + static_cast<size_t>(dim) * n),
                           embc::ErrorBound(0.01)};
    const embc::MatchStats m = embc::match_stats(q, embc::VlzConfig{window});
    *lit = m.literal_count;
    *ref = m.reference_count;
  })
}

int ref_huff_encode(const int32_t* codes, uint64_t n, uint8_t** out, uint64_t* len, char* err,
                    size_t errcap) {
  GUARD({
    const embc::HuffStream s = embc::huff_encode_codes(std::span<const int32_t>(codes, n));
    *out = dup(s.bytes);
    *len = s.bytes.size();
  })
}

int ref_huff_decode(const uint8_t* in, uint64_t len, int32_t** out, uint64_t* n, char* err,
                    size_t errcap) {
  GUARD({
    const std::vector<int32_t> v = embc::huff_decode(embc::HuffStream{std::vector<uint8_t>(in, in + len)});
    *out = dup(v);
    *n = v.size();
  })
}

int ref_huff_codebook(const int32_t* codes, uint64_t n, int32_t* syms, uint8_t* lens, uint32_t* cws,
                      uint32_t* nsym, char* err, size_t errcap) {
  GUARD({
    const embc::Codebook b = embc::Codebook::build(std::span<const int32_t>(codes, n));
    for (size_t i = 0; i < b.entries().size(); ++i) {
      syms[i] = b.entries()[i].symbol;
      lens[i] = b.entries()[i].length;
      cws[i] = b.code_of(i);
    }
    *nsym = static_cast<uint32_t>(b.entries().size());
  })
}

int ref_huff_from_histogram(const int32_t* sym, const uint64_t* cnt, uint32_t n, int32_t* out_sym,
                            uint8_t* out_len, char* err, size_t errcap) {
  GUARD({
    std::vector<std::pair<int32_t, uint64_t>> h;
    for (uint32_t i = 0; i < n; ++i) h.emplace_back(sym[i], cnt[i]);
    const embc::Codebook b = embc::Codebook::from_histogram(std::move(h));
    for (size_t i = 0; i < b.entries().size(); ++i) {
      out_sym[i] = b.entries()[i].symbol;
      out_len[i] = b.entries()[i].length;
    }
  })
}

// pack() over serialized chunks (each re-parsed into a CompressedChunk).
int ref_pack(const uint8_t* const* chunks, const uint64_t* lens, uint32_t k, uint8_t** out,
             uint64_t* len, char* err, size_t errcap) {
  GUARD({
    std::vector<embc::CompressedChunk> cs;
    for (uint32_t i = 0; i < k; ++i)
      cs.push_back(embc::parse_chunk(std::span<const uint8_t>(chunks[i], lens[i])));
    const embc::PackedSendBuffer b = embc::pack(cs);
    *out = dup(b.bytes);
    *len = b.bytes.size();
  })
}

// unpack(): returns the re-serialized chunks concatenated plus their lengths.
int ref_unpack(const uint8_t* buf, uint64_t len, uint8_t** out, uint64_t** lens, uint32_t* k,
               char* err, size_t errcap) {
  GUARD({
    embc::PackedSendBuffer b{std::vector<uint8_t>(buf, buf + len)};
    const std::vector<embc::CompressedChunk> cs = embc::unpack(b);
    std::vector<uint8_t> all;
    std::vector<uint64_t> ls;
    for (const auto& c : cs) {
      const auto s = embc::serialize_chunk(c);
      all.insert(all.end(), s.begin(), s.end());
      ls.push_back(s.size());
    }
    *out = dup(all);
    *lens = dup(ls);
    *k = static_cast<uint32_t>(cs.size());
  })
}

int ref_metadata(const uint8_t* chunk, uint64_t len, uint8_t* out25, char* err, size_t errcap) {
  GUARD({
    const embc::CompressedChunk c = embc::parse_chunk(std::span<const uint8_t>(chunk, len));
    const std::vector<uint8_t> m = embc::serialize_metadata(embc::metadata_for(c));
    std::memcpy(out25, m.data(), m.size());
  })
}

int ref_parse_metadata(const uint8_t* in, uint64_t len, uint64_t* clen, uint8_t* codec, double* eb,
                       uint32_t* dim, uint32_t* count, char* err, size_t errcap) {
  GUARD({
    const embc::ChunkMetadata m = embc::parse_metadata(std::span<const uint8_t>(in, len));
    *clen = m.compressed_len;
    *codec = m.codec;
    *eb = m.eb;
    *dim = m.dim;
    *count = m.vector_count;
  })
}

// ---- datagen (datagen.hpp) -------------------------------------------------

int ref_gen_table(int32_t id, uint32_t rows, uint32_t dim, int dist, double mu, double sigma,
                  double lo, double hi, double zipf, uint64_t seed, double* out, char* err,
                  size_t errcap) {
  GUARD({
    const auto v = embc::gen_table(make_spec(id, rows, dim, dist, mu, sigma, lo, hi, zipf, seed));
    std::memcpy(out, v.data(), sizeof(double) * v.size());
  })
}

int ref_lookup_indices(int32_t id, uint32_t rows, uint32_t dim, int dist, double mu, double sigma,
                       double lo, double hi, double zipf, uint64_t seed, uint32_t batch,
                       uint64_t stream, uint32_t* out, char* err, size_t errcap) {
  GUARD({
    const auto v = embc::gen_lookup_indices(
        make_spec(id, rows, dim, dist, mu, sigma, lo, hi, zipf, seed), batch, stream);
    std::memcpy(out, v.data(), sizeof(uint32_t) * v.size());
  })
}

uint64_t ref_mix_seed(uint64_t seed, uint64_t salt) { return embc::detail::mix_seed(seed, salt); }

// ---- policy (policy.hpp) -------------------------------------------------

int ref_pattern_counts(const double* x, uint32_t dim, uint32_t rows, double eb, uint64_t* orig,
                       uint64_t* quant, char* err, size_t errcap) {
  GUARD({
    embc::EmbeddingBatch b{0, dim, std::vector<double>(x, x + static_cast<size_t>(dim) * rows)};
    const auto c = embc::detail::pattern_counts(b, embc::ErrorBound(eb));
    *orig = c.original;
    *quant = c.quantized;
  })
}

double ref_decay_multiplier(uint64_t it, int fn, double start, uint64_t end, uint32_t steps) {
  embc::DecayConfig d;
  d.function = static_cast<embc::DecayConfig::Fn>(fn);
  d.start_scale = start;
  d.decay_end = end;
  d.step_count = steps;
  return embc::decay_multiplier(it, d);
}

int ref_classify(double survival, double global_eb, double alpha, double beta, double l_thr,
                 double s_thr, int* cls, double* eb, char* err, size_t errcap) {
  GUARD({
    embc::PolicyConfig p;
    p.global_eb = global_eb;
    p.alpha = alpha;
    p.beta = beta;
    p.large_threshold = l_thr;
    p.small_threshold = s_thr;
    const embc::TableClass c = embc::classify_table(survival, p);
    *cls = static_cast<int>(c);
    *eb = p.eb_for(c);
  })
}

double ref_estimate_speedup(double ratio, double bw, double comp, double decomp) {
  return embc::estimate_speedup(ratio, bw, comp, decomp);
}

// ---- CPU baseline timing: encode_chunks + pack, then parallel decode -------
// Jobs share one contiguous value array (job i starts at offs[i] doubles).
int ref_codec_timed(const double* values, const uint64_t* offs, const uint32_t* dims,
                    const uint32_t* ns, const double* ebs, const uint8_t* codecs, uint32_t njobs,
                    unsigned workers, int reps, double* comp_s, double* decomp_s,
                    uint64_t* packed_len, char* err, size_t errcap) {
  GUARD({
    std::vector<embc::EmbeddingBatch> batches(njobs);
    for (uint32_t j = 0; j < njobs; ++j) {
      batches[j].dim = dims[j];
      batches[j].values.assign(values + offs[j], values + offs[j] + static_cast<size_t>(dims[j]) * ns[j]);
    }
    std::vector<embc::EncodeJob> jobs(njobs);
    for (uint32_t j = 0; j < njobs; ++j)
      jobs[j] = embc::EncodeJob{&batches[j], ebs[j], static_cast<embc::Codec>(codecs[j]), {}};
    double best_c = 1e30, best_d = 1e30;
    for (int r = 0; r < reps; ++r) {
      auto t0 = std::chrono::steady_clock::now();
      std::vector<embc::CompressedChunk> chunks = embc::encode_chunks(jobs, workers);
      embc::PackedSendBuffer buf = embc::pack(chunks);
      auto t1 = std::chrono::steady_clock::now();
      std::vector<embc::CompressedChunk> back = embc::unpack(buf);
      std::vector<embc::EmbeddingBatch> out(back.size());
      embc::parallel_for(back.size(), workers, [&](size_t i) { out[i] = embc::decode_chunk(back[i]); });
      auto t2 = std::chrono::steady_clock::now();
      best_c = std::min(best_c, std::chrono::duration<double>(t1 - t0).count());
      best_d = std::min(best_d, std::chrono::duration<double>(t2 - t1).count());
      *packed_len = buf.bytes.size();
    }
    *comp_s = best_c;
    *decomp_s = best_d;
  })
}

// ---- simulator (commsim.hpp), one table per rank, pinned profiles ----------
// Returns per-iteration byte accounting and the deterministic digest.
int ref_simulate(uint32_t ranks, uint32_t batch, uint32_t iterations, uint64_t seed, int compression,
                 double global_eb, double start_scale, uint64_t decay_end, uint32_t steps,
                 const uint32_t* t_rows, const uint32_t* t_dim, const int* t_dist,
                 const double* t_mu, const double* t_sigma, const double* t_lo, const double* t_hi,
                 const double* t_zipf, uint32_t ntables, const uint8_t* prof_codec,
                 const double* prof_eb, uint64_t* out_uncompressed, uint64_t* out_payload,
                 uint64_t* out_metadata, double* out_max_err, uint64_t* out_digest,
                 uint64_t* report_digest, char* err, size_t errcap) {
  GUARD({
    embc::SimConfig cfg;
    cfg.ranks = ranks;
    cfg.batch = batch;
    cfg.iterations = iterations;
    cfg.seed = seed;
    cfg.compression = compression != 0;
    cfg.policy.global_eb = global_eb;
    cfg.policy.decay.start_scale = start_scale;
    cfg.policy.decay.decay_end = decay_end;
    cfg.policy.decay.step_count = steps;
    for (uint32_t t = 0; t < ntables; ++t)
      cfg.tables.push_back(make_spec(static_cast<int32_t>(t), t_rows[t], t_dim[t], t_dist[t], t_mu[t],
                                     t_sigma[t], t_lo[t], t_hi[t], t_zipf[t], t + 1));
    std::map<int32_t, embc::TableProfile> profiles;
    for (uint32_t r = 0; r < ranks; ++r) {
      embc::TableProfile p;
      p.table_id = static_cast<int32_t>(r);
      p.codec = static_cast<embc::Codec>(prof_codec[r]);
      p.eb = prof_eb[r];
      profiles[p.table_id] = p;
    }
    const embc::SimReport rep = embc::run_training_schedule(cfg, profiles);
    for (size_t i = 0; i < rep.iterations.size(); ++i) {
      out_uncompressed[i] = rep.iterations[i].uncompressed_bytes;
      out_payload[i] = rep.iterations[i].payload_bytes;
      out_metadata[i] = rep.iterations[i].metadata_bytes;
      out_max_err[i] = rep.iterations[i].max_abs_error;
      out_digest[i] = rep.iterations[i].delivered_digest;
    }
    *report_digest = rep.deterministic_digest();
  })
}

// ---- presets and profiles (config.hpp) ---------------------------------------
// load_tables + load_policy of a reference preset file (config.hpp:184-228).
int ref_load_preset(const char* path, uint32_t cap, uint32_t* count, uint32_t* rows, uint32_t* dim,
                    int* dist, double* mu, double* sigma, double* lo, double* hi, double* zipf,
                    uint64_t* seed, double* policy5, int* decay_fn, double* decay_start,
                    uint64_t* decay_end, uint32_t* decay_steps, uint32_t* batch, uint32_t* ranks,
                    char* err, size_t errcap) {
  GUARD({
    const embc::KeyValueConfig kv = embc::KeyValueConfig::parse_file(path);
    const std::vector<embc::TableSpec> t = embc::load_tables(kv);
    const embc::PolicyConfig p = embc::load_policy(kv);
    *count = static_cast<uint32_t>(t.size());
    for (size_t i = 0; i < t.size() && i < cap; ++i) {
      rows[i] = t[i].rows;
      dim[i] = t[i].dim;
      dist[i] = t[i].dist == embc::ValueDist::gaussian ? 0 : 1;
      mu[i] = t[i].mu;
      sigma[i] = t[i].sigma;
      lo[i] = t[i].lo;
      hi[i] = t[i].hi;
      zipf[i] = t[i].zipf_s;
      seed[i] = t[i].seed;
    }
    policy5[0] = p.global_eb;
    policy5[1] = p.alpha;
    policy5[2] = p.beta;
    policy5[3] = p.large_threshold;
    policy5[4] = p.small_threshold;
    *decay_fn = static_cast<int>(p.decay.function);
    *decay_start = p.decay.start_scale;
    *decay_end = p.decay.decay_end;
    *decay_steps = p.decay.step_count;
    *batch = static_cast<uint32_t>(kv.get_u64("batch", 0));
    *ranks = static_cast<uint32_t>(kv.get_u64("ranks", 0));
  })
}

// offline_analysis (policy.hpp:278-302) of per-table samples, persisted with
// write_profiles (config.hpp:247-271).  Samples share one value array.
int ref_offline_analysis(const double* values, const uint64_t* offs, const uint32_t* dims,
                         const uint32_t* ns, const int32_t* table_ids, uint32_t nsamples,
                         double global_eb, double alpha, double beta, double l_thr, double s_thr,
                         double bandwidth, uint32_t window, const char* out_path, char* err,
                         size_t errcap) {
  GUARD({
    std::vector<embc::EmbeddingBatch> samples(nsamples);
    for (uint32_t j = 0; j < nsamples; ++j) {
      samples[j].table_id = table_ids[j];
      samples[j].dim = dims[j];
      samples[j].values.assign(values + offs[j], values + offs[j] + static_cast<size_t>(dims[j]) * ns[j]);
    }
    embc::PolicyConfig p;
    p.global_eb = global_eb;
    p.alpha = alpha;
    p.beta = beta;
    p.large_threshold = l_thr;
    p.small_threshold = s_thr;
    const auto profiles = embc::offline_analysis(samples, p, bandwidth, embc::VlzConfig{window});
    embc::write_profiles(out_path, profiles);
  })
}

// read_profiles (config.hpp:273-303) into arrays (ratios 0 when not measured).
int ref_read_profiles(const char* path, uint32_t cap, uint32_t* count, int32_t* table_id,
                      uint64_t* n_orig, uint64_t* n_quant, double* survival, int* cls, int* codec,
                      double* eb, double* ratio_vlz, double* ratio_huf, char* err, size_t errcap) {
  GUARD({
    const auto profiles = embc::read_profiles(path);
    *count = static_cast<uint32_t>(profiles.size());
    uint32_t i = 0;
    for (const auto& [id, p] : profiles) {
      if (i >= cap) break;
      table_id[i] = id;
      n_orig[i] = p.n_original_patterns;
      n_quant[i] = p.n_quantized_patterns;
      survival[i] = p.survival_ratio;
      cls[i] = static_cast<int>(p.cls);
      codec[i] = static_cast<int>(p.codec);
      eb[i] = p.eb;
      ratio_vlz[i] = ratio_huf[i] = 0.0;
      for (const auto& m : p.measured) (m.codec == embc::Codec::vlz ? ratio_vlz : ratio_huf)[i] = m.ratio;
      ++i;
    }
  })
}

// detail::format_double (csv.hpp:31-37) into buf (NUL-terminated).
void ref_format_double(double v, char* buf, size_t cap) {
  const std::string s = embc::detail::format_double(v);
  std::snprintf(buf, cap, "%s", s.c_str());
}

// pack(encode_chunks(jobs, workers)) bytes (container.hpp:242-256, :304-311).
int ref_encode_pack(const double* values, const uint64_t* offs, const uint32_t* dims,
                    const uint32_t* ns, const double* ebs, const uint8_t* codecs, uint32_t njobs,
                    uint32_t window, unsigned workers, uint8_t** out, uint64_t* len, char* err,
                    size_t errcap) {
  GUARD({
    std::vector<embc::EmbeddingBatch> batches(njobs);
    for (uint32_t j = 0; j < njobs; ++j) {
      batches[j].dim = dims[j];
      batches[j].values.assign(values + offs[j], values + offs[j] + static_cast<size_t>(dims[j]) * ns[j]);
    }
    std::vector<embc::EncodeJob> jobs(njobs);
    for (uint32_t j = 0; j < njobs; ++j)
      jobs[j] = embc::EncodeJob{&batches[j], ebs[j], static_cast<embc::Codec>(codecs[j]),
                                embc::VlzConfig{window}};
    const embc::PackedSendBuffer buf = embc::pack(embc::encode_chunks(jobs, workers));
    *out = dup(buf.bytes);
    *len = buf.bytes.size();
  })
}

}  // extern "C"
