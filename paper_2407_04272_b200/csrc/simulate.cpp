// simulate.cpp -- the reference's Simulator (commsim.hpp:200-435) with the codec
// on the GPU: R ranks of one forward all-to-all per iteration, every rank's
// chunks compressed and packed by embc_encode, every received chunk unpacked,
// checked against its metadata record and decoded by embc_decode into the
// reference's doubles.  Ranks run one after another on one device; the two
// stages are separated exactly as the reference's barriers separate them
// (all ranks compress, then all ranks decode), so every byte count, error and
// digest is the reference's: IterationStats (commsim.hpp:77-96) and
// SimReport::deterministic_digest (:146-163) are reproduced bit for bit.
// The transport is a device-to-device copy of each packed send buffer
// (the reference moves them through shared slots); the NCCL exchange itself is
// exchange.cpp.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/embc_cuda.h"

namespace {

constexpr uint64_t kFnvSeed = 0xCBF29CE484222325ull;

uint64_t fnv1a(const void* data, size_t n, uint64_t h = kFnvSeed) {  // bytes.hpp:177-185
  const auto* p = static_cast<const uint8_t*>(data);
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001B3ull;
  }
  return h;
}

struct SimError {
  embc_status st;
  int reason;
  std::string msg;
};

void fail(embc_error* err, const SimError& e) {
  if (!err) return;
  std::memset(err, 0, sizeof(*err));
  err->status = e.st;
  err->reason = e.reason;
  std::snprintf(err->message, sizeof(err->message), "%s", e.msg.c_str());
}

#define SIM_CUDA(x)                                                                          \
  do {                                                                                       \
    const cudaError_t ce_ = (x);                                                             \
    if (ce_ != cudaSuccess) throw SimError{EMBC_ERR_CUDA, 0, std::string("simulate: ") + #x + \
                                                                 ": " + cudaGetErrorString(ce_)}; \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  void ensure(size_t bytes) {
    if (bytes <= n) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    SIM_CUDA(cudaMalloc(&p, bytes));
    n = bytes;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

// A rank's table (datagen.hpp:146-179): fp32-exact values and its sampler.
struct Table {
  embc_sim_table spec;
  uint64_t seed;
  std::vector<float> values;
  std::vector<float> gather(uint32_t batch, uint64_t stream) const {
    std::vector<uint32_t> idx(batch);
    const embc_status st = embc_gen_lookup_indices(spec.rows, spec.zipf_s, seed, batch, stream, idx.data());
    if (st != EMBC_OK) throw SimError{st, 0, "simulate: lookup index generation failed"};
    std::vector<float> out(static_cast<size_t>(batch) * spec.dim);
    for (uint32_t i = 0; i < batch; ++i)
      std::memcpy(out.data() + static_cast<size_t>(i) * spec.dim, values.data() + static_cast<size_t>(idx[i]) * spec.dim,
                  sizeof(float) * spec.dim);
    return out;
  }
};

std::string err_text(embc_ctx* ctx, embc_status st) {
  embc_error e{};
  embc_get_error(ctx, &e);
  return e.message[0] ? std::string(e.message) : ("status " + std::to_string(st));
}

}  // namespace

extern "C" embc_status embc_simulate(int device, const embc_sim_config* cfg, const embc_sim_table* tables,
                                     uint32_t ntables, const uint8_t* prof_codec, const double* prof_eb,
                                     embc_sim_iteration* out, uint64_t* report_digest, embc_error* err) {
  embc_ctx* ctx = nullptr;
  cudaStream_t s = nullptr;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  try {
    // SimConfig::validate (commsim.hpp:46-62)
    if (!cfg || !out || !report_digest) throw SimError{EMBC_ERR_ARGUMENT, 0, "simulate: null argument"};
    if (cfg->ranks < 1) throw SimError{EMBC_ERR_CONFIG, 0, "ranks must be >= 1"};
    if (cfg->batch < 1) throw SimError{EMBC_ERR_CONFIG, 0, "batch must be >= 1"};
    if (ntables < 1 || !tables) throw SimError{EMBC_ERR_CONFIG, 0, "at least one table spec is required"};
    if (cfg->compression && (!prof_codec || !prof_eb))
      throw SimError{EMBC_ERR_ARGUMENT, 0, "simulate: profiles are required with compression"};
    const uint32_t R = cfg->ranks, B = cfg->batch;
    SIM_CUDA(cudaSetDevice(device));
    embc_status st = embc_ctx_create(device, &ctx);
    if (st != EMBC_OK) throw SimError{st, 0, "simulate: context creation failed"};
    SIM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    SIM_CUDA(cudaEventCreate(&ev[0]));
    SIM_CUDA(cudaEventCreate(&ev[1]));
    // Simulator::rank_table_spec (commsim.hpp:207-213): specs cycled over ranks, re-seeded per rank
    std::vector<Table> tab(R);
    for (uint32_t r = 0; r < R; ++r) {
      tab[r].spec = tables[r % ntables];
      tab[r].seed = embc_mix_seed(cfg->seed, 0x7AB1Eull ^ r);
      const embc_sim_table& t = tab[r].spec;
      if (t.rows < 1 || t.dim < 1) throw SimError{EMBC_ERR_VALUE, 0, "table rows and dim must be >= 1"};
      tab[r].values.resize(static_cast<size_t>(t.rows) * t.dim);
      st = embc_gen_table(t.rows, t.dim, t.dist, t.mu, t.sigma, t.lo, t.hi, tab[r].seed, tab[r].values.data());
      if (st != EMBC_OK) throw SimError{st, 0, "simulate: table generation failed"};
    }
    auto stream_id = [&](uint64_t it, uint32_t src, uint32_t dst) {  // commsim.hpp:282-284
      return (it * R + src) * R + dst + 1;
    };
    DevBuf d_in, d_send, d_out, d_aux;
    std::vector<DevBuf> d_bufs(R);
    std::vector<std::vector<uint8_t>> h_bufs(R), h_meta(R);
    uint64_t rep = kFnvSeed;
    auto mix = [&rep](uint64_t v) { rep = fnv1a(&v, sizeof(v), rep); };
    mix(R);
    mix(B);
    mix(cfg->compression ? 1 : 0);
    for (uint32_t it = 0; it < cfg->iterations; ++it) {
      embc_sim_iteration& S = out[it];
      std::memset(&S, 0, sizeof(S));
      S.iteration = it;
      S.delivery_conserved = 1;
      uint64_t dig = kFnvSeed;
      // ---- stage 1 on every rank: gather, compress + pack + metadata
      std::vector<std::vector<std::vector<float>>> outgoing(R);
      for (uint32_t r = 0; r < R; ++r) {
        const uint32_t dim = tab[r].spec.dim;
        outgoing[r].resize(R);
        for (uint32_t d = 0; d < R; ++d) outgoing[r][d] = tab[r].gather(B, stream_id(it, r, d));
        const size_t nv = static_cast<size_t>(B) * dim;
        double eb = cfg->global_eb;
        if (cfg->compression) {  // eb_at (policy.hpp:336-342) for table id = rank
          double m = 1.0;
          st = embc_decay_multiplier(it, cfg->decay_fn, cfg->decay_start_scale, cfg->decay_end, cfg->decay_steps, &m);
          if (st != EMBC_OK) throw SimError{st, 0, "simulate: decay configuration"};
          eb = prof_eb[r] * m;
          if (!(std::isfinite(eb) && eb > 0.0)) {
            char b[96];
            std::snprintf(b, sizeof(b), "error bound must be finite and > 0, got %f", eb);
            throw SimError{EMBC_ERR_VALUE, 0, b};
          }
          S.eb_max = std::max(S.eb_max, eb);
        }
        d_in.ensure(sizeof(float) * nv * R);
        for (uint32_t d = 0; d < R; ++d)
          SIM_CUDA(cudaMemcpyAsync(static_cast<float*>(d_in.p) + nv * d, outgoing[r][d].data(), sizeof(float) * nv,
                                   cudaMemcpyHostToDevice, s));
        for (uint32_t d = 0; d < R; ++d)
          if (d != r) S.uncompressed_bytes += 4ull * nv;  // EmbeddingBatch::wire_bytes
        if (cfg->compression) {
          std::vector<embc_job> jobs(R);
          for (uint32_t d = 0; d < R; ++d) {
            embc_job& j = jobs[d];
            std::memset(&j, 0, sizeof(j));
            j.src = static_cast<const float*>(d_in.p) + nv * d;
            j.dim = dim;
            j.n = B;
            j.eb = eb;
            j.window = 255;  // VlzConfig{}
            j.codec = prof_codec[r];
            j.src_kind = EMBC_SRC_F32;
          }
          const uint64_t bound = embc_encode_bound(jobs.data(), R, EMBC_LAYOUT_PACKED);
          d_bufs[r].ensure(bound + 16);
          const size_t mbytes = (25ull * R + 7) & ~7ull;
          d_aux.ensure(mbytes + 8);
          uint8_t* d_meta = static_cast<uint8_t*>(d_aux.p);
          uint64_t* d_total = reinterpret_cast<uint64_t*>(d_meta + mbytes);
          SIM_CUDA(cudaEventRecord(ev[0], s));
          st = embc_encode(ctx, jobs.data(), R, EMBC_LAYOUT_PACKED, static_cast<uint8_t*>(d_bufs[r].p), bound + 16,
                           nullptr, nullptr, d_meta, d_total, s);
          SIM_CUDA(cudaEventRecord(ev[1], s));
          if (st == EMBC_OK) st = embc_sync(ctx, s);
          if (st != EMBC_OK)
            throw SimError{st, 0, "rank " + std::to_string(r) + " compress stage: " + err_text(ctx, st)};
          float ms = 0.f;
          SIM_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
          S.comp_time = std::max(S.comp_time, ms * 1e-3);
          uint64_t total = 0;
          SIM_CUDA(cudaMemcpy(&total, d_total, 8, cudaMemcpyDeviceToHost));
          h_bufs[r].resize(total);
          h_meta[r].resize(25ull * R);
          SIM_CUDA(cudaMemcpy(h_bufs[r].data(), d_bufs[r].p, total, cudaMemcpyDeviceToHost));
          SIM_CUDA(cudaMemcpy(h_meta[r].data(), d_meta, 25ull * R, cudaMemcpyDeviceToHost));
          for (uint32_t d = 0; d < R; ++d) {
            if (d == r) continue;
            uint64_t clen = 0;
            std::memcpy(&clen, h_meta[r].data() + 25ull * d, 8);
            S.payload_bytes += clen;
            S.metadata_bytes += 25;
          }
        }
      }
      // ---- stage 4 on every rank: unpack every sender's buffer, check the
      // metadata, decode this rank's chunk into doubles, verify and digest
      for (uint32_t r = 0; r < R; ++r) {
        double max_err = 0.0;
        uint64_t rdig = kFnvSeed;
        float dec_ms = 0.f;
        for (uint32_t src = 0; src < R; ++src) {
          const uint32_t dim = tab[src].spec.dim;
          const size_t nv = static_cast<size_t>(B) * dim;
          std::vector<double> got(nv);
          const std::vector<float>& truth = outgoing[src][r];
          if (cfg->compression) {
            std::vector<uint64_t> off(R + 1), len(R + 1);
            uint32_t cnt = 0;
            embc_error ue{};
            st = embc_unpack(h_bufs[src].data(), h_bufs[src].size(), off.data(), len.data(), R + 1, &cnt, &ue);
            auto where = [&](const std::string& m) {
              return "rank " + std::to_string(r) + " decompress stage (from rank " + std::to_string(src) + "): " + m;
            };
            if (st != EMBC_OK) throw SimError{st, ue.reason, where(ue.message)};
            if (cnt != R)
              throw SimError{EMBC_ERR_FORMAT, 0,
                             where("send buffer from rank " + std::to_string(src) + " holds " + std::to_string(cnt) +
                                   " chunks, expected " + std::to_string(R))};
            // ChunkMetadata of (src -> r) against the chunk (commsim.hpp:371-376)
            uint64_t mlen = 0;
            uint32_t mcount = 0, mdim = 0;
            const uint8_t* m = h_meta[src].data() + 25ull * r;
            std::memcpy(&mlen, m, 8);
            std::memcpy(&mdim, m + 17, 4);
            std::memcpy(&mcount, m + 21, 4);
            uint32_t ccount = 0;
            if (len[r] >= 22) std::memcpy(&ccount, h_bufs[src].data() + off[r] + 18, 4);
            if (mlen != len[r] || mcount != ccount)
              throw SimError{EMBC_ERR_FORMAT, EMBC_R_META_MISMATCH,
                             where("metadata from rank " + std::to_string(src) + " disagrees with its chunk")};
            // the rank's copy of the sender's buffer, then the decode of its chunk
            d_send.ensure(h_bufs[src].size() + 16);
            SIM_CUDA(cudaMemcpyAsync(d_send.p, d_bufs[src].p, h_bufs[src].size(), cudaMemcpyDeviceToDevice, s));
            d_out.ensure(sizeof(double) * nv + 16);
            embc_chunk_ref ref{};
            ref.offset = off[r];
            ref.length = len[r];
            ref.out = d_out.p;
            ref.dim = mdim;
            ref.count = mcount;
            ref.codec = m[8];
            SIM_CUDA(cudaEventRecord(ev[0], s));
            st = embc_decode(ctx, static_cast<const uint8_t*>(d_send.p), &ref, 1, EMBC_OUT_F64, 0, s);
            SIM_CUDA(cudaEventRecord(ev[1], s));
            if (st == EMBC_OK) st = embc_sync(ctx, s);
            if (st != EMBC_OK) throw SimError{st, 0, where(err_text(ctx, st))};
            float ms = 0.f;
            SIM_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
            dec_ms += ms;
            SIM_CUDA(cudaMemcpy(got.data(), d_out.p, sizeof(double) * nv, cudaMemcpyDeviceToHost));
          } else {
            // baseline: raw float32 values, delivered exactly (commsim.hpp:337-351, :384-400)
            for (size_t i = 0; i < nv; ++i) got[i] = static_cast<double>(truth[i]);
          }
          for (size_t i = 0; i < nv; ++i)
            max_err = std::max(max_err, std::abs(got[i] - static_cast<double>(truth[i])));
          rdig = fnv1a(got.data(), sizeof(double) * nv, rdig);
        }
        if (cfg->compression) S.decomp_time = std::max(S.decomp_time, dec_ms * 1e-3);
        S.max_abs_error = std::max(S.max_abs_error, max_err);
        dig = fnv1a(&rdig, sizeof(rdig), dig);
      }
      // reduce (commsim.hpp:438-487)
      S.delivered_digest = dig;
      if (!cfg->compression) {
        S.payload_bytes = S.uncompressed_bytes;
        S.metadata_bytes = 0;
      }
      S.wire_bytes = S.payload_bytes + S.metadata_bytes;
      if (cfg->compression && S.max_abs_error > S.eb_max) {
        char b[160];
        std::snprintf(b, sizeof(b), "iteration %u: reconstruction error %f exceeds error bound %f", it,
                      S.max_abs_error, S.eb_max);
        throw SimError{EMBC_ERR_VALUE, 0, b};
      }
      if (!cfg->compression && S.max_abs_error != 0.0)
        throw SimError{EMBC_ERR_VALUE, 0, "iteration " + std::to_string(it) + ": baseline delivery must be exact"};
      // SimReport::deterministic_digest (commsim.hpp:146-163)
      uint64_t ebits = 0, ebits2 = 0;
      std::memcpy(&ebits, &S.eb_max, 8);
      std::memcpy(&ebits2, &S.max_abs_error, 8);
      mix(S.iteration);
      mix(ebits);
      mix(S.uncompressed_bytes);
      mix(S.payload_bytes);
      mix(S.metadata_bytes);
      mix(ebits2);
      mix(S.delivery_conserved ? 1 : 0);
      mix(S.delivered_digest);
    }
    *report_digest = rep;
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    cudaStreamDestroy(s);
    embc_ctx_destroy(ctx);
    return EMBC_OK;
  } catch (const SimError& e) {
    fail(err, e);
    if (ev[0]) cudaEventDestroy(ev[0]);
    if (ev[1]) cudaEventDestroy(ev[1]);
    if (s) cudaStreamDestroy(s);
    if (ctx) embc_ctx_destroy(ctx);
    return e.st;
  }
}
