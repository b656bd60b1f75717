// C++ drop-in API test: include/embc_b200.hpp over libembc_cuda.so, written the
// way the reference's container_test.cc exercises embc:: (golden chunk bytes,
// round trip within the error bound, ValueError on non-finite input).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <fstream>
#include <sstream>
#include <vector>

#include "embc_b200.hpp"

static int failures = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++failures;                                                  \
    }                                                              \
  } while (0)

// Reads a whole file.
static std::string slurp(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  std::ostringstream b;
  b << f.rdbuf();
  return b.str();
}

int main(int argc, char** argv) {
  const std::string root = argc > 1 ? argv[1] : ".";
  embc_b200::Context ctx(0);
  // container_test.cc:37-68: raw chunk of codes {1, -2} at eb 0.02
  const float host[2] = {0.04f, -0.08f};
  float* d = nullptr;
  cudaMalloc(&d, sizeof(host));
  cudaMemcpy(d, host, sizeof(host), cudaMemcpyHostToDevice);
  embc_b200::EncodeJob job{d, 2, 1, 0.02, embc_b200::Codec::raw};
  const std::vector<uint8_t> bytes = embc_b200::encode_chunk(ctx, job);
  const uint8_t expect[38] = {'E', 'M', 'B', 'C', 0x01, 0x00, 0x7B, 0x14, 0xAE, 0x47, 0xE1, 0x7A, 0x94,
                              0x3F, 0x02, 0, 0, 0, 0x01, 0, 0, 0, 0x08, 0, 0, 0, 0, 0, 0, 0,
                              0x01, 0, 0, 0, 0xFE, 0xFF, 0xFF, 0xFF};
  CHECK(bytes.size() == 38 && std::memcmp(bytes.data(), expect, 38) == 0);

  // every codec round-trips within the bound (container_test.cc:125-142)
  std::vector<float> x(64 * 8);
  for (size_t i = 0; i < x.size(); ++i) x[i] = static_cast<float>(0.2 * std::sin(0.37 * static_cast<double>(i % 97)));
  float* dx = nullptr;
  float* dy = nullptr;
  cudaMalloc(&dx, x.size() * 4);
  cudaMalloc(&dy, x.size() * 4);
  cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
  for (auto codec : {embc_b200::Codec::raw, embc_b200::Codec::vlz, embc_b200::Codec::huffman}) {
    embc_b200::EncodeJob j{dx, 8, 64, 0.013, codec};
    const auto c = embc_b200::encode_chunk(ctx, j);
    uint8_t* dc = nullptr;
    cudaMalloc(&dc, c.size());
    cudaMemcpy(dc, c.data(), c.size(), cudaMemcpyHostToDevice);
    const embc_b200::ChunkRef ref{0, c.size(), dy, 8, 64, codec};
    embc_b200::decode_chunks(ctx, dc, std::span<const embc_b200::ChunkRef>(&ref, 1));
    std::vector<float> y(x.size());
    cudaMemcpy(y.data(), dy, y.size() * 4, cudaMemcpyDeviceToHost);
    double worst = 0.0;
    for (size_t i = 0; i < x.size(); ++i) worst = std::fmax(worst, std::fabs(static_cast<double>(y[i]) - x[i]));
    CHECK(worst <= 0.013 * (1 + 1e-6));
    cudaFree(dc);
  }

  // quantizer_test.cc:67-74: non-finite value -> ValueError naming the index
  const float bad[3] = {0.0f, std::numeric_limits<float>::infinity(), 1.0f};
  cudaMemcpy(dx, bad, sizeof(bad), cudaMemcpyHostToDevice);
  bool threw = false;
  try {
    embc_b200::encode_chunk(ctx, embc_b200::EncodeJob{dx, 1, 3, 0.01, embc_b200::Codec::vlz});
  } catch (const embc_b200::ValueError& e) {
    threw = std::strcmp(e.what(), "non-finite value at index 1") == 0;
  }
  CHECK(threw);

  // malformed chunk -> FormatError (container_test.cc:89-96)
  std::vector<uint8_t> broken(bytes);
  broken[0] = 'X';
  uint8_t* db = nullptr;
  cudaMalloc(&db, broken.size());
  cudaMemcpy(db, broken.data(), broken.size(), cudaMemcpyHostToDevice);
  threw = false;
  try {
    const embc_b200::ChunkRef ref{0, broken.size(), dy, 2, 1, embc_b200::Codec::raw};
    embc_b200::decode_chunks(ctx, db, std::span<const embc_b200::ChunkRef>(&ref, 1));
  } catch (const embc_b200::FormatError& e) {
    threw = std::strcmp(e.what(), "bad chunk magic") == 0;
  }
  CHECK(threw);

  // controller arithmetic (policy_test.cc:236-244)
  CHECK(std::fabs(0.03 * embc_b200::decay_multiplier(0, 0, 2.0, 1000, 4) - 0.06) < 1e-15);
  CHECK(embc_b200::decay_multiplier(1000, 0, 2.0, 1000, 4) == 1.0);
  CHECK(embc_b200::classify_table(0.5, 0.03, 5.0 / 3.0, 3.0, 0.7, 0.95) == embc_b200::TableClass::large);

  // encode_chunks([]) + pack: the 4-byte rank count (container.hpp:242-256)
  {
    uint8_t* dp = nullptr;
    cudaMalloc(&dp, 16);
    cudaMemset(dp, 0xAB, 16);
    const auto r = embc_b200::encode_chunks(ctx, std::span<const embc_b200::EncodeJob>(), dp, 16, true);
    uint8_t h[8];
    cudaMemcpy(h, dp, 8, cudaMemcpyDeviceToHost);
    CHECK(r.total == 4 && h[0] == 0 && h[3] == 0 && h[4] == 0xAB);
    cudaFree(dp);
  }

  // the reference-shaped encode_chunks (host chunks in job order) + pack table
  // + unpack (container.hpp:258-292)
  cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
  {
    const embc_b200::EncodeJob jobs[3] = {{dx, 8, 64, 0.01, embc_b200::Codec::vlz},
                                          {dx, 8, 32, 0.02, embc_b200::Codec::huffman},
                                          {dx, 4, 16, 0.01, embc_b200::Codec::raw}};
    const auto chunks = embc_b200::encode_chunks(ctx, jobs);
    CHECK(chunks.size() == 3 && chunks[2].size() == embc_b200::kHeaderSize + 4 * 64);
    const uint64_t cap = embc_b200::encode_bound(jobs, true);
    uint8_t* dp = nullptr;
    cudaMalloc(&dp, cap);
    const auto r = embc_b200::encode_chunks(ctx, jobs, dp, cap, true);
    std::vector<uint8_t> packed(r.total);
    cudaMemcpy(packed.data(), dp, r.total, cudaMemcpyDeviceToHost);
    const auto table = embc_b200::unpack(packed);
    CHECK(table.size() == 3);
    for (size_t j = 0; j < 3 && j < table.size(); ++j)
      CHECK(std::memcmp(packed.data() + table[j].first, chunks[j].data(), chunks[j].size()) == 0 &&
            table[j].second == chunks[j].size());
    packed.push_back(0);
    threw = false;
    try {
      embc_b200::unpack(packed);
    } catch (const embc_b200::FormatError& e) {
      threw = std::strcmp(e.what(), "send buffer has 1 unclaimed trailing bytes") == 0;
    }
    CHECK(threw);
    cudaFree(dp);
  }

  // controller: profiles written by the reference (configs/profiles_kg.cfg)
  // read back and re-written byte for byte (config.hpp:247-303); eb_at in the
  // decay (policy.hpp:336-342); GPU offline_analysis of table 0's iteration-0
  // sample == the reference's profile (policy.hpp:278-302)
  {
    const std::string src = root + "/configs/profiles_kg.cfg";
    const auto prof = embc_b200::read_profiles(src);
    CHECK(prof.size() == 26);
    embc_b200::write_profiles("/tmp/embc_api_test_profiles.cfg", prof);
    CHECK(slurp("/tmp/embc_api_test_profiles.cfg") == slurp(src));
    embc_b200::PolicyConfig cfg;
    cfg.global_eb = 0.03;
    cfg.decay.start_scale = 2.0;
    cfg.decay.decay_end = 500;
    cfg.decay.step_count = 4;
    CHECK(embc_b200::eb_at(0, 300, prof, cfg) == prof.at(0).eb * (2.0 - 2.0 / 3.0));
    CHECK(embc_b200::eb_at(99, 600, prof, cfg) == 0.03);
    // KAGGLE table 0: rows 8, gaussian sigma 0.004, zipf 1.8 (kaggle_like.cfg), dim 16, batch 2048
    const uint32_t rows = 8, dim = 16, B = 2048;
    const uint64_t seed = embc_mix_seed(1, 0x7AB1Eull ^ 0);
    std::vector<float> tab(rows * dim);
    std::vector<uint32_t> idx(B);
    CHECK(embc_gen_table(rows, dim, 0, 0.0, 0.004, 0.0, 1.0, seed, tab.data()) == EMBC_OK);
    CHECK(embc_gen_lookup_indices(rows, 1.8, seed, B, 0, idx.data()) == EMBC_OK);
    float *dt = nullptr, *ds = nullptr;
    uint32_t* di = nullptr;
    cudaMalloc(&dt, tab.size() * 4);
    cudaMalloc(&ds, 4ull * B * dim);
    cudaMalloc(&di, 4ull * B);
    cudaMemcpy(dt, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(di, idx.data(), 4ull * B, cudaMemcpyHostToDevice);
    CHECK(embc_gather_rows(dt, dim, di, B, ds, nullptr) == EMBC_OK);
    const embc_b200::Sample smp{0, ds, dim, B};
    embc_b200::PolicyConfig acfg;
    acfg.global_eb = 0.03;
    const auto got = embc_b200::offline_analysis(ctx, std::span<const embc_b200::Sample>(&smp, 1), acfg, 1e-300);
    const auto& g0 = got.at(0);
    const auto& w0 = prof.at(0);
    CHECK(g0.n_original_patterns == w0.n_original_patterns && g0.n_quantized_patterns == w0.n_quantized_patterns);
    CHECK(g0.cls == w0.cls && g0.eb == w0.eb && g0.codec == w0.codec);
    CHECK(g0.measured.size() == 2 && g0.measured[0].ratio == w0.measured[0].ratio &&
          g0.measured[1].ratio == w0.measured[1].ratio);
    cudaFree(dt);
    cudaFree(ds);
    cudaFree(di);
  }

  // the compressed all-to-all on a one-rank NCCL communicator: forward and
  // backward deliver exactly decode(encode(chunk)); the baseline is exact
  {
    const auto id = embc_b200::Exchange::unique_id();
    embc_b200::Exchange ex(0, 0, 1, id, 2);
    const uint32_t T = 3, dim = 8, B = 64;
    std::vector<float*> look(T), out(T), bout(T);
    std::vector<const float*> clook(T);
    for (uint32_t t = 0; t < T; ++t) {
      cudaMalloc(&look[t], 4ull * B * dim);
      cudaMalloc(&out[t], 4ull * B * dim);
      cudaMalloc(&bout[t], 4ull * B * dim);
      cudaMemcpy(look[t], x.data() + t * 8, 4ull * B * dim - 4 * 8 * t, cudaMemcpyHostToDevice);
      cudaMemset(reinterpret_cast<char*>(look[t]) + 4ull * B * dim - 4 * 8 * t, 0, 4 * 8 * t);
      clook[t] = look[t];
    }
    const double ebs[T] = {0.01, 0.02, 0.005};
    const uint8_t codecs[T] = {1, 2, 0};
    const auto st = ex.fwd(dim, B, clook, ebs, codecs, out);
    cudaDeviceSynchronize();
    CHECK(st.sent_values == uint64_t(T) * B * dim && st.payload_bytes == 0);
    for (uint32_t t = 0; t < T; ++t) {
      const embc_b200::EncodeJob j{look[t], dim, B, ebs[t], static_cast<embc_b200::Codec>(codecs[t])};
      const auto c = embc_b200::encode_chunk(ctx, j);
      uint8_t* dc = nullptr;
      cudaMalloc(&dc, c.size());
      cudaMemcpy(dc, c.data(), c.size(), cudaMemcpyHostToDevice);
      const embc_b200::ChunkRef ref{0, c.size(), dy, dim, B, j.codec};
      embc_b200::decode_chunks(ctx, dc, std::span<const embc_b200::ChunkRef>(&ref, 1));
      std::vector<float> want(B * dim), got(B * dim);
      cudaMemcpy(want.data(), dy, 4ull * B * dim, cudaMemcpyDeviceToHost);
      cudaMemcpy(got.data(), out[t], 4ull * B * dim, cudaMemcpyDeviceToHost);
      CHECK(std::memcmp(want.data(), got.data(), 4ull * B * dim) == 0);
      cudaFree(dc);
    }
    const auto bst = ex.bwd(dim, B, clook, ebs, codecs, bout);
    CHECK(bst.recv_values == uint64_t(T) * B * dim);
    std::vector<float> a(B * dim), b(B * dim);
    for (uint32_t t = 0; t < T; ++t) {
      cudaMemcpy(a.data(), out[t], 4ull * B * dim, cudaMemcpyDeviceToHost);
      cudaMemcpy(b.data(), bout[t], 4ull * B * dim, cudaMemcpyDeviceToHost);
      CHECK(std::memcmp(a.data(), b.data(), 4ull * B * dim) == 0);  // same chunk, same codec both ways
    }
    ex.baseline_fwd(dim, B, clook, out);
    cudaDeviceSynchronize();
    for (uint32_t t = 0; t < T; ++t) {
      cudaMemcpy(a.data(), out[t], 4ull * B * dim, cudaMemcpyDeviceToHost);
      cudaMemcpy(b.data(), look[t], 4ull * B * dim, cudaMemcpyDeviceToHost);
      CHECK(std::memcmp(a.data(), b.data(), 4ull * B * dim) == 0);
    }
    for (uint32_t t = 0; t < T; ++t) {
      cudaFree(look[t]);
      cudaFree(out[t]);
      cudaFree(bout[t]);
    }
  }

  cudaFree(d);
  cudaFree(dx);
  cudaFree(dy);
  cudaFree(db);
  std::printf(failures ? "api_test: %d failures\n" : "api_test: ok\n", failures);
  return failures ? 1 : 0;
}
