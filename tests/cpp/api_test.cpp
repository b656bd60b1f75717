// C++ drop-in API test: include/embc_b200.hpp over libembc_cuda.so, written the
// way the reference's container_test.cc exercises embc:: (golden chunk bytes,
// round trip within the error bound, ValueError on non-finite input).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
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

int main() {
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

  cudaFree(d);
  cudaFree(dx);
  cudaFree(dy);
  cudaFree(db);
  std::printf(failures ? "api_test: %d failures\n" : "api_test: ok\n", failures);
  return failures ? 1 : 0;
}
