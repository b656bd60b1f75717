// host_policy.cpp -- the dual-level adaptive error-bound controller's
// arithmetic (table-wise class bounds and iteration-wise decay) and the
// synthetic workload generator, host C++ with the reference's exact formulas.
//
// Controller: policy.hpp:58-102 (configs), :188-208 (classify, Eq. 2),
//             :308-331 (decay_multiplier).
// Workload:   datagen.hpp:63-126 (splitmix64 / mix_seed / u01 / Box-Muller /
//             gen_table), :89-110 (ZipfSampler), :130-142 (draw_indices).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numbers>
#include <random>
#include <vector>

#include "../../include/embc_cuda.h"

namespace {

uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

uint64_t mix(uint64_t seed, uint64_t salt) { return splitmix64(seed ^ splitmix64(salt)); }

// top 53 bits -> [0, 1)
double unit(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }

double box_muller(std::mt19937_64& g, double mu, double sigma) {
  const double a = (static_cast<double>(g() >> 11) + 1.0) * 0x1.0p-53;  // (0, 1]
  const double b = unit(g);
  return mu + sigma * std::sqrt(-2.0 * std::log(a)) * std::cos(2.0 * std::numbers::pi * b);
}

}  // namespace

extern "C" {

uint64_t embc_mix_seed(uint64_t seed, uint64_t salt) { return mix(seed, salt); }

embc_status embc_gen_table(uint32_t rows, uint32_t dim, int dist, double mu, double sigma,
                           double lo, double hi, uint64_t seed, float* h_out) {
  if (rows < 1 || dim < 1) return EMBC_ERR_VALUE;  // TableSpec::validate
  if (dist == 0 && !(sigma > 0.0)) return EMBC_ERR_VALUE;
  if (dist == 1 && !(lo < hi)) return EMBC_ERR_VALUE;
  if (!h_out) return EMBC_ERR_ARGUMENT;
  std::mt19937_64 g(mix(seed, 0xEBC0A11ull));
  const uint64_t n = static_cast<uint64_t>(rows) * dim;
  for (uint64_t i = 0; i < n; ++i) {
    const double x = dist == 0 ? box_muller(g, mu, sigma) : lo + (hi - lo) * unit(g);
    h_out[i] = static_cast<float>(x);
  }
  return EMBC_OK;
}

embc_status embc_gen_lookup_indices(uint32_t rows, double zipf_s, uint64_t seed, uint32_t batch,
                                    uint64_t stream_id, uint32_t* h_out) {
  if (rows < 1 || zipf_s < 0.0) return EMBC_ERR_VALUE;
  if (!h_out && batch) return EMBC_ERR_ARGUMENT;
  // inverse CDF over (k+1)^-s, normalised, last entry pinned to 1
  std::vector<double> cdf(rows);
  double total = 0.0;
  for (uint32_t k = 0; k < rows; ++k) {
    total += std::pow(static_cast<double>(k) + 1.0, -zipf_s);
    cdf[k] = total;
  }
  for (double& c : cdf) c /= total;
  cdf.back() = 1.0;
  std::mt19937_64 g(mix(seed, 0xEBC10C0ull ^ stream_id));
  for (uint32_t i = 0; i < batch; ++i) {
    const double u = unit(g);
    h_out[i] = static_cast<uint32_t>(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
  }
  return EMBC_OK;
}

embc_status embc_decay_multiplier(uint64_t it, int fn, double s, uint64_t end, uint32_t steps,
                                  double* out) {
  if (!out) return EMBC_ERR_ARGUMENT;
  if (!(s >= 1.0) || steps < 1) return EMBC_ERR_CONFIG;  // DecayConfig::validate
  if (fn < 0 || fn > 2) return EMBC_ERR_CONFIG;
  if (end == 0 || it >= end || s == 1.0) {
    *out = 1.0;
    return EMBC_OK;
  }
  const double span = s - 1.0;
  if (fn == 0) {
    if (steps == 1) {
      *out = s;
      return EMBC_OK;
    }
    const uint64_t stair = it * steps / end;
    *out = s - span * static_cast<double>(stair) / static_cast<double>(steps - 1);
  } else {
    const double t = static_cast<double>(it) / static_cast<double>(end);
    *out = fn == 1 ? s - span * t : 1.0 + span * (1.0 - std::log1p((std::numbers::e - 1.0) * t));
  }
  return EMBC_OK;
}

embc_status embc_classify_table(double survival, double global_eb, double alpha, double beta,
                                double large_thr, double small_thr, int* cls, double* eb) {
  if (!cls || !eb) return EMBC_ERR_ARGUMENT;
  // PolicyConfig::validate (policy.hpp:83-93)
  if (!(global_eb > 0.0 && std::isfinite(global_eb)) || !(alpha >= 1.0) || !(beta >= 1.0) ||
      !(0.0 < large_thr && large_thr < small_thr && small_thr <= 1.0))
    return EMBC_ERR_CONFIG;
  int c = 1;
  if (survival > small_thr) c = 2;
  else if (survival < large_thr) c = 0;
  *cls = c;
  *eb = c == 0 ? global_eb * alpha : c == 2 ? global_eb / beta : global_eb;
  return EMBC_OK;
}

embc_status embc_estimate_speedup(double ratio, double bw, double comp, double decomp,
                                  double* out) {
  if (!out) return EMBC_ERR_ARGUMENT;
  if (!(ratio > 0.0 && bw > 0.0 && comp > 0.0 && decomp > 0.0)) return EMBC_ERR_VALUE;
  *out = 1.0 / (1.0 / ratio + bw * (1.0 / comp + 1.0 / decomp));
  return EMBC_OK;
}

}  // extern "C"
