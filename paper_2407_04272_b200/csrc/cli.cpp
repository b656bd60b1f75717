// cli.cpp -- embc_gpu: the reference's command-line front end
// (tools/embc_main.cpp: analyze / compress / decompress / bench / simulate /
// report) over the GPU codec (include/embc_b200.hpp, libembc_cuda.so).
// File formats are the reference's: key = value configs and profiles
// (config.hpp), .embv value files (valuefile.hpp:28-64), .embc chunk files
// (container.hpp:74-115), CSV with a "# schema:" line (csv.hpp).  Codec
// timings are GPU timings (CUDA events), so auto codec selection and the
// bench / analyze throughput columns describe this GPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/embc_b200.hpp"

namespace {

using namespace embc_b200;

// ---- key = value configuration (config.hpp:37-139 semantics) --------------
class KeyValue {
 public:
  static KeyValue parse_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw ConfigError("cannot open config file '" + path + "'");
    KeyValue kv;
    std::string line;
    size_t no = 0;
    while (std::getline(in, line)) {
      ++no;
      const std::string t = trim(line);
      if (t.empty() || t[0] == '#') continue;
      const size_t eq = t.find('=');
      if (eq == std::string::npos) throw ConfigError(path + ":" + std::to_string(no) + ": expected 'key = value'");
      const std::string k = trim(t.substr(0, eq));
      if (k.empty()) throw ConfigError(path + ":" + std::to_string(no) + ": empty key");
      kv.v_[k] = trim(t.substr(eq + 1));
    }
    return kv;
  }
  bool has(const std::string& k) const { return v_.count(k) != 0; }
  std::string str(const std::string& k) const {
    const auto it = v_.find(k);
    if (it == v_.end()) throw ConfigError("missing config key '" + k + "'");
    return it->second;
  }
  std::string str(const std::string& k, const std::string& d) const { return has(k) ? str(k) : d; }
  double f64(const std::string& k) const {
    const std::string s = str(k);
    double out = 0.0;
    const auto [p, ec] = std::from_chars(s.data(), s.data() + s.size(), out);
    if (ec != std::errc() || p != s.data() + s.size())
      throw ConfigError("key '" + k + "' expects a number, got '" + s + "'");
    return out;
  }
  double f64(const std::string& k, double d) const { return has(k) ? f64(k) : d; }
  uint64_t u64(const std::string& k) const {
    const std::string s = str(k);
    uint64_t out = 0;
    const auto [p, ec] = std::from_chars(s.data(), s.data() + s.size(), out);
    if (ec != std::errc() || p != s.data() + s.size())
      throw ConfigError("key '" + k + "' expects a non-negative integer, got '" + s + "'");
    return out;
  }
  uint64_t u64(const std::string& k, uint64_t d) const { return has(k) ? u64(k) : d; }
  bool flag(const std::string& k, bool d) const {
    if (!has(k)) return d;
    const std::string s = str(k);
    if (s == "on" || s == "true" || s == "1" || s == "yes") return true;
    if (s == "off" || s == "false" || s == "0" || s == "no") return false;
    throw ConfigError("key '" + k + "' expects on/off, got '" + s + "'");
  }

 private:
  static std::string trim(const std::string& s) {
    const auto b = s.find_first_not_of(" \t\r");
    if (b == std::string::npos) return "";
    return s.substr(b, s.find_last_not_of(" \t\r") - b + 1);
  }
  std::map<std::string, std::string> v_;
};

struct TableSpec {  // datagen.hpp:36-59
  int32_t table_id = 0;
  uint32_t rows = 1, dim = 1;
  int dist = 0;  // 0 gaussian, 1 uniform
  double mu = 0.0, sigma = 0.1, lo = 0.0, hi = 1.0, zipf = 0.0;
  uint64_t seed = 1;
};

PolicyConfig load_policy(const KeyValue& kv) {  // config.hpp:179-193
  PolicyConfig p;
  p.global_eb = kv.f64("policy.global_eb", p.global_eb);
  p.alpha = kv.f64("policy.alpha", p.alpha);
  p.beta = kv.f64("policy.beta", p.beta);
  p.large_threshold = kv.f64("policy.l_thr", p.large_threshold);
  p.small_threshold = kv.f64("policy.s_thr", p.small_threshold);
  const std::string fn = kv.str("policy.decay.function", "stepwise");
  if (fn == "stepwise") p.decay.function = DecayConfig::Fn::stepwise;
  else if (fn == "linear") p.decay.function = DecayConfig::Fn::linear;
  else if (fn == "logarithmic") p.decay.function = DecayConfig::Fn::logarithmic;
  else throw ConfigError("unknown decay function '" + fn + "'");
  p.decay.start_scale = kv.f64("policy.decay.start_scale", p.decay.start_scale);
  p.decay.decay_end = kv.u64("policy.decay.end", p.decay.decay_end);
  p.decay.step_count = static_cast<uint32_t>(kv.u64("policy.decay.steps", p.decay.step_count));
  p.validate();
  return p;
}

std::vector<TableSpec> load_tables(const KeyValue& kv) {  // config.hpp:195-225
  const uint64_t n = kv.u64("tables.count");
  if (n == 0) throw ConfigError("tables.count must be >= 1");
  std::vector<TableSpec> out;
  for (uint64_t i = 0; i < n; ++i) {
    const std::string p = "table." + std::to_string(i) + ".";
    TableSpec t;
    t.table_id = static_cast<int32_t>(i);
    t.rows = static_cast<uint32_t>(kv.u64(p + "rows"));
    t.dim = static_cast<uint32_t>(kv.u64(p + "dim"));
    const std::string d = kv.str(p + "dist", "gaussian");
    if (d == "gaussian") {
      t.mu = kv.f64(p + "mu", 0.0);
      t.sigma = kv.f64(p + "sigma", 0.1);
    } else if (d == "uniform") {
      t.dist = 1;
      t.lo = kv.f64(p + "lo", 0.0);
      t.hi = kv.f64(p + "hi", 1.0);
    } else {
      throw ConfigError("table " + std::to_string(i) + ": unknown distribution '" + d + "'");
    }
    t.zipf = kv.f64(p + "zipf", 0.0);
    t.seed = kv.u64(p + "seed", i + 1);
    if (t.rows < 1) throw ValueError("table rows must be >= 1");
    if (t.dim < 1) throw ValueError("table dim must be >= 1");
    if (t.dist == 0 && !(t.sigma > 0.0)) throw ValueError("gaussian sigma must be > 0, got " + std::to_string(t.sigma));
    if (t.dist == 1 && !(t.lo < t.hi)) throw ValueError("uniform bounds must satisfy lo < hi");
    if (t.zipf < 0.0) throw ValueError("zipf exponent must be >= 0");
    out.push_back(t);
  }
  return out;
}

// seeded_tables (embc_main.cpp:45-51)
std::vector<TableSpec> seeded(const KeyValue& kv, uint64_t seed) {
  auto t = load_tables(kv);
  for (auto& s : t) s.seed = embc_mix_seed(seed, 0x7AB1Eull ^ static_cast<uint32_t>(s.table_id));
  return t;
}

// Table(spec).lookup_batch(batch, stream) on the host generator (datagen.hpp:146-179)
std::vector<float> lookup_batch(const TableSpec& s, uint32_t batch, uint64_t stream) {
  std::vector<float> table(static_cast<size_t>(s.rows) * s.dim);
  if (embc_gen_table(s.rows, s.dim, s.dist, s.mu, s.sigma, s.lo, s.hi, s.seed, table.data()) != EMBC_OK)
    throw ValueError("table generation failed");
  std::vector<uint32_t> idx(batch);
  if (embc_gen_lookup_indices(s.rows, s.zipf, s.seed, batch, stream, idx.data()) != EMBC_OK)
    throw ValueError("lookup generation failed");
  std::vector<float> out(static_cast<size_t>(batch) * s.dim);
  for (uint32_t i = 0; i < batch; ++i)
    std::memcpy(out.data() + static_cast<size_t>(i) * s.dim, table.data() + static_cast<size_t>(idx[i]) * s.dim,
                4 * s.dim);
  return out;
}

struct Dev {  // a device allocation
  void* p = nullptr;
  explicit Dev(size_t n) {
    if (cudaMalloc(&p, n ? n : 1) != cudaSuccess) throw Error("cudaMalloc failed");
  }
  ~Dev() { cudaFree(p); }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

// ---- CSV (csv.hpp) ----------------------------------------------------------
struct Csv {
  std::ostream& o;
  size_t n;
  Csv(std::ostream& out, const std::string& schema, const std::vector<std::string>& cols) : o(out), n(cols.size()) {
    o << "# schema: " << schema << "\n";
    row(cols);
  }
  void row(const std::vector<std::string>& f) {
    if (f.size() != n)
      throw Error("csv row has " + std::to_string(f.size()) + " fields, expected " + std::to_string(n));
    for (size_t i = 0; i < f.size(); ++i) o << (i ? "," : "") << f[i];
    o << "\n";
  }
};

std::string fmt(double v) { return format_double(v); }

std::vector<uint8_t> read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Error("cannot open file '" + path + "'");
  return std::vector<uint8_t>((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}

void write_file(const std::string& path, const std::vector<uint8_t>& d) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw Error("cannot write file '" + path + "'");
  out.write(reinterpret_cast<const char*>(d.data()), static_cast<std::streamsize>(d.size()));
  if (!out) throw Error("short write to '" + path + "'");
}

// .embv value file (valuefile.hpp:28-64): "EMBV", u8 1, u32 dim, u32 count, f64 values
struct Values {
  uint32_t dim = 0, count = 0;
  std::vector<double> v;
};

Values parse_values(const std::vector<uint8_t>& d) {
  auto need = [&](size_t pos, size_t n) {
    if (d.size() < pos + n)
      throw FormatError("truncated input: need " + std::to_string(n) + " bytes at offset " + std::to_string(pos) +
                        ", have " + std::to_string(d.size() > pos ? d.size() - pos : 0));
  };
  need(0, 4);
  if (std::memcmp(d.data(), "EMBV", 4) != 0) throw FormatError("bad value file magic");
  need(4, 1);
  if (d[4] != 1) throw FormatError("unsupported value file version " + std::to_string(d[4]));
  need(5, 8);
  Values b;
  std::memcpy(&b.dim, d.data() + 5, 4);
  std::memcpy(&b.count, d.data() + 9, 4);
  const size_t n = static_cast<size_t>(b.dim) * b.count;
  if (d.size() - 13 != 8 * n)
    throw FormatError("value file holds " + std::to_string((d.size() - 13) / 8) + " values, header claims " +
                      std::to_string(n));
  b.v.resize(n);
  std::memcpy(b.v.data(), d.data() + 13, 8 * n);
  return b;
}

std::vector<uint8_t> serialize_values(const Values& b) {
  std::vector<uint8_t> d(13 + 8 * b.v.size());
  std::memcpy(d.data(), "EMBV", 4);
  d[4] = 1;
  std::memcpy(d.data() + 5, &b.dim, 4);
  std::memcpy(d.data() + 9, &b.count, 4);
  std::memcpy(d.data() + 13, b.v.data(), 8 * b.v.size());
  return d;
}

Codec codec_from(const std::string& s) {
  if (s == "raw") return Codec::raw;
  if (s == "vlz") return Codec::vlz;
  if (s == "huffman") return Codec::huffman;
  throw ConfigError("unknown codec '" + s + "'");
}

// ---- subcommands --------------------------------------------------------------
struct DevSample {
  Dev d;
  Sample s;
  DevSample(const TableSpec& t, const std::vector<float>& v) : d(4 * v.size()) {
    cudaMemcpy(d.p, v.data(), 4 * v.size(), cudaMemcpyHostToDevice);
    s = Sample{t.table_id, d.as<float>(), t.dim, static_cast<uint32_t>(v.size() / t.dim)};
  }
};

int cmd_analyze(const std::string& config, std::optional<uint64_t> seed_flag, std::optional<double> bw_flag,
                const std::string& profiles_out, const std::string& csv_out, const std::string& dump_dir) {
  const KeyValue kv = KeyValue::parse_file(config);
  const PolicyConfig policy = load_policy(kv);
  const uint64_t seed = seed_flag ? *seed_flag : kv.u64("seed", 1);
  const double bw = bw_flag.value_or(kv.f64("bandwidth", 4e9));
  const uint32_t batch = static_cast<uint32_t>(kv.u64("batch", 128));
  const auto tables = seeded(kv, seed);
  Context ctx(0);
  std::vector<std::unique_ptr<DevSample>> ds;
  std::vector<Sample> samples;
  for (const auto& t : tables) {
    ds.push_back(std::make_unique<DevSample>(t, lookup_batch(t, batch, 0)));
    samples.push_back(ds.back()->s);
  }
  const auto profiles = offline_analysis(ctx, samples, policy, bw, 255, true);
  std::cout << "table  survival  homo      class   eb        codec\n";
  for (const auto& [id, p] : profiles)
    std::cout << id << "  " << fmt(p.survival_ratio) << "  " << fmt(p.homo_index) << "  " << table_class_name(p.cls)
              << "  " << fmt(p.eb) << "  " << codec_name(p.codec) << "\n";
  if (!profiles_out.empty()) {
    write_profiles(profiles_out, profiles);
    std::cout << "profiles written to " << profiles_out << "\n";
  }
  if (!csv_out.empty()) {
    std::ofstream out(csv_out);
    if (!out) throw Error("cannot write '" + csv_out + "'");
    Csv csv(out, "embc.analyze.v1", {"table_id", "survival_ratio", "homo_index", "class", "eb", "cr_vlz", "cr_huff", "codec"});
    for (const auto& [id, p] : profiles) {
      double cv = 0.0, ch = 0.0;
      for (const auto& m : p.measured) (m.codec == Codec::vlz ? cv : ch) = m.ratio;
      csv.row({std::to_string(id), fmt(p.survival_ratio), fmt(p.homo_index), table_class_name(p.cls), fmt(p.eb),
               fmt(cv), fmt(ch), codec_name(p.codec)});
    }
    std::cout << "csv written to " << csv_out << "\n";
  }
  if (!dump_dir.empty()) {  // sample batches as raw-codes chunks at their profile bound
    std::filesystem::create_directories(dump_dir);
    for (const Sample& s : samples) {
      const auto& p = profiles.at(s.table_id);
      const EncodeJob job{s.d_values, s.dim, s.rows, p.eb, Codec::raw, 255};
      write_file(dump_dir + "/table_" + std::to_string(s.table_id) + ".embc", encode_chunk(ctx, job));
    }
    std::cout << "sample batches dumped to " << dump_dir << "\n";
  }
  return 0;
}

int cmd_compress(const std::string& in, const std::string& out, double eb, const std::string& codec_name_s,
                 uint32_t window, double bw) {
  const Values b = parse_values(read_file(in));
  if (b.dim == 0) throw ValueError("embedding batch dim must be >= 1");
  if (!(std::isfinite(eb) && eb > 0.0)) throw ValueError("error bound must be finite and > 0, got " + std::to_string(eb));
  if (window < 1 || window > 65536) throw ValueError("vlz window must be in [1, 65536], got " + std::to_string(window));
  Context ctx(0);
  const size_t n = b.v.size();
  // the values are doubles: quantize them on the device, then encode the codes
  Dev dx(8 * n), dc(4 * n);
  cudaMemcpy(dx.p, b.v.data(), 8 * n, cudaMemcpyHostToDevice);
  ctx.check(embc_quantize(ctx.get(), dx.p, 1, n, eb, dc.as<int32_t>(), nullptr));
  ctx.sync();
  Codec codec;
  if (codec_name_s == "auto") {
    // select_codec (policy.hpp:239-274) on the fp32 view when exact, else by ratio
    std::vector<float> f(n);
    bool exact = true;
    for (size_t i = 0; i < n; ++i) {
      f[i] = static_cast<float>(b.v[i]);
      exact = exact && static_cast<double>(f[i]) == b.v[i];
    }
    Dev df(4 * n);
    cudaMemcpy(df.p, f.data(), 4 * n, cudaMemcpyHostToDevice);
    const Codec cands[2] = {Codec::vlz, Codec::huffman};
    codec = select_codec(ctx, Sample{0, df.as<float>(), b.dim, b.count}, eb, cands, bw, window, exact, nullptr);
  } else {
    codec = codec_from(codec_name_s);
  }
  embc_job j{};
  j.src = dc.p;
  j.dim = b.dim;
  j.n = b.count;
  j.eb = eb;
  j.window = window;
  j.codec = static_cast<uint8_t>(codec);
  j.src_kind = EMBC_SRC_I32;
  const uint64_t cap = embc_encode_bound(&j, 1, EMBC_LAYOUT_CHUNKS);
  Dev dout(cap), dtot(8);
  ctx.check(embc_encode(ctx.get(), &j, 1, EMBC_LAYOUT_CHUNKS, dout.as<uint8_t>(), cap, nullptr, nullptr, nullptr,
                        dtot.as<uint64_t>(), nullptr));
  ctx.sync();
  uint64_t total = 0;
  cudaMemcpy(&total, dtot.p, 8, cudaMemcpyDeviceToHost);
  std::vector<uint8_t> chunk(total);
  cudaMemcpy(chunk.data(), dout.p, total, cudaMemcpyDeviceToHost);
  write_file(out, chunk);
  std::cout << "codec " << codec_name(codec) << ", " << b.count << " x " << b.dim << " values, ratio "
            << fmt(4.0 * static_cast<double>(n) / static_cast<double>(total - kHeaderSize)) << "\n";
  return 0;
}

int cmd_decompress(const std::string& in, const std::string& out) {
  const std::vector<uint8_t> c = read_file(in);
  // the header fields the device decode is planned with (parse_chunk re-checks all of them)
  uint32_t dim = 0, count = 0;
  uint8_t codec = 0;
  double eb = 0.0;
  if (c.size() >= kHeaderSize) {
    codec = c[5];
    std::memcpy(&eb, c.data() + 6, 8);
    std::memcpy(&dim, c.data() + 14, 4);
    std::memcpy(&count, c.data() + 18, 4);
  }
  Context ctx(0);
  Dev din(c.size() + 16), dout(8ull * dim * count + 8);
  cudaMemcpy(din.p, c.data(), c.size(), cudaMemcpyHostToDevice);
  embc_chunk_ref r{};
  r.offset = 0;
  r.length = c.size();
  r.out = dout.p;
  r.dim = dim;
  r.count = count;
  r.codec = codec > 2 ? 0 : codec;
  if (codec > 2) {  // parse_chunk's own message (container.hpp:100-102)
    throw FormatError("unknown codec tag " + std::to_string(codec));
  }
  ctx.check(embc_decode(ctx.get(), din.as<uint8_t>(), &r, 1, EMBC_OUT_F64, 0, nullptr));
  ctx.sync();
  Values b;
  b.dim = dim;
  b.count = count;
  b.v.resize(static_cast<size_t>(dim) * count);
  cudaMemcpy(b.v.data(), dout.p, 8 * b.v.size(), cudaMemcpyDeviceToHost);
  write_file(out, serialize_values(b));
  std::cout << "decoded " << count << " x " << dim << " values (codec " << codec_name(static_cast<Codec>(codec))
            << ", eb " << fmt(eb) << ")\n";
  return 0;
}

int cmd_bench(const std::string& config, std::optional<uint64_t> seed_flag, std::optional<double> bw_flag,
              uint32_t window, const std::string& csv_out) {
  const KeyValue kv = KeyValue::parse_file(config);
  const PolicyConfig policy = load_policy(kv);
  const uint64_t seed = seed_flag ? *seed_flag : kv.u64("seed", 1);
  const double bw = bw_flag.value_or(kv.f64("bandwidth", 4e9));
  const uint32_t batch = static_cast<uint32_t>(kv.u64("batch", 128));
  const auto tables = seeded(kv, seed);
  std::ostream* out = &std::cout;
  std::ofstream file;
  if (!csv_out.empty()) {
    file.open(csv_out);
    if (!file) throw Error("cannot write '" + csv_out + "'");
    out = &file;
  }
  Csv csv(*out, "embc.bench.v1", {"table_id", "codec", "eb", "compression_ratio", "comp_bps", "decomp_bps", "est_speedup"});
  Context ctx(0);
  const Codec cands[3] = {Codec::raw, Codec::vlz, Codec::huffman};
  for (const auto& t : tables) {
    DevSample s(t, lookup_batch(t, batch, 0));
    std::vector<ThroughputSample> m;
    select_codec(ctx, s.s, policy.global_eb, cands, bw, window, true, &m);
    for (const auto& x : m)
      csv.row({std::to_string(t.table_id), codec_name(x.codec), fmt(policy.global_eb), fmt(x.ratio), fmt(x.comp_bps),
               fmt(x.decomp_bps), fmt(estimate_speedup(x.ratio, bw, x.comp_bps, x.decomp_bps))});
  }
  if (!csv_out.empty()) std::cout << "csv written to " << csv_out << "\n";
  return 0;
}

int cmd_simulate(const std::string& config, uint64_t seed, const std::string& csv_out, const std::string& prof_path,
                 std::optional<uint64_t> ranks_f, std::optional<double> bw_f, std::optional<double> lat_f,
                 std::optional<uint64_t> iters_f, std::optional<std::string> comp_f) {
  const KeyValue kv = KeyValue::parse_file(config);
  // load_sim_config (config.hpp:227-243) + the command-line overrides (embc_main.cpp:187-202)
  uint32_t ranks = static_cast<uint32_t>(kv.u64("ranks", 4));
  double bw = kv.f64("bandwidth", 4e9), lat = kv.f64("latency", 0.0);
  uint32_t iters = static_cast<uint32_t>(kv.u64("iterations", 1));
  const uint32_t batch = static_cast<uint32_t>(kv.u64("batch", 128));
  bool comp = kv.flag("compression", true);
  (void)kv.u64("workers", 1);
  const PolicyConfig policy = load_policy(kv);
  std::vector<TableSpec> tables = load_tables(kv);
  if (ranks_f) ranks = static_cast<uint32_t>(*ranks_f);
  if (bw_f) bw = *bw_f;
  if (lat_f) lat = *lat_f;
  if (iters_f) iters = static_cast<uint32_t>(*iters_f);
  if (comp_f) {
    if (*comp_f == "on") comp = true;
    else if (*comp_f == "off") comp = false;
    else throw ConfigError("--compression expects on|off");
  }
  if (ranks < 2) throw ConfigError("simulation needs at least 2 ranks");
  if (!(bw > 0.0)) throw ConfigError("bandwidth must be > 0");
  if (lat < 0.0) throw ConfigError("latency must be >= 0");
  if (iters < 1) throw ConfigError("iterations must be >= 1");
  if (batch < 1) throw ConfigError("batch must be >= 1");
  // profiles: from the file, or analyze_sim_tables (commsim.hpp:493-503) on the GPU
  std::map<int32_t, TableProfile> profiles;
  if (!prof_path.empty()) {
    profiles = read_profiles(prof_path);
  } else {
    Context ctx(0);
    std::vector<std::unique_ptr<DevSample>> ds;
    std::vector<Sample> samples;
    for (uint32_t r = 0; r < ranks; ++r) {
      TableSpec t = tables[r % tables.size()];
      t.table_id = static_cast<int32_t>(r);
      t.seed = embc_mix_seed(seed, 0x7AB1Eull ^ r);
      ds.push_back(std::make_unique<DevSample>(t, lookup_batch(t, batch, 0)));
      samples.push_back(ds.back()->s);
    }
    profiles = offline_analysis(ctx, samples, policy, bw, 255, true);
  }
  embc_sim_config c{};
  c.ranks = ranks;
  c.batch = batch;
  c.iterations = iters;
  c.compression = comp ? 1 : 0;
  c.seed = seed;
  c.global_eb = policy.global_eb;
  c.decay_fn = static_cast<int32_t>(policy.decay.function);
  c.decay_steps = policy.decay.step_count;
  c.decay_start_scale = policy.decay.start_scale;
  c.decay_end = policy.decay.decay_end;
  std::vector<embc_sim_table> st(tables.size());
  for (size_t i = 0; i < tables.size(); ++i) {
    st[i].rows = tables[i].rows;
    st[i].dim = tables[i].dim;
    st[i].dist = tables[i].dist;
    st[i].mu = tables[i].mu;
    st[i].sigma = tables[i].sigma;
    st[i].lo = tables[i].lo;
    st[i].hi = tables[i].hi;
    st[i].zipf_s = tables[i].zipf;
  }
  std::vector<uint8_t> pc(ranks);
  std::vector<double> pe(ranks);
  for (uint32_t r = 0; r < ranks; ++r) {
    const auto it = profiles.find(static_cast<int32_t>(r));
    pc[r] = it != profiles.end() ? static_cast<uint8_t>(it->second.codec) : 0;
    pe[r] = it != profiles.end() ? it->second.eb : policy.global_eb;
  }
  std::vector<embc_sim_iteration> its(iters);
  uint64_t digest = 0;
  embc_error err{};
  const embc_status s = embc_simulate(0, &c, st.data(), static_cast<uint32_t>(st.size()), pc.data(), pe.data(),
                                      its.data(), &digest, &err);
  throw_for(s, err);
  // modeled times (commsim.hpp:466-475) and the aggregate model (:176-197)
  double unc = 0, pay = 0, wire = 0, comp_t = 0, dec_t = 0, maxerr = 0;
  bool conserved = true;
  std::vector<std::vector<std::string>> rows;
  for (const auto& it : its) {
    const double rl = ranks * lat;
    const double base = static_cast<double>(it.uncompressed_bytes) / bw + rl;
    const double wt = static_cast<double>(it.wire_bytes) / bw + rl;
    const double sp = comp ? base / (it.comp_time + it.decomp_time + wt) : 1.0;
    rows.push_back({std::to_string(it.iteration), fmt(it.eb_max), std::to_string(it.uncompressed_bytes),
                    std::to_string(it.payload_bytes), std::to_string(it.metadata_bytes), std::to_string(it.wire_bytes),
                    fmt(it.comp_time), fmt(it.decomp_time), fmt(base), fmt(wt), fmt(sp), fmt(it.max_abs_error)});
    unc += static_cast<double>(it.uncompressed_bytes);
    pay += static_cast<double>(it.payload_bytes);
    wire += static_cast<double>(it.wire_bytes);
    comp_t += it.comp_time;
    dec_t += it.decomp_time;
    maxerr = std::max(maxerr, it.max_abs_error);
    conserved = conserved && it.delivery_conserved;
  }
  if (!csv_out.empty()) {
    std::ofstream out(csv_out);
    if (!out) throw Error("cannot write '" + csv_out + "'");
    Csv csv(out, "embc.simulate.v1",
            {"iteration", "eb_max", "uncompressed_bytes", "payload_bytes", "metadata_bytes", "wire_bytes", "comp_time_s",
             "decomp_time_s", "modeled_base_time_s", "modeled_wire_time_s", "modeled_speedup", "max_abs_error"});
    for (const auto& r : rows) csv.row(r);
  }
  auto ratio = [&](uint64_t b, uint64_t e) {
    uint64_t u = 0, p = 0;
    for (const auto& it : its)
      if (it.iteration >= b && it.iteration < e) {
        u += it.uncompressed_bytes;
        p += it.payload_bytes;
      }
    return p == 0 ? 1.0 : static_cast<double>(u) / static_cast<double>(p);
  };
  std::cout << "== embc simulate (GPU codec) ==\n"
            << "ranks " << ranks << "  iterations " << iters << "  batch " << batch << "  compression "
            << (comp ? "on" : "off") << "  bandwidth " << fmt(bw) << " B/s  latency " << fmt(lat) << " s\n"
            << "wire bytes:        " << static_cast<uint64_t>(unc) << " -> " << static_cast<uint64_t>(wire)
            << " (payload " << static_cast<uint64_t>(pay) << " + metadata " << static_cast<uint64_t>(wire - pay) << ")\n"
            << "compression ratio: " << fmt(ratio(0, ~0ull)) << " overall";
  const uint64_t dend = policy.decay.decay_end;
  if (dend > 0 && !its.empty()) {
    if (its.front().iteration < dend) std::cout << " | initial phase " << fmt(ratio(0, dend));
    if (its.back().iteration >= dend) std::cout << " | later phase " << fmt(ratio(dend, ~0ull));
  }
  std::cout << "\nmax abs error:     " << fmt(maxerr) << " (delivery conserved: " << (conserved ? "yes" : "NO") << ")\n";
  if (comp) {
    const double base = unc / bw + its.size() * ranks * lat, wt = wire / bw + its.size() * ranks * lat;
    const double cr = pay > 0 ? unc / pay : 1.0;
    const double cb = unc / std::max(comp_t, 1e-12), db = unc / std::max(dec_t, 1e-12);
    std::cout << "codec time:        compress " << fmt(comp_t) << " s, decompress " << fmt(dec_t) << " s\n"
              << "modeled speedup:   " << fmt(base / (comp_t + dec_t + wt)) << " (closed-form estimate "
              << fmt(estimate_speedup(cr, bw, cb, db)) << ")\n";
  } else {
    std::cout << "modeled speedup:   1 (baseline)\n";
  }
  std::cout << "report digest:     " << digest << "\n";
  if (!csv_out.empty()) std::cout << "csv written to " << csv_out << "\n";
  return 0;
}

bool is_number(const std::string& s) {
  return !s.empty() && s.find_first_not_of("0123456789+-.eE") == std::string::npos &&
         s.find_first_of("0123456789") != std::string::npos;
}

int cmd_report(const std::vector<std::string>& paths) {  // pretty-printed csv with column means
  for (const auto& path : paths) {
    std::ifstream in(path);
    if (!in) throw Error("cannot open csv file '" + path + "'");
    std::string schema, line;
    std::vector<std::string> header;
    std::vector<std::vector<std::string>> rows;
    bool seen = false;
    while (std::getline(in, line)) {
      if (!line.empty() && line.back() == '\r') line.pop_back();
      if (line.empty()) continue;
      if (line[0] == '#') {
        if (line.rfind("# schema: ", 0) == 0) schema = line.substr(10);
        continue;
      }
      std::vector<std::string> f;
      std::stringstream ss(line);
      std::string x;
      while (std::getline(ss, x, ',')) f.push_back(x);
      if (!line.empty() && line.back() == ',') f.push_back("");
      if (!seen) {
        header = f;
        seen = true;
      } else {
        rows.push_back(f);
      }
    }
    std::cout << "== " << path;
    if (!schema.empty()) std::cout << " (" << schema << ")";
    std::cout << " ==\n";
    if (header.empty()) {
      std::cout << "(empty)\n";
      continue;
    }
    std::vector<size_t> w(header.size());
    for (size_t c = 0; c < header.size(); ++c) w[c] = header[c].size();
    for (const auto& r : rows)
      for (size_t c = 0; c < r.size() && c < w.size(); ++c) w[c] = std::max(w[c], r[c].size());
    auto print = [&](const std::vector<std::string>& r) {
      for (size_t c = 0; c < r.size(); ++c) {
        const size_t pad = c < w.size() && w[c] > r[c].size() ? w[c] - r[c].size() : 0;
        std::cout << (c ? "  " : "") << r[c] << std::string(pad, ' ');
      }
      std::cout << "\n";
    };
    print(header);
    for (const auto& r : rows) print(r);
    if (!rows.empty()) {
      std::vector<std::string> means(header.size());
      bool any = false;
      for (size_t c = 0; c < header.size(); ++c) {
        double sum = 0.0;
        size_t n = 0;
        for (const auto& r : rows)
          if (c < r.size() && is_number(r[c])) {
            sum += std::stod(r[c]);
            ++n;
          }
        if (n == rows.size()) {
          means[c] = "mean " + fmt(sum / static_cast<double>(n));
          any = true;
        }
      }
      if (any) print(means);
    }
  }
  return 0;
}

// ---- argument parsing ------------------------------------------------------------
struct Args {
  std::map<std::string, std::string> opt;
  std::vector<std::string> pos;
  bool has(const std::string& k) const { return opt.count(k) != 0; }
  std::string get(const std::string& k, const std::string& d = "") const { return has(k) ? opt.at(k) : d; }
  std::string req(const std::string& k) const {
    if (!has(k)) throw ConfigError(k + " is required");
    return opt.at(k);
  }
};

uint64_t to_u64(const std::string& k, const std::string& v) {
  uint64_t out = 0;
  const auto [p, ec] = std::from_chars(v.data(), v.data() + v.size(), out);
  if (ec != std::errc() || p != v.data() + v.size()) throw ConfigError(k + ": expected an integer, got '" + v + "'");
  return out;
}
double to_f64(const std::string& k, const std::string& v) {
  double out = 0.0;
  const auto [p, ec] = std::from_chars(v.data(), v.data() + v.size(), out);
  if (ec != std::errc() || p != v.data() + v.size()) throw ConfigError(k + ": expected a number, got '" + v + "'");
  return out;
}

const char* kUsage =
    "embc_gpu: embedding-lookup compression toolkit (GPU codec)\n"
    "usage: embc_gpu <command> [options]\n"
    "  analyze    --config C [--seed S] [--bandwidth B] [--out PROFILES] [--csv F] [--dump-dir D]\n"
    "  compress   --in VALUES.embv --out CHUNK.embc --eb E [--codec auto|raw|vlz|huffman] [--window W] [--bandwidth B]\n"
    "  decompress --in CHUNK.embc --out VALUES.embv\n"
    "  bench      --config C [--seed S] [--bandwidth B] [--window W] [--out F]\n"
    "  simulate   --config C --seed S [--out F] [--profiles P] [--ranks R] [--bandwidth B] [--latency L]\n"
    "             [--iterations N] [--workers W] [--compression on|off]\n"
    "  report     FILE.csv...\n";

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h") {
    std::cout << kUsage;
    return argc < 2 ? 1 : 0;
  }
  const std::string cmd = argv[1];
  static const std::map<std::string, std::vector<std::string>> known = {
      {"analyze", {"--config", "--seed", "--bandwidth", "--out", "--csv", "--dump-dir"}},
      {"compress", {"--in", "--out", "--eb", "--codec", "--window", "--bandwidth"}},
      {"decompress", {"--in", "--out"}},
      {"bench", {"--config", "--seed", "--bandwidth", "--window", "--out"}},
      {"simulate", {"--config", "--seed", "--out", "--profiles", "--ranks", "--bandwidth", "--latency", "--iterations",
                    "--workers", "--compression"}},
      {"report", {}}};
  try {
    const auto k = known.find(cmd);
    if (k == known.end()) throw ConfigError("unknown command '" + cmd + "'\n" + kUsage);
    Args a;
    for (int i = 2; i < argc; ++i) {
      const std::string s = argv[i];
      if (s.rfind("--", 0) == 0) {
        if (std::find(k->second.begin(), k->second.end(), s) == k->second.end())
          throw ConfigError("unknown option " + s + " for " + cmd);
        if (i + 1 >= argc) throw ConfigError(s + " needs a value");
        a.opt[s] = argv[++i];
      } else {
        a.pos.push_back(s);
      }
    }
    auto opt_u64 = [&](const std::string& n) -> std::optional<uint64_t> {
      if (!a.has(n)) return std::nullopt;
      return to_u64(n, a.get(n));
    };
    auto opt_f64 = [&](const std::string& n) -> std::optional<double> {
      if (!a.has(n)) return std::nullopt;
      return to_f64(n, a.get(n));
    };
    if (cmd == "analyze")
      return cmd_analyze(a.req("--config"), opt_u64("--seed"), opt_f64("--bandwidth"), a.get("--out"), a.get("--csv"),
                         a.get("--dump-dir"));
    if (cmd == "compress") {
      const std::string codec = a.get("--codec", "auto");
      if (codec != "auto" && codec != "raw" && codec != "vlz" && codec != "huffman")
        throw ConfigError("--codec: " + codec + " not in {auto,raw,vlz,huffman}");
      return cmd_compress(a.req("--in"), a.req("--out"), to_f64("--eb", a.req("--eb")), codec,
                          static_cast<uint32_t>(opt_u64("--window").value_or(255)), opt_f64("--bandwidth").value_or(4e9));
    }
    if (cmd == "decompress") return cmd_decompress(a.req("--in"), a.req("--out"));
    if (cmd == "bench")
      return cmd_bench(a.req("--config"), opt_u64("--seed"), opt_f64("--bandwidth"),
                       static_cast<uint32_t>(opt_u64("--window").value_or(255)), a.get("--out"));
    if (cmd == "simulate") {
      std::optional<std::string> comp;
      if (a.has("--compression")) comp = a.get("--compression");
      (void)opt_u64("--workers");
      return cmd_simulate(a.req("--config"), to_u64("--seed", a.req("--seed")), a.get("--out"), a.get("--profiles"),
                          opt_u64("--ranks"), opt_f64("--bandwidth"), opt_f64("--latency"), opt_u64("--iterations"),
                          comp);
    }
    if (a.pos.empty()) throw ConfigError("report needs at least one csv file");
    return cmd_report(a.pos);
  } catch (const std::exception& e) {
    std::cerr << "embc: " << e.what() << "\n";
    return 2;
  }
}
