// libace.so — the reference's C++ ACE API (include/ace/b200_api.hpp) over the
// B200 C ABI (include/ace_b200.h).  Host responsibilities only: seeded W
// generation (construction time, must match glibc libm bit-for-bit, so it
// cannot move to the device), argument validation, exception mapping, and
// label tallies.  Every hash / count / score / threshold runs on the GPU.
#include <bit>
#include <fstream>
#include <type_traits>
#include <charconv>
#include <thread>
#include <optional>
#include <string_view>
#include <cstdlib>
#include <iterator>
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numbers>
#include <string>

#include "ace/b200_api.hpp"
#include "ace_b200.h"
#include "ace_host.h"

namespace ace {

namespace {

[[noreturn]] void raise(ace_status st) {
  const std::string msg = ace_last_error();
  switch (st) {
    case ACE_E_CONTRACT: throw ContractViolation(msg);
    case ACE_E_UNSUPPORTED: throw UnsupportedOperation(msg);
    case ACE_E_INCONSISTENT: throw InconsistentDelete(msg);
    case ACE_E_DATA: throw DataError(msg);
    default: throw std::runtime_error(msg);
  }
}

inline void ok(ace_status st) {
  if (st != ACE_OK) raise(st);
}

// Stream seed of direction (table, b): srp.cpp:17-20.
std::uint64_t seed_of(std::uint64_t master, std::size_t table, std::size_t b, std::uint32_t k) {
  return rng::mix_seed(master, table * k + b);
}

std::vector<double> generate_w(const SrpConfig& c) {
  std::vector<double> w(static_cast<std::size_t>(c.k_bits) * c.num_tables * c.dim);
  for (std::size_t t = 0; t < c.num_tables; ++t)
    for (std::size_t b = 0; b < c.k_bits; ++b) {
      rng::NormalStream g(seed_of(c.seed, t, b, c.k_bits));
      double* out = w.data() + (t * c.k_bits + b) * c.dim;
      for (std::size_t i = 0; i < c.dim; ++i) out[i] = g.next();
    }
  return w;
}

}  // namespace

// ---- rng: restatement of rng.hpp:10-58 ------------------------------------
namespace rng {
std::uint64_t splitmix64(std::uint64_t& state) {
  std::uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t index) {
  std::uint64_t s = seed ^ (0x9e3779b97f4a7c15ULL * (index + 1));
  return splitmix64(s);
}
double unit_double(std::uint64_t bits) { return static_cast<double>((bits >> 11) + 1) * 0x1.0p-53; }
std::uint64_t bounded(std::uint64_t bits, std::uint64_t bound) {
  return static_cast<std::uint64_t>((static_cast<unsigned __int128>(bits) * bound) >> 64);
}
double NormalStream::next() {
  if (cached_valid_) {
    cached_valid_ = false;
    return cached_;
  }
  const double u1 = unit_double(splitmix64(s_));
  const double u2 = unit_double(splitmix64(s_));
  const double radius = std::sqrt(-2.0 * std::log(u1));
  const double angle = 2.0 * std::numbers::pi * u2;
  cached_ = radius * std::sin(angle);
  cached_valid_ = true;
  return radius * std::cos(angle);
}
}  // namespace rng

// ---- SrpFamily --------------------------------------------------------------
SrpFamily::SrpFamily(const SrpConfig& cfg) : cfg_(cfg) {
  // srp.cpp:25-32
  if (cfg_.dim == 0) throw ContractViolation("SrpFamily: dim must be >= 1");
  if (cfg_.k_bits < 1 || cfg_.k_bits > 30) throw ContractViolation("SrpFamily: k_bits must be in [1, 30]");
  if (cfg_.num_tables < 1) throw ContractViolation("SrpFamily: num_tables must be >= 1");
  if (cfg_.noise_scale < 0.0) throw ContractViolation("SrpFamily: noise_scale must be >= 0");
  w_ = std::make_shared<const std::vector<double>>(generate_w(cfg_));
  dev_ = std::make_shared<std::shared_ptr<::AceFamily>>();
  noise_seed_ = rng::mix_seed(cfg_.seed, 0x6e6f697365ULL);  // srp.cpp:34, the aux stream
}

std::vector<double> SrpFamily::draw_noise(std::size_t count) const {
  const std::uint64_t tick0 = noise_ctr_.v.fetch_add(count, std::memory_order_relaxed);
  std::vector<double> out(count);
  if (count) ace_noise_terms(noise_seed_, tick0, count, cfg_.noise_scale, out.data());
  return out;
}

std::vector<std::uint32_t> SrpFamily::noisy_ids(const void* x, int dtype, std::size_t n, std::size_t t0,
                                                std::size_t nt, std::size_t b0, std::size_t nb) const {
  const auto noise = draw_noise(n * nt * nb);
  std::vector<std::uint32_t> ids(n * nt);
  if (n && nt)
    ok(ace_family_buckets_noisy(device(), x, dtype, n, cfg_.dim, ACE_HOST, static_cast<std::uint32_t>(t0),
                                static_cast<std::uint32_t>(nt), static_cast<std::uint32_t>(b0),
                                static_cast<std::uint32_t>(nb), noise.data(), ACE_HOST, ids.data(), ACE_HOST));
  return ids;
}

::AceFamily* SrpFamily::device() const {
  if (!*dev_) {
    ::AceFamily* f = nullptr;
    ok(ace_family_create(cfg_.dim, cfg_.k_bits, cfg_.num_tables, cfg_.noise_scale, w_->data(), &f));
    *dev_ = std::shared_ptr<::AceFamily>(f, [](::AceFamily* p) { ace_family_destroy(p); });
  }
  return dev_->get();
}

void SrpFamily::check(std::size_t table, std::size_t b, std::span<const double> x) const {
  // srp.cpp:66-76
  if (x.size() != cfg_.dim)
    throw ContractViolation("SrpFamily: expected vector of length " + std::to_string(cfg_.dim) +
                            ", received " + std::to_string(x.size()));
  if (table >= cfg_.num_tables) throw ContractViolation("SrpFamily: table index out of range");
  if (b >= cfg_.k_bits) throw ContractViolation("SrpFamily: bit index out of range");
}

std::uint32_t SrpFamily::bucket(std::size_t table, std::span<const double> x) const {
  check(table, 0, x);
  if (cfg_.noise_scale > 0.0) return noisy_ids(x.data(), ACE_F64, 1, table, 1, 0, cfg_.k_bits)[0];
  std::vector<std::uint32_t> ids(cfg_.num_tables);
  ok(ace_family_buckets(device(), x.data(), ACE_F64, 1, cfg_.dim, ACE_HOST, ids.data(), ACE_HOST,
                        nullptr));
  return ids[table];
}

std::uint32_t SrpFamily::bit(std::size_t table, std::size_t b, std::span<const double> x) const {
  check(table, b, x);
  if (cfg_.noise_scale > 0.0) return noisy_ids(x.data(), ACE_F64, 1, table, 1, b, 1)[0];  // one tick
  return (bucket(table, x) >> (cfg_.k_bits - 1 - b)) & 1u;
}

std::vector<std::uint32_t> SrpFamily::buckets(std::span<const float> rows, std::size_t n) const {
  if (rows.size() != n * cfg_.dim) throw ContractViolation("SrpFamily::buckets: rows size != n * dim");
  if (cfg_.noise_scale > 0.0) return noisy_ids(rows.data(), ACE_F32, n, 0, cfg_.num_tables, 0, cfg_.k_bits);
  std::vector<std::uint32_t> ids(n * cfg_.num_tables);
  if (n)
    ok(ace_family_buckets(device(), rows.data(), ACE_F32, n, cfg_.dim, ACE_HOST, ids.data(),
                          ACE_HOST, nullptr));
  return ids;
}

std::vector<double> SrpFamily::direction(std::size_t table, std::size_t b) const {
  if (table >= cfg_.num_tables || b >= cfg_.k_bits)
    throw ContractViolation("SrpFamily: direction index out of range");
  const double* row = w_->data() + (table * cfg_.k_bits + b) * cfg_.dim;
  return std::vector<double>(row, row + cfg_.dim);
}

void SrpFamily::reset_noise_stream(std::uint64_t aux_seed) const {
  // srp.cpp:126-129
  noise_seed_ = aux_seed;
  noise_ctr_.v.store(0, std::memory_order_relaxed);
}

// collision_probability (srp.cpp:130-146): closed-form statistic, not on the
// hashing path; kept for API completeness.
double collision_probability(std::span<const double> x, std::span<const double> y) {
  if (x.size() != y.size()) throw ContractViolation("collision_probability: length mismatch");
  double xy = 0.0, xx = 0.0, yy = 0.0;
  for (std::size_t i = 0; i < x.size(); ++i) {
    xy += x[i] * y[i];
    xx += x[i] * x[i];
    yy += y[i] * y[i];
  }
  if (xx == 0.0 || yy == 0.0)
    throw std::domain_error("collision_probability: zero-norm vector, cosine undefined");
  double c = xy / (std::sqrt(xx) * std::sqrt(yy));
  c = c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);
  return 1.0 - std::acos(c) / std::numbers::pi;
}

// ---- AceSketch --------------------------------------------------------------
AceSketch::AceSketch(const SrpFamily& family, CounterWidth width) : family_(family), width_(width) {
  ok(ace_sketch_create(family_.device(), static_cast<std::uint32_t>(width_), &dev_));
}

AceSketch::AceSketch(const AceSketch& o) : family_(o.family_), width_(o.width_) {
  ok(ace_sketch_clone(o.dev_, &dev_));
}

AceSketch& AceSketch::operator=(const AceSketch& o) {
  if (this == &o) return *this;
  ::AceSketch* d = nullptr;
  ok(ace_sketch_clone(o.dev_, &d));
  ace_sketch_destroy(dev_);
  dev_ = d;
  family_ = o.family_;
  width_ = o.width_;
  return *this;
}

AceSketch::AceSketch(AceSketch&& o) noexcept : family_(o.family_), width_(o.width_), dev_(o.dev_) {
  o.dev_ = nullptr;
}

AceSketch& AceSketch::operator=(AceSketch&& o) noexcept {
  if (this != &o) {
    ace_sketch_destroy(dev_);
    family_ = o.family_;
    width_ = o.width_;
    dev_ = o.dev_;
    o.dev_ = nullptr;
  }
  return *this;
}

AceSketch::~AceSketch() { ace_sketch_destroy(dev_); }

void AceSketch::check_dim(std::span<const double> x) const {
  // sketch.cpp:19-24
  if (x.size() != family_.config().dim)
    throw ContractViolation("AceSketch: expected vector of length " +
                            std::to_string(family_.config().dim) + ", received " +
                            std::to_string(x.size()));
}

void AceSketch::insert(std::span<const double> x) {
  check_dim(x);
  if (family_.config().noise_scale > 0.0) {
    const auto ids = family_.noisy_ids(x.data(), ACE_F64, 1, 0, family_.config().num_tables, 0,
                                       family_.config().k_bits);
    ok(ace_sketch_insert_ids(dev_, ids.data(), 1, ACE_HOST));
    return;
  }
  ok(ace_sketch_insert(dev_, x.data(), ACE_F64, 1, x.size(), ACE_HOST, nullptr));
}

void AceSketch::remove(std::span<const double> x) {
  check_dim(x);
  if (family_.config().noise_scale > 0.0)  // sketch.cpp:76-79
    throw UnsupportedOperation(
        "AceSketch: delete is unsupported with noisy hashes (buckets are not reproducible)");
  ok(ace_sketch_remove(dev_, x.data(), ACE_F64, 1, x.size(), ACE_HOST, nullptr));
}

ScoreEstimate AceSketch::score(std::span<const double> q) const {
  check_dim(q);
  double v = 0.0;
  if (family_.config().noise_scale > 0.0) {
    const auto ids = family_.noisy_ids(q.data(), ACE_F64, 1, 0, family_.config().num_tables, 0,
                                       family_.config().k_bits);
    ok(ace_sketch_score_ids(dev_, ids.data(), 1, ACE_HOST, &v, nullptr, ACE_HOST));
    return {v, family_.config().k_bits, family_.config().num_tables};
  }
  ok(ace_sketch_score(dev_, q.data(), ACE_F64, 1, q.size(), ACE_HOST, &v, nullptr, ACE_HOST,
                      nullptr));
  return {v, family_.config().k_bits, family_.config().num_tables};
}

void AceSketch::insert_batch(std::span<const float> rows, std::size_t n) {
  const auto d = family_.config().dim;
  if (rows.size() != n * d) throw ContractViolation("AceSketch::insert_batch: rows size != n * dim");
  if (n && family_.config().noise_scale > 0.0) {
    const auto ids = family_.buckets(rows, n);  // noisy: ticks in row order
    ok(ace_sketch_insert_ids(dev_, ids.data(), n, ACE_HOST));
    return;
  }
  if (n) ok(ace_sketch_insert(dev_, rows.data(), ACE_F32, n, d, ACE_HOST, nullptr));
}

std::vector<double> AceSketch::score_batch(std::span<const float> rows, std::size_t n) const {
  const auto d = family_.config().dim;
  if (rows.size() != n * d) throw ContractViolation("AceSketch::score_batch: rows size != n * dim");
  std::vector<double> out(n);
  if (n && family_.config().noise_scale > 0.0) {
    const auto ids = family_.buckets(rows, n);
    ok(ace_sketch_score_ids(dev_, ids.data(), n, ACE_HOST, out.data(), nullptr, ACE_HOST));
    return out;
  }
  if (n)
    ok(ace_sketch_score(dev_, rows.data(), ACE_F32, n, d, ACE_HOST, out.data(), nullptr, ACE_HOST,
                        nullptr));
  return out;
}

std::uint64_t AceSketch::size() const {
  std::uint64_t n = 0;
  ok(ace_sketch_info(dev_, &n, nullptr, nullptr));
  return n;
}

double AceSketch::mean() const {
  double m = 0.0;
  ok(ace_sketch_info(dev_, nullptr, &m, nullptr));
  return m;
}

bool AceSketch::saturated() const {
  int s = 0;
  ok(ace_sketch_info(dev_, nullptr, nullptr, &s));
  return s != 0;
}

std::size_t AceSketch::counter_bytes() const {
  return num_counters() * (width_ == CounterWidth::k16 ? 2 : 4);
}

std::uint64_t AceSketch::counter(std::size_t table, std::size_t bucket) const {
  if (table >= family_.config().num_tables || bucket >= family_.num_buckets())
    throw ContractViolation("AceSketch: counter index out of range");
  std::uint64_t v = 0;
  ok(ace_sketch_counter(dev_, static_cast<std::uint32_t>(table), bucket, &v));
  return v;
}

std::vector<std::uint64_t> AceSketch::counters_flat() const {
  std::vector<std::uint64_t> out(num_counters());
  ok(ace_sketch_counters(dev_, out.data()));
  return out;
}

AceSketch AceSketch::restore(const SrpFamily& family, CounterWidth width,
                             std::vector<std::uint64_t> counters, std::uint64_t n, double mean,
                             bool saturated) {
  AceSketch s(family, width);
  ok(ace_sketch_restore(s.dev_, counters.data(), counters.size(), n, mean, saturated ? 1 : 0));
  return s;
}

// ---- detection --------------------------------------------------------------
DetectionReport detect_batch(const AceSketch& sketch, const Dataset& data, unsigned) {
  // detect.cpp:14-16
  if (data.rows == 0) throw ContractViolation("detect_batch: empty dataset");
  if (data.cols != sketch.family().config().dim)
    throw ContractViolation("detect_batch: data dimension mismatch");
  std::vector<std::uint32_t> bits((data.rows + 31) / 32);
  AceBatchReport r{};
  if (sketch.family().config().noise_scale > 0.0) {
    // noisy variant: scores with fresh noise (ticks in row order: the
    // reference's threads=1 order), then the reference's own statistics
    // (detect.cpp:44-60, sequential binary64 sums over the N scores)
    const auto t0 = std::chrono::steady_clock::now();
    const auto ids = sketch.family().noisy_ids(data.values.data(), ACE_F64, data.rows, 0,
                                               sketch.family().config().num_tables, 0,
                                               sketch.family().config().k_bits);
    std::vector<double> sc(data.rows);
    ok(ace_sketch_score_ids(sketch.device(), ids.data(), data.rows, ACE_HOST, sc.data(), nullptr, ACE_HOST));
    double sum = 0.0;
    for (double v : sc) sum += v;
    const double mean = sum / static_cast<double>(data.rows);
    double var = 0.0;
    for (double v : sc) var += (v - mean) * (v - mean);
    const double sd = std::sqrt(var / static_cast<double>(data.rows));
    r.score_mean = mean;
    r.score_stddev = sd;
    r.threshold = mean - sd;
    for (std::size_t i = 0; i < data.rows; ++i)
      if (sc[i] < r.threshold) {
        bits[i >> 5] |= 1u << (i & 31);
        ++r.reported;
      }
    r.elapsed_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  } else {
    ok(ace_sketch_detect_batch(sketch.device(), data.values.data(), ACE_F64, data.rows, data.cols,
                               ACE_HOST, bits.data(), nullptr, ACE_HOST, &r, nullptr));
  }
  DetectionReport rep;
  rep.reported = r.reported;
  rep.threshold = r.threshold;
  rep.score_mean = r.score_mean;
  rep.score_stddev = r.score_stddev;
  rep.elapsed_seconds = r.elapsed_seconds;
  rep.has_labels = data.labels.has_value();
  rep.total_labeled_anomalies = data.labeled_anomalies();
  if (rep.has_labels)  // label tallies, detect.cpp:59-68
    for (std::size_t i = 0; i < data.rows; ++i) {
      const bool flagged = (bits[i >> 5] >> (i & 31)) & 1u;
      const bool anomalous = (*data.labels)[i] != 0;
      if (flagged && anomalous) ++rep.correctly_reported;
      if (!flagged && anomalous) ++rep.missed;
    }
  return rep;
}

std::pair<ScoreEstimate, bool> detect_stream(const AceSketch& sketch, std::span<const double> q,
                                             double alpha) {
  // detect.cpp:79-83
  if (alpha < 0.0) throw ContractViolation("detect_stream: alpha must be >= 0");
  const auto& c = sketch.family().config();
  if (c.noise_scale > 0.0 || q.size() != c.dim) {
    if (sketch.size() == 0) throw ContractViolation("detect_stream: empty sketch");
    const ScoreEstimate e = sketch.score(q);
    return {e, e.value <= sketch.mean() - alpha};
  }
  // one call: score on the device, flag against the state it saw
  double v = 0.0;
  std::uint8_t f = 0;
  ok(ace_sketch_detect_stream(sketch.device(), q.data(), ACE_F64, 1, q.size(), ACE_HOST, alpha, &v, &f));
  return {ScoreEstimate{v, c.k_bits, c.num_tables}, f != 0};
}

std::vector<std::uint8_t> stream_batch(AceSketch& sketch, std::span<const float> rows, std::size_t n,
                                       double alpha) {
  const auto d = sketch.family().config().dim;
  if (rows.size() != n * d) throw ContractViolation("stream_batch: rows size != n * dim");
  std::vector<std::uint32_t> bits((n + 31) / 32);
  std::vector<std::uint8_t> flags(n);
  if (!n) return flags;
  ok(ace_sketch_stream_batch(sketch.device(), rows.data(), ACE_F32, n, d, ACE_HOST, alpha,
                             bits.data(), nullptr, ACE_HOST, nullptr, nullptr));
  for (std::size_t i = 0; i < n; ++i) flags[i] = (bits[i >> 5] >> (i & 31)) & 1u;
  return flags;
}

AceSketch build_sketch(const Dataset& data, std::uint32_t k_bits, std::uint32_t num_tables,
                       std::uint64_t seed, double noise_scale, CounterWidth width) {
  // estimators.cpp:79-92
  if (data.rows == 0) throw ContractViolation("build_sketch: empty dataset");
  SrpConfig cfg;
  cfg.dim = data.cols;
  cfg.k_bits = k_bits;
  cfg.num_tables = num_tables;
  cfg.seed = seed;
  cfg.noise_scale = noise_scale;
  AceSketch sketch{SrpFamily(cfg), width};
  if (noise_scale > 0.0) {  // rows in index order, ticks in row / table / bit order
    const auto ids = sketch.family().noisy_ids(data.values.data(), ACE_F64, data.rows, 0, num_tables, 0, k_bits);
    ok(ace_sketch_insert_ids(sketch.device(), ids.data(), data.rows, ACE_HOST));
    return sketch;
  }
  ok(ace_sketch_insert(sketch.device(), data.values.data(), ACE_F64, data.rows, data.cols, ACE_HOST,
                       nullptr));
  return sketch;
}

// ---- ACE1 sketch files (reference io.cpp:184-244) --------------------------
namespace io {
namespace {

// ---- CSV (reference io.cpp:20-49, 89-182) ----
std::string_view trim_csv(std::string_view s) {
  while (!s.empty() && (s.front() == ' ' || s.front() == '\t' || s.front() == '\r')) s.remove_prefix(1);
  while (!s.empty() && (s.back() == ' ' || s.back() == '\t' || s.back() == '\r')) s.remove_suffix(1);
  return s;
}

bool parse_cell(std::string_view token, double& out) {
  token = trim_csv(token);
  if (token.empty()) return false;
  const char* b = token.data();
  const char* e = b + token.size();
  auto [ptr, ec] = std::from_chars(b, e, out);
  return ec == std::errc{} && ptr == e;
}

// One non-empty line, parsed: its cells' values and the first unparsable cell.
struct ParsedLine {
  std::size_t line_number = 0;
  std::vector<double> cells;
  std::vector<std::string_view> raw;  // kept only when a cell fails to parse
  long bad = -1;                      // first unparsable cell, or -1
};

void parse_line(std::string_view view, ParsedLine& pl) {
  std::size_t start = 0;
  for (std::size_t i = 0; i <= view.size(); ++i) {
    if (i == view.size() || view[i] == ',') {
      const std::string_view cell = view.substr(start, i - start);
      double v = 0.0;
      if (!parse_cell(cell, v) && pl.bad < 0) pl.bad = static_cast<long>(pl.cells.size());
      pl.cells.push_back(v);
      pl.raw.push_back(cell);
      start = i + 1;
    }
  }
}

constexpr char kMagic[4] = {'A', 'C', 'E', '1'};

template <typename T>
void put_le(std::ostream& out, T v) {
  unsigned char b[sizeof(T)];
  for (std::size_t i = 0; i < sizeof(T); ++i)
    b[i] = static_cast<unsigned char>((static_cast<std::make_unsigned_t<T>>(v) >> (8 * i)) & 0xff);
  out.write(reinterpret_cast<const char*>(b), sizeof(T));
}

template <typename T>
T get_le(std::istream& in) {
  unsigned char b[sizeof(T)];
  in.read(reinterpret_cast<char*>(b), sizeof(T));
  if (!in) throw DataError("sketch file truncated");
  std::make_unsigned_t<T> v = 0;
  for (std::size_t i = 0; i < sizeof(T); ++i) v |= static_cast<std::make_unsigned_t<T>>(b[i]) << (8 * i);
  return static_cast<T>(v);
}
}  // namespace

Dataset load_dataset(const std::string& path, std::optional<int> label_column) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw DataError("cannot open dataset file: " + path);
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  // line table (std::getline semantics: '\n' separated, a final line without
  // '\n' still counts; trimming removes '\r')
  std::vector<std::pair<std::size_t, std::size_t>> lines;
  for (std::size_t pos = 0; pos < text.size();) {
    std::size_t nl = text.find('\n', pos);
    if (nl == std::string::npos) nl = text.size();
    lines.emplace_back(pos, nl - pos);
    pos = nl + 1;
  }
  // parse every line on all host threads (pure per line)
  std::vector<ParsedLine> parsed(lines.size());
  const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(),
                                                      static_cast<unsigned>(lines.size() / 4096 + 1)));
  std::vector<std::thread> pool;
  for (unsigned w = 0; w < nt; ++w)
    pool.emplace_back([&, w] {
      for (std::size_t i = w; i < lines.size(); i += nt) {
        const std::string_view view = trim_csv(std::string_view(text).substr(lines[i].first, lines[i].second));
        parsed[i].line_number = i + 1;
        if (!view.empty()) parse_line(view, parsed[i]);
      }
    });
  for (auto& t : pool) t.join();
  // the reference's validation, in line order
  Dataset data;
  data.name = path;
  std::vector<std::size_t> zero_rows;
  bool first_data_line = true;
  for (std::size_t i = 0; i < lines.size(); ++i) {
    const ParsedLine& pl = parsed[i];
    if (pl.cells.empty()) continue;  // blank line
    if (first_data_line && pl.bad == 0) continue;  // header line
    if (pl.bad >= 0)
      throw DataError("unparsable cell at row " + std::to_string(pl.line_number) + ", column " +
                      std::to_string(pl.bad + 1) + ": '" + std::string(trim_csv(pl.raw[pl.bad])) + "'");
    std::optional<std::size_t> label_index;
    if (label_column) {
      const int raw = *label_column;
      const long resolved = raw >= 0 ? raw : static_cast<long>(pl.cells.size()) + raw;
      if (resolved < 0 || resolved >= static_cast<long>(pl.cells.size()))
        throw DataError("label column " + std::to_string(raw) + " out of range at row " +
                        std::to_string(pl.line_number));
      label_index = static_cast<std::size_t>(resolved);
    }
    const std::size_t nf = pl.cells.size() - (label_index ? 1 : 0);
    if (first_data_line) {
      data.cols = nf;
      if (label_column) data.labels.emplace();
      first_data_line = false;
    } else if (nf != data.cols) {
      throw DataError("ragged row " + std::to_string(pl.line_number) + ": expected " + std::to_string(data.cols) +
                      " feature columns, found " + std::to_string(nf));
    }
    bool all_zero = true;
    for (std::size_t c = 0; c < pl.cells.size(); ++c)
      if ((!label_index || c != *label_index) && pl.cells[c] != 0.0) {
        all_zero = false;
        break;
      }
    if (all_zero) {
      zero_rows.push_back(pl.line_number);
      continue;
    }
    if (label_index) {
      const double lv = pl.cells[*label_index];
      if (lv != 0.0 && lv != 1.0)
        throw DataError("label at row " + std::to_string(pl.line_number) + " is not 0 or 1");
      data.labels->push_back(lv != 0.0 ? 1 : 0);
    }
    for (std::size_t c = 0; c < pl.cells.size(); ++c)
      if (!label_index || c != *label_index) data.values.push_back(pl.cells[c]);
    ++data.rows;
  }
  if (!zero_rows.empty()) {
    std::string rows;
    for (std::size_t i = 0; i < zero_rows.size(); ++i) rows += (i ? "," : "") + std::to_string(zero_rows[i]);
    throw DataError("all-zero feature rows rejected (cosine undefined): " + rows);
  }
  if (data.rows == 0) throw DataError("empty dataset file: " + path);
  return data;
}

void save_sketch(const AceSketch& sketch, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw DataError("cannot open sketch file for write: " + path);
  const auto& cfg = sketch.family().config();
  out.write(kMagic, 4);
  put_le(out, static_cast<std::uint32_t>(cfg.dim));
  put_le(out, cfg.k_bits);
  put_le(out, cfg.num_tables);
  put_le(out, static_cast<std::uint32_t>(sketch.counter_width()));
  put_le(out, cfg.seed);
  put_le(out, std::bit_cast<std::uint64_t>(cfg.noise_scale));
  put_le(out, sketch.size());
  put_le(out, std::bit_cast<std::uint64_t>(sketch.mean()));
  put_le(out, static_cast<std::uint8_t>(sketch.saturated() ? 1 : 0));
  const auto counters = sketch.counters_flat();
  if (sketch.counter_width() == CounterWidth::k16) {
    for (auto c : counters) put_le(out, static_cast<std::uint16_t>(c));
  } else {
    for (auto c : counters) put_le(out, static_cast<std::uint32_t>(c));
  }
  if (!out) throw DataError("write failed: " + path);
}

AceSketch load_sketch(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw DataError("cannot open sketch file: " + path);
  char magic[4];
  in.read(magic, 4);
  if (!in || std::memcmp(magic, kMagic, 4) != 0) throw DataError("bad magic in sketch file: " + path);
  SrpConfig cfg;
  cfg.dim = get_le<std::uint32_t>(in);
  cfg.k_bits = get_le<std::uint32_t>(in);
  cfg.num_tables = get_le<std::uint32_t>(in);
  const std::uint32_t width_bits = get_le<std::uint32_t>(in);
  cfg.seed = get_le<std::uint64_t>(in);
  cfg.noise_scale = std::bit_cast<double>(get_le<std::uint64_t>(in));
  const std::uint64_t n = get_le<std::uint64_t>(in);
  const double mean = std::bit_cast<double>(get_le<std::uint64_t>(in));
  const bool saturated = get_le<std::uint8_t>(in) != 0;
  if (width_bits != 16 && width_bits != 32)
    throw DataError("sketch file counter width must be 16 or 32, got " + std::to_string(width_bits));
  const CounterWidth width = width_bits == 16 ? CounterWidth::k16 : CounterWidth::k32;
  const SrpFamily family{cfg};
  const std::size_t total = static_cast<std::size_t>(cfg.num_tables) << cfg.k_bits;
  std::vector<std::uint64_t> counters(total);
  for (auto& c : counters)
    c = width == CounterWidth::k16 ? get_le<std::uint16_t>(in) : get_le<std::uint32_t>(in);
  return AceSketch::restore(family, width, std::move(counters), n, mean, saturated);
}
}  // namespace io

}  // namespace ace

// CSV ingestion for non-C++ hosts (the Python mirror): ace::io::load_dataset.
// Returns 0 and malloc'd values (rows x cols f64) / labels (rows u8, only with
// a label column), ACE_E_DATA with the message in ace_host_last_error(), or
// ACE_E_CONTRACT for null arguments.  Free with ace_free().
namespace {
thread_local std::string g_host_err;
}
extern "C" const char* ace_host_last_error(void) { return g_host_err.c_str(); }
extern "C" void ace_free(void* p) { std::free(p); }
extern "C" int ace_load_dataset_csv(const char* path, int has_label, int label_column, double** values,
                                    uint64_t* rows, uint64_t* cols, uint8_t** labels) {
  if (!path || !values || !rows || !cols || !labels) return ACE_E_CONTRACT;
  try {
    const auto d = ace::io::load_dataset(path, has_label ? std::optional<int>(label_column) : std::nullopt);
    *rows = d.rows;
    *cols = d.cols;
    *values = static_cast<double*>(std::malloc(sizeof(double) * std::max<size_t>(1, d.values.size())));
    std::memcpy(*values, d.values.data(), sizeof(double) * d.values.size());
    *labels = nullptr;
    if (d.labels) {
      *labels = static_cast<uint8_t*>(std::malloc(std::max<size_t>(1, d.labels->size())));
      std::memcpy(*labels, d.labels->data(), d.labels->size());
    }
    return 0;
  } catch (const ace::DataError& e) {
    g_host_err = e.what();
    return ACE_E_DATA;
  } catch (const std::exception& e) {
    g_host_err = e.what();
    return ACE_E_CONTRACT;
  }
}

// Noise terms of the noisy variant, ticks tick0 .. tick0+count-1 (srp.cpp:97-101):
// noise_scale * NormalStream(mix_seed(noise_seed, tick)).next(), glibc libm,
// computed on all host threads (each term is independent of the others).
extern "C" int ace_noise_terms(uint64_t noise_seed, uint64_t tick0, uint64_t count, double noise_scale,
                               double* out) {
  if (count && !out) return ACE_E_CONTRACT;
  const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(),
                                                      static_cast<unsigned>(count / 65536 + 1)));
  std::vector<std::thread> pool;
  for (unsigned w = 0; w < nt; ++w)
    pool.emplace_back([=] {
      for (uint64_t i = w; i < count; i += nt) {
        ace::rng::NormalStream g(ace::rng::mix_seed(noise_seed, tick0 + i));
        out[i] = noise_scale * g.next();
      }
    });
  for (auto& t : pool) t.join();
  return 0;
}

// W generation for non-C++ hosts (the Python mirror): the same generator as
// SrpFamily's constructor.
extern "C" int ace_generate_directions(uint64_t seed, uint64_t dim, uint32_t k_bits,
                                       uint32_t num_tables, double* w) {
  if (!w || dim == 0 || k_bits < 1 || k_bits > 30 || num_tables < 1) return 1;
  ace::SrpConfig c;
  c.dim = dim;
  c.k_bits = k_bits;
  c.num_tables = num_tables;
  c.seed = seed;
  const auto v = ace::generate_w(c);
  std::memcpy(w, v.data(), v.size() * sizeof(double));
  return 0;
}
