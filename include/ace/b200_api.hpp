// ace/b200_api.hpp — the ACE C++ API (same names, signatures and error
// behaviour as the reference's proj/include/ace/{errors,rng,srp,sketch,
// dataset,detect,estimators}.hpp), implemented over the B200 C ABI
// (ace_b200.h).  The per-header drop-ins (ace/srp.hpp, ace/sketch.hpp, ...)
// all include this file.
//
// Hashing, counting, scoring and detection run on the GPU; there is no CPU
// compute path.  Host code generates W (seeded, construction time only) and
// finalises nothing the device can do.  Batch extensions (insert_batch,
// score_batch, buckets, detect_batch over fp32 rows, stream_batch) take
// row-major fp32 matrices, the north-star input format.
#pragma once

#include <atomic>
#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

struct AceFamily;
struct AceSketch;

namespace ace {

// ---- errors (reference errors.hpp:9-26) -----------------------------------
struct ContractViolation : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InconsistentDelete : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct UnsupportedOperation : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---- deterministic streams (reference rng.hpp:10-73) ----------------------
namespace rng {
std::uint64_t splitmix64(std::uint64_t& state);
std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t index);
double unit_double(std::uint64_t bits);
std::uint64_t bounded(std::uint64_t bits, std::uint64_t bound);

class NormalStream {
 public:
  explicit NormalStream(std::uint64_t seed) : s_(seed) {}
  double next();

 private:
  std::uint64_t s_;
  double cached_ = 0.0;
  bool cached_valid_ = false;
};

class UniformStream {
 public:
  explicit UniformStream(std::uint64_t seed) : s_(seed) {}
  std::uint64_t next_u64() { return splitmix64(s_); }
  double next_unit() { return unit_double(splitmix64(s_)); }
  std::uint64_t next_bounded(std::uint64_t bound) { return bounded(splitmix64(s_), bound); }

 private:
  std::uint64_t s_;
};
}  // namespace rng

// ---- dataset (reference dataset.hpp:14-31) --------------------------------
struct Dataset {
  std::vector<double> values;
  std::size_t rows = 0;
  std::size_t cols = 0;
  std::optional<std::vector<std::uint8_t>> labels;
  std::string name;

  std::span<const double> row(std::size_t i) const { return {values.data() + i * cols, cols}; }
  std::size_t labeled_anomalies() const {
    std::size_t k = 0;
    if (labels)
      for (std::uint8_t v : *labels) k += v != 0;
    return k;
  }
};

// ---- SRP family (reference srp.hpp:10-79) ---------------------------------
struct SrpConfig {
  std::size_t dim = 0;
  std::uint32_t k_bits = 15;
  std::uint32_t num_tables = 50;
  std::uint64_t seed = 0;
  double noise_scale = 0.0;
  bool cache_projections = true;
};

class SrpFamily {
 public:
  explicit SrpFamily(const SrpConfig& cfg);
  SrpFamily(const SrpFamily& other) = default;
  SrpFamily& operator=(const SrpFamily& other) = default;

  std::uint32_t bit(std::size_t table, std::size_t b, std::span<const double> x) const;
  std::uint32_t bucket(std::size_t table, std::span<const double> x) const;
  // Batch extension: ids[t * n + i] for n fp32 rows (row-major, dim cols).
  std::vector<std::uint32_t> buckets(std::span<const float> rows, std::size_t n) const;

  const SrpConfig& config() const { return cfg_; }
  std::size_t num_buckets() const { return std::size_t{1} << cfg_.k_bits; }
  std::vector<double> direction(std::size_t table, std::size_t b) const;
  std::size_t projection_bytes() const { return cfg_.cache_projections ? w_->size() * sizeof(double) : 0; }
  void reset_noise_stream(std::uint64_t aux_seed) const;

  friend bool operator==(const SrpFamily& a, const SrpFamily& b) {
    return a.cfg_.dim == b.cfg_.dim && a.cfg_.k_bits == b.cfg_.k_bits &&
           a.cfg_.num_tables == b.cfg_.num_tables && a.cfg_.seed == b.cfg_.seed &&
           a.cfg_.noise_scale == b.cfg_.noise_scale;
  }

  // Device handle (created on first use; shared by copies).
  ::AceFamily* device() const;

  // Noisy variant (noise_scale > 0, srp.cpp:93-104): reserves `count` ticks of
  // this family's noise stream and returns the terms noise_scale * N(0,1).
  std::vector<double> draw_noise(std::size_t count) const;
  // Bucket ids (table-major, nt x n) of n points with a noisy family, bits
  // [b0, b0+nb) of tables [t0, t0+nt), ticks in point / table / bit order.
  std::vector<std::uint32_t> noisy_ids(const void* x, int dtype, std::size_t n, std::size_t t0, std::size_t nt,
                                       std::size_t b0, std::size_t nb) const;

 private:
  struct NoiseCounter {  // the reference's atomic tick counter; copies take the current value
    std::atomic<std::uint64_t> v{0};
    NoiseCounter() = default;
    NoiseCounter(const NoiseCounter& o) : v(o.v.load(std::memory_order_relaxed)) {}
    NoiseCounter& operator=(const NoiseCounter& o) {
      v.store(o.v.load(std::memory_order_relaxed), std::memory_order_relaxed);
      return *this;
    }
  };
  void check(std::size_t table, std::size_t b, std::span<const double> x) const;
  SrpConfig cfg_;
  mutable std::uint64_t noise_seed_ = 0;
  mutable NoiseCounter noise_ctr_;
  std::shared_ptr<const std::vector<double>> w_;  // (K*L) x d, host copy
  std::shared_ptr<std::shared_ptr<::AceFamily>> dev_;  // created on first use, shared by copies
};

double collision_probability(std::span<const double> x, std::span<const double> y);

// ---- sketch (reference sketch.hpp:11-84) ----------------------------------
enum class CounterWidth : std::uint32_t { k16 = 16, k32 = 32 };

struct ScoreEstimate {
  double value = 0.0;
  std::uint32_t k_bits = 0;
  std::uint32_t num_tables = 0;
};

class AceSketch {
 public:
  explicit AceSketch(const SrpFamily& family, CounterWidth width = CounterWidth::k16);
  AceSketch(const AceSketch& other);
  AceSketch& operator=(const AceSketch& other);
  AceSketch(AceSketch&&) noexcept;
  AceSketch& operator=(AceSketch&&) noexcept;
  ~AceSketch();

  void insert(std::span<const double> x);
  void remove(std::span<const double> x);
  ScoreEstimate score(std::span<const double> q) const;

  // Batch extensions over n fp32 rows (row-major, dim columns).
  void insert_batch(std::span<const float> rows, std::size_t n);
  std::vector<double> score_batch(std::span<const float> rows, std::size_t n) const;

  std::uint64_t size() const;
  double mean() const;
  bool saturated() const;
  const SrpFamily& family() const { return family_; }
  CounterWidth counter_width() const { return width_; }

  std::uint64_t counter(std::size_t table, std::size_t bucket) const;
  std::size_t num_counters() const { return family_.config().num_tables * family_.num_buckets(); }
  std::size_t counter_bytes() const;
  std::size_t memory_bytes() const { return counter_bytes() + kHeaderBytes; }

  static constexpr std::size_t kHeaderBytes = 53;

  static AceSketch restore(const SrpFamily& family, CounterWidth width,
                           std::vector<std::uint64_t> counters, std::uint64_t n, double mean,
                           bool saturated);
  std::vector<std::uint64_t> counters_flat() const;

  ::AceSketch* device() const { return dev_; }

 private:
  void check_dim(std::span<const double> x) const;
  SrpFamily family_;
  CounterWidth width_;
  ::AceSketch* dev_ = nullptr;
};

// ---- detection (reference detect.hpp:12-36) -------------------------------
struct DetectionReport {
  std::size_t reported = 0;
  std::size_t correctly_reported = 0;
  std::size_t missed = 0;
  std::size_t total_labeled_anomalies = 0;
  bool has_labels = false;
  double threshold = 0.0;
  double score_mean = 0.0;
  double score_stddev = 0.0;
  double elapsed_seconds = 0.0;
};

DetectionReport detect_batch(const AceSketch& sketch, const Dataset& data, unsigned threads = 0);
std::pair<ScoreEstimate, bool> detect_stream(const AceSketch& sketch, std::span<const double> q,
                                             double alpha);

// Streaming extension: score a whole batch against the current counts with
// detect_stream's rule, then insert it (config-5 order).  flags[i] in {0,1}.
std::vector<std::uint8_t> stream_batch(AceSketch& sketch, std::span<const float> rows,
                                       std::size_t n, double alpha);

// ---- estimators: build_sketch (reference estimators.hpp:38-41) -------------
AceSketch build_sketch(const Dataset& data, std::uint32_t k_bits, std::uint32_t num_tables,
                       std::uint64_t seed, double noise_scale = 0.0,
                       CounterWidth width = CounterWidth::k16);

// ---- ACE1 sketch files (reference io.hpp:23-27) ---------------------------
namespace io {
// CSV ingestion (reference io.hpp:16-21, io.cpp:89-182): comma-separated
// numeric text, one row per instance; a header line is detected by a
// non-numeric first token; label_column (0-based, negative from the end)
// splits off a 0/1 label column; all-zero feature rows are rejected with
// their line numbers.  Lines are parsed on all host threads; validation and
// error messages follow the reference's line order exactly.
Dataset load_dataset(const std::string& path, std::optional<int> label_column = std::nullopt);

// Binary sketch persistence ("ACE1", 53-byte little-endian header, counters
// table-major).  Round-trips counters, n, mean and configuration bit-exactly;
// the bytes are the reference's for the same state.
void save_sketch(const AceSketch& sketch, const std::string& path);
AceSketch load_sketch(const std::string& path);
}  // namespace io

}  // namespace ace
