// ref_driver.cpp — extern "C" harness around the UNMODIFIED reference ACE
// library, compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libaceref.so (git-ignored; travels to the GPU box prebuilt).
//
// TEST / BASELINE INFRASTRUCTURE ONLY: used by tests/ to pin the C oracle and
// generate golden digests, and by bench.py's cpu_baseline and --impl
// reference legs to time the reference's own CPU implementation.  Every call
// below goes through the reference's public API (proj/include/ace/*.hpp).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <optional>
#include <exception>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "ace/detect.hpp"
#include "ace/errors.hpp"
#include "ace/estimators.hpp"
#include "ace/io.hpp"
#include "ace/sketch.hpp"
#include "ace/srp.hpp"

namespace {

thread_local std::string g_err;

ace::SrpConfig make_cfg(uint64_t dim, uint32_t k, uint32_t l, uint64_t seed) {
  ace::SrpConfig c;
  c.dim = dim;
  c.k_bits = k;
  c.num_tables = l;
  c.seed = seed;
  return c;
}

struct RefSketch {
  ace::AceSketch sketch;
  RefSketch(const ace::SrpFamily& f, ace::CounterWidth w) : sketch(f, w) {}
  explicit RefSketch(ace::AceSketch s) : sketch(std::move(s)) {}
};

std::vector<double> row_f64(const float* x, uint64_t dim, uint64_t i) {
  std::vector<double> r(dim);
  for (uint64_t c = 0; c < dim; ++c) r[c] = static_cast<double>(x[i * dim + c]);
  return r;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// W via SrpFamily::direction (srp.cpp:115-123), row t*K+b.
int ref_directions(uint64_t seed, uint64_t dim, uint32_t k, uint32_t l, double* w) {
  try {
    ace::SrpFamily fam(make_cfg(dim, k, l, seed));
    for (uint32_t t = 0; t < l; ++t)
      for (uint32_t b = 0; b < k; ++b) {
        auto v = fam.direction(t, b);
        std::memcpy(w + (static_cast<uint64_t>(t) * k + b) * dim, v.data(), dim * sizeof(double));
      }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Bucket ids via SrpFamily::bucket (srp.cpp:106-113), table-major ids[t*n+i],
// rows as (double) of fp32 X; `threads` workers (bucket is const, thread-safe).
int ref_buckets(uint64_t seed, uint64_t dim, uint32_t k, uint32_t l, const float* x,
                uint64_t n, uint32_t* ids, int threads) {
  try {
    const ace::SrpFamily fam(make_cfg(dim, k, l, seed));
    if (threads < 1) threads = 1;
    std::vector<std::thread> pool;
    const uint64_t chunk = (n + threads - 1) / threads;
    for (int w = 0; w < threads; ++w) {
      const uint64_t lo = std::min<uint64_t>(n, w * chunk), hi = std::min<uint64_t>(n, lo + chunk);
      pool.emplace_back([&, lo, hi] {
        for (uint64_t i = lo; i < hi; ++i) {
          const auto r = row_f64(x, dim, i);
          for (uint32_t t = 0; t < l; ++t) ids[static_cast<uint64_t>(t) * n + i] = fam.bucket(t, r);
        }
      });
    }
    for (auto& t : pool) t.join();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

void* ref_sketch_new(uint64_t seed, uint64_t dim, uint32_t k, uint32_t l, uint32_t width) {
  try {
    const ace::SrpFamily fam(make_cfg(dim, k, l, seed));
    return new RefSketch(fam, width == 16 ? ace::CounterWidth::k16 : ace::CounterWidth::k32);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_sketch_free(void* h) { delete static_cast<RefSketch*>(h); }

// Noisy variant (srp.cpp:93-104): a sketch over a noisy family; its family
// copy's aux stream can be re-seeded (reset_noise_stream, srp.cpp:126-129).
void* ref_sketch_new_noisy(uint64_t seed, uint64_t dim, uint32_t k, uint32_t l, uint32_t width, double noise) {
  try {
    auto c = make_cfg(dim, k, l, seed);
    c.noise_scale = noise;
    const ace::SrpFamily fam(c);
    return new RefSketch(fam, width == 16 ? ace::CounterWidth::k16 : ace::CounterWidth::k32);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_sketch_reset_noise(void* h, uint64_t aux) {
  static_cast<RefSketch*>(h)->sketch.family().reset_noise_stream(aux);
}

// A noisy family's bucket calls in order: for each row i, tables t0..t0+nt-1
// (bucket) or, with b >= 0, the single bit (t, b) of each table.  ids[t*n+i].
// A sequence of calls on one noisy family: op j = (row, table, b), b < 0
// meaning bucket(table, row) and b >= 0 bit(table, b, row).
int ref_noisy_sequence(uint64_t seed, uint64_t dim, uint32_t k, uint32_t l, double noise, uint64_t aux,
                       const double* x, const int32_t* ops, uint64_t nops, uint32_t* out) {
  try {
    auto c = make_cfg(dim, k, l, seed);
    c.noise_scale = noise;
    const ace::SrpFamily fam(c);
    fam.reset_noise_stream(aux);
    for (uint64_t j = 0; j < nops; ++j) {
      std::span<const double> row(x + static_cast<uint64_t>(ops[3 * j]) * dim, dim);
      const auto t = static_cast<std::size_t>(ops[3 * j + 1]);
      out[j] = ops[3 * j + 2] < 0 ? fam.bucket(t, row) : fam.bit(t, static_cast<std::size_t>(ops[3 * j + 2]), row);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_noisy_calls(uint64_t seed, uint64_t dim, uint32_t k, uint32_t l, double noise, int reset, uint64_t aux,
                    const double* x, uint64_t n, uint32_t t0, uint32_t nt, int b, uint32_t* ids) {
  try {
    auto c = make_cfg(dim, k, l, seed);
    c.noise_scale = noise;
    const ace::SrpFamily fam(c);
    if (reset) fam.reset_noise_stream(aux);
    for (uint64_t i = 0; i < n; ++i) {
      std::span<const double> row(x + i * dim, dim);
      for (uint32_t t = 0; t < nt; ++t)
        ids[static_cast<uint64_t>(t) * n + i] = b < 0 ? fam.bucket(t0 + t, row) : fam.bit(t0 + t, b, row);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// AceSketch::insert (sketch.cpp:50-72) for each row in order.
int ref_sketch_insert(void* h, const float* x, uint64_t n, uint64_t dim) {
  try {
    auto& s = static_cast<RefSketch*>(h)->sketch;
    for (uint64_t i = 0; i < n; ++i) s.insert(row_f64(x, dim, i));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_sketch_insert_f64(void* h, const double* x, uint64_t n, uint64_t dim) {
  try {
    auto& s = static_cast<RefSketch*>(h)->sketch;
    for (uint64_t i = 0; i < n; ++i) s.insert(std::span<const double>(x + i * dim, dim));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// AceSketch::remove (sketch.cpp:74-106); returns -2 on InconsistentDelete.
int ref_sketch_remove(void* h, const float* x, uint64_t n, uint64_t dim) {
  try {
    auto& s = static_cast<RefSketch*>(h)->sketch;
    for (uint64_t i = 0; i < n; ++i) s.remove(row_f64(x, dim, i));
    return 0;
  } catch (const ace::InconsistentDelete& e) {
    g_err = e.what();
    return -2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// AceSketch::score (sketch.cpp:108-116).
int ref_sketch_score(void* h, const float* x, uint64_t n, uint64_t dim, double* scores) {
  try {
    auto& s = static_cast<RefSketch*>(h)->sketch;
    for (uint64_t i = 0; i < n; ++i) scores[i] = s.score(row_f64(x, dim, i)).value;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

uint64_t ref_sketch_size(void* h) { return static_cast<RefSketch*>(h)->sketch.size(); }
double ref_sketch_mean(void* h) { return static_cast<RefSketch*>(h)->sketch.mean(); }
int ref_sketch_saturated(void* h) { return static_cast<RefSketch*>(h)->sketch.saturated(); }

void ref_sketch_counters(void* h, uint64_t* out) {
  const auto flat = static_cast<RefSketch*>(h)->sketch.counters_flat();
  std::memcpy(out, flat.data(), flat.size() * sizeof(uint64_t));
}

// detect_batch (detect.cpp:12-74) on the rows; also returns the per-row flags
// (score < threshold, the reference's own rule at detect.cpp:60, recomputed
// from AceSketch::score since the report carries only counts).
int ref_detect_batch(void* h, const float* x, uint64_t n, uint64_t dim, unsigned threads,
                     double* mean, double* sd, double* thr, uint64_t* reported,
                     double* elapsed, uint8_t* flags) {
  try {
    auto& s = static_cast<RefSketch*>(h)->sketch;
    ace::Dataset data;
    data.rows = n;
    data.cols = dim;
    data.values.resize(n * dim);
    for (uint64_t i = 0; i < n * dim; ++i) data.values[i] = static_cast<double>(x[i]);
    const auto rep = ace::detect_batch(s, data, threads);
    *mean = rep.score_mean;
    *sd = rep.score_stddev;
    *thr = rep.threshold;
    *reported = rep.reported;
    *elapsed = rep.elapsed_seconds;
    if (flags)
      for (uint64_t i = 0; i < n; ++i) flags[i] = s.score(data.row(i)).value < rep.threshold;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Streaming batch: detect_stream (detect.cpp:76-84) for every row against the
// counts at batch start (empty sketch -> flag 0, where detect_stream throws),
// then insert the rows in order.
int ref_stream_batch(void* h, const float* x, uint64_t n, uint64_t dim, double alpha,
                     double* scores, uint8_t* flags) {
  try {
    auto& s = static_cast<RefSketch*>(h)->sketch;
    for (uint64_t i = 0; i < n; ++i) {
      const auto r = row_f64(x, dim, i);
      if (s.size() == 0) {
        if (scores) scores[i] = s.score(r).value;
        if (flags) flags[i] = 0;
      } else {
        const auto [est, flag] = ace::detect_stream(s, r, alpha);
        if (scores) scores[i] = est.value;
        if (flags) flags[i] = flag;
      }
    }
    for (uint64_t i = 0; i < n; ++i) s.insert(row_f64(x, dim, i));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// CPU baseline timing: insert rows on 1 core (single-writer), then score them
// with detect_batch on `threads` cores (0 = hardware_concurrency).  Seconds.
int ref_time_build_detect(uint64_t seed, const float* x, uint64_t n, uint64_t dim, uint32_t k,
                          uint32_t l, unsigned threads, double* t_insert, double* t_detect,
                          uint64_t* reported) {
  try {
    const ace::SrpFamily fam(make_cfg(dim, k, l, seed));
    ace::AceSketch s(fam, ace::CounterWidth::k32);
    ace::Dataset data;
    data.rows = n;
    data.cols = dim;
    data.values.resize(n * dim);
    for (uint64_t i = 0; i < n * dim; ++i) data.values[i] = static_cast<double>(x[i]);
    const auto t0 = std::chrono::steady_clock::now();
    for (uint64_t i = 0; i < n; ++i) s.insert(data.row(i));
    const auto t1 = std::chrono::steady_clock::now();
    const auto rep = ace::detect_batch(s, data, threads);
    const auto t2 = std::chrono::steady_clock::now();
    *t_insert = std::chrono::duration<double>(t1 - t0).count();
    *t_detect = std::chrono::duration<double>(t2 - t1).count();
    *reported = rep.reported;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// CPU baseline of the streaming driver in config 5's order: per batch, every
// row scored by detect_stream (detect.cpp:76-84) against the counts at batch
// start on `threads` cores (the sketch is only read: const, thread-safe), then
// the batch inserted in row order on one core (single writer, sketch.hpp:
// 23-24), as ace_cli.cpp:173-186 does per query with the insert deferred to
// the batch end.  Seconds of scoring and of inserting over all n rows.
int ref_time_stream(uint64_t seed, const float* x, uint64_t n, uint64_t dim, uint32_t k, uint32_t l,
                    uint64_t batch, double alpha, unsigned threads, double* t_score, double* t_insert,
                    uint64_t* reported) {
  try {
    const ace::SrpFamily fam(make_cfg(dim, k, l, seed));
    ace::AceSketch s(fam, ace::CounterWidth::k32);
    if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
    std::vector<double> xd(n * dim);
    for (uint64_t i = 0; i < n * dim; ++i) xd[i] = static_cast<double>(x[i]);
    double ts = 0.0, ti = 0.0;
    uint64_t rep = 0;
    std::vector<uint64_t> rep_t(threads);
    for (uint64_t b0 = 0; b0 < n; b0 += batch) {
      const uint64_t m = std::min(batch, n - b0);
      const auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> pool;
      for (unsigned t = 0; t < threads; ++t) {
        rep_t[t] = 0;
        pool.emplace_back([&, t] {
          for (uint64_t i = b0 + t; i < b0 + m; i += threads) {
            std::span<const double> r(xd.data() + i * dim, dim);
            if (s.size() == 0) {
              (void)s.score(r);
            } else {
              const auto res = ace::detect_stream(s, r, alpha);
              rep_t[t] += res.second ? 1 : 0;
            }
          }
        });
      }
      for (auto& th : pool) th.join();
      const auto t1 = std::chrono::steady_clock::now();
      for (uint64_t i = b0; i < b0 + m; ++i) s.insert(std::span<const double>(xd.data() + i * dim, dim));
      const auto t2 = std::chrono::steady_clock::now();
      ts += std::chrono::duration<double>(t1 - t0).count();
      ti += std::chrono::duration<double>(t2 - t1).count();
      for (unsigned t = 0; t < threads; ++t) rep += rep_t[t];
    }
    *t_score = ts;
    *t_insert = ti;
    *reported = rep;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Per-point API baseline in ace_cli stream --adapt's order (ace_cli.cpp:
// 173-183): a sketch built from the first n_build rows (untimed), then for
// each of the next n_query rows detect_stream (detect.cpp:76-84) followed by
// insert (sketch.cpp:50-72), one call at a time on one core.  Seconds of the
// query loop; scores / flags optional.
int ref_time_point(uint64_t seed, const float* x, uint64_t n_build, uint64_t n_query, uint64_t dim,
                   uint32_t k, uint32_t l, double alpha, double* seconds, uint64_t* reported,
                   double* scores, uint8_t* flags) {
  try {
    const ace::SrpFamily fam(make_cfg(dim, k, l, seed));
    ace::AceSketch s(fam, ace::CounterWidth::k32);
    std::vector<double> xd((n_build + n_query) * dim);
    for (uint64_t i = 0; i < xd.size(); ++i) xd[i] = static_cast<double>(x[i]);
    for (uint64_t i = 0; i < n_build; ++i) s.insert(std::span<const double>(xd.data() + i * dim, dim));
    uint64_t rep = 0;
    const auto t0 = std::chrono::steady_clock::now();
    for (uint64_t i = n_build; i < n_build + n_query; ++i) {
      std::span<const double> r(xd.data() + i * dim, dim);
      const auto [est, flag] = ace::detect_stream(s, r, alpha);
      if (scores) scores[i - n_build] = est.value;
      if (flags) flags[i - n_build] = flag ? 1 : 0;
      rep += flag ? 1 : 0;
      s.insert(r);
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *reported = rep;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// ACE1 sketch files through the reference's io (io.cpp:184-244): 0 ok,
// -3 DataError (message in ref_last_error), -1 other.
int ref_save_sketch(void* h, const char* path) {
  try {
    ace::io::save_sketch(static_cast<RefSketch*>(h)->sketch, path);
    return 0;
  } catch (const ace::DataError& e) {
    g_err = e.what();
    return -3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

void* ref_load_sketch(const char* path, int* status) {
  try {
    auto* r = new RefSketch(ace::io::load_sketch(path));
    *status = 0;
    return r;
  } catch (const ace::DataError& e) {
    g_err = e.what();
    *status = -3;
  } catch (const std::exception& e) {
    g_err = e.what();
    *status = -1;
  }
  return nullptr;
}

// ace::io::load_dataset (io.cpp:89-182): 0 ok with malloc'd values/labels
// (free with ref_free), -3 DataError (message in ref_last_error).
int ref_load_dataset(const char* path, int has_label, int label_column, double** values, uint64_t* rows,
                     uint64_t* cols, uint8_t** labels) {
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
    g_err = e.what();
    return -3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

void ref_free(void* p) { std::free(p); }

void ref_sketch_config(void* h, uint64_t* dim, uint32_t* k, uint32_t* l, uint64_t* seed, uint32_t* width) {
  const auto& s = static_cast<RefSketch*>(h)->sketch;
  const auto& c = s.family().config();
  *dim = c.dim;
  *k = c.k_bits;
  *l = c.num_tables;
  *seed = c.seed;
  *width = static_cast<uint32_t>(s.counter_width());
}

}  // extern "C"
