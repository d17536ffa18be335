// Per-point API timing through the drop-in headers: ace_cli stream --adapt's
// loop (ace_cli.cpp:173-183) — detect_stream (detect.hpp:34-36) then insert
// (sketch.hpp:33) for one query at a time — after an untimed build from the
// first n_build rows.  Built by paper_1706_06664_b200/build.py, driven by
// bench.py --api point.
//
//   ace_point_bench DIM K L SEED ALPHA N_BUILD N_WARM N_QUERY ROWS.f32 [OUT.bin]
//
// ROWS.f32: (N_BUILD + N_WARM + N_QUERY) x DIM float32, row-major; the first
// N_WARM queries are untimed.  Prints one line "seconds reported p50_us
// p99_us detect_us launches" over the N_QUERY timed queries (detect_us: mean
// time inside detect_stream; launches: kernels libace_dev.so launched);
// OUT.bin (optional) receives the timed queries' scores (f64) followed by
// their flags (u8) for the parity test.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <span>
#include <vector>

#include "ace_b200.h"
#include "ace/detect.hpp"
#include "ace/sketch.hpp"
#include "ace/srp.hpp"

int main(int argc, char** argv) {
  if (argc < 10) {
    std::fprintf(stderr, "usage: %s DIM K L SEED ALPHA N_BUILD N_WARM N_QUERY ROWS.f32 [OUT.bin]\n", argv[0]);
    return 2;
  }
  ace::SrpConfig c;
  c.dim = std::strtoull(argv[1], nullptr, 10);
  c.k_bits = static_cast<std::uint32_t>(std::strtoul(argv[2], nullptr, 10));
  c.num_tables = static_cast<std::uint32_t>(std::strtoul(argv[3], nullptr, 10));
  c.seed = std::strtoull(argv[4], nullptr, 10);
  const double alpha = std::strtod(argv[5], nullptr);
  const std::size_t n_build = std::strtoull(argv[6], nullptr, 10);
  const std::size_t n_warm = std::strtoull(argv[7], nullptr, 10);
  const std::size_t n_query = std::strtoull(argv[8], nullptr, 10);
  const std::size_t dim = c.dim;
  std::vector<float> rows((n_build + n_warm + n_query) * dim);
  {
    std::ifstream f(argv[9], std::ios::binary);
    if (!f.read(reinterpret_cast<char*>(rows.data()), static_cast<std::streamsize>(rows.size() * 4))) {
      std::fprintf(stderr, "short read of %s\n", argv[9]);
      return 2;
    }
  }
  std::vector<double> xd(rows.begin(), rows.end());
  const ace::SrpFamily fam(c);
  ace::AceSketch s(fam, ace::CounterWidth::k32);
  if (n_build) s.insert_batch(std::span<const float>(rows.data(), n_build * dim), n_build);
  for (std::size_t i = 0; i < n_warm; ++i) {  // untimed queries, the same loop
    std::span<const double> r(xd.data() + (n_build + i) * dim, dim);
    (void)ace::detect_stream(s, r, alpha);
    s.insert(r);
  }
  const std::size_t q0 = n_build + n_warm;
  std::vector<double> scores(n_query);
  std::vector<std::uint8_t> flags(n_query);
  std::vector<double> lat(n_query);
  std::uint64_t reported = 0;
  double t_detect = 0.0;  // microseconds inside detect_stream calls
  const std::uint64_t launches0 = ace_kernel_launches();
  const auto t0 = std::chrono::steady_clock::now();
  for (std::size_t i = 0; i < n_query; ++i) {
    const auto a = std::chrono::steady_clock::now();
    std::span<const double> r(xd.data() + (q0 + i) * dim, dim);
    const auto [est, flag] = ace::detect_stream(s, r, alpha);
    t_detect += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - a).count();
    scores[i] = est.value;
    flags[i] = flag ? 1 : 0;
    reported += flag ? 1 : 0;
    s.insert(r);
    lat[i] = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - a).count();
  }
  (void)s.size();  // the last deferred insert lands inside the timed region
  const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  const std::uint64_t launches = ace_kernel_launches() - launches0;
  std::sort(lat.begin(), lat.end());
  const double p50 = n_query ? lat[n_query / 2] : 0.0;
  const double p99 = n_query ? lat[std::min(n_query - 1, n_query * 99 / 100)] : 0.0;
  std::printf("%.9f %llu %.3f %.3f %.3f %llu\n", sec, static_cast<unsigned long long>(reported), p50, p99,
              n_query ? t_detect / static_cast<double>(n_query) : 0.0, static_cast<unsigned long long>(launches));
  if (argc > 10) {
    std::ofstream o(argv[10], std::ios::binary);
    o.write(reinterpret_cast<const char*>(scores.data()), static_cast<std::streamsize>(n_query * 8));
    o.write(reinterpret_cast<const char*>(flags.data()), static_cast<std::streamsize>(n_query));
  }
  return 0;
}
