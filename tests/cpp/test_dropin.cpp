// Drop-in check: the reference's own known-answer tests (proj/tests/
// test_srp.cpp, test_sketch.cpp, test_detect.cpp), restated against the
// B200 implementation through the unchanged reference header names
// (#include "ace/srp.hpp" etc.).  Built by paper_1706_06664_b200/build.py,
// run on the GPU by tests/test_cpp_dropin_gpu.py.  Prints PASS/FAIL lines;
// exit code = number of failures.
#include <cmath>
#include <cstdlib>
#include <fstream>
#include <iterator>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "ace/detect.hpp"
#include "ace/errors.hpp"
#include "ace/estimators.hpp"
#include "ace/io.hpp"
#include "ace/rng.hpp"
#include "ace/sketch.hpp"
#include "ace/srp.hpp"

namespace {

int failures = 0;

void check(bool ok, const std::string& what) {
  std::printf("%s %s\n", ok ? "PASS" : "FAIL", what.c_str());
  if (!ok) ++failures;
}

template <class E>
void expect_throw(const std::function<void()>& f, const std::string& what) {
  bool thrown = false;
  try {
    f();
  } catch (const E&) {
    thrown = true;
  } catch (...) {
  }
  check(thrown, what);
}

ace::SrpConfig cfg(std::size_t d, std::uint32_t k, std::uint32_t l, std::uint64_t s) {
  ace::SrpConfig c;
  c.dim = d;
  c.k_bits = k;
  c.num_tables = l;
  c.seed = s;
  return c;
}

std::vector<double> normals(std::size_t d, std::uint64_t seed) {
  ace::rng::NormalStream g(seed);
  std::vector<double> v(d);
  for (auto& x : v) x = g.next();
  return v;
}

}  // namespace

int main() {
  // test_srp.cpp: bit on its own direction is 1
  {
    const ace::SrpFamily f{cfg(5, 3, 4, 99)};
    bool ok = true;
    for (std::size_t j = 0; j < 4; ++j)
      for (std::size_t b = 0; b < 3; ++b) ok &= f.bit(j, b, f.direction(j, b)) == 1;
    check(ok, "bit on own direction is 1");
  }
  // sign(0) -> 1, zero vector -> bucket 0b11
  {
    const ace::SrpFamily f{cfg(4, 2, 3, 7)};
    const std::vector<double> z(4, 0.0);
    bool ok = true;
    for (std::size_t j = 0; j < 3; ++j) ok &= f.bit(j, 0, z) == 1 && f.bucket(j, z) == 0b11;
    check(ok, "zero vector hashes to all ones");
  }
  // bit on e1 equals sign of w[0]
  {
    const ace::SrpFamily f{cfg(2, 1, 1, 1234)};
    const std::vector<double> e1 = {1.0, 0.0};
    check(f.bit(0, 0, e1) == (f.direction(0, 0)[0] >= 0.0 ? 1u : 0u), "bit on e1 = sign(w0)");
  }
  // bit 0 is the MSB
  {
    const ace::SrpFamily f{cfg(3, 4, 2, 77)};
    const std::vector<double> e1 = {1.0, 0.0, 0.0};
    bool ok = true;
    for (std::size_t j = 0; j < 2; ++j) {
      std::uint32_t expect = 0;
      for (std::size_t b = 0; b < 4; ++b) expect = (expect << 1) | (f.direction(j, b)[0] >= 0.0 ? 1u : 0u);
      ok &= f.bucket(j, e1) == expect;
    }
    check(ok, "bit 0 is the most significant bit");
  }
  // scaling invariance, K=1 range
  {
    const ace::SrpFamily f{cfg(8, 6, 10, 11)};
    auto x = normals(8, 21);
    auto y = x;
    for (auto& v : y) v *= 3.75;
    bool ok = true;
    for (std::size_t j = 0; j < 10; ++j) ok &= f.bucket(j, x) == f.bucket(j, y);
    check(ok, "bucket invariant under positive scaling");
    const ace::SrpFamily g{cfg(6, 1, 8, 5)};
    auto q = normals(6, 42);
    ok = true;
    for (std::size_t j = 0; j < 8; ++j) ok &= g.bucket(j, q) <= 1;
    check(ok, "K=1 buckets in {0,1}");
  }
  // validation
  expect_throw<ace::ContractViolation>([] { ace::SrpFamily f{cfg(0, 2, 2, 0)}; }, "dim 0 rejected");
  expect_throw<ace::ContractViolation>([] { ace::SrpFamily f{cfg(2, 31, 2, 0)}; }, "K=31 rejected");
  expect_throw<ace::ContractViolation>(
      [] {
        const ace::SrpFamily f{cfg(3, 2, 2, 0)};
        std::vector<double> w = {1.0, 2.0};
        f.bucket(0, w);
      },
      "dimension mismatch rejected");
  // test_sketch.cpp: first insert n=1, mean=1; double insert mean=2
  {
    ace::AceSketch s{ace::SrpFamily{cfg(4, 5, 8, 1)}};
    const std::vector<double> x = {1.0, -2.0, 0.5, 3.0};
    s.insert(x);
    check(s.size() == 1 && std::fabs(s.mean() - 1.0) < 1e-12 && s.score(x).value == 1.0,
          "first insert: n=1, mean=1, score=1");
    ace::AceSketch t{ace::SrpFamily{cfg(3, 4, 6, 2)}};
    const std::vector<double> y = {0.3, 1.0, -1.0};
    t.insert(y);
    t.insert(y);
    check(std::fabs(t.mean() - 2.0) < 1e-12, "double insert: mean=2");
  }
  // per-table sums == n, 0 <= score <= n, empty sketch scores 0
  {
    const ace::SrpFamily f{cfg(6, 5, 7, 3)};
    ace::AceSketch s{f, ace::CounterWidth::k32};
    check(s.score(normals(6, 1)).value == 0.0, "empty sketch scores 0");
    for (int i = 0; i < 300; ++i) s.insert(normals(6, 100 + i));
    bool ok = true;
    for (std::size_t j = 0; j < 7; ++j) {
      std::uint64_t tot = 0;
      for (std::size_t b = 0; b < f.num_buckets(); b += 1) tot += s.counters_flat()[j * f.num_buckets() + b];
      ok &= tot == 300;
    }
    check(ok, "per-table counter sums == n");
    const auto e = s.score(normals(6, 5));
    check(e.value >= 0 && e.value <= 300 && e.k_bits == 5 && e.num_tables == 7, "score range, K, L");
  }
  // counter bytes
  {
    const ace::SrpFamily f{cfg(2, 15, 50, 0)};
    check(ace::AceSketch(f).counter_bytes() == 3276800u, "k16 counter bytes 3,276,800");
    check(ace::AceSketch(f, ace::CounterWidth::k32).counter_bytes() == 6553600u, "k32 counter bytes 6,553,600");
  }
  // saturation sticky at 65535 (k16)
  {
    ace::AceSketch s{ace::SrpFamily{cfg(2, 1, 1, 9)}};
    const std::vector<double> x = {1.0, 1.0};
    std::vector<float> rows(2 * 70000, 1.0f);
    s.insert_batch(rows, 70000);
    const auto c = s.counters_flat();
    check(s.saturated() && (c[0] == 65535 || c[1] == 65535), "k16 saturation is sticky at 65535");
  }
  // remove: exact inverse; InconsistentDelete on a never-inserted point
  {
    const ace::SrpFamily f{cfg(5, 4, 6, 8)};
    ace::AceSketch s{f, ace::CounterWidth::k32};
    for (int i = 0; i < 50; ++i) s.insert(normals(5, 300 + i));
    const double m = s.mean();
    s.insert(normals(5, 999));
    s.remove(normals(5, 999));
    check(s.size() == 50 && std::fabs(s.mean() - m) < 1e-9 * m, "insert then remove restores n and mean");
    ace::AceSketch e{f, ace::CounterWidth::k32};
    expect_throw<ace::InconsistentDelete>([&] { e.remove(normals(5, 1)); }, "delete of unseen item throws");
  }
  // test_detect.cpp: identical points -> sigma 0, nothing flagged
  {
    ace::Dataset d;
    d.rows = 200;
    d.cols = 3;
    d.values.assign(600, 0.0);
    for (std::size_t i = 0; i < 200; ++i) {
      d.values[3 * i] = 1.0;
      d.values[3 * i + 1] = 2.0;
      d.values[3 * i + 2] = -1.0;
    }
    const auto s = ace::build_sketch(d, 8, 10, 4, 0.0, ace::CounterWidth::k32);
    const auto r = ace::detect_batch(s, d);
    check(r.score_stddev == 0.0 && r.reported == 0, "identical points: sigma 0, no flags");
  }
  // antipodal pair scores 1 each
  {
    ace::Dataset d;
    d.rows = 2;
    d.cols = 4;
    d.values = {1.0, 2.0, -3.0, 0.5, -1.0, -2.0, 3.0, -0.5};
    const auto s = ace::build_sketch(d, 15, 50, 6, 0.0, ace::CounterWidth::k32);
    check(s.score(d.row(0)).value == 1.0 && s.score(d.row(1)).value == 1.0, "antipodal pair scores 1");
  }
  // far outliers flagged
  {
    ace::Dataset d;
    d.cols = 8;
    ace::rng::NormalStream g(77);
    for (int i = 0; i < 2000; ++i)
      for (int c = 0; c < 8; ++c) d.values.push_back(5.0 + 0.3 * g.next());
    for (int i = 0; i < 10; ++i)
      for (int c = 0; c < 8; ++c) d.values.push_back(c % 2 ? -40.0 : 40.0 * (i % 3 - 1));
    d.rows = d.values.size() / 8;
    d.labels = std::vector<std::uint8_t>(d.rows, 0);
    for (std::size_t i = 2000; i < d.rows; ++i) (*d.labels)[i] = 1;
    const auto s = ace::build_sketch(d, 15, 50, 10, 0.0, ace::CounterWidth::k32);
    const auto r = ace::detect_batch(s, d);
    check(r.has_labels && r.correctly_reported == 10 && r.missed == 0, "far outliers all flagged");
  }
  // stream: inclusive <=, alpha > mean never flags, empty throws, alpha < 0 throws
  {
    const ace::SrpFamily f{cfg(4, 6, 12, 5)};
    ace::AceSketch s{f, ace::CounterWidth::k32};
    expect_throw<ace::ContractViolation>([&] { ace::detect_stream(s, normals(4, 1), 0.5); },
                                         "detect_stream on empty sketch throws");
    for (int i = 0; i < 100; ++i) s.insert(normals(4, 500 + i));
    expect_throw<ace::ContractViolation>([&] { ace::detect_stream(s, normals(4, 1), -0.1); },
                                         "negative alpha throws");
    const auto q = normals(4, 3);
    const auto [est, flag] = ace::detect_stream(s, q, 0.0);
    check(flag == (est.value <= s.mean()), "stream rule score <= mean - alpha");
    check(!ace::detect_stream(s, q, s.mean() + 1.0).second, "alpha > mean never flags");
  }
  // copy semantics: deep copy
  {
    const ace::SrpFamily f{cfg(3, 3, 4, 12)};
    ace::AceSketch a{f, ace::CounterWidth::k32};
    a.insert(normals(3, 1));
    ace::AceSketch b = a;
    b.insert(normals(3, 2));
    check(a.size() == 1 && b.size() == 2, "AceSketch copy is deep");
  }
  // test_srp.cpp:169-194 / test_sketch.cpp:118-126: the noisy variant
  {
    auto c = cfg(6, 4, 2, 1);
    c.noise_scale = 1.5;
    const ace::SrpFamily f{c};
    const auto x = normals(6, 3);
    f.reset_noise_stream(99);
    const auto first = f.bucket(0, x);
    f.reset_noise_stream(99);
    check(f.bucket(0, x) == first, "noisy bucket reproducible after reset_noise_stream");
    const std::size_t m = 4000;
    const auto y = normals(10, 9);
    double previous = 1.0;
    bool below = true, falling = true;
    for (const double noise : {0.5, 2.0, 8.0}) {
      auto cn = cfg(10, 1, m, 77);
      cn.noise_scale = noise;
      const ace::SrpFamily g{cn};
      g.reset_noise_stream(4242);
      std::size_t hits = 0;
      for (std::size_t j = 0; j < m; ++j) hits += g.bit(j, 0, y) == g.bit(j, 0, y);
      const double rate = static_cast<double>(hits) / m;
      below = below && rate < 1.0;
      falling = falling && rate < previous;
      previous = rate;
    }
    check(below && falling, "noisy self-collision rate < 1 and decreasing in noise");
    ace::AceSketch s{f};
    s.insert(std::vector<double>{1, 2, 3, 4, 5, 6});
    check(s.size() == 1, "noisy insert counts the point");
    expect_throw<ace::UnsupportedOperation>([&] { s.remove(std::vector<double>{1, 2, 3, 4, 5, 6}); },
                                            "noisy remove reports UnsupportedOperation");
  }
  // test_io.cpp: ACE1 save/load round-trips state and scores bit-exactly
  {
    const char* tmp = std::getenv("TMPDIR");
    const std::string dir = tmp ? tmp : "/tmp";
    const std::string path = dir + "/ace_dropin_sketch.ace";
    ace::Dataset data;
    data.rows = 120;
    data.cols = 6;
    for (std::size_t i = 0; i < data.rows; ++i) {
      const auto r = normals(6, 1000 + i);
      data.values.insert(data.values.end(), r.begin(), r.end());
    }
    const auto sketch = ace::build_sketch(data, 10, 20, 99);
    ace::io::save_sketch(sketch, path);
    const auto loaded = ace::io::load_sketch(path);
    check(loaded.size() == sketch.size(), "ACE1: size round-trips");
    check(loaded.mean() == sketch.mean(), "ACE1: mean round-trips bit-exactly");
    check(loaded.saturated() == sketch.saturated(), "ACE1: saturation flag round-trips");
    check(loaded.counter_width() == sketch.counter_width(), "ACE1: counter width round-trips");
    check(loaded.family().config().seed == 99, "ACE1: seed round-trips");
    check(loaded.counters_flat() == sketch.counters_flat(), "ACE1: counters round-trip");
    bool same = true;
    for (std::size_t i = 0; i < 100; ++i)
      same = same && loaded.score(data.row(i % data.rows)).value == sketch.score(data.row(i % data.rows)).value;
    check(same, "ACE1: scores of the loaded sketch are identical");
    {
      std::ofstream bad(dir + "/ace_dropin_bad.ace", std::ios::binary);
      bad << "NOPEnotasketch";
    }
    expect_throw<ace::DataError>([&] { ace::io::load_sketch(dir + "/ace_dropin_bad.ace"); },
                                 "ACE1: bad magic throws DataError");
    std::ifstream in(path, std::ios::binary);
    std::string bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    {
      std::ofstream tr(dir + "/ace_dropin_trunc.ace", std::ios::binary);
      tr.write(bytes.data(), static_cast<std::streamsize>(bytes.size() - 7));
    }
    expect_throw<ace::DataError>([&] { ace::io::load_sketch(dir + "/ace_dropin_trunc.ace"); },
                                 "ACE1: truncated payload throws DataError");
  }
  std::printf("%d failure(s)\n", failures);
  return failures;
}
