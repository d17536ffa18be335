// Synthetic workload generators for the five BASELINE.json configurations.
//
// Test/bench input only — not part of the ACE hot path.  Every value is a pure
// function of (seed, row, column): a counter-based hash feeds uniforms, and the
// transcendental functions (ln, exp, cos) are evaluated with basic IEEE
// operations only (+, -, *, /, sqrt, exact scaling by powers of two).  Compiled
// by gcc with -ffp-contract=off and by nvcc with --fmad=false, the host and the
// device therefore produce bit-identical float rows, so full-size inputs can be
// generated on the GPU while any prefix can be regenerated on the host for the
// CPU oracle.
//
// Configurations (BASELINE.json "configs"; choices for the ambiguities listed
// in SURVEY.md Appendix C are recorded in DESIGN.md §2):
//   1: 8 isotropic Gaussian clusters, centres U[-5,5]^40, sigma 1; 1% of rows
//      are outliers U[-15,15]^40.                              d=40
//   2: KDD-like mixed record: 3 categorical fields (cardinality 3/66/10,
//      Zipf(1.2)) one-hot -> 79 cols; 38 log-normal(0,2) cols z-scored with
//      the analytic moments; 3 zero pad cols; 3% outliers (continuous x20,
//      categories uniform).                                    d=120
//   3: i.i.d. N(0,1); 0.5% outliers shifted +6 on 16 distinct coords. d=128
//   4: rank-32 Gaussian-factor signal (unit variance per coord) + N(0, 0.1^2)
//      noise; 1% outliers full-rank N(0,1).                    d=4096
//   5: 16 clusters sigma 1, centres U[-5,5]^64 drifting 1e-7*t*(+-1) per
//      coord; outliers in bursts of 256 rows (burst prob 0.5%), U[-20,20]^64.
//      d=64
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define DG_FN __host__ __device__ static inline
#else
#define DG_FN static inline
#endif

#define DG_PHI 0x9e3779b97f4a7c15ULL

enum {
  DG_S_CLUSTER = 1,
  DG_S_OUTLIER = 2,
  DG_S_VALUE = 3,
  DG_S_CENTER = 4,
  DG_S_FACTOR = 5,
  DG_S_BASIS = 6,
  DG_S_CAT = 7,
  DG_S_SHIFT = 8,
  DG_S_DRIFT = 9,
  DG_S_NOISE = 10
};

DG_FN uint64_t dg_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

DG_FN uint64_t dg_key(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
  uint64_t h = dg_mix(seed + stream * DG_PHI);
  h = dg_mix(h ^ (a * 0xd1b54a32d192ed03ULL + DG_PHI));
  return dg_mix(h ^ (b * 0x8cb92ba72f3d8dd7ULL + 0x632be59bd9b4e019ULL));
}

// Uniform in (0, 1].
DG_FN double dg_unit(uint64_t h) {
  return (double)((h >> 11) + 1) * (1.0 / 9007199254740992.0);
}

DG_FN double dg_bits_to_double(uint64_t b) {
  union {
    uint64_t u;
    double d;
  } c;
  c.u = b;
  return c.d;
}
DG_FN uint64_t dg_double_to_bits(double d) {
  union {
    uint64_t u;
    double d;
  } c;
  c.d = d;
  return c.u;
}

// Natural log of a positive normal double: x = m * 2^e, m in [1,2),
// ln m = 2 atanh((m-1)/(m+1)) by its odd series.
DG_FN double dg_ln(double x) {
  const uint64_t b = dg_double_to_bits(x);
  const int e = (int)((b >> 52) & 0x7ff) - 1023;
  const double m = dg_bits_to_double((b & 0x000fffffffffffffULL) |
                                     0x3ff0000000000000ULL);
  const double s = (m - 1.0) / (m + 1.0);
  const double s2 = s * s;
  double acc = 1.0 / 27.0;
  for (int k = 25; k >= 1; k -= 2) acc = 1.0 / (double)k + s2 * acc;
  return (double)e * 0.6931471805599453094 + 2.0 * s * acc;
}

// 2^k for |k| < 1000, exact.
DG_FN double dg_pow2(int k) {
  return dg_bits_to_double((uint64_t)(k + 1023) << 52);
}

DG_FN double dg_exp(double y) {
  const double inv_ln2 = 1.4426950408889634074;
  double kf = y * inv_ln2;
  int k = (int)(kf < 0 ? kf - 0.5 : kf + 0.5);
  const double r = y - (double)k * 0.6931471805599453094;
  double acc = 1.0;
  for (int n = 18; n >= 1; --n) acc = 1.0 + r * acc / (double)n;
  return acc * dg_pow2(k);
}

// cos(2*pi*t) for t in (0, 1].
DG_FN double dg_cos2pi(double t) {
  double v = t - (double)(int64_t)(t + 0.5);  // [-0.5, 0.5]
  double a = v < 0 ? -v : v;
  double sign = 1.0;
  if (a > 0.25) {
    a = 0.5 - a;
    sign = -1.0;
  }
  const double x = 6.283185307179586477 * a;  // [0, pi/2]
  const double x2 = x * x;
  double acc = 1.0;
  for (int n = 22; n >= 2; n -= 2) acc = 1.0 - x2 * acc / (double)(n * (n - 1));
  return sign * acc;
}

// Standard normal from two independent hashes (Box-Muller, cosine branch).
DG_FN double dg_normal(uint64_t h1, uint64_t h2) {
  const double u1 = dg_unit(h1);
  const double u2 = dg_unit(h2);
  return sqrt(-2.0 * dg_ln(u1)) * dg_cos2pi(u2);
}

DG_FN double dg_normal_at(uint64_t seed, uint64_t stream, uint64_t a,
                          uint64_t b) {
  return dg_normal(dg_key(seed, stream, a, 2 * b),
                   dg_key(seed, stream, a, 2 * b + 1));
}

DG_FN double dg_uniform_at(uint64_t seed, uint64_t stream, uint64_t a,
                           uint64_t b, double lo, double hi) {
  return lo + (hi - lo) * dg_unit(dg_key(seed, stream, a, b));
}

// ---------------------------------------------------------------------------
// Per-configuration shape and per-row generation.

typedef struct {
  int cfg;
  uint64_t seed;
  uint64_t dim;
  // cfg 4 only: 32 x 4096 factor basis, row-major, doubles (host or device
  // pointer as appropriate for the caller).
  const double* basis;
  // cfg 2 only: unnormalised Zipf(1.2) cumulative weights per field, and the
  // analytic log-normal(0,2) moments.
  double zipf_cum[3][66];
  double ln_mean, ln_sd;
} dg_params;

DG_FN uint64_t dg_dim(int cfg) {
  switch (cfg) {
    case 1: return 40;
    case 2: return 120;
    case 3: return 128;
    case 4: return 4096;
    case 5: return 64;
    default: return 0;
  }
}

DG_FN int dg_is_outlier(const dg_params* p, uint64_t row) {
  switch (p->cfg) {
    case 1: return dg_unit(dg_key(p->seed, DG_S_OUTLIER, row, 0)) <= 0.01;
    case 2: return dg_unit(dg_key(p->seed, DG_S_OUTLIER, row, 0)) <= 0.03;
    case 3: return dg_unit(dg_key(p->seed, DG_S_OUTLIER, row, 0)) <= 0.005;
    case 4: return dg_unit(dg_key(p->seed, DG_S_OUTLIER, row, 0)) <= 0.01;
    case 5: return dg_unit(dg_key(p->seed, DG_S_OUTLIER, row / 256, 0)) <= 0.005;
    default: return 0;
  }
}

// Zipf(1.2) category in [0, card) by inverse CDF over the cumulative
// unnormalised weights (k+1)^-1.2 = exp(-1.2 ln(k+1)).
DG_FN int dg_zipf(const double* cum, double u, int card) {
  const double target = u * cum[card - 1];
  for (int k = 0; k < card; ++k)
    if (target <= cum[k]) return k;
  return card - 1;
}

DG_FN void dg_init(dg_params* p, int cfg, uint64_t seed, const double* basis) {
  const int card[3] = {3, 66, 10};
  p->cfg = cfg;
  p->seed = dg_mix(seed + (uint64_t)cfg * 0x2545f4914f6cdd1dULL);
  p->dim = dg_dim(cfg);
  p->basis = basis;
  for (int f = 0; f < 3; ++f) {
    double c = 0.0;
    for (int k = 0; k < 66; ++k) {
      if (k < card[f]) c += dg_exp(-1.2 * dg_ln((double)(k + 1)));
      p->zipf_cum[f][k] = c;
    }
  }
  const double e2 = dg_exp(2.0), e4 = dg_exp(4.0);
  p->ln_mean = e2;
  p->ln_sd = sqrt((e4 - 1.0) * e4);
}

// Writes row `row` (dim floats) into out; returns the outlier label.
DG_FN int dg_row(const dg_params* p, uint64_t row, float* out) {
  const uint64_t s = p->seed;
  const int outl = dg_is_outlier(p, row);
  switch (p->cfg) {
    case 1: {
      const uint64_t c = dg_key(s, DG_S_CLUSTER, row, 0) % 8;
      for (uint64_t k = 0; k < 40; ++k) {
        double v;
        if (outl)
          v = dg_uniform_at(s, DG_S_VALUE, row, k, -15.0, 15.0);
        else
          v = dg_uniform_at(s, DG_S_CENTER, c, k, -5.0, 5.0) +
              dg_normal_at(s, DG_S_VALUE, row, k);
        out[k] = (float)v;
      }
      break;
    }
    case 2: {
      const int card[3] = {3, 66, 10};
      int off = 0;
      for (int f = 0; f < 3; ++f) {
        const double u = dg_unit(dg_key(s, DG_S_CAT, row, (uint64_t)f));
        int cat;
        if (outl) {
          cat = (int)(u * card[f]);
          if (cat >= card[f]) cat = card[f] - 1;
        } else {
          cat = dg_zipf(p->zipf_cum[f], u, card[f]);
        }
        for (int k = 0; k < card[f]; ++k) out[off + k] = (k == cat) ? 1.0f : 0.0f;
        off += card[f];
      }
      // log-normal(0, 2): mean e^2, variance (e^4 - 1) e^4.
      const double e2 = p->ln_mean, sd = p->ln_sd;
      for (int k = 0; k < 38; ++k) {
        const double z = dg_normal_at(s, DG_S_VALUE, row, (uint64_t)k);
        double v = (dg_exp(2.0 * z) - e2) / sd;
        if (outl) v = v * 20.0;
        out[off + k] = (float)v;
      }
      off += 38;
      for (; off < 120; ++off) out[off] = 0.0f;
      break;
    }
    case 3: {
      for (uint64_t k = 0; k < 128; ++k)
        out[k] = (float)dg_normal_at(s, DG_S_VALUE, row, k);
      if (outl) {
        const uint64_t h = dg_key(s, DG_S_SHIFT, row, 0);
        const uint64_t a = h & 127, b = ((h >> 7) & 127) | 1;
        for (uint64_t j = 0; j < 16; ++j) {
          const uint64_t k = (a + j * b) & 127;
          out[k] = (float)((double)out[k] + 6.0);
        }
      }
      break;
    }
    case 4: {
      if (outl) {
        for (uint64_t k = 0; k < 4096; ++k)
          out[k] = (float)dg_normal_at(s, DG_S_VALUE, row, k);
      } else {
        double f[32];
        for (int r = 0; r < 32; ++r)
          f[r] = dg_normal_at(s, DG_S_FACTOR, row, (uint64_t)r);
        const double inv = 1.0 / sqrt(32.0);
        for (uint64_t k = 0; k < 4096; ++k) {
          double acc = 0.0;
          for (int r = 0; r < 32; ++r) acc += f[r] * p->basis[(uint64_t)r * 4096 + k];
          out[k] = (float)(acc * inv + 0.1 * dg_normal_at(s, DG_S_NOISE, row, k));
        }
      }
      break;
    }
    case 5: {
      const uint64_t c = dg_key(s, DG_S_CLUSTER, row, 0) % 16;
      const double drift = 1e-7 * (double)row;
      for (uint64_t k = 0; k < 64; ++k) {
        double v;
        if (outl) {
          v = dg_uniform_at(s, DG_S_VALUE, row, k, -20.0, 20.0);
        } else {
          const double dir =
              (dg_key(s, DG_S_DRIFT, c, k) & 1) ? 1.0 : -1.0;
          v = dg_uniform_at(s, DG_S_CENTER, c, k, -5.0, 5.0) + drift * dir +
              dg_normal_at(s, DG_S_VALUE, row, k);
        }
        out[k] = (float)v;
      }
      break;
    }
    default:
      break;
  }
  return outl;
}

// Factor basis for cfg 4: 32 x 4096 standard normals.
DG_FN double dg_basis_entry(uint64_t seed, uint64_t r, uint64_t k) {
  return dg_normal_at(seed, DG_S_BASIS, r, k);
}
