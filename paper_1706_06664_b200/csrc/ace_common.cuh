// Shared definitions of the ACE device library (libace_dev.so).
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "ace_b200.h"

namespace ace_dev {

// Device-resident per-sketch state; host reads it back after each call.
struct DevState {
  unsigned long long T;          // sum of insert numerators = n * L * mean
  unsigned long long n;          // points inserted
  unsigned long long sum_lo, sum_hi;  // sum_i S_i         (u128)
  unsigned long long sq_lo, sq_hi;    // sum_i S_i^2       (u128)
  unsigned long long reported;
  unsigned long long ambiguous;
  unsigned long long rechecked;
  unsigned long long flipped;
  unsigned long long near_ties;      // |p| < 1e-6 |x| |w| (BASELINE.json near-tie measure), exact
  unsigned long long near_count;     // tc path: near-tie items pushed
  unsigned long long near_overflow;  // tc path: list overflowed (rows rechecked in full)
  unsigned long long batch_sum;      // stream: sum of the batch's pre-insert S_i
  unsigned int ticket_a, ticket_b;   // detect tail: blocks done with the score / flag phases
  unsigned long long underflow;  // remove: counters that would go negative
  int saturated;
  int replayed;
  long long s_cut;               // flag iff S <= s_cut
  long long s_lo, s_hi;          // ambiguity band in S units (inclusive)
  double mean, sd, thr;          // detect_batch statistics
  double cut;                    // stream cut (mean - alpha)
  double mean_before;
  // stream cut per batch (stream_apply_kernel): recorded by the batch's
  // phase A from the state before its insert, read by its phase B one launch
  // later (two slots, alternating); not reset per call
  double cut_ring[2], mean_ring[2];
  int live_ring[2];
  unsigned int ticket_s;         // phase-A blocks done (the last one commits T and n)
  unsigned long long dT_acc;     // phase-A increments of T pending the last block's commit
  unsigned int ticket_r;         // recheck_near_kernel: blocks done (the last one cleans the overflow state)
  // stream_group_kernel: T and n before each group (two slots, alternating),
  // recorded by the group's last phase-A CTA, read by its phase B one launch later
  unsigned long long gbase[2][2];
  unsigned int ticket_g;
};

// T / den correctly rounded to binary64 (round half to even), T, den < 2^64:
// the exact sketch mean T / (n L) with a single rounding.  Long division
// produces 53 mantissa bits plus a round bit; the remainder is the sticky bit.
__host__ __device__ inline int ace_bits64(uint64_t v) {
#ifdef __CUDA_ARCH__
  return 64 - __clzll(static_cast<long long>(v));
#else
  return v ? 64 - __builtin_clzll(v) : 0;
#endif
}
__host__ __device__ inline double ace_div_rn(uint64_t T, uint64_t den) {
  if (T == 0 || den == 0) return 0.0;
  const uint64_t q = T / den;
  uint64_t r = T % den;  // < den
  uint64_t m;
  int e;
  bool sticky;
  const int bq = ace_bits64(q);
  if (bq >= 54) {
    const int sh = bq - 54;
    sticky = (sh > 0 && (q & ((1ull << sh) - 1ull)) != 0) || r != 0;
    m = q >> sh;
    e = sh;
  } else {
    m = q;
    e = 0;
    while (ace_bits64(m) < 54) {
      // r < den < 2^64: 2r may need 65 bits
      const bool carry = (r >> 63) != 0;
      r <<= 1;
      const uint64_t bit = (carry || r >= den) ? 1ull : 0ull;
      if (bit) r -= den;
      m = (m << 1) | bit;
      --e;
    }
    sticky = r != 0;
  }
  uint64_t mant = m >> 1;
  if ((m & 1ull) && (sticky || (mant & 1ull))) ++mant;
  if (mant == (1ull << 53)) {
    mant >>= 1;
    ++e;
  }
  return ldexp(static_cast<double>(mant), e + 1);
}

// Fast-path projection operands of a family (SIMT tile layout).
//   Columns are grouped in tiles of kTileCols; tile j holds tables
//   [j*tpt, (j+1)*tpt) with tpt = floor(kTileCols / K), column c of the tile
//   being direction (j*tpt + c/K)*K + c%K; unused columns are zero.
constexpr int kTileCols = 128;

struct FamilyDev {
  uint64_t dim;
  uint64_t dpad;     // dim rounded up to the K-chunk
  uint32_t k_bits, tables, rows;  // rows = K*L
  uint32_t tpt, ntiles, ncols;    // ncols = ntiles * kTileCols
  double* w64;       // rows x dim, binary64 (the reference's W)
  float* w32t;       // dpad x ncols, fp32, zero padded
  float* wnorm;      // ncols, upper bound of ||w|| (0 on pad columns)
  double* wnorm64;   // rows, ||w|| as the oracle computes it (sequential binary64 fold, IEEE sqrt)
};

void set_error(const std::string& msg);
extern std::atomic<unsigned long long> g_launches;

inline void count_launch(unsigned long long k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

}  // namespace ace_dev
