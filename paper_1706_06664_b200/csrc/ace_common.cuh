// Shared definitions of the ACE device library (libace_dev.so).
#pragma once
#include <cuda_runtime.h>
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
};

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
};

void set_error(const std::string& msg);
extern std::atomic<unsigned long long> g_launches;

inline void count_launch(unsigned long long k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

}  // namespace ace_dev
