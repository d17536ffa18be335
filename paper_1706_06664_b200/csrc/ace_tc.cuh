// tcgen05 projection path (ace_hash_tc.cu).
#pragma once
#include "ace_common.cuh"

namespace ace_dev {

// Fast-path operands of the tensor-core projection:
//   W rows normalised to ||w|| = 2^14 (binary64), split into fp16 hi + lo;
//   directions packed densely (tile j = directions 128j..128j+127, tables may
//   straddle tiles), stored per (tile j, K-chunk kc) as two 128-row x 64-col blocks
//   in the canonical K-major SWIZZLE_128B shared-memory image (16 KB each),
//   so one cp.async.bulk per block lands them ready for tcgen05.mma.
struct TcFamily {
  uint16_t* w16 = nullptr;   // [ntiles][nkc][2][128*64] fp16 (swizzled)
  uint32_t nkc = 0;          // K-chunks of 64: dpad64 / 64
  uint32_t ntiles = 0;       // 128-direction tiles (directions packed densely)
  int enabled = 0;
};

struct TcArgs {
  const void* x;
  int x_f64;
  uint64_t n, ld, dim;
  uint32_t k_bits, tables, tpt, ntiles, nkc;
  const uint16_t* w16;
  uint16_t* x16;              // converted x tiles (pre-pass output), SW128 image
  float* rowthr;              // per-row error threshold (pre-pass output)
  float margin_c;             // relative error bound
  uint32_t* ids;              // table-major, stride n
  unsigned long long* near_list;  // (row << 32) | direction
  unsigned long long near_cap;
  uint32_t* overflow_rows;    // bitmap over rows; rows rechecked in full
  DevState* st;
  int dbg;  // experiments: 1 = skip epilogue work, 2 = skip MMAs, 4 = skip convert, 8 = half W
  unsigned long long* prof;  // instrumentation: wait cycles per barrier kind (or null)
};

cudaError_t tc_prepare_family(const FamilyDev& f, TcFamily* tc);
void tc_free_family(TcFamily* tc);
// X -> fp16 hi/lo SW128 tile image + per-row thresholds (must precede the hash)
cudaError_t launch_convert_x(const TcArgs& a, cudaStream_t s);
cudaError_t launch_hash_tc(const TcArgs& a, cudaStream_t s);
// Exact FP64 recheck of the near-tie list (patches ids) + rows that
// overflowed the list (all projections recomputed).
cudaError_t launch_recheck(const TcArgs& a, const double* w64, cudaStream_t s);
size_t tc_smem_bytes(uint32_t nkc);
bool tc_supported(uint64_t dim);

}  // namespace ace_dev
