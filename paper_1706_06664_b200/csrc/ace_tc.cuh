// tcgen05 projection path: ace_hash_tc.cu (d <= 256, raw fp32 rows through
// tensor-map TMA, fp16 split in-kernel) and ace_hash_tck.cu (d > 256,
// K-streamed).
#pragma once
#include <cuda.h>

#include "ace_common.cuh"

namespace ace_dev {

// Fast-path operands of the tensor-core projection:
//   W rows normalised to ||w|| = 2^14 (binary64), split into fp16 hi + lo;
//   directions packed densely (tile j = directions tw*j .. tw*j+tw-1, tables
//   may straddle tiles; the K-streamed kernel packs whole tables per tile),
//   stored per (tile j, K-chunk kc) as two tw-row x 64-col blocks in the
//   canonical K-major SWIZZLE_128B shared-memory image, so one cp.async.bulk
//   per block lands them ready for tcgen05.mma.
struct TcFamily {
  uint16_t* w16 = nullptr;     // [ntiles][nkc][2][tw*64] fp16 (swizzled)
  float* w32 = nullptr;        // K-streamed recheck: W rounded to fp32, [rows][dim]
  uint32_t nkc = 0;            // K-chunks of 64: dpad64 / 64
  uint32_t ntiles = 0;         // direction tiles
  uint32_t tw = 128;           // direction tile width (MMA N)
  uint32_t tpt = 0;            // K-streamed: whole tables per direction tile
  int enabled = 0;
};

struct TcArgs {
  const void* x;              // the caller's rows (fp32 or fp64): the exact recheck reads these
  int x_f64;
  uint64_t n, ld, dim;
  uint32_t k_bits, tables, tpt, ntiles, nkc;
  uint32_t tw;                // direction tile width (MMA N)
  const uint16_t* w16;
  uint16_t* x16;              // K-streamed: converted x tiles (SW128 image)
  float* rowthr;              // K-streamed: per-row error threshold
  float margin_c;             // relative error bound
  uint32_t* ids;              // table-major, stride ids_ld
  uint64_t ids_ld;            // ids row stride per table (>= n; a chunk of a longer batch writes into it)
  int ids16;                  // ids stored as u16 (K <= 16; the stream driver), else u32
  unsigned long long* near_list;  // (row << 32) | direction; one segment per CTA
  unsigned long long near_cap;    // total entries (near_cap / grid per CTA)
  const double* w64;              // the reference's W (binary64) for the exact recheck
  const double* wnorm64;          // ||w|| per direction (near-tie measure)
  uint32_t* counters;             // fused insert target (fused_insert != 0)
  int fused_insert;               // 32-bit sketch, K > 20: insert buckets in the epilogue
  uint32_t* seg_counts;           // K-streamed: near ties pushed per CTA
  const float* w32;               // K-streamed recheck: W rounded to fp32 [rows][dim]
  uint32_t* overflow_rows;        // bitmap over rows; rows rechecked in full
  DevState* st;
  uint32_t grid_cap;              // d <= 256: at most this many CTAs (0 = one per SM); the stream pipeline
};

cudaError_t tc_prepare_family(const FamilyDev& f, TcFamily* tc);
void tc_free_family(TcFamily* tc);
bool tc_supported(uint64_t dim);
// d <= 256: the projection kernel reads raw fp32 rows through a tensor map
// (16-byte aligned base and row stride); otherwise launch_hash_tc first
// stages the rows as fp32 into `stage` (fp64 input, odd strides).
bool tc_direct_ok(const void* x, int x_f64, uint64_t ld);
cudaError_t launch_hash_tc(const TcArgs& a, void* stage, cudaStream_t s);
size_t tc_stage_bytes(uint64_t n, uint64_t dim);
// Rows whose near ties overflowed their CTA's list: every bucket recomputed
// exactly (counters moved when the insert was fused).
cudaError_t launch_recheck(const TcArgs& a, cudaStream_t s);
// d <= 256: the near ties hash_tc_kernel listed (per-CTA segments, lengths in
// TcArgs::seg_counts, tc_grid(n) entries) and the overflowed rows, decided
// exactly in one launch after the projection
uint32_t tc_grid(uint64_t n, uint32_t cap = 0);
cudaError_t launch_recheck_near(const TcArgs& a, cudaStream_t s);
// K-streamed kernel for d > 256 (nkc > 4): its own conversion, projection and
// near-tie recheck (per-CTA list segments, counts in TcArgs::seg_counts)
bool tc_kstream(uint32_t nkc);
uint32_t tck_grid(uint64_t n);
float tc_margin(uint32_t nkc, bool x_f64);
float tck_margin(uint32_t nkc, bool x_f64);
cudaError_t tck_prepare(uint32_t tw);
cudaError_t launch_convert_x_wide(const TcArgs& a, cudaStream_t s);
cudaError_t launch_hash_tck(const TcArgs& a, cudaStream_t s);
cudaError_t launch_recheck_segs(const TcArgs& a, cudaStream_t s);
int tc_sms();

}  // namespace ace_dev
