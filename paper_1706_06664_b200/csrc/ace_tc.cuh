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
  float* w32 = nullptr;      // near-tie recheck (recheck_segs_kernel): W rounded to fp32, [rows][dim]
  uint32_t nkc = 0;          // K-chunks of 64: dpad64 / 64
  uint32_t ntiles = 0;       // direction tiles of tw directions (packed densely)
  uint32_t tw = 128;         // direction tile width: 192 (d <= 128) or 128; K-streamed: 256 or 128
  uint32_t tpt = 0;          // K-streamed: whole tables per direction tile (tw / K)
  int enabled = 0;
};

struct TcArgs {
  const void* x;
  int x_f64;
  uint64_t n, ld, dim;
  uint32_t k_bits, tables, tpt, ntiles, nkc;
  uint32_t tw;                // direction tile width (MMA N): 128 or 192
  const uint16_t* w16;
  uint16_t* x16;              // converted x tiles (pre-pass output), SW128 image
  float* rowthr;              // per-row error threshold (pre-pass output)
  uint32_t* lomask;           // per point tile: bit s set iff some x lo part of K16 step s is nonzero
                              // (pre-pass output, zeroed before it; null = all steps need the lo pass)
  float margin_c;             // relative error bound
  uint32_t* ids;              // table-major, stride ids_ld
  uint64_t ids_ld;            // ids row stride per table (>= n; a chunk of a longer batch writes into it)
  unsigned long long* near_list;  // (row << 32) | direction; one segment per CTA
  unsigned long long near_cap;    // total entries (the kernel uses near_cap / grid per CTA)
  const double* w64;              // the reference's W (binary64) for the exact recheck
  uint32_t* counters;             // fused insert target (fused_insert != 0)
  int fused_insert;               // 32-bit sketch: insert buckets in the epilogue
  int fuse_convert;               // convert X inside the projection kernel (no pre-pass)
  uint32_t* seg_counts;           // near ties pushed per CTA (K-streamed kernel, ext_recheck)
  const float* w32;               // recheck_segs_kernel: W rounded to fp32 [rows][dim]
  int ext_recheck;                // hash_tc_kernel: leave the near-tie list to recheck_segs_kernel
  uint32_t* overflow_rows;    // bitmap over rows; rows rechecked in full
  DevState* st;
  uint16_t tab_end[64];      // tables completed by the end of direction tile j
  int dbg;  // experiments: 1 = skip epilogue work, 2 = skip MMAs, 4 = skip convert, 8 = half W, 16 = TMEM loads only
  unsigned long long* prof;  // instrumentation: wait cycles per barrier kind (or null)
};

cudaError_t tc_prepare_family(const FamilyDev& f, TcFamily* tc);
// per-tile table ranges (TcArgs::tab_end) from k_bits, tables, ntiles
void tc_fill_tables(TcArgs* a);
void tc_free_family(TcFamily* tc);
// X -> fp16 hi/lo SW128 tile image + per-row thresholds (must precede the hash)
cudaError_t launch_convert_x(const TcArgs& a, cudaStream_t s);
cudaError_t launch_hash_tc(const TcArgs& a, cudaStream_t s);
// Rows whose near ties overflowed their CTA's list: every bucket recomputed
// exactly (counters moved when the insert was fused).  The listed near ties
// are rechecked inside hash_tc_kernel itself.
cudaError_t launch_recheck(const TcArgs& a, const double* w64, cudaStream_t s);
size_t tc_smem_bytes(uint32_t nkc);
bool tc_supported(uint64_t dim);
bool tc_fuse_ok_dim(uint64_t dim, uint32_t nkc);
// K-streamed kernel for d > 256 (nkc > 4): its own conversion, projection and
// near-tie recheck (per-CTA list segments, counts in TcArgs::seg_counts)
bool tc_kstream(uint32_t nkc);
uint32_t tck_grid(uint64_t n);
float tck_margin(uint32_t nkc, bool x_f64);
cudaError_t launch_convert_x_wide(const TcArgs& a, cudaStream_t s);
cudaError_t launch_hash_tck(const TcArgs& a, cudaStream_t s);
cudaError_t launch_recheck_segs(const TcArgs& a, cudaStream_t s);

}  // namespace ace_dev
