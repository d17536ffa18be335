// Kernel entry points of libace_dev.so (implemented in ace_kernels.cu).
#pragma once
#include "ace_common.cuh"

namespace ace_dev {

struct HashArgs {
  const void* x;
  int x_f64;
  uint64_t n, ld;          // rows, row stride (elements)
  FamilyDev fam;
  float margin_c;          // relative error bound of the fast projection
  uint32_t* ids;           // table-major, ids[t * ids_stride + i]
  uint64_t ids_stride;
  uint64_t id_base;        // ids written at column id_base + i
  // fused insert (batch build): counters += 1 at each bucket
  uint32_t* counters;      // L x 2^K
  int insert;
  uint32_t cap;            // 0xffff (k16) or 0xffffffff (k32)
  DevState* st;
};

// ||w|| per direction as the oracle computes it (sequential binary64 fold of
// w*w, IEEE sqrt): the near-tie measure |p| < 1e-6 |x| |w|.  Synchronous.
cudaError_t launch_wnorm64(const double* w64, uint64_t dim, uint32_t rows, double* out);

// SIMT FP32 projection + FP64 near-tie recheck + bucket packing (+ insert).
cudaError_t launch_hash_simt(const HashArgs& a, cudaStream_t s);
size_t hash_simt_smem_bytes();

// Counter updates from ids (streaming insert / remove), warp-aggregated.
//   sign = +1 insert, -1 remove (remove assumes validation passed).
//   track_t = false (32-bit, no saturation possible): T is recomputed as
//   sum c^2 instead of accumulated from returned pre-add values.
cudaError_t launch_apply_ids(const uint32_t* ids, uint64_t n, uint32_t tables,
                             uint32_t k_bits, uint32_t* counters, uint32_t cap,
                             int sign, DevState* st, cudaStream_t s, bool track_t = true,
                             uint64_t ids_stride = 0);  // 0: n
// build (deferred insert, gather = 1: 32-bit, K <= 16) + detect_batch tail in
// one cooperative launch: counts, ids replaced by final counts, scores, exact
// threshold, flags, sequential replay when ambiguous.  gather = 0: scores
// gathered from the final counters, then threshold and flags.
cudaError_t launch_detect_tail(uint32_t* ids, uint64_t n, uint32_t tables, uint32_t k_bits, uint32_t* counters,
                               int gather, uint64_t* sums, double* scores, uint32_t* flag_bits, DevState* st,
                               cudaStream_t s);
// Noisy hashing (srp.cpp:93-104), exact: tables [t0, t0+nt), bits [b0, b0+nb)
// of each; noise[(i*nt + tt)*nb + (b-b0)] pre-scaled terms in tick order.
cudaError_t launch_noisy_buckets(const void* x, int x_f64, uint64_t n, uint64_t ld, uint64_t dim, const double* w64,
                                 uint32_t k_bits, uint32_t t0, uint32_t nt, uint32_t b0, uint32_t nb,
                                 const double* noise, uint32_t* ids, cudaStream_t s);
// Remove validation: counts, per counter, how many removals target it and
// flags underflow (any count < demand).  scratch: L x 2^K u32, zeroed here.
cudaError_t launch_remove_check(const uint32_t* ids, uint64_t n, uint32_t tables,
                                uint32_t k_bits, const uint32_t* counters,
                                uint32_t* scratch, DevState* st, cudaStream_t s);

// Sticky saturation for k16: clamp to cap, set st->saturated.
cudaError_t launch_cap(uint32_t* counters, uint64_t num, uint32_t cap, DevState* st,
                       cudaStream_t s);

// Scores: S_i = sum_t counters[t*2^K + ids[t*stride+i]]; optional outputs;
// accumulates sum S and sum S^2 into st (u128).
cudaError_t launch_score(const uint32_t* ids, uint64_t ids_stride, uint64_t n,
                         uint32_t tables, uint32_t k_bits, const uint32_t* counters,
                         uint64_t* sums, double* scores, DevState* st, cudaStream_t s);

// Streaming: score against current counts, flag score <= mean - alpha.
cudaError_t launch_stream_score(const uint32_t* ids, uint64_t n, uint32_t tables,
                                uint32_t k_bits, const uint32_t* counters,
                                double alpha, uint32_t* flag_bits, double* scores,
                                DevState* st, cudaStream_t s, uint64_t ids_stride = 0);  // 0: n

// Streaming (32-bit, unsaturable, K <= 16), no grid barrier: one launch runs
// phase B of the previous batch (scores from cnt_in [L][n_prev], flags
// against slot_b's cut) and phase A of batch b (counts at batch start into
// cnt_out [L][n], insert, T exact; the cut of batch b recorded in slot_a).
// n = 0: phase B only; n_prev = 0: phase A only.
// The stream over one group of batches per launch (stream_group_kernel):
// u16 ids [tables][ids_ld] of n rows in batches of `batch`; co ([batches]
// [tables][batch] u32), dT ([batches][2 tables] u64) and done ([batches] u32,
// all 0 between launches) are scratch; flags receive the group's flag words.
// hash_ctas != 0 selects stream_solo_kernel: one CTA per table plus scoring
// CTAs on the SMs a projection kernel capped at hash_ctas CTAs leaves free, so
// the next group's projection runs beside this group's stream kernel.
bool stream_group_ok(uint32_t tables, uint32_t k_bits, uint64_t batch);
bool stream_solo_ok(uint32_t tables, uint32_t k_bits, uint64_t batch, uint32_t hash_ctas);
cudaError_t launch_stream_group(const uint16_t* ids, uint64_t ids_ld, uint64_t n, uint64_t batch, uint32_t tables,
                                uint32_t k_bits, uint32_t* counters, uint32_t* co, unsigned long long* dT,
                                unsigned int* done, unsigned int* claim, uint32_t* flags, double alpha, DevState* st,
                                cudaStream_t s, uint32_t hash_ctas = 0);
// The stream driver hashes into u16 ids (ids16) where the pair kernel runs
// (K <= 15, batches of at most 2 x 65,535 rows, two CTAs per table fit).
bool stream_pair_ok(uint32_t tables, uint32_t k_bits, uint64_t batch);
cudaError_t launch_stream_apply(const uint32_t* ids, uint64_t n, uint64_t ids_stride, uint32_t tables, uint32_t k_bits,
                                uint32_t* counters, uint32_t* cnt_out, uint32_t slot_a, const uint32_t* cnt_in,
                                uint64_t n_prev, uint32_t* flag_bits, double* scores, uint32_t slot_b, double alpha,
                                DevState* st, cudaStream_t s, int ids16 = 0);

// Per-point path (AceSketch::insert / score / detect_stream one query at a
// time, sketch.hpp:33,42, detect.hpp:34-36): up to kPointMaxRows rows passed
// by value in the launch parameters (no staging copy); one cluster of CTAs
// runs the exact binary64 folds (srp.cpp:78-113, one thread per (row,
// direction), W transposed so loads coalesce) and ORs the bucket bits into
// CTA 0's shared memory; CTA 0 then gathers (score: S_i into host-mapped
// memory, the ids kept for an insert of the same rows) or inserts (c += 1,
// T += 2c + 1, n += rows; 32-bit unsaturable sketches only) and snapshots n
// and T into host-mapped memory.  One launch per call.
constexpr uint32_t kPointMaxRows = 32;
constexpr uint32_t kPointXBytes = 3072;   // rows by value: n * dim * sizeof(elem)
constexpr uint32_t kPointXSmall = 512;    // a smaller parameter block when the rows fit
enum { kPointScore = 0, kPointInsert = 1, kPointInsertCached = 2 };
struct PointHdr {
  const double* w64t;           // dim x rows: W transposed (binary64)
  uint64_t dim;
  uint32_t k_bits, tables, rows, n;
  int x_f64;
  int mode;                     // kPointScore / kPointInsert / kPointInsertCached
  uint32_t pend_n;              // kPointScore: a deferred insert of the cached ids (rows) applied first
  uint32_t* counters;
  DevState* st;
  uint32_t* cache;              // n x tables: ids of the last score (read by kPointInsertCached)
  double* scores;               // host-mapped [n] (score)
  unsigned long long* sums;     // host-mapped [n] (score)
  unsigned long long* snap;     // host-mapped: n, T after the call
};
template <uint32_t XB>
struct PointArgs {
  PointHdr h;
  alignas(16) unsigned char x[XB];  // n x dim, dense, fp32 or fp64
};
template <uint32_t XB>
cudaError_t launch_point(const PointArgs<XB>& a, cudaStream_t s);

// Sum of squares of all counters (T after restore with exact state).
cudaError_t launch_sum_squares(const uint32_t* counters, uint64_t num,
                               unsigned long long* out, cudaStream_t s);

}  // namespace ace_dev
