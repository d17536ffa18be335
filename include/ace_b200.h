/*
 * ace_b200.h — C ABI of the B200-native ACE hot path (libace_dev.so).
 *
 * The reference exposes this path only as a C++ class API
 * (/root/reference/proj/include/ace/{srp,sketch,detect,estimators}.hpp); it has
 * no FFI.  These entry points are what that API binds to in this framework:
 * the drop-in C++ headers under include/ace/ (libace.so) and the Python mirror
 * (paper_1706_06664_b200.ace) both call exactly these functions.  No C++ or
 * torch types cross the boundary: plain pointers, sizes and status codes.
 *
 * Conventions
 *   - Every function returns an ace_status; on failure ace_last_error()
 *     returns a thread-local message.  Status codes map one-to-one onto the
 *     reference's exception types (proj/include/ace/errors.hpp:9-26).
 *   - Point matrices are row-major, `n` rows of `dim` values with row stride
 *     `ld` elements, dtype ACE_F32 (the north-star input) or ACE_F64 (the
 *     reference's std::span<const double> per-point API).  `where` says
 *     whether a pointer is host (ACE_HOST; pageable or pinned) or device
 *     (ACE_DEVICE) memory.
 *   - Bucket ids are table-major: ids[t * n + i] (t < L, i < n).
 *   - Flags are bitmaps: bit (i % 32) of word i / 32.
 *   - All device work of a sketch runs on its own CUDA stream (single
 *     writer, sketch.hpp:23-24); calls are synchronous unless stated.
 */
#ifndef ACE_B200_H_
#define ACE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ACE_OK = 0,
  ACE_E_CONTRACT = 1,      /* ContractViolation (std::invalid_argument)   */
  ACE_E_UNSUPPORTED = 2,   /* UnsupportedOperation                         */
  ACE_E_INCONSISTENT = 3,  /* InconsistentDelete (sketch unchanged)        */
  ACE_E_DATA = 4,          /* DataError                                    */
  ACE_E_CUDA = 5,          /* CUDA runtime failure / no device             */
  ACE_E_NOMEM = 6          /* device allocation failure                    */
} ace_status;

enum { ACE_F32 = 0, ACE_F64 = 1 };
enum { ACE_HOST = 0, ACE_DEVICE = 1 };

typedef struct AceFamily AceFamily; /* SrpFamily: W on device   */
typedef struct AceSketch AceSketch; /* AceSketch: counters, n, mean */

/* Hash statistics of one call (exactness guard, SURVEY.md §7 hard part 1). */
typedef struct {
  uint64_t projections; /* n * K * L                                      */
  uint64_t rechecked;   /* projections inside the fast-path error margin,
                           recomputed as the reference's FP64 fold        */
  uint64_t flipped;     /* rechecked projections whose fast sign was wrong */
  uint64_t near_ties;   /* projections with |<x,w>| < 1e-6 |x| |w| (the
                           BASELINE.json near-tie measure, evaluated on the
                           exact fold as the oracle does)                  */
} AceHashStats;

/* detect_batch result (detect.hpp:12-22 DetectionReport + exactness info). */
typedef struct {
  double score_mean;
  double score_stddev;
  double threshold;
  uint64_t reported;
  uint64_t ambiguous;   /* points whose score lies within the rigorous
                           rounding band of the threshold               */
  int replayed;         /* 1 if the reference's sequential sums were
                           replayed on the device to settle them         */
  double elapsed_seconds;
} AceBatchReport;

/* Streaming batch result (detect.hpp:34-36 detect_stream, per batch). */
typedef struct {
  double mean_before;   /* sketch mean used for the cut                  */
  double cut;           /* mean_before - alpha                           */
  uint64_t reported;
  uint64_t ambiguous;   /* scores within 1e-9 relative of the cut        */
} AceStreamReport;

/* ---- library ----------------------------------------------------------- */
const char* ace_last_error(void);
/* Version / build tag, e.g. "ace-b200 sm_100a". */
const char* ace_version(void);
/* 1 if a CUDA device is usable, 0 otherwise (no error set). */
int ace_device_available(void);

/* ---- SrpFamily (srp.hpp:26-75) ----------------------------------------- */
/* Uploads the (K*L) x dim binary64 projection matrix W (row t*K+b, as
 * produced by SrpFamily's constructor, srp.cpp:36-48) and derives the
 * fast-path operands.  Validation as srp.cpp:25-32; noise_scale > 0 is
 * ACE_E_UNSUPPORTED (no device noise path). */
ace_status ace_family_create(uint64_t dim, uint32_t k_bits, uint32_t num_tables,
                             double noise_scale, const double* w_host,
                             AceFamily** out);
ace_status ace_family_destroy(AceFamily* fam);
/* Projection kernel selection: 0 = automatic (tcgen05 when the shape is
 * supported), 1 = SIMT FP32 kernel, 2 = tcgen05 kernel (ACE_E_UNSUPPORTED if
 * the shape is not).  For testing both paths; results are identical. */
ace_status ace_family_set_kernel(AceFamily* fam, int which);
/* Which kernel the next hash will use (1 SIMT, 2 tcgen05). */
int ace_family_kernel(const AceFamily* fam);
/* Bucket ids of n points for all L tables (SrpFamily::bucket,
 * srp.cpp:106-113, batched).  ids: L*n uint32, table-major, in `ids_where`
 * memory. */
ace_status ace_family_buckets(AceFamily* fam, const void* x, int dtype,
                              uint64_t n, uint64_t ld, int x_where,
                              uint32_t* ids, int ids_where, AceHashStats* stats);

/* Noisy (private) hashing, SrpFamily::bit with noise_scale > 0
 * (srp.cpp:93-104), exact: for tables [t0, t0+nt) and bits [b0, b0+nb) of
 * each, value = RN(p + noise[(i*nt + t-t0)*nb + b-b0]) with p the binary64
 * left fold and noise the pre-scaled terms noise_scale * N(0,1) drawn on the
 * host in tick order (ace_noise_terms, include/ace_host.h); bit = value >= 0,
 * packed MSB-first into ids[(t-t0)*n + i].  The regular hashing entry points
 * return ACE_E_UNSUPPORTED for a noisy family. */
ace_status ace_family_buckets_noisy(AceFamily* fam, const void* x, int dtype,
                                    uint64_t n, uint64_t ld, int x_where,
                                    uint32_t t0, uint32_t nt, uint32_t b0, uint32_t nb,
                                    const double* noise, int noise_where,
                                    uint32_t* ids, int ids_where);

/* ---- AceSketch (sketch.hpp:25-84) -------------------------------------- */
/* counter_width 16 or 32 (CounterWidth, sketch.hpp:11). */
ace_status ace_sketch_create(AceFamily* fam, uint32_t counter_width,
                             AceSketch** out);
ace_status ace_sketch_clone(const AceSketch* src, AceSketch** out);
ace_status ace_sketch_destroy(AceSketch* sk);
/* Zero counters, n, mean. */
ace_status ace_sketch_reset(AceSketch* sk);
/* Use an external CUDA stream (cudaStream_t) instead of the sketch's own;
 * NULL restores the private stream. */
ace_status ace_sketch_set_stream(AceSketch* sk, void* cuda_stream);
/* Per-sketch execution options (results are identical under every setting):
 *   ACE_OPT_H2D_CHUNKS    pinned host rows of a large batch are copied in this
 *                         many chunks, each hashed as it lands (default 8;
 *                         1 = one copy, then the work);
 *   ACE_OPT_DEFER_INSERT  build + detect: fuse the insert into the detect
 *                         tail's count-and-gather pass: 0 = when the batch is
 *                         large enough (default), 1 = whenever the sketch
 *                         allows it (32-bit, K <= 16), -1 = never;
 *   ACE_OPT_STREAM_GROUP  ace_sketch_stream_run: batches hashed by one
 *                         projection launch (default 4; 1..64; throughput vs
 *                         per-batch latency);
 *   ACE_OPT_STREAM_PIPE   ace_sketch_stream_run: P > 0 = the projection of
 *                         group g + 1 runs on P SMs beside the stream kernel
 *                         of group g (one CTA per table plus scoring CTAs on
 *                         the other SMs; K <= 15, batches of at most 65,536
 *                         rows, more than one group, tables + 4 + P <= SM
 *                         count, else ignored); 0 = projection and stream
 *                         kernels one after the other on the whole GPU (lower
 *                         per-batch latency); -1 (default) = P = SM count -
 *                         tables - 8.  Same results. */
enum { ACE_OPT_H2D_CHUNKS = 1, ACE_OPT_DEFER_INSERT = 2, ACE_OPT_STREAM_GROUP = 3, ACE_OPT_STREAM_PIPE = 4 };
ace_status ace_sketch_set_option(AceSketch* sk, int option, int64_t value);

/* AceSketch::insert (sketch.cpp:50-72) for n rows, in row order.
 * A few host rows (n <= 32, n * dim * size <= 3 KB) of a 32-bit sketch with
 * stats == NULL take the per-point path: one kernel launch carrying the rows
 * by value, and the call returns without waiting (every later call on the
 * sketch is ordered after it; x may be reused at once). */
ace_status ace_sketch_insert(AceSketch* sk, const void* x, int dtype, uint64_t n,
                             uint64_t ld, int x_where, AceHashStats* stats);
/* Insert / score n points given by their bucket ids (L x n, table-major,
 * ids < 2^K; host ids are validated): the counter, mean and score logic of
 * AceSketch::insert / score without hashing (the noisy variant's path). */
ace_status ace_sketch_insert_ids(AceSketch* sk, const uint32_t* ids, uint64_t n, int where);
ace_status ace_sketch_score_ids(AceSketch* sk, const uint32_t* ids, uint64_t n, int where,
                                double* scores, uint64_t* sums, int out_where);
/* AceSketch::remove (sketch.cpp:74-106) for n rows.  The batch is
 * all-or-nothing: if any target counter would reach below zero the call
 * returns ACE_E_INCONSISTENT and the sketch is unchanged. */
ace_status ace_sketch_remove(AceSketch* sk, const void* x, int dtype, uint64_t n,
                             uint64_t ld, int x_where, AceHashStats* stats);
/* AceSketch::score (sketch.cpp:108-116) for n rows: scores[i] = S_i / L.
 * scores and/or sums (uint64 S_i) may be NULL. */
ace_status ace_sketch_score(AceSketch* sk, const void* x, int dtype, uint64_t n,
                            uint64_t ld, int x_where, double* scores,
                            uint64_t* sums, int out_where, AceHashStats* stats);
/* detect_stream (detect.cpp:76-84) for each of n queries against the
 * current sketch (nothing inserted): scores[i] (host, may be NULL) and
 * flags[i] = scores[i] <= mean - alpha (host bytes, may be NULL).
 * alpha < 0 or an empty sketch is ACE_E_CONTRACT, checked in the
 * reference's order.  A few host queries take the per-point path (one
 * launch, results in mapped host memory, one wait). */
ace_status ace_sketch_detect_stream(AceSketch* sk, const void* q, int dtype,
                                    uint64_t n, uint64_t ld, int q_where,
                                    double alpha, double* scores,
                                    uint8_t* flags);
/* detect_batch (detect.cpp:12-74): score every row against the current
 * counts, mean / population stddev, flag score < mean - stddev.
 * flag_bits ((n+31)/32 words) and scores may be NULL. */
ace_status ace_sketch_detect_batch(AceSketch* sk, const void* x, int dtype,
                                   uint64_t n, uint64_t ld, int x_where,
                                   uint32_t* flag_bits, double* scores,
                                   int out_where, AceBatchReport* report,
                                   AceHashStats* stats);
/* The batch pipeline build_sketch + detect_batch (estimators.cpp:79-92 then
 * detect.cpp:12-74) in one call: insert all n rows, then detect over the
 * same rows, hashing each row once. */
ace_status ace_sketch_build_detect(AceSketch* sk, const void* x, int dtype,
                                   uint64_t n, uint64_t ld, int x_where,
                                   uint32_t* flag_bits, double* scores,
                                   int out_where, AceBatchReport* report,
                                   AceHashStats* stats);
/* Streaming batch in the reference's streaming order (detect.cpp:76-84 +
 * ace_cli.cpp:177-183, insert deferred to the batch end): every row is
 * scored against the counts at batch start and flagged iff
 * score <= mean - alpha (nothing is flagged while the sketch is empty),
 * then all rows are inserted in order.  alpha < 0 is ACE_E_CONTRACT. */
ace_status ace_sketch_stream_batch(AceSketch* sk, const void* x, int dtype,
                                   uint64_t n, uint64_t ld, int x_where,
                                   double alpha, uint32_t* flag_bits,
                                   double* scores, int out_where,
                                   AceStreamReport* report, AceHashStats* stats);

/* The streaming driver over many batches: rows [0, n) in consecutive
 * batches of `batch` rows (a positive multiple of 32), each handled exactly
 * like ace_sketch_stream_batch, all queued on the sketch's stream with no
 * host synchronisation until the end.  flag_bits: (n+31)/32 words;
 * batch_ms (host, ceil(n/batch) floats, may be NULL): per-batch device
 * latency from CUDA events; report->reported / ambiguous are run totals. */
ace_status ace_sketch_stream_run(AceSketch* sk, const void* x, int dtype,
                                 uint64_t n, uint64_t ld, int x_where,
                                 uint64_t batch, double alpha,
                                 uint32_t* flag_bits, int out_where,
                                 float* batch_ms, AceStreamReport* report,
                                 AceHashStats* stats);

/* State (sketch.hpp:44-69). */
ace_status ace_sketch_info(const AceSketch* sk, uint64_t* n, double* mean,
                           int* saturated);
/* One counter (AceSketch::counter): a 4-byte device read. */
ace_status ace_sketch_counter(const AceSketch* sk, uint32_t table,
                              uint64_t bucket, uint64_t* value);
/* counters: L * 2^K values, array-major (counters_flat), host memory. */
ace_status ace_sketch_counters(const AceSketch* sk, uint64_t* counters);
ace_status ace_sketch_counters_u32(const AceSketch* sk, uint32_t* counters,
                                   int where);
/* AceSketch::restore (sketch.cpp:132-150). */
ace_status ace_sketch_restore(AceSketch* sk, const uint64_t* counters,
                              uint64_t num_counters, uint64_t n, double mean,
                              int saturated);
/* Device-resident counters (read-only view for zero-copy consumers). */
const uint32_t* ace_sketch_device_counters(const AceSketch* sk);
/* Number of kernels this library has launched since load (diagnostics). */
uint64_t ace_kernel_launches(void);
/* Phase timing with CUDA events on the sketch's stream (off by default):
 * after each call, ms[0] = hash (+ recheck + insert), ms[1] = score,
 * ms[2] = threshold + flags (batch) or stream flags + insert (stream),
 * ms[3] = x conversion pre-pass (0 where the projection kernel converts the
 * raw rows itself, d <= 256), ms[4] = tcgen05 projection kernel.  After
 * ace_sketch_stream_run: ms[0] = ms[4] = all hashing (projection launches
 * with their near-tie passes), ms[2] = all stream kernels (phases A and B). */
ace_status ace_sketch_set_timing(AceSketch* sk, int enable);
ace_status ace_sketch_timings(const AceSketch* sk, double* ms5);

#ifdef __cplusplus
}
#endif
#endif /* ACE_B200_H_ */
