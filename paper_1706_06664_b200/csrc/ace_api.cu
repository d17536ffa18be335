// C ABI of libace_dev.so (include/ace_b200.h): handles, staging, pipelines.
// Each entry point cites the reference function it stands in for.
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include "ace_kernels.cuh"
#include "ace_tc.cuh"

namespace ace_dev {

thread_local std::string g_err;
std::atomic<unsigned long long> g_launches{0};

void set_error(const std::string& msg) { g_err = msg; }

}  // namespace ace_dev

using namespace ace_dev;

namespace {

constexpr uint32_t kMaxKBits = 30;  // srp.cpp:15

ace_status fail(ace_status code, const std::string& msg) {
  set_error(msg);
  return code;
}

#define ACE_CUDA(call)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(e_ == cudaErrorMemoryAllocation ? ACE_E_NOMEM : ACE_E_CUDA,              \
                  std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call);    \
  } while (0)

// Growable device buffer.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    size_t grow = std::max(want, static_cast<size_t>(1) << 20);
    cudaError_t e = cudaMalloc(&p, grow);
    if (e == cudaSuccess) bytes = grow;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

}  // namespace

struct AceSketch;

struct AceFamily {
  FamilyDev d{};
  double noise_scale = 0.0;  // > 0: noisy variant, hashed only through the *_noisy / *_ids entry points
  TcFamily tc{};
  double* w64t = nullptr;  // per-point path: W transposed (dim x rows), dims the point kernel takes
  int kernel = 0;  // 0 auto, 1 SIMT, 2 tcgen05
  float margin_c = 0.f;
  std::atomic<int> refs{1};
  // scratch state of the family-level hashing calls (ace_family_buckets*):
  // stream, staging and id buffers reused across calls, no counters; it
  // holds no reference on the family (family_release frees it)
  std::mutex scratch_mu;
  AceSketch* scratch = nullptr;
  bool use_tc() const { return tc.enabled && kernel != 1; }
};

struct AceSketch {
  AceFamily* fam = nullptr;
  uint32_t width = 32;
  uint32_t cap = 0xffffffffu;
  uint64_t num_counters = 0;
  uint32_t* counters = nullptr;
  DevState* st = nullptr;    // device
  DevState* hst = nullptr;   // pinned host mirror
  // per-point path (point_kernel): host-mapped results, the ids of the last
  // point score (kPointMaxRows x L words), and the rows inserted
  // asynchronously since the host mirror was last refreshed
  struct PointHost {
    double scores[kPointMaxRows];
    unsigned long long sums[kPointMaxRows];
    unsigned long long snap[2];
    uint32_t counter;  // ace_sketch_counter
  };
  PointHost* pth = nullptr;
  uint32_t* pbits = nullptr;  // [kPointMaxRows * L] ids of the last point score
  unsigned long long pending_rows = 0;
  std::vector<unsigned char> pcache_x;  // rows (dense) whose ids the last point score left in the cache
  uint64_t pcache_n = 0;
  int pcache_dtype = 0;
  bool pcache_valid = false;
  // insert(q) right after a point score of q: deferred (no launch) and
  // applied from the cached ids by the next point kernel, or by
  // flush_point() before any other work is queued on the sketch
  uint32_t pins_pend = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  // chunked host-input pipeline (batch_detect): H2D copies on their own
  // stream, one event per chunk
  cudaStream_t cstream = nullptr;
  cudaEvent_t cstart = nullptr;
  std::vector<cudaEvent_t> cev;
  // stream driver with pinned host rows: two staging halves, copied on
  // cstream; copy-done and hash-done events per half
  DevBuf sstage[2];
  cudaEvent_t s_copied[2] = {nullptr, nullptr}, s_used[2] = {nullptr, nullptr};
  DevBuf ids, sums, stage, flags, scores, demand, near, overflow, x16, rowthr, segc, xf32;
  DevBuf cnt[2];            // stream: counts at batch start (double-buffered)
  DevBuf gco, gdT, gdone;   // group stream kernel: counts at batch start, T increments, batches done
  int h2d_chunks = 8;       // pinned host rows of a large batch: copy chunks hashed as they land
  int defer_mode = 0;       // ACE_OPT_DEFER_INSERT
  // stream driver: batches hashed by one projection launch (hashing does not
  // depend on the counts), amortising the persistent kernel's fill and drain
  int stream_group = 4;     // ACE_OPT_STREAM_GROUP
  // stream driver pipeline: the projection of group g + 1 (capped at this many
  // CTAs) runs beside the stream kernel of group g (one CTA per table on the
  // other SMs, on pstream); 0 = one after the other on the whole GPU
  int stream_pipe = -1;     // ACE_OPT_STREAM_PIPE (-1 = automatic)
  cudaStream_t pstream = nullptr;
  cudaEvent_t p_hashed[2] = {nullptr, nullptr}, p_streamed[2] = {nullptr, nullptr};
  // build + detect over the same rows: run_hash leaves the insert to the
  // fused count-and-gather pass of the detect tail (detect_tail_kernel)
  bool defer_insert = false, insert_deferred = false;
  // restore (e.g. an ACE1 file) reports the restored mean exactly until the
  // next update, as the reference does (its mean is a stored recurrence)
  bool mean_pinned = false;
  double pinned_mean = 0.0;
  // phase timing (ace_sketch_set_timing)
  bool timing = false;
  cudaEvent_t ev[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  // stream driver phase totals (timing on): [0] hashing (projection + near-tie
  // rows + memsets), [1] stream kernels (phases A / B); valid after a stream_run
  double stream_ms[2] = {0.0, 0.0};
  bool stream_timed = false;
  bool ev_used[7] = {false, false, false, false, false, false, false};
  void mark(int i) {
    if (timing) {
      cudaEventRecord(ev[i], stream);
      ev_used[i] = true;
    }
  }
  // CUDA graph of the device work of a repeated batch call (build/detect with
  // the same arguments): captured on the second identical call, replayed after
  struct GraphKey {
    const void* x = nullptr;
    const void* flags = nullptr;
    const void* scores = nullptr;
    uint64_t n = 0, ld = 0;
    int dtype = 0, where = 0, out_where = 0, build = 0, ff = 0;
    cudaStream_t stream = nullptr;
    const void* bufs[13] = {};  // the sketch's scratch buffers (a reallocation invalidates the graph)
    bool operator==(const GraphKey& o) const {
      for (int i = 0; i < 13; ++i)
        if (bufs[i] != o.bufs[i]) return false;
      return x == o.x && flags == o.flags && scores == o.scores && n == o.n && ld == o.ld && dtype == o.dtype &&
             where == o.where && out_where == o.out_where && build == o.build && ff == o.ff && stream == o.stream;
    }
  };
  GraphKey gkey, gseen;
  // stream driver graph (ace_sketch_stream_run with device rows)
  struct StreamKey {
    const void* x = nullptr;
    const void* flags = nullptr;
    uint64_t n = 0, ld = 0, batch = 0;
    double alpha = 0.0;
    int dtype = 0, out_where = 0, group = 0;
    bool lat = false, ff = false;
    cudaStream_t stream = nullptr;
    const void* bufs[9] = {};
    bool operator==(const StreamKey& o) const {
      for (int i = 0; i < 9; ++i)
        if (bufs[i] != o.bufs[i]) return false;
      return x == o.x && flags == o.flags && n == o.n && ld == o.ld && batch == o.batch && alpha == o.alpha &&
             dtype == o.dtype && out_where == o.out_where && group == o.group && lat == o.lat && ff == o.ff &&
             stream == o.stream;
    }
  };
  StreamKey sgkey, sgseen;
  bool sgseen_valid = false;
  cudaGraphExec_t sgexec = nullptr;
  unsigned long long sglaunches = 0;
  std::vector<cudaEvent_t> lat_a, lat_b;  // per-batch latency events of the stream driver
  bool gseen_valid = false;
  cudaGraphExec_t gexec = nullptr;
  unsigned long long glaunches = 0;
  void drop_graph() {
    if (gexec) cudaGraphExecDestroy(gexec);
    gexec = nullptr;
    gseen_valid = false;
    if (sgexec) cudaGraphExecDestroy(sgexec);
    sgexec = nullptr;
    sgseen_valid = false;
  }
};

namespace {

void family_release(AceFamily* f) {
  if (!f) return;
  if (f->refs.fetch_sub(1) == 1) {
    if (f->scratch) {  // its destroy releases the family once more
      AceSketch* s = f->scratch;
      f->scratch = nullptr;
      f->refs.store(1);
      ace_sketch_destroy(s);
      return;
    }
    cudaFree(f->d.w64);
    cudaFree(f->d.w32t);
    cudaFree(f->d.wnorm);
    cudaFree(f->d.wnorm64);
    cudaFree(f->w64t);
    tc_free_family(&f->tc);
    delete f;
  }
}

ace_status check_x(const AceFamily* f, const void* x, int dtype, uint64_t n, uint64_t ld,
                   int where, bool noisy_ok = false) {
  if (f->noise_scale > 0.0 && !noisy_ok)
    return fail(ACE_E_UNSUPPORTED,
                "ace: a noisy family hashes through ace_family_buckets_noisy (noise terms drawn in tick order on "
                "the host) and the ids entry points");
  if (dtype != ACE_F32 && dtype != ACE_F64) return fail(ACE_E_CONTRACT, "ace: dtype must be ACE_F32 or ACE_F64");
  if (where != ACE_HOST && where != ACE_DEVICE) return fail(ACE_E_CONTRACT, "ace: bad memory location");
  if (n > 0 && !x) return fail(ACE_E_CONTRACT, "ace: null point matrix");
  if (ld < f->d.dim)
    return fail(ACE_E_CONTRACT, "AceSketch: expected vector of length " + std::to_string(f->d.dim) +
                                    ", received row stride " + std::to_string(ld));
  return ACE_OK;
}

// Device view of the point matrix (copies host input into the staging buffer).
ace_status stage_x(AceSketch* sk, DevBuf& stage, cudaStream_t s, const void* x, int dtype,
                   uint64_t n, uint64_t ld, int where, const void** xd, uint64_t* ldd) {
  if (where == ACE_DEVICE || n == 0) {
    *xd = x;
    *ldd = ld;
    return ACE_OK;
  }
  const size_t esz = dtype == ACE_F64 ? 8 : 4;
  const uint64_t dim = sk ? sk->fam->d.dim : 0;
  (void)dim;
  ACE_CUDA(stage.ensure(n * ld * esz));
  ACE_CUDA(cudaMemcpyAsync(stage.p, x, n * ld * esz, cudaMemcpyHostToDevice, s));
  *xd = stage.p;
  *ldd = ld;
  return ACE_OK;
}

HashArgs make_hash_args(const AceFamily* f, const void* xd, int dtype, uint64_t n, uint64_t ld,
                        uint32_t* ids, uint64_t stride, DevState* st) {
  HashArgs a{};
  a.x = xd;
  a.x_f64 = dtype == ACE_F64;
  a.n = n;
  a.ld = ld;
  a.fam = f->d;
  a.margin_c = f->margin_c;
  a.ids = ids;
  a.ids_stride = stride;
  a.id_base = 0;
  a.counters = nullptr;
  a.insert = 0;
  a.cap = 0xffffffffu;
  a.st = st;
  return a;
}

// Zero the per-call accumulators (sum_lo .. underflow are contiguous).
cudaError_t zero_call_fields(AceSketch* sk) {
  char* base = reinterpret_cast<char*>(sk->st);
  const size_t off = offsetof(DevState, sum_lo);
  const size_t end = offsetof(DevState, underflow) + sizeof(unsigned long long);
  return cudaMemsetAsync(base + off, 0, end - off, sk->stream);
}

ace_status flush_point(const AceSketch* sk);
#define ACE_FLUSH(sk)                       \
  do {                                      \
    const ace_status fr_ = flush_point(sk); \
    if (fr_ != ACE_OK) return fr_;          \
  } while (0)

ace_status pull_state(AceSketch* sk) {
  ACE_FLUSH(sk);
  ACE_CUDA(cudaMemcpyAsync(sk->hst, sk->st, sizeof(DevState), cudaMemcpyDeviceToHost, sk->stream));
  ACE_CUDA(cudaStreamSynchronize(sk->stream));
  sk->pending_rows = 0;
  return ACE_OK;
}

double host_mean(const DevState& s, uint32_t tables) {
  if (s.n == 0) return 0.0;
  return ace_div_rn(s.T, s.n * tables);
}

void fill_stats(AceHashStats* stats, const DevState& s, uint64_t n, const AceFamily* f) {
  if (!stats) return;
  stats->projections = n * f->d.rows;
  stats->rechecked = s.rechecked;
  stats->flipped = s.flipped;
  stats->near_ties = s.near_ties;
}

ace_status copy_out(void* dst, const void* src, size_t bytes, int where, cudaStream_t s) {
  if (!dst || bytes == 0) return ACE_OK;
  ACE_CUDA(cudaMemcpyAsync(dst, src, bytes,
                           where == ACE_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
  return ACE_OK;
}

// 32-bit sketches cannot saturate while n stays below 2^32 - 1, so their
// insert merge may skip the pre-add values and recompute T = sum c^2; T (a
// u64, at most L n^2 when every point shares one bucket) must not wrap either.
bool fire_and_forget_ok(const AceSketch* sk, uint64_t n) {
  const unsigned long long tot = sk->hst->n + sk->pending_rows + n;
  const unsigned __int128 worst = static_cast<unsigned __int128>(tot) * tot * sk->fam->d.tables;
  return sk->width == 32 && !sk->hst->saturated && tot < 0xffffffffull && (worst >> 64) == 0;
}

// The barrier-free stream kernel (stream_apply_kernel): 32-bit unsaturable
// sketches with K <= 16; others score, insert and cap with separate kernels.
bool stream_apply_ok(const AceSketch* sk, bool ff) { return ff && sk->width == 32 && sk->fam->d.k_bits <= 16; }

// The per-point kernel takes up to kPointMaxRows host rows of a noise-free
// family by value in its launch parameters.
bool point_ok(const AceSketch* sk, int dtype, uint64_t n, int where) {
  const size_t esz = dtype == ACE_F64 ? 8 : 4;
  return sk->pth && sk->fam->w64t && where == ACE_HOST && n >= 1 && n <= kPointMaxRows &&
         sk->fam->noise_scale == 0.0 && n * sk->fam->d.dim * esz <= kPointXBytes &&
         n * sk->fam->d.tables <= 12288;  // the ids fit CTA 0's default shared memory
}

// The last point score hashed exactly these rows (its ids are in the cache).
bool point_cached(const AceSketch* sk, const void* x, int dtype, uint64_t n, uint64_t ld) {
  if (!sk->pcache_valid || sk->pcache_dtype != dtype || sk->pcache_n != n) return false;
  const size_t esz = dtype == ACE_F64 ? 8 : 4, row = sk->fam->d.dim * esz;
  for (uint64_t i = 0; i < n; ++i)
    if (memcmp(sk->pcache_x.data() + i * row, static_cast<const unsigned char*>(x) + i * ld * esz, row) != 0)
      return false;
  return true;
}

template <uint32_t XB>
ace_status run_point_t(AceSketch* sk, const void* x, int dtype, uint64_t n, uint64_t ld, int insert) {
  const AceFamily* f = sk->fam;
  PointArgs<XB> a;
  PointHdr& h = a.h;
  h.w64t = f->w64t;
  h.dim = f->d.dim;
  h.k_bits = f->d.k_bits;
  h.tables = f->d.tables;
  h.rows = f->d.rows;
  h.n = static_cast<uint32_t>(n);
  h.x_f64 = dtype == ACE_F64;
  h.counters = sk->counters;
  h.st = sk->st;
  h.cache = sk->pbits;
  h.scores = sk->pth->scores;
  h.sums = sk->pth->sums;
  h.snap = sk->pth->snap;
  const size_t esz = h.x_f64 ? 8 : 4, row = f->d.dim * esz, bytes = n * row;
  for (uint64_t i = 0; i < n; ++i)
    memcpy(a.x + i * row, static_cast<const unsigned char*>(x) + i * ld * esz, row);
  // an insert of the rows the last score hashed reuses their ids (the
  // per-point loop detect_stream(q); insert(q)): bucket ids depend on the
  // rows and the family only
  const bool cached = insert && !sk->pins_pend && point_cached(sk, x, dtype, n, ld);
  h.mode = insert ? (cached ? kPointInsertCached : kPointInsert) : kPointScore;
  h.pend_n = 0;
  if (!insert) {  // a deferred insert rides along, applied before the gather
    h.pend_n = sk->pins_pend;
    sk->pins_pend = 0;
  } else {
    ACE_FLUSH(sk);
  }
  sk->pcache_valid = false;
  ACE_CUDA(launch_point(a, sk->stream));
  if (!insert) {
    sk->pcache_x.assign(a.x, a.x + bytes);
    sk->pcache_n = n;
    sk->pcache_dtype = dtype;
    sk->pcache_valid = true;
  }
  return ACE_OK;
}

// One point_kernel launch over host rows x (insert: 32-bit unsaturable
// sketches, see fire_and_forget_ok).  Asynchronous; results land in sk->pth.
ace_status run_point(AceSketch* sk, const void* x, int dtype, uint64_t n, uint64_t ld, int insert) {
  const size_t esz = dtype == ACE_F64 ? 8 : 4;
  if (n * sk->fam->d.dim * esz <= kPointXSmall) return run_point_t<kPointXSmall>(sk, x, dtype, n, ld, insert);
  return run_point_t<kPointXBytes>(sk, x, dtype, n, ld, insert);
}

// Apply a deferred point insert before other work is queued on the sketch.
ace_status flush_point(const AceSketch* csk) {
  AceSketch* sk = const_cast<AceSketch*>(csk);
  if (!sk->pins_pend) return ACE_OK;
  PointArgs<kPointXSmall> a;
  PointHdr& h = a.h;
  h = PointHdr{};
  h.k_bits = sk->fam->d.k_bits;
  h.tables = sk->fam->d.tables;
  h.rows = sk->fam->d.rows;
  h.n = sk->pins_pend;
  h.mode = kPointInsertCached;
  h.counters = sk->counters;
  h.st = sk->st;
  h.cache = sk->pbits;
  h.snap = sk->pth->snap;
  sk->pins_pend = 0;
  ACE_CUDA(launch_point(a, sk->stream));
  return ACE_OK;
}

// Wait for a point_kernel score; the host mirror takes its n and T (the only
// state an unsaturable insert changes).
ace_status finish_point_score(AceSketch* sk) {
  ACE_CUDA(cudaStreamSynchronize(sk->stream));
  sk->hst->n = sk->pth->snap[0];
  sk->hst->T = sk->pth->snap[1];
  sk->pending_rows = 0;
  return ACE_OK;
}


ace_status ensure_stream_bufs(AceSketch* sk, uint64_t rows) {
  const size_t cnt_bytes = static_cast<size_t>(rows) * sk->fam->d.tables * sizeof(uint32_t);
  ACE_CUDA(sk->cnt[0].ensure(cnt_bytes));
  ACE_CUDA(sk->cnt[1].ensure(cnt_bytes));
  return ACE_OK;
}

ace_status ensure_group_bufs(AceSketch* sk, uint64_t group_batches, uint64_t batch, uint64_t ids_ld, bool pipe) {
  const uint64_t L = sk->fam->d.tables;
  ACE_CUDA(sk->gco.ensure(static_cast<size_t>(group_batches) * L * batch * sizeof(uint32_t)));
  ACE_CUDA(sk->gdT.ensure(static_cast<size_t>(group_batches) * 2 * L * sizeof(unsigned long long)));
  const void* before = sk->gdone.p;
  // done[batches] then claim[batches]
  ACE_CUDA(sk->gdone.ensure(static_cast<size_t>(group_batches) * 2 * sizeof(unsigned int)));
  if (sk->gdone.p != before) ACE_CUDA(cudaMemsetAsync(sk->gdone.p, 0, sk->gdone.bytes, sk->stream));
  // pipelined: two id buffers (the projection fills one while the stream kernel reads the other)
  ACE_CUDA(sk->ids.ensure(static_cast<size_t>(ids_ld) * L * sizeof(uint16_t) * (pipe ? 2u : 1u)));
  if (pipe) {
    if (!sk->pstream) ACE_CUDA(cudaStreamCreateWithFlags(&sk->pstream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      if (!sk->p_hashed[i]) ACE_CUDA(cudaEventCreateWithFlags(&sk->p_hashed[i], cudaEventDisableTiming));
      if (!sk->p_streamed[i]) ACE_CUDA(cudaEventCreateWithFlags(&sk->p_streamed[i], cudaEventDisableTiming));
    }
  }
  return ACE_OK;
}

// hash n rows into sk->ids (table-major, stride n); optional fused insert.
// Chunk mode (ids_out != null): the rows are rows [r0, r0 + n) of a longer
// batch whose ids (stride ids_ld) the caller has sized.
ace_status run_hash(AceSketch* sk, const void* xd, int dtype, uint64_t n, uint64_t ld, int insert,
                    uint32_t* ids_out = nullptr, uint64_t ids_ld = 0, bool ids16 = false, uint32_t grid_cap = 0) {
  const AceFamily* f = sk->fam;
  if (!ids_out) {
    ACE_CUDA(sk->ids.ensure(static_cast<size_t>(n) * f->d.tables * sizeof(uint32_t)));
    ids_out = sk->ids.as<uint32_t>();
    ids_ld = n;
  }
  for (bool& u : sk->ev_used) u = false;
  sk->stream_timed = false;
  sk->mark(0);
  if (f->use_tc()) {
    const bool kstream = tc_kstream(f->tc.nkc);
    TcArgs t{};
    t.x = xd;
    t.x_f64 = dtype == ACE_F64;
    t.n = n;
    t.ld = ld;
    t.dim = f->d.dim;
    t.k_bits = f->d.k_bits;
    t.tables = f->d.tables;
    t.tpt = f->tc.tpt;
    t.ntiles = f->tc.ntiles;
    t.nkc = f->tc.nkc;
    t.tw = f->tc.tw;
    t.w16 = f->tc.w16;
    t.margin_c = kstream ? tck_margin(f->tc.nkc, t.x_f64 != 0) : tc_margin(f->tc.nkc, t.x_f64 != 0);
    t.ids = ids_out;
    t.ids_ld = ids_ld;
    t.ids16 = ids16 ? 1 : 0;  // callers ask for u16 ids only on this path (stream driver, K <= 15)
    t.grid_cap = kstream ? 0u : grid_cap;
    // near-tie list: the K-streamed path's bound (large d, dense data) leaves
    // far more near ties per row, size its list accordingly
    uint64_t cap = kstream ? n * f->d.rows / 48 : n * f->d.rows / 1024;
    cap = std::min<uint64_t>(std::max<uint64_t>(cap, 1u << 20), kstream ? (1u << 27) : (1u << 25));
    {
      // the kernel's near-tie list is all ~0 between launches (entries are
      // reset as they are rechecked); fill a newly allocated one
      const void* before = sk->near.p;
      ACE_CUDA(sk->near.ensure(cap * sizeof(unsigned long long)));
      if (sk->near.p != before) ACE_CUDA(cudaMemsetAsync(sk->near.p, 0xff, sk->near.bytes, sk->stream));
    }
    {
      // the overflow-row bitmap is all 0 and the overflow flag clear between
      // launches (recheck_near_kernel cleans what it used; the K-streamed path
      // clears them per launch); fill a newly allocated bitmap
      const void* before = sk->overflow.p;
      ACE_CUDA(sk->overflow.ensure(((n + 31) / 32) * sizeof(uint32_t)));
      if (sk->overflow.p != before) ACE_CUDA(cudaMemsetAsync(sk->overflow.p, 0, sk->overflow.bytes, sk->stream));
      if (kstream) {
        ACE_CUDA(cudaMemsetAsync(sk->overflow.p, 0, ((n + 31) / 32) * sizeof(uint32_t), sk->stream));
        ACE_CUDA(cudaMemsetAsync(&sk->st->near_count, 0, 2 * sizeof(unsigned long long), sk->stream));
      }
    }
    t.near_list = sk->near.as<unsigned long long>();
    t.near_cap = sk->near.bytes / sizeof(unsigned long long);
    t.overflow_rows = sk->overflow.as<uint32_t>();
    t.st = sk->st;
    t.w64 = f->d.w64;
    t.wnorm64 = f->d.wnorm64;
    t.counters = sk->counters;
    if (kstream) {
      // d > 256: K-streamed kernel with its own conversion and recheck
      const uint64_t tiles = (n + 127) / 128;
      ACE_CUDA(sk->x16.ensure(tiles * f->tc.nkc * 2 * 16384));
      ACE_CUDA(sk->rowthr.ensure(tiles * 128 * sizeof(float)));
      t.x16 = sk->x16.as<uint16_t>();
      t.rowthr = sk->rowthr.as<float>();
      ACE_CUDA(sk->segc.ensure(static_cast<size_t>(tck_grid(n)) * sizeof(uint32_t)));
      t.seg_counts = sk->segc.as<uint32_t>();
      t.w32 = f->tc.w32;
      sk->mark(4);
      ACE_CUDA(launch_convert_x_wide(t, sk->stream));
      sk->mark(6);
      ACE_CUDA(launch_hash_tck(t, sk->stream));
      sk->mark(5);
      ACE_CUDA(launch_recheck_segs(t, sk->stream));
      ACE_CUDA(launch_recheck(t, sk->stream));
      if (insert && sk->defer_insert)
        sk->insert_deferred = true;
      else if (insert)
        ACE_CUDA(launch_apply_ids(ids_out, n, f->d.tables, f->d.k_bits, sk->counters, sk->cap, +1, sk->st,
                                  sk->stream, !fire_and_forget_ok(sk, n), ids_ld));
      if (insert && sk->width == 16)
        ACE_CUDA(launch_cap(sk->counters, sk->num_counters, sk->cap, sk->st, sk->stream));
      sk->mark(1);
      return ACE_OK;
    }
    // Fused epilogue insert (global REDs) only where the separate insert would
    // use global atomics too (K > 20); otherwise the shared-memory histogram
    // (split into 2^15-bin parts for K > 15) absorbs hot buckets far better.
    const bool fused = insert && sk->width == 32 && fire_and_forget_ok(sk, n) && f->d.k_bits > 20;
    t.fused_insert = fused ? 1 : 0;
    if (!tc_direct_ok(xd, t.x_f64, ld)) ACE_CUDA(sk->xf32.ensure(tc_stage_bytes(n, f->d.dim)));
    ACE_CUDA(sk->segc.ensure(static_cast<size_t>(tc_grid(n)) * sizeof(uint32_t)));
    t.seg_counts = sk->segc.as<uint32_t>();
    sk->mark(4);
    sk->mark(6);
    ACE_CUDA(launch_hash_tc(t, sk->xf32.p, sk->stream));
    sk->mark(5);
    ACE_CUDA(launch_recheck_near(t, sk->stream));
    if (fused) {
      // T = sum of squared counters (exact: 32-bit, unsaturated)
      ACE_CUDA(cudaMemsetAsync(&sk->st->T, 0, sizeof(unsigned long long), sk->stream));
      ACE_CUDA(launch_sum_squares(sk->counters, sk->num_counters, &sk->st->T, sk->stream));
    } else if (insert && sk->defer_insert) {
      sk->insert_deferred = true;
    } else if (insert) {
      ACE_CUDA(launch_apply_ids(ids_out, n, f->d.tables, f->d.k_bits, sk->counters, sk->cap, +1, sk->st,
                                sk->stream, !fire_and_forget_ok(sk, n), ids_ld));
    }
  } else {
    HashArgs a = make_hash_args(f, xd, dtype, n, ld, ids_out, ids_ld, sk->st);
    a.insert = insert;
    a.counters = sk->counters;
    a.cap = sk->cap;
    ACE_CUDA(launch_hash_simt(a, sk->stream));
  }
  if (insert && sk->width == 16)
    ACE_CUDA(launch_cap(sk->counters, sk->num_counters, sk->cap, sk->st, sk->stream));
  sk->mark(1);
  return ACE_OK;
}

// Device part of the detect tail: score from sk->ids; threshold + flags.
ace_status run_detect_device(AceSketch* sk, uint64_t n, uint32_t* flag_bits, double* scores, int out_where,
                             uint32_t** dflags_out, double** dscores_out);
// Host part: outputs to host memory, state read-back, report.
ace_status finish_detect(AceSketch* sk, uint64_t n, uint32_t* flag_bits, double* scores, int out_where,
                         const uint32_t* dflags, const double* dscores, AceBatchReport* report);

ace_status run_detect_device(AceSketch* sk, uint64_t n, uint32_t* flag_bits, double* scores, int out_where,
                             uint32_t** dflags_out, double** dscores_out) {
  const AceFamily* f = sk->fam;
  ACE_CUDA(sk->sums.ensure(n * sizeof(uint64_t)));
  ACE_CUDA(sk->flags.ensure(((n + 31) / 32) * sizeof(uint32_t)));
  double* dscores = nullptr;
  if (scores) {
    if (out_where == ACE_DEVICE) {
      dscores = scores;
    } else {
      ACE_CUDA(sk->scores.ensure(n * sizeof(double)));
      dscores = sk->scores.as<double>();
    }
  }
  uint32_t* dflags = (flag_bits && out_where == ACE_DEVICE) ? flag_bits : sk->flags.as<uint32_t>();
  // one cooperative launch: (deferred insert: counts, ids replaced by their
  // final counts,) scores, exact threshold, flags (+ replay when ambiguous)
  const int gather = sk->insert_deferred ? 1 : 0;
  sk->insert_deferred = false;
  sk->mark(1);
  sk->mark(2);
  ACE_CUDA(launch_detect_tail(sk->ids.as<uint32_t>(), n, f->d.tables, f->d.k_bits, sk->counters, gather,
                              sk->sums.as<uint64_t>(), dscores, dflags, sk->st, sk->stream));
  sk->mark(3);
  *dflags_out = dflags;
  *dscores_out = dscores;
  return ACE_OK;
}

ace_status finish_detect(AceSketch* sk, uint64_t n, uint32_t* flag_bits, double* scores, int out_where,
                         const uint32_t* dflags, const double* dscores, AceBatchReport* report) {
  if (flag_bits && out_where == ACE_HOST) {
    ace_status r = copy_out(flag_bits, dflags, ((n + 31) / 32) * sizeof(uint32_t), ACE_HOST, sk->stream);
    if (r != ACE_OK) return r;
  }
  if (scores && out_where == ACE_HOST) {
    ace_status r = copy_out(scores, dscores, n * sizeof(double), ACE_HOST, sk->stream);
    if (r != ACE_OK) return r;
  }
  ace_status r = pull_state(sk);
  if (r != ACE_OK) return r;
  const DevState& s = *sk->hst;
  if (s.sum_hi != 0) return fail(ACE_E_DATA, "detect_batch: score sum exceeds 2^64");
  if (report) {
    report->score_mean = s.mean;
    report->score_stddev = s.sd;
    report->threshold = s.thr;
    report->reported = s.reported;
    report->ambiguous = s.ambiguous;
    report->replayed = s.replayed;
  }
  return ACE_OK;
}

}  // namespace

extern "C" {

const char* ace_last_error(void) { return g_err.c_str(); }

const char* ace_version(void) { return "ace-b200 0.1 sm_100a"; }

int ace_device_available(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n > 0;
}

uint64_t ace_kernel_launches(void) { return g_launches.load(); }

// SrpFamily::SrpFamily (srp.cpp:24-49): validation + W upload.
ace_status ace_family_create(uint64_t dim, uint32_t k_bits, uint32_t num_tables, double noise_scale,
                             const double* w_host, AceFamily** out) {
  if (!out) return fail(ACE_E_CONTRACT, "ace_family_create: null out");
  *out = nullptr;
  if (dim == 0) return fail(ACE_E_CONTRACT, "SrpFamily: dim must be >= 1");
  if (k_bits < 1 || k_bits > kMaxKBits)
    return fail(ACE_E_CONTRACT, "SrpFamily: k_bits must be in [1, " + std::to_string(kMaxKBits) + "]");
  if (num_tables < 1) return fail(ACE_E_CONTRACT, "SrpFamily: num_tables must be >= 1");
  if (noise_scale < 0.0) return fail(ACE_E_CONTRACT, "SrpFamily: noise_scale must be >= 0");
  if (!w_host) return fail(ACE_E_CONTRACT, "ace_family_create: null W");
  if (!ace_device_available()) return fail(ACE_E_CUDA, "ace: no CUDA device available");

  AceFamily* f = new AceFamily();
  f->noise_scale = noise_scale;
  FamilyDev& d = f->d;
  d.dim = dim;
  d.k_bits = k_bits;
  d.tables = num_tables;
  d.rows = k_bits * num_tables;
  d.tpt = static_cast<uint32_t>(kTileCols) / k_bits;
  d.ntiles = (num_tables + d.tpt - 1) / d.tpt;
  d.ncols = d.ntiles * kTileCols;
  d.dpad = (dim + 31) / 32 * 32;
  // fast-path error bound: fp32 FMA fold of fp32-rounded W and x against
  // the binary64 fold, relative to ||w|| ||x||.
  // (at least 2e-6: every projection below the BASELINE near-tie measure
  // 1e-6 |x| |w| is then rechecked and counted)
  f->margin_c = static_cast<float>(std::max((static_cast<double>(dim) + 6.0) * 0x1.0p-24 * 1.01, 2e-6));

  std::vector<float> w32t(static_cast<size_t>(d.dpad) * d.ncols, 0.0f);
  std::vector<float> wn(d.ncols, 0.0f);
  for (uint32_t j = 0; j < d.ntiles; ++j)
    for (uint32_t c = 0; c < d.tpt * k_bits; ++c) {
      const uint32_t table = j * d.tpt + c / k_bits;
      if (table >= num_tables) continue;
      const uint64_t r = static_cast<uint64_t>(table) * k_bits + c % k_bits;
      double ss = 0.0;
      for (uint64_t i = 0; i < dim; ++i) {
        const double w = w_host[r * dim + i];
        w32t[i * d.ncols + j * kTileCols + c] = static_cast<float>(w);
        ss += w * w;
      }
      float nb = static_cast<float>(std::sqrt(ss) * (1.0 + 1e-12));
      wn[j * kTileCols + c] = std::nextafter(nb, INFINITY);
    }
  auto cleanup = [&]() { family_release(f); };
  f->tc = TcFamily{};
  cudaError_t e;
  if ((e = cudaMalloc(&d.w64, sizeof(double) * d.rows * dim)) != cudaSuccess ||
      (e = cudaMalloc(&d.w32t, sizeof(float) * w32t.size())) != cudaSuccess ||
      (e = cudaMalloc(&d.wnorm, sizeof(float) * wn.size())) != cudaSuccess ||
      (e = cudaMalloc(&d.wnorm64, sizeof(double) * d.rows)) != cudaSuccess ||
      (e = cudaMemcpy(d.w64, w_host, sizeof(double) * d.rows * dim, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(d.w32t, w32t.data(), sizeof(float) * w32t.size(), cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(d.wnorm, wn.data(), sizeof(float) * wn.size(), cudaMemcpyHostToDevice)) != cudaSuccess) {
    cleanup();
    return fail(e == cudaErrorMemoryAllocation ? ACE_E_NOMEM : ACE_E_CUDA,
                std::string("ace_family_create: ") + cudaGetErrorString(e));
  }
  if (dim * sizeof(float) <= kPointXBytes) {  // a row fits the per-point kernel's parameters
    std::vector<double> wt(static_cast<size_t>(d.rows) * dim);
    for (uint64_t r = 0; r < d.rows; ++r)
      for (uint64_t i = 0; i < dim; ++i) wt[i * d.rows + r] = w_host[r * dim + i];
    if ((e = cudaMalloc(&f->w64t, sizeof(double) * wt.size())) != cudaSuccess ||
        (e = cudaMemcpy(f->w64t, wt.data(), sizeof(double) * wt.size(), cudaMemcpyHostToDevice)) != cudaSuccess) {
      cleanup();
      return fail(e == cudaErrorMemoryAllocation ? ACE_E_NOMEM : ACE_E_CUDA,
                  std::string("ace_family_create: ") + cudaGetErrorString(e));
    }
  }
  if ((e = launch_wnorm64(d.w64, d.dim, d.rows, d.wnorm64)) != cudaSuccess) {
    cleanup();
    return fail(ACE_E_CUDA, std::string("ace_family_create: ") + cudaGetErrorString(e));
  }
  if ((e = tc_prepare_family(d, &f->tc)) != cudaSuccess) {
    cleanup();
    return fail(ACE_E_CUDA, std::string("ace_family_create (tcgen05 operands): ") + cudaGetErrorString(e));
  }
  *out = f;
  return ACE_OK;
}

ace_status ace_family_set_kernel(AceFamily* fam, int which) {
  if (!fam) return fail(ACE_E_CONTRACT, "ace_family_set_kernel: null family");
  if (which < 0 || which > 2) return fail(ACE_E_CONTRACT, "ace_family_set_kernel: which must be 0, 1 or 2");
  if (which == 2 && !fam->tc.enabled)
    return fail(ACE_E_UNSUPPORTED, "ace_family_set_kernel: tcgen05 path does not support dim " +
                                       std::to_string(fam->d.dim));
  fam->kernel = which;
  return ACE_OK;
}

int ace_family_kernel(const AceFamily* fam) { return fam && fam->use_tc() ? 2 : 1; }

ace_status ace_family_destroy(AceFamily* fam) {
  family_release(fam);
  return ACE_OK;
}

ace_status sketch_create(AceFamily* fam, uint32_t counter_width, AceSketch** out, bool counters);

// The family's scratch state for one hashing call: the shared one when free,
// else (a concurrent caller holds it) a private one for this call.
struct ScratchLease {
  AceFamily* f = nullptr;
  AceSketch* sk = nullptr;
  bool shared = false;
  ~ScratchLease() {
    if (shared) f->scratch_mu.unlock();
    else if (sk) ace_sketch_destroy(sk);
  }
};

ace_status lease_scratch(AceFamily* f, ScratchLease& l) {
  l.f = f;
  if (f->scratch_mu.try_lock()) {
    l.shared = true;
    if (!f->scratch) {
      ace_status r = sketch_create(f, 32, &f->scratch, false);
      if (r != ACE_OK) return r;
      f->refs.fetch_sub(1);  // held by the family itself
    }
    l.sk = f->scratch;
    ACE_CUDA(zero_call_fields(l.sk));
    return ACE_OK;
  }
  return sketch_create(f, 32, &l.sk, false);
}

// SrpFamily::bucket (srp.cpp:106-113) for every row and table.
ace_status ace_family_buckets(AceFamily* fam, const void* x, int dtype, uint64_t n, uint64_t ld,
                              int x_where, uint32_t* ids, int ids_where, AceHashStats* stats) {
  if (!fam) return fail(ACE_E_CONTRACT, "ace_family_buckets: null family");
  ace_status r = check_x(fam, x, dtype, n, ld, x_where);
  if (r != ACE_OK) return r;
  ScratchLease lease;
  r = lease_scratch(fam, lease);
  if (r != ACE_OK) return r;
  AceSketch* sk = lease.sk;
  const void* xd;
  uint64_t ldd;
  r = stage_x(sk, sk->stage, sk->stream, x, dtype, n, ld, x_where, &xd, &ldd);
  if (r == ACE_OK) r = run_hash(sk, xd, dtype, n, ldd, 0);
  if (r == ACE_OK && n)
    r = copy_out(ids, sk->ids.p, static_cast<size_t>(n) * fam->d.tables * sizeof(uint32_t),
                 ids_where, sk->stream);
  if (r == ACE_OK) r = pull_state(sk);
  if (r == ACE_OK) fill_stats(stats, *sk->hst, n, fam);
  return r;
}

// Noisy hashing (SrpFamily::bit with noise_scale > 0, srp.cpp:93-104): the
// host draws the noise terms in tick order, the device folds exactly.
ace_status ace_family_buckets_noisy(AceFamily* fam, const void* x, int dtype, uint64_t n, uint64_t ld, int x_where,
                                    uint32_t t0, uint32_t nt, uint32_t b0, uint32_t nb, const double* noise,
                                    int noise_where, uint32_t* ids, int ids_where) {
  if (!fam) return fail(ACE_E_CONTRACT, "ace_family_buckets_noisy: null family");
  ace_status r = check_x(fam, x, dtype, n, ld, x_where, true);
  if (r != ACE_OK) return r;
  if (t0 + nt > fam->d.tables || b0 + nb > fam->d.k_bits || nb == 0)
    return fail(ACE_E_CONTRACT, "ace_family_buckets_noisy: table or bit range out of range");
  if (n == 0 || nt == 0) return ACE_OK;
  if (!noise || !ids) return fail(ACE_E_CONTRACT, "ace_family_buckets_noisy: null noise or ids");
  ScratchLease lease;
  r = lease_scratch(fam, lease);
  if (r != ACE_OK) return r;
  AceSketch* sk = lease.sk;
  const void* xd;
  uint64_t ldd;
  r = stage_x(sk, sk->stage, sk->stream, x, dtype, n, ld, x_where, &xd, &ldd);
  const double* nd = noise;
  const size_t nbytes = static_cast<size_t>(n) * nt * nb * sizeof(double);
  if (r == ACE_OK && noise_where == ACE_HOST) {
    cudaError_t e = sk->scores.ensure(nbytes);
    if (e == cudaSuccess) e = cudaMemcpyAsync(sk->scores.p, noise, nbytes, cudaMemcpyHostToDevice, sk->stream);
    if (e != cudaSuccess) r = fail(ACE_E_CUDA, cudaGetErrorString(e));
    nd = sk->scores.as<double>();
  }
  if (r == ACE_OK) {
    cudaError_t e = sk->ids.ensure(static_cast<size_t>(n) * nt * sizeof(uint32_t));
    if (e == cudaSuccess)
      e = launch_noisy_buckets(xd, dtype == ACE_F64, n, ldd, fam->d.dim, fam->d.w64, fam->d.k_bits, t0, nt, b0, nb, nd,
                               sk->ids.as<uint32_t>(), sk->stream);
    if (e != cudaSuccess) r = fail(ACE_E_CUDA, cudaGetErrorString(e));
  }
  if (r == ACE_OK)
    r = copy_out(ids, sk->ids.p, static_cast<size_t>(n) * nt * sizeof(uint32_t), ids_where, sk->stream);
  if (r == ACE_OK && cudaStreamSynchronize(sk->stream) != cudaSuccess) r = fail(ACE_E_CUDA, "ace_family_buckets_noisy");
  return r;
}

// AceSketch::AceSketch (sketch.cpp:10-17): zeroed table-major counters.
ace_status ace_sketch_create(AceFamily* fam, uint32_t counter_width, AceSketch** out) {
  return sketch_create(fam, counter_width, out, true);
}

ace_status sketch_create(AceFamily* fam, uint32_t counter_width, AceSketch** out, bool counters) {
  if (!out || !fam) return fail(ACE_E_CONTRACT, "ace_sketch_create: null argument");
  *out = nullptr;
  if (counter_width != 16 && counter_width != 32)
    return fail(ACE_E_CONTRACT, "AceSketch: counter width must be 16 or 32");
  AceSketch* sk = new AceSketch();
  sk->fam = fam;
  fam->refs.fetch_add(1);
  sk->width = counter_width;
  sk->cap = counter_width == 16 ? 0xffffu : 0xffffffffu;
  sk->num_counters = counters ? static_cast<uint64_t>(fam->d.tables) << fam->d.k_bits : 0;
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&sk->own, cudaStreamNonBlocking)) != cudaSuccess ||
      (counters && (e = cudaMalloc(&sk->counters, sk->num_counters * sizeof(uint32_t))) != cudaSuccess) ||
      (e = cudaMalloc(&sk->st, sizeof(DevState))) != cudaSuccess ||
      (e = cudaMallocHost(&sk->hst, sizeof(DevState))) != cudaSuccess ||
      (counters && (e = cudaHostAlloc(&sk->pth, sizeof(AceSketch::PointHost), cudaHostAllocMapped)) != cudaSuccess) ||
      (counters && (e = cudaMalloc(&sk->pbits, kPointMaxRows * fam->d.tables * sizeof(uint32_t))) != cudaSuccess)) {
    ace_sketch_destroy(sk);
    return fail(e == cudaErrorMemoryAllocation ? ACE_E_NOMEM : ACE_E_CUDA,
                std::string("ace_sketch_create: ") + cudaGetErrorString(e));
  }
  sk->stream = sk->own;
  memset(sk->hst, 0, sizeof(DevState));
  if (sk->pbits &&
      (e = cudaMemsetAsync(sk->pbits, 0, kPointMaxRows * fam->d.tables * sizeof(uint32_t), sk->stream)) !=
          cudaSuccess) {
    ace_sketch_destroy(sk);
    return fail(ACE_E_CUDA, std::string("ace_sketch_create: ") + cudaGetErrorString(e));
  }
  ace_status r = ace_sketch_reset(sk);
  if (r != ACE_OK) {
    ace_sketch_destroy(sk);
    return r;
  }
  *out = sk;
  return ACE_OK;
}

// Stream-ordered: later calls on the sketch's stream see the zeroed state; the
// host mirror is cleared at once (its next refresh comes after these memsets).
ace_status ace_sketch_reset(AceSketch* sk) {
  if (!sk) return fail(ACE_E_CONTRACT, "ace_sketch_reset: null sketch");
  sk->mean_pinned = false;
  if (sk->num_counters) ACE_CUDA(cudaMemsetAsync(sk->counters, 0, sk->num_counters * sizeof(uint32_t), sk->stream));
  ACE_CUDA(cudaMemsetAsync(sk->st, 0, sizeof(DevState), sk->stream));
  memset(sk->hst, 0, sizeof(DevState));
  sk->pending_rows = 0;
  sk->pins_pend = 0;
  return ACE_OK;
}

ace_status ace_sketch_clone(const AceSketch* src, AceSketch** out) {
  if (!src || !out) return fail(ACE_E_CONTRACT, "ace_sketch_clone: null argument");
  ACE_FLUSH(src);
  ace_status r = ace_sketch_create(src->fam, src->width, out);
  if (r != ACE_OK) return r;
  AceSketch* d = *out;
  ACE_CUDA(cudaStreamSynchronize(src->stream));
  ACE_CUDA(cudaMemcpyAsync(d->counters, src->counters, src->num_counters * sizeof(uint32_t),
                           cudaMemcpyDeviceToDevice, d->stream));
  ACE_CUDA(cudaMemcpyAsync(d->st, src->st, sizeof(DevState), cudaMemcpyDeviceToDevice, d->stream));
  d->mean_pinned = src->mean_pinned;
  d->pinned_mean = src->pinned_mean;
  return pull_state(d);
}

ace_status ace_sketch_destroy(AceSketch* sk) {
  if (!sk) return ACE_OK;
  if (sk->stream) cudaStreamSynchronize(sk->stream);
  sk->drop_graph();
  sk->ids.release();
  sk->sums.release();
  sk->stage.release();
  sk->flags.release();
  sk->scores.release();
  sk->demand.release();
  sk->near.release();
  sk->overflow.release();
  sk->x16.release();
  sk->rowthr.release();
  sk->segc.release();
  sk->xf32.release();
  sk->cnt[0].release();
  sk->cnt[1].release();
  sk->gco.release();
  sk->gdT.release();
  sk->gdone.release();
  if (sk->counters) cudaFree(sk->counters);
  if (sk->st) cudaFree(sk->st);
  if (sk->hst) cudaFreeHost(sk->hst);
  if (sk->pth) cudaFreeHost(sk->pth);
  if (sk->pbits) cudaFree(sk->pbits);
  if (sk->own) cudaStreamDestroy(sk->own);
  sk->sstage[0].release();
  sk->sstage[1].release();
  for (int i = 0; i < 2; ++i) {
    if (sk->s_copied[i]) cudaEventDestroy(sk->s_copied[i]);
    if (sk->s_used[i]) cudaEventDestroy(sk->s_used[i]);
  }
  if (sk->cstream) cudaStreamDestroy(sk->cstream);
  for (int i = 0; i < 2; ++i) {
    if (sk->p_hashed[i]) cudaEventDestroy(sk->p_hashed[i]);
    if (sk->p_streamed[i]) cudaEventDestroy(sk->p_streamed[i]);
  }
  if (sk->pstream) cudaStreamDestroy(sk->pstream);
  if (sk->cstart) cudaEventDestroy(sk->cstart);
  for (cudaEvent_t e : sk->cev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t& e : sk->ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : sk->lat_a) cudaEventDestroy(e);
  for (cudaEvent_t e : sk->lat_b) cudaEventDestroy(e);
  family_release(sk->fam);
  delete sk;
  cudaGetLastError();  // teardown errors are not the next call's launch error
  return ACE_OK;
}

ace_status ace_sketch_set_stream(AceSketch* sk, void* cuda_stream) {
  if (!sk) return fail(ACE_E_CONTRACT, "ace_sketch_set_stream: null sketch");
  ACE_FLUSH(sk);
  ACE_CUDA(cudaStreamSynchronize(sk->stream));
  sk->stream = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : sk->own;
  return ACE_OK;
}

ace_status ace_sketch_set_option(AceSketch* sk, int option, int64_t value) {
  if (!sk) return fail(ACE_E_CONTRACT, "ace_sketch_set_option: null sketch");
  switch (option) {
    case ACE_OPT_H2D_CHUNKS:
      if (value < 1 || value > 64) return fail(ACE_E_CONTRACT, "ace_sketch_set_option: chunks must be in [1, 64]");
      sk->h2d_chunks = static_cast<int>(value);
      break;
    case ACE_OPT_DEFER_INSERT:
      if (value < -1 || value > 1) return fail(ACE_E_CONTRACT, "ace_sketch_set_option: defer mode must be -1, 0 or 1");
      sk->defer_mode = static_cast<int>(value);
      break;
    case ACE_OPT_STREAM_GROUP:
      if (value < 1 || value > 64) return fail(ACE_E_CONTRACT, "ace_sketch_set_option: group must be in [1, 64]");
      sk->stream_group = static_cast<int>(value);
      break;
    case ACE_OPT_STREAM_PIPE:
      if (value < -1 || value > 1024) return fail(ACE_E_CONTRACT, "ace_sketch_set_option: pipe CTAs must be in [-1, 1024]");
      sk->stream_pipe = static_cast<int>(value);
      break;
    default:
      return fail(ACE_E_CONTRACT, "ace_sketch_set_option: unknown option " + std::to_string(option));
  }
  sk->drop_graph();
  return ACE_OK;
}

// AceSketch::insert (sketch.cpp:50-72), rows in order.
ace_status ace_sketch_insert(AceSketch* sk, const void* x, int dtype, uint64_t n, uint64_t ld,
                             int x_where, AceHashStats* stats) {
  if (!sk) return fail(ACE_E_CONTRACT, "ace_sketch_insert: null sketch");
  ace_status r = check_x(sk->fam, x, dtype, n, ld, x_where);
  if (r != ACE_OK) return r;
  sk->mean_pinned = false;
  if (!stats && point_ok(sk, dtype, n, x_where) && fire_and_forget_ok(sk, n)) {
    // a few host rows, no stats asked: one launch, no wait (stream-ordered
    // before every later call on the sketch; the rows travel by value) --
    // or none, when the last point score hashed exactly these rows
    if (!sk->pins_pend && point_cached(sk, x, dtype, n, ld)) {
      sk->pins_pend = static_cast<uint32_t>(n);
      sk->pcache_valid = false;
      sk->pending_rows += n;
      return ACE_OK;
    }
    r = run_point(sk, x, dtype, n, ld, 1);
    if (r == ACE_OK) sk->pending_rows += n;
    return r;
  }
  ACE_FLUSH(sk);
  ACE_CUDA(zero_call_fields(sk));
  const void* xd;
  uint64_t ldd;
  r = stage_x(sk, sk->stage, sk->stream, x, dtype, n, ld, x_where, &xd, &ldd);
  if (r == ACE_OK && n) r = run_hash(sk, xd, dtype, n, ldd, 1);
  if (r == ACE_OK) r = pull_state(sk);
  if (r == ACE_OK) fill_stats(stats, *sk->hst, n, sk->fam);
  return r;
}

namespace {
ace_status stage_ids(AceSketch* sk, const uint32_t* ids, uint64_t n, int where, const uint32_t** out) {
  const AceFamily* f = sk->fam;
  if (where != ACE_HOST && where != ACE_DEVICE) return fail(ACE_E_CONTRACT, "ace: bad memory location");
  if (n > 0 && !ids) return fail(ACE_E_CONTRACT, "ace: null ids");
  const uint64_t total = n * f->d.tables;
  if (where == ACE_HOST) {
    const uint32_t lim = f->d.k_bits >= 32 ? 0xffffffffu : (1u << f->d.k_bits) - 1u;
    for (uint64_t i = 0; i < total; ++i)
      if (ids[i] > lim) return fail(ACE_E_CONTRACT, "ace: bucket id out of range [0, 2^K)");
    ACE_CUDA(sk->ids.ensure(total * sizeof(uint32_t)));
    ACE_CUDA(cudaMemcpyAsync(sk->ids.p, ids, total * sizeof(uint32_t), cudaMemcpyHostToDevice, sk->stream));
    *out = sk->ids.as<uint32_t>();
  } else {
    *out = ids;  // device ids are taken as valid
  }
  return ACE_OK;
}
}  // namespace

// Insert n points given by their bucket ids (L x n, table-major; e.g. from
// ace_family_buckets_noisy): AceSketch::insert's counter and mean update
// (sketch.cpp:55-71) without hashing.
ace_status ace_sketch_insert_ids(AceSketch* sk, const uint32_t* ids, uint64_t n, int where) {
  if (!sk) return fail(ACE_E_CONTRACT, "ace_sketch_insert_ids: null sketch");
  ACE_FLUSH(sk);
  if (n == 0) return ACE_OK;
  const uint32_t* d = nullptr;
  ace_status r = stage_ids(sk, ids, n, where, &d);
  if (r != ACE_OK) return r;
  sk->mean_pinned = false;
  ACE_CUDA(zero_call_fields(sk));
  ACE_CUDA(launch_apply_ids(d, n, sk->fam->d.tables, sk->fam->d.k_bits, sk->counters, sk->cap, +1, sk->st,
                            sk->stream, !fire_and_forget_ok(sk, n)));
  if (sk->width == 16) ACE_CUDA(launch_cap(sk->counters, sk->num_counters, sk->cap, sk->st, sk->stream));
  return pull_state(sk);
}

// Scores of n points given by their bucket ids (AceSketch::score's gather,
// sketch.cpp:108-116).
ace_status ace_sketch_score_ids(AceSketch* sk, const uint32_t* ids, uint64_t n, int where, double* scores,
                                uint64_t* sums, int out_where) {
  if (!sk) return fail(ACE_E_CONTRACT, "ace_sketch_score_ids: null sketch");
  ACE_FLUSH(sk);
  if (n == 0) return ACE_OK;
  const uint32_t* d = nullptr;
  ace_status r = stage_ids(sk, ids, n, where, &d);
  if (r != ACE_OK) return r;
  ACE_CUDA(zero_call_fields(sk));
  double* dsc = nullptr;
  uint64_t* dsum = nullptr;
  if (scores) {
    if (out_where == ACE_DEVICE) dsc = scores;
    else {
      ACE_CUDA(sk->scores.ensure(n * sizeof(double)));
      dsc = sk->scores.as<double>();
    }
  }
  if (sums) {
    if (out_where == ACE_DEVICE) dsum = sums;
    else {
      ACE_CUDA(sk->sums.ensure(n * sizeof(uint64_t)));
      dsum = sk->sums.as<uint64_t>();
    }
  }
  ACE_CUDA(launch_score(d, n, n, sk->fam->d.tables, sk->fam->d.k_bits, sk->counters, dsum, dsc, sk->st, sk->stream));
  if (out_where == ACE_HOST) {
    if (scores && (r = copy_out(scores, dsc, n * sizeof(double), ACE_HOST, sk->stream)) != ACE_OK) return r;
    if (sums && (r = copy_out(sums, dsum, n * sizeof(uint64_t), ACE_HOST, sk->stream)) != ACE_OK) return r;
  }
  return pull_state(sk);
}

// AceSketch::remove (sketch.cpp:74-106), all-or-nothing over the batch.
ace_status ace_sketch_remove(AceSketch* sk, const void* x, int dtype, uint64_t n, uint64_t ld,
                             int x_where, AceHashStats* stats) {
  if (!sk) return fail(ACE_E_CONTRACT, "ace_sketch_remove: null sketch");
  ACE_FLUSH(sk);
  ace_status r = check_x(sk->fam, x, dtype, n, ld, x_where);
  if (r != ACE_OK) return r;
  if (n == 0) return ACE_OK;
  if (sk->width == 16 && sk->hst->saturated)
    return fail(ACE_E_UNSUPPORTED, "AceSketch: delete from a saturated 16-bit sketch has no exact inverse");
  ACE_CUDA(zero_call_fields(sk));
  const void* xd;
  uint64_t ldd;
  r = stage_x(sk, sk->stage, sk->stream, x, dtype, n, ld, x_where, &xd, &ldd);
  if (r == ACE_OK) r = run_hash(sk, xd, dtype, n, ldd, 0);
  if (r != ACE_OK) return r;
  ACE_CUDA(sk->demand.ensure(sk->num_counters * sizeof(uint32_t)));
  ACE_CUDA(launch_remove_check(sk->ids.as<uint32_t>(), n, sk->fam->d.tables, sk->fam->d.k_bits,
                               sk->counters, sk->demand.as<uint32_t>(), sk->st, sk->stream));
  r = pull_state(sk);
  if (r != ACE_OK) return r;
  if (sk->hst->underflow)
    return fail(ACE_E_INCONSISTENT,
                "AceSketch: delete target counter is zero (item was never inserted)");
  sk->mean_pinned = false;
  ACE_CUDA(launch_apply_ids(sk->ids.as<uint32_t>(), n, sk->fam->d.tables, sk->fam->d.k_bits,
                            sk->counters, sk->cap, -1, sk->st, sk->stream));
  r = pull_state(sk);
  if (r == ACE_OK) fill_stats(stats, *sk->hst, n, sk->fam);
  return r;
}

// AceSketch::score (sketch.cpp:108-116) for every row.
ace_status ace_sketch_score(AceSketch* sk, const void* x, int dtype, uint64_t n, uint64_t ld,
                            int x_where, double* scores, uint64_t* sums, int out_where,
                            AceHashStats* stats) {
  if (!sk) return fail(ACE_E_CONTRACT, "ace_sketch_score: null sketch");
  ace_status r = check_x(sk->fam, x, dtype, n, ld, x_where);
  if (r != ACE_OK) return r;
  if (n == 0) return ACE_OK;
  if (!stats && out_where == ACE_HOST && point_ok(sk, dtype, n, x_where)) {
    if ((r = run_point(sk, x, dtype, n, ld, 0)) != ACE_OK || (r = finish_point_score(sk)) != ACE_OK) return r;
    if (scores) memcpy(scores, sk->pth->scores, n * sizeof(double));
    if (sums) memcpy(sums, sk->pth->sums, n * sizeof(uint64_t));
    return ACE_OK;
  }
  ACE_FLUSH(sk);
  ACE_CUDA(zero_call_fields(sk));
  const void* xd;
  uint64_t ldd;
  r = stage_x(sk, sk->stage, sk->stream, x, dtype, n, ld, x_where, &xd, &ldd);
  if (r == ACE_OK) r = run_hash(sk, xd, dtype, n, ldd, 0);
  if (r != ACE_OK) return r;
  double* dsc = nullptr;
  uint64_t* dsum = nullptr;
  if (scores) {
    if (out_where == ACE_DEVICE) dsc = scores;
    else {
      ACE_CUDA(sk->scores.ensure(n * sizeof(double)));
      dsc = sk->scores.as<double>();
    }
  }
  if (sums) {
    if (out_where == ACE_DEVICE) dsum = sums;
    else {
      ACE_CUDA(sk->sums.ensure(n * sizeof(uint64_t)));
      dsum = sk->sums.as<uint64_t>();
    }
  }
  ACE_CUDA(launch_score(sk->ids.as<uint32_t>(), n, n, sk->fam->d.tables, sk->fam->d.k_bits,
                        sk->counters, dsum, dsc, sk->st, sk->stream));
  if (out_where == ACE_HOST) {
    if (scores && (r = copy_out(scores, dsc, n * sizeof(double), ACE_HOST, sk->stream)) != ACE_OK) return r;
    if (sums && (r = copy_out(sums, dsum, n * sizeof(uint64_t), ACE_HOST, sk->stream)) != ACE_OK) return r;
  }
  r = pull_state(sk);
  if (r == ACE_OK) fill_stats(stats, *sk->hst, n, sk->fam);
  return r;
}

}  // extern "C"

namespace {

bool host_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// build (optional) + detect over one batch.  The device work is replayed from
// a CUDA graph when the same call repeats (same buffers, sizes and stream;
// captured on the second identical call, once every buffer is sized), so the
// dozen launches and memsets of the pipeline cost one graph launch.
ace_status batch_detect(AceSketch* sk, const void* x, int dtype, uint64_t n, uint64_t ld, int x_where,
                        uint32_t* flag_bits, double* scores, int out_where, AceBatchReport* report, int build) {
  if (build) sk->mean_pinned = false;
  // Deferred insert (counts and gather fused into the detect tail) where the
  // tables fit one shared-memory histogram and the batch is large enough for
  // the gathers to dominate (cfg 2: 0.541 -> 0.525 ms; a loss on small
  // batches such as cfg 1)
  sk->defer_insert = build && sk->defer_mode >= 0 && sk->width == 32 && sk->fam->use_tc() &&
                     sk->fam->d.k_bits <= 16 && (sk->defer_mode == 1 || n * sk->fam->d.tables >= (16ull << 20)) &&
                     fire_and_forget_ok(sk, n);
  sk->insert_deferred = false;
  AceSketch::GraphKey key;
  key.x = x;
  key.flags = flag_bits;
  key.scores = scores;
  key.n = n;
  key.ld = ld;
  key.dtype = dtype;
  key.where = x_where;
  key.out_where = out_where;
  key.build = build;
  key.ff = build ? (fire_and_forget_ok(sk, n) ? 1 : 0) : 2;
  key.stream = sk->stream;
  const DevBuf* bufs[12] = {&sk->ids, &sk->sums, &sk->stage, &sk->flags, &sk->scores, &sk->demand, &sk->near,
                            &sk->overflow, &sk->x16, &sk->rowthr, &sk->segc, &sk->xf32};
  for (int i = 0; i < 12; ++i) key.bufs[i] = bufs[i]->p;
  const bool pinned = x_where == ACE_HOST && host_pinned(x);
  const bool eligible = !sk->timing && (x_where == ACE_DEVICE || pinned);
  const void* xd = nullptr;
  uint64_t ldd = 0;
  uint32_t* dflags = nullptr;
  double* dscores = nullptr;
  // Pinned host rows of a large batch: the H2D copy runs in chunks on a copy
  // stream and each chunk is converted and hashed as it lands, so the hashing
  // hides behind the transfer (sk->h2d_chunks, 8 by default; 1 = one copy,
  // then the work).
  const int chunks_env = sk->h2d_chunks;
  if (pinned && chunks_env > 1 && !sk->timing && sk->fam->use_tc() && !tc_kstream(sk->fam->tc.nkc) &&
      n >= static_cast<uint64_t>(chunks_env) * 16384u) {
    // chunk boundaries: chunks_env - 1 equal chunks and a last one of a quarter
    // of their size (only the last chunk's hashing follows the transfer)
    const uint64_t rows_c = ((n * 4 + (4 * chunks_env - 3) - 1) / (4 * chunks_env - 3) + 127) / 128 * 128;
    const size_t esz = dtype == ACE_F64 ? 8 : 4;
    ACE_CUDA(zero_call_fields(sk));
    ACE_CUDA(sk->stage.ensure(n * ld * esz));
    ACE_CUDA(sk->ids.ensure(static_cast<size_t>(n) * sk->fam->d.tables * sizeof(uint32_t)));
    if (!sk->cstream) ACE_CUDA(cudaStreamCreateWithFlags(&sk->cstream, cudaStreamNonBlocking));
    if (!sk->cstart) ACE_CUDA(cudaEventCreateWithFlags(&sk->cstart, cudaEventDisableTiming));
    const uint64_t nch = (n + rows_c - 1) / rows_c;
    while (sk->cev.size() < nch) {
      cudaEvent_t e;
      ACE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      sk->cev.push_back(e);
    }
    // the copies overwrite the staging buffer: after earlier work on the stream
    ACE_CUDA(cudaEventRecord(sk->cstart, sk->stream));
    ACE_CUDA(cudaStreamWaitEvent(sk->cstream, sk->cstart, 0));
    for (uint64_t c = 0; c < nch; ++c) {
      const uint64_t r0 = c * rows_c, rows = std::min(rows_c, n - r0);
      ACE_CUDA(cudaMemcpyAsync(static_cast<char*>(sk->stage.p) + r0 * ld * esz,
                               static_cast<const char*>(x) + r0 * ld * esz, rows * ld * esz, cudaMemcpyHostToDevice,
                               sk->cstream));
      ACE_CUDA(cudaEventRecord(sk->cev[c], sk->cstream));
    }
    for (uint64_t c = 0; c < nch; ++c) {
      const uint64_t r0 = c * rows_c, rows = std::min(rows_c, n - r0);
      ACE_CUDA(cudaStreamWaitEvent(sk->stream, sk->cev[c], 0));
      ace_status r = run_hash(sk, static_cast<const char*>(sk->stage.p) + r0 * ld * esz, dtype, rows, ld, build,
                              sk->ids.as<uint32_t>() + r0, n);
      if (r != ACE_OK) return r;
    }
    ace_status r = run_detect_device(sk, n, flag_bits, scores, out_where, &dflags, &dscores);
    sk->defer_insert = false;
    if (r != ACE_OK) return r;
    return finish_detect(sk, n, flag_bits, scores, out_where, dflags, dscores, report);
  }
  auto device_work = [&]() -> ace_status {
    ACE_CUDA(zero_call_fields(sk));
    ace_status r = stage_x(sk, sk->stage, sk->stream, x, dtype, n, ld, x_where, &xd, &ldd);
    if (r == ACE_OK) r = run_hash(sk, xd, dtype, n, ldd, build);
    if (r == ACE_OK) r = run_detect_device(sk, n, flag_bits, scores, out_where, &dflags, &dscores);
    return r;
  };
  ace_status r = ACE_OK;
  if (eligible && sk->gexec && key == sk->gkey) {
    ACE_CUDA(cudaGraphLaunch(sk->gexec, sk->stream));
    count_launch(sk->glaunches);
    // pointers the host part needs (same as at capture)
    dflags = (flag_bits && out_where == ACE_DEVICE) ? flag_bits : sk->flags.as<uint32_t>();
    dscores = scores ? (out_where == ACE_DEVICE ? scores : sk->scores.as<double>()) : nullptr;
  } else if (eligible && sk->gseen_valid && key == sk->gseen) {
    sk->drop_graph();
    const unsigned long long l0 = ace_kernel_launches();
    ACE_CUDA(cudaStreamBeginCapture(sk->stream, cudaStreamCaptureModeThreadLocal));
    r = device_work();
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(sk->stream, &g);
    if (r != ACE_OK) {
      if (g) cudaGraphDestroy(g);
      return r;
    }
    if (ce != cudaSuccess) return fail(ACE_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    const cudaError_t ie = cudaGraphInstantiate(&sk->gexec, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) {
      sk->gexec = nullptr;
      return fail(ACE_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ie));
    }
    sk->glaunches = ace_kernel_launches() - l0;
    sk->gkey = key;
    ACE_CUDA(cudaGraphLaunch(sk->gexec, sk->stream));
  } else {
    r = device_work();
    if (r != ACE_OK) return r;
    sk->gseen = key;
    sk->gseen_valid = eligible;
  }
  sk->defer_insert = false;
  return finish_detect(sk, n, flag_bits, scores, out_where, dflags, dscores, report);
}

}  // namespace

extern "C" {

// detect_batch (detect.cpp:12-74).
ace_status ace_sketch_detect_batch(AceSketch* sk, const void* x, int dtype, uint64_t n, uint64_t ld,
                                   int x_where, uint32_t* flag_bits, double* scores, int out_where,
                                   AceBatchReport* report, AceHashStats* stats) {
  if (!sk) return fail(ACE_E_CONTRACT, "detect_batch: null sketch");
  ACE_FLUSH(sk);
  if (n == 0) return fail(ACE_E_CONTRACT, "detect_batch: empty dataset");
  if (ld < sk->fam->d.dim) return fail(ACE_E_CONTRACT, "detect_batch: data dimension mismatch");
  ace_status r = check_x(sk->fam, x, dtype, n, ld, x_where);
  if (r != ACE_OK) return r;
  const auto t0 = std::chrono::steady_clock::now();
  r = batch_detect(sk, x, dtype, n, ld, x_where, flag_bits, scores, out_where, report, 0);
  if (r == ACE_OK) {
    fill_stats(stats, *sk->hst, n, sk->fam);
    if (report)
      report->elapsed_seconds =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  return r;
}

// build_sketch (estimators.cpp:79-92) followed by detect_batch (detect.cpp:12-74).
ace_status ace_sketch_build_detect(AceSketch* sk, const void* x, int dtype, uint64_t n, uint64_t ld,
                                   int x_where, uint32_t* flag_bits, double* scores, int out_where,
                                   AceBatchReport* report, AceHashStats* stats) {
  if (!sk) return fail(ACE_E_CONTRACT, "build_sketch: null sketch");
  ACE_FLUSH(sk);
  if (n == 0) return fail(ACE_E_CONTRACT, "build_sketch: empty dataset");
  ace_status r = check_x(sk->fam, x, dtype, n, ld, x_where);
  if (r != ACE_OK) return r;
  const auto t0 = std::chrono::steady_clock::now();
  r = batch_detect(sk, x, dtype, n, ld, x_where, flag_bits, scores, out_where, report, 1);
  if (r == ACE_OK) {
    fill_stats(stats, *sk->hst, n, sk->fam);
    if (report)
      report->elapsed_seconds =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  return r;
}

// detect_stream (detect.cpp:76-84) for a batch, then insert (ace_cli.cpp:177-183).
ace_status ace_sketch_stream_batch(AceSketch* sk, const void* x, int dtype, uint64_t n, uint64_t ld,
                                   int x_where, double alpha, uint32_t* flag_bits, double* scores,
                                   int out_where, AceStreamReport* report, AceHashStats* stats) {
  if (!sk) return fail(ACE_E_CONTRACT, "detect_stream: null sketch");
  ACE_FLUSH(sk);
  if (!(alpha >= 0.0)) return fail(ACE_E_CONTRACT, "detect_stream: alpha must be >= 0");
  ace_status r = check_x(sk->fam, x, dtype, n, ld, x_where);
  if (r != ACE_OK) return r;
  sk->mean_pinned = false;
  if (n == 0) return ACE_OK;
  const AceFamily* f = sk->fam;
  ACE_CUDA(zero_call_fields(sk));
  const void* xd;
  uint64_t ldd;
  r = stage_x(sk, sk->stage, sk->stream, x, dtype, n, ld, x_where, &xd, &ldd);
  if (r == ACE_OK) r = run_hash(sk, xd, dtype, n, ldd, 0);
  if (r != ACE_OK) return r;
  ACE_CUDA(sk->flags.ensure(((n + 31) / 32) * sizeof(uint32_t)));
  double* dsc = nullptr;
  if (scores) {
    if (out_where == ACE_DEVICE) dsc = scores;
    else {
      ACE_CUDA(sk->scores.ensure(n * sizeof(double)));
      dsc = sk->scores.as<double>();
    }
  }
  uint32_t* dflags = (flag_bits && out_where == ACE_DEVICE) ? flag_bits : sk->flags.as<uint32_t>();
  if (stream_apply_ok(sk, fire_and_forget_ok(sk, n))) {
    // phase A (counts at batch start, insert), then phase B (scores, flags)
    if ((r = ensure_stream_bufs(sk, n)) != ACE_OK) return r;
    const uint32_t slot = 0u;  // a one-batch call: its phase B reads slot 0 right after
    uint32_t* cnt = sk->cnt[slot].as<uint32_t>();
    ACE_CUDA(launch_stream_apply(sk->ids.as<uint32_t>(), n, n, f->d.tables, f->d.k_bits, sk->counters, cnt, slot,
                                 nullptr, 0, nullptr, nullptr, 0, alpha, sk->st, sk->stream));
    sk->mark(2);
    ACE_CUDA(launch_stream_apply(nullptr, 0, 0, f->d.tables, f->d.k_bits, sk->counters, nullptr, 0, cnt, n, dflags, dsc,
                                 slot, alpha, sk->st, sk->stream));
  } else {
    ACE_CUDA(cudaMemsetAsync(&sk->st->batch_sum, 0, sizeof(unsigned long long), sk->stream));
    ACE_CUDA(launch_stream_score(sk->ids.as<uint32_t>(), n, f->d.tables, f->d.k_bits, sk->counters,
                                 alpha, dflags, dsc, sk->st, sk->stream));
    sk->mark(2);
    ACE_CUDA(launch_apply_ids(sk->ids.as<uint32_t>(), n, f->d.tables, f->d.k_bits, sk->counters,
                              sk->cap, +1, sk->st, sk->stream, !fire_and_forget_ok(sk, n)));
    if (sk->width == 16) ACE_CUDA(launch_cap(sk->counters, sk->num_counters, sk->cap, sk->st, sk->stream));
  }
  sk->mark(3);
  if (out_where == ACE_HOST) {
    if (flag_bits &&
        (r = copy_out(flag_bits, dflags, ((n + 31) / 32) * sizeof(uint32_t), ACE_HOST, sk->stream)) != ACE_OK)
      return r;
    if (scores && (r = copy_out(scores, dsc, n * sizeof(double), ACE_HOST, sk->stream)) != ACE_OK) return r;
  }
  r = pull_state(sk);
  if (r != ACE_OK) return r;
  fill_stats(stats, *sk->hst, n, f);
  if (report) {
    report->mean_before = sk->hst->mean_before;
    report->cut = sk->hst->cut;
    report->reported = sk->hst->reported;
    report->ambiguous = sk->hst->ambiguous;
  }
  return ACE_OK;
}

// The streaming driver (ace_cli.cpp:173-186 with the insert deferred to each
// batch end) over many batches, queued without host synchronisation.
ace_status ace_sketch_stream_run(AceSketch* sk, const void* x, int dtype, uint64_t n, uint64_t ld, int x_where,
                                 uint64_t batch, double alpha, uint32_t* flag_bits, int out_where,
                                 float* batch_ms, AceStreamReport* report, AceHashStats* stats) {
  if (!sk) return fail(ACE_E_CONTRACT, "detect_stream: null sketch");
  ACE_FLUSH(sk);
  if (!(alpha >= 0.0)) return fail(ACE_E_CONTRACT, "detect_stream: alpha must be >= 0");
  if (batch == 0 || batch % 32 != 0) return fail(ACE_E_CONTRACT, "stream_run: batch must be a positive multiple of 32");
  ace_status r = check_x(sk->fam, x, dtype, n, ld, x_where);
  if (r != ACE_OK) return r;
  sk->mean_pinned = false;
  if (n == 0) return ACE_OK;
  const AceFamily* f = sk->fam;
  const size_t esz = dtype == ACE_F64 ? 8 : 4;
  const uint64_t nb = (n + batch - 1) / batch;
  const bool ff = fire_and_forget_ok(sk, n);
  const bool fast = stream_apply_ok(sk, ff);
  const uint64_t G = static_cast<uint64_t>(sk->stream_group);
  // u16 bucket ids between the projection and the pair stream kernel: half
  // the id traffic (K <= 15, the d <= 256 tensor-core projection)
  const bool ids16 = fast && stream_pair_ok(f->d.tables, f->d.k_bits, batch) && f->use_tc() && !tc_kstream(f->tc.nkc);
  // one stream launch per hashing group (stream_group_kernel): the tables'
  // counts stay in shared memory across the group's batches
  const bool gfast = ids16 && stream_group_ok(f->d.tables, f->d.k_bits, batch);
  const uint64_t gl = std::min(G, nb);                    // batches per group
  const uint64_t gld = (std::min(gl * batch, n) + 7) / 8 * 8;  // u16 id stride (16-byte rows)
  ACE_CUDA(sk->flags.ensure(((n + 31) / 32) * sizeof(uint32_t)));
  uint32_t* dflags = (flag_bits && out_where == ACE_DEVICE) ? flag_bits : sk->flags.as<uint32_t>();
  if (fast && !gfast && (r = ensure_stream_bufs(sk, std::min(batch, n))) != ACE_OK) return r;
  // pipelined groups (ACE_OPT_STREAM_PIPE): the projection of group g + 1 on
  // `pipe` SMs beside the stream kernel of group g on the others
  // automatic: every SM but one per table and eight for scoring (cfg 5: 90 of 148)
  const int sms_all = tc_sms();
  const int pipe_req = sk->stream_pipe >= 0 ? sk->stream_pipe : std::max(0, sms_all - static_cast<int>(f->d.tables) - 8);
  const uint32_t pipe = (gfast && nb > G && pipe_req > 0 &&
                         stream_solo_ok(f->d.tables, f->d.k_bits, batch, static_cast<uint32_t>(pipe_req)))
                            ? static_cast<uint32_t>(pipe_req)
                            : 0u;
  if (gfast && (r = ensure_group_bufs(sk, gl, batch, gld, pipe != 0)) != ACE_OK) return r;
  // per-batch latency: from the start of the batch's work (its group's
  // hashing for a group's first batch) to the end of the launch that writes
  // its flags; events kept by the sketch across calls
  if (batch_ms) {
    while (sk->lat_a.size() < nb) {
      cudaEvent_t e0, e1;
      ACE_CUDA(cudaEventCreate(&e0));
      ACE_CUDA(cudaEventCreate(&e1));
      sk->lat_a.push_back(e0);
      sk->lat_b.push_back(e1);
    }
  }
  std::vector<cudaEvent_t> tev;  // timing on: (start, end) pairs, hashing then stream kernels
  std::vector<int> tkind;
  auto tmark = [&](int kind, bool end, cudaStream_t ts = nullptr) -> cudaError_t {
    if (!sk->timing) return cudaSuccess;
    cudaEvent_t e;
    cudaError_t err = cudaEventCreate(&e);
    if (err != cudaSuccess) return err;
    tev.push_back(e);
    if (!end) tkind.push_back(kind);
    return cudaEventRecord(e, ts ? ts : sk->stream);
  };
  // pinned host rows: H2D copies of the next group overlap this group's work
  const bool overlap = x_where == ACE_HOST && host_pinned(x) && nb > G;
  if (overlap) {
    const size_t gbytes = static_cast<size_t>(G * batch) * ld * esz;
    ACE_CUDA(sk->sstage[0].ensure(gbytes));
    ACE_CUDA(sk->sstage[1].ensure(gbytes));
    if (!sk->cstream) ACE_CUDA(cudaStreamCreateWithFlags(&sk->cstream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      if (!sk->s_copied[i]) ACE_CUDA(cudaEventCreateWithFlags(&sk->s_copied[i], cudaEventDisableTiming));
      if (!sk->s_used[i]) ACE_CUDA(cudaEventCreateWithFlags(&sk->s_used[i], cudaEventDisableTiming));
    }
  }
  // All device work of the call.  Consecutive batches alternate the two cut
  // slots (slot = batch index & 1): a batch's phase B reads the slot its
  // phase A wrote one launch earlier.
  auto device_work = [&]() -> ace_status {
    ACE_CUDA(zero_call_fields(sk));
    if (overlap) {
      // the staging halves are free once earlier work on the stream is done
      ACE_CUDA(cudaEventRecord(sk->s_used[0], sk->stream));
      ACE_CUDA(cudaEventRecord(sk->s_used[1], sk->stream));
      ACE_CUDA(cudaStreamWaitEvent(sk->cstream, sk->s_used[0], 0));
      const uint64_t rows0 = std::min(G * batch, n);
      ACE_CUDA(cudaMemcpyAsync(sk->sstage[0].p, x, rows0 * ld * esz, cudaMemcpyHostToDevice, sk->cstream));
      ACE_CUDA(cudaEventRecord(sk->s_copied[0], sk->cstream));
    }
    // the batch whose phase B is still due (fast path)
    const uint32_t* p_cnt = nullptr;
    uint64_t p_rows = 0, p_b = 0;
    uint32_t* p_flags = nullptr;
    uint32_t p_slot = 0;
    for (uint64_t g0 = 0; g0 < nb; g0 += G) {
      const uint64_t gb = std::min(G, nb - g0), gr0 = g0 * batch, grows = std::min(gb * batch, n - gr0);
      // pipelined: id buffer g & 1, free once the stream kernel of group g - 2 has read it
      const int pb = pipe ? static_cast<int>((g0 / G) & 1u) : 0;
      uint16_t* gids = gfast ? sk->ids.as<uint16_t>() + static_cast<size_t>(pb) * gld * f->d.tables : nullptr;
      if (pipe && g0 >= 2 * G) ACE_CUDA(cudaStreamWaitEvent(sk->stream, sk->p_streamed[pb], 0));
      if (batch_ms)
        for (uint64_t b = g0; b < (gfast ? g0 + gb : g0 + 1); ++b) ACE_CUDA(cudaEventRecord(sk->lat_a[b], sk->stream));
      const void* xg = static_cast<const char*>(x) + gr0 * ld * esz;
      const void* xd;
      uint64_t ldd;
      ace_status rr;
      if (overlap) {
        // group g's rows were copied into staging half g & 1 ahead of time;
        // start the copy of group g + 1 into the other half once the hash of
        // group g - 1 (its previous user) has run
        const int hb = static_cast<int>((g0 / G) & 1u);
        ACE_CUDA(cudaStreamWaitEvent(sk->stream, sk->s_copied[hb], 0));
        xd = sk->sstage[hb].p;
        ldd = ld;
        ACE_CUDA(tmark(0, false));
        if ((rr = run_hash(sk, xd, dtype, grows, ldd, 0, reinterpret_cast<uint32_t*>(gids), gfast ? gld : 0, ids16,
                           pipe)) != ACE_OK)
          return rr;
        ACE_CUDA(tmark(0, true));
        ACE_CUDA(cudaEventRecord(sk->s_used[hb], sk->stream));
        const uint64_t g1 = g0 + G;
        if (g1 < nb) {
          const uint64_t r1 = g1 * batch, rows1 = std::min(G * batch, n - r1);
          ACE_CUDA(cudaStreamWaitEvent(sk->cstream, sk->s_used[hb ^ 1], 0));
          ACE_CUDA(cudaMemcpyAsync(sk->sstage[hb ^ 1].p, static_cast<const char*>(x) + r1 * ld * esz,
                                   rows1 * ld * esz, cudaMemcpyHostToDevice, sk->cstream));
          ACE_CUDA(cudaEventRecord(sk->s_copied[hb ^ 1], sk->cstream));
        }
      } else {
        if ((rr = stage_x(sk, sk->stage, sk->stream, xg, dtype, grows, ld, x_where, &xd, &ldd)) != ACE_OK) return rr;
        ACE_CUDA(tmark(0, false));
        if ((rr = run_hash(sk, xd, dtype, grows, ldd, 0, reinterpret_cast<uint32_t*>(gids), gfast ? gld : 0, ids16,
                           pipe)) != ACE_OK)
          return rr;
        ACE_CUDA(tmark(0, true));
      }
      if (gfast) {
        // pipelined: on pstream, after this group's projection; the last
        // group's stream kernel has the GPU to itself (pair kernel)
        cudaStream_t ss = pipe ? sk->pstream : sk->stream;
        if (pipe) {
          ACE_CUDA(cudaEventRecord(sk->p_hashed[pb], sk->stream));
          ACE_CUDA(cudaStreamWaitEvent(ss, sk->p_hashed[pb], 0));
        }
        ACE_CUDA(tmark(1, false, ss));
        ACE_CUDA(launch_stream_group(gids, gld, grows, batch, f->d.tables, f->d.k_bits, sk->counters,
                                     sk->gco.as<uint32_t>(), sk->gdT.as<unsigned long long>(),
                                     sk->gdone.as<unsigned int>(), sk->gdone.as<unsigned int>() + gl,
                                     dflags + gr0 / 32, alpha, sk->st, ss,
                                     g0 + G < nb ? pipe : 0u));
        ACE_CUDA(tmark(1, true, ss));
        if (batch_ms)
          for (uint64_t b = g0; b < g0 + gb; ++b) ACE_CUDA(cudaEventRecord(sk->lat_b[b], ss));
        if (pipe) {
          ACE_CUDA(cudaEventRecord(sk->p_streamed[pb], ss));
          // join: the caller's stream continues after the last stream kernel
          if (g0 + G >= nb) ACE_CUDA(cudaStreamWaitEvent(sk->stream, sk->p_streamed[pb], 0));
        }
        continue;
      }
      for (uint64_t b = g0; b < g0 + gb; ++b) {
        const uint64_t r0 = b * batch, rows = std::min(batch, n - r0);
        if (batch_ms && b != g0) ACE_CUDA(cudaEventRecord(sk->lat_a[b], sk->stream));
        const uint32_t* ids = ids16 ? reinterpret_cast<const uint32_t*>(sk->ids.as<uint16_t>() + (r0 - gr0))
                                    : sk->ids.as<uint32_t>() + (r0 - gr0);
        if (fast) {
          const uint32_t slot = static_cast<uint32_t>(b & 1u);
          uint32_t* cnt = sk->cnt[slot].as<uint32_t>();
          ACE_CUDA(tmark(1, false));
          ACE_CUDA(launch_stream_apply(ids, rows, grows, f->d.tables, f->d.k_bits, sk->counters, cnt, slot, p_cnt,
                                       p_rows, p_flags, nullptr, p_slot, alpha, sk->st, sk->stream, ids16 ? 1 : 0));
          ACE_CUDA(tmark(1, true));
          if (batch_ms && p_rows) ACE_CUDA(cudaEventRecord(sk->lat_b[p_b], sk->stream));
          p_cnt = cnt;
          p_rows = rows;
          p_b = b;
          p_flags = dflags + r0 / 32;
          p_slot = slot;
          continue;
        }
        ACE_CUDA(cudaMemsetAsync(&sk->st->batch_sum, 0, sizeof(unsigned long long), sk->stream));
        ACE_CUDA(launch_stream_score(ids, rows, f->d.tables, f->d.k_bits, sk->counters, alpha, dflags + r0 / 32,
                                     nullptr, sk->st, sk->stream, grows));
        ACE_CUDA(launch_apply_ids(ids, rows, f->d.tables, f->d.k_bits, sk->counters, sk->cap, +1, sk->st, sk->stream,
                                  !ff, grows));
        if (sk->width == 16) ACE_CUDA(launch_cap(sk->counters, sk->num_counters, sk->cap, sk->st, sk->stream));
        if (batch_ms) ACE_CUDA(cudaEventRecord(sk->lat_b[b], sk->stream));
      }
    }
    if (fast && !gfast && p_rows) {  // the last batch's phase B
      ACE_CUDA(tmark(1, false));
      ACE_CUDA(launch_stream_apply(nullptr, 0, 0, f->d.tables, f->d.k_bits, sk->counters, nullptr, 0, p_cnt, p_rows,
                                   p_flags, nullptr, p_slot, alpha, sk->st, sk->stream));
      ACE_CUDA(tmark(1, true));
      if (batch_ms) ACE_CUDA(cudaEventRecord(sk->lat_b[p_b], sk->stream));
    }
    if (flag_bits && out_where == ACE_HOST) {
      ace_status rr2 = copy_out(flag_bits, dflags, ((n + 31) / 32) * sizeof(uint32_t), ACE_HOST, sk->stream);
      if (rr2 != ACE_OK) return rr2;
    }
    return ACE_OK;
  };
  // Repeated calls with the same arguments (device rows) replay a CUDA graph
  // of all the device work (captured on the second identical call): the
  // thousands of launches of a long stream cost one graph launch.
  AceSketch::StreamKey key;
  key.x = x;
  key.flags = flag_bits;
  key.n = n;
  key.ld = ld;
  key.batch = batch;
  key.alpha = alpha;
  key.dtype = dtype;
  key.out_where = out_where;
  key.lat = batch_ms != nullptr;
  key.group = sk->stream_group * 4096 + sk->stream_pipe;
  key.stream = sk->stream;
  key.ff = ff;
  const DevBuf* sb[9] = {&sk->ids, &sk->flags, &sk->cnt[0], &sk->cnt[1], &sk->near, &sk->overflow,
                         &sk->gco, &sk->gdT, &sk->gdone};
  for (int i = 0; i < 9; ++i) key.bufs[i] = sb[i]->p;
  // (per-batch latency events are recorded only outside graphs)
  const bool eligible = x_where == ACE_DEVICE && !sk->timing && fast && !batch_ms;
  if (eligible && sk->sgexec && key == sk->sgkey) {
    ACE_CUDA(cudaGraphLaunch(sk->sgexec, sk->stream));
    count_launch(sk->sglaunches);
  } else if (eligible && sk->sgseen_valid && key == sk->sgseen) {
    if (sk->sgexec) cudaGraphExecDestroy(sk->sgexec);
    sk->sgexec = nullptr;
    const unsigned long long l0 = ace_kernel_launches();
    ACE_CUDA(cudaStreamBeginCapture(sk->stream, cudaStreamCaptureModeThreadLocal));
    r = device_work();
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(sk->stream, &g);
    if (r != ACE_OK) {
      if (g) cudaGraphDestroy(g);
      return r;
    }
    if (ce != cudaSuccess) return fail(ACE_E_CUDA, std::string("stream graph capture: ") + cudaGetErrorString(ce));
    const cudaError_t ie = cudaGraphInstantiate(&sk->sgexec, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) {
      sk->sgexec = nullptr;
      return fail(ACE_E_CUDA, std::string("stream graph instantiate: ") + cudaGetErrorString(ie));
    }
    sk->sglaunches = ace_kernel_launches() - l0;
    sk->sgkey = key;
    ACE_CUDA(cudaGraphLaunch(sk->sgexec, sk->stream));
  } else {
    if ((r = device_work()) != ACE_OK) return r;
    sk->sgseen = key;
    sk->sgseen_valid = eligible;
  }
  r = pull_state(sk);
  if (r != ACE_OK) return r;
  if (sk->timing) {
    sk->stream_ms[0] = sk->stream_ms[1] = 0.0;
    for (size_t k = 0; k < tkind.size(); ++k) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tev[2 * k], tev[2 * k + 1]);
      sk->stream_ms[tkind[k]] += ms;
    }
    for (auto& e : tev) cudaEventDestroy(e);
    sk->stream_timed = true;
  }
  if (batch_ms) {
    for (uint64_t b = 0; b < nb; ++b) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, sk->lat_a[b], sk->lat_b[b]);
      batch_ms[b] = ms;
    }
  }
  fill_stats(stats, *sk->hst, n, f);
  if (report) {
    report->mean_before = sk->hst->mean_before;
    report->cut = sk->hst->cut;
    report->reported = sk->hst->reported;
    report->ambiguous = sk->hst->ambiguous;
  }
  return ACE_OK;
}

// detect_stream (detect.cpp:76-84) for each of n queries against the current
// sketch: score, flag = score <= mean - alpha.  Host outputs.
ace_status ace_sketch_detect_stream(AceSketch* sk, const void* q, int dtype, uint64_t n, uint64_t ld, int q_where,
                                    double alpha, double* scores, uint8_t* flags) {
  if (!sk) return fail(ACE_E_CONTRACT, "ace_sketch_detect_stream: null sketch");
  if (alpha < 0.0) return fail(ACE_E_CONTRACT, "detect_stream: alpha must be >= 0");
  ace_status r = check_x(sk->fam, q, dtype, n, ld, q_where);
  if (r != ACE_OK) {
    // the reference reports an empty sketch before it scores (detect.cpp:80-81)
    const std::string msg = g_err;
    if (pull_state(sk) == ACE_OK && sk->hst->n == 0) return fail(ACE_E_CONTRACT, "detect_stream: empty sketch");
    return fail(r, msg);
  }
  if (n == 0) return ACE_OK;
  std::vector<double> tmp;
  double* sc = scores;
  if (!sc) {
    tmp.resize(n);
    sc = tmp.data();
  }
  if (point_ok(sk, dtype, n, q_where)) {
    if ((r = run_point(sk, q, dtype, n, ld, 0)) != ACE_OK || (r = finish_point_score(sk)) != ACE_OK) return r;
    memcpy(sc, sk->pth->scores, n * sizeof(double));
  } else if ((r = ace_sketch_score(sk, q, dtype, n, ld, q_where, sc, nullptr, ACE_HOST, nullptr)) != ACE_OK) {
    return r;
  }
  if (sk->hst->n == 0) return fail(ACE_E_CONTRACT, "detect_stream: empty sketch");
  const double mean = sk->mean_pinned ? sk->pinned_mean : host_mean(*sk->hst, sk->fam->d.tables);
  if (flags)
    for (uint64_t i = 0; i < n; ++i) flags[i] = sc[i] <= mean - alpha ? 1 : 0;
  return ACE_OK;
}

// One counter (AceSketch::counter, sketch.hpp): a 4-byte read into pinned
// memory, not the whole array.
ace_status ace_sketch_counter(const AceSketch* sk, uint32_t table, uint64_t bucket, uint64_t* value) {
  if (!sk || !value) return fail(ACE_E_CONTRACT, "ace_sketch_counter: null argument");
  ACE_FLUSH(sk);
  if (!sk->pth || table >= sk->fam->d.tables || bucket >= (1ull << sk->fam->d.k_bits))
    return fail(ACE_E_CONTRACT, "AceSketch: counter index out of range");
  const uint32_t* src = sk->counters + (static_cast<uint64_t>(table) << sk->fam->d.k_bits) + bucket;
  ACE_CUDA(cudaMemcpyAsync(&sk->pth->counter, src, sizeof(uint32_t), cudaMemcpyDeviceToHost, sk->stream));
  ACE_CUDA(cudaStreamSynchronize(sk->stream));
  *value = sk->pth->counter;
  return ACE_OK;
}

// size / mean / saturated (sketch.hpp:44-46).
ace_status ace_sketch_info(const AceSketch* sk, uint64_t* n, double* mean, int* saturated) {
  if (!sk) return fail(ACE_E_CONTRACT, "ace_sketch_info: null sketch");
  AceSketch* m = const_cast<AceSketch*>(sk);
  ace_status r = pull_state(m);
  if (r != ACE_OK) return r;
  if (n) *n = sk->hst->n;
  if (mean) *mean = sk->mean_pinned ? sk->pinned_mean : host_mean(*sk->hst, sk->fam->d.tables);
  if (saturated) *saturated = sk->hst->saturated;
  return ACE_OK;
}

// counters_flat (sketch.cpp:126-130).
ace_status ace_sketch_counters(const AceSketch* sk, uint64_t* counters) {
  if (!sk || !counters) return fail(ACE_E_CONTRACT, "ace_sketch_counters: null argument");
  ACE_FLUSH(sk);
  std::vector<uint32_t> tmp(sk->num_counters);
  ACE_CUDA(cudaMemcpyAsync(tmp.data(), sk->counters, sk->num_counters * sizeof(uint32_t),
                           cudaMemcpyDeviceToHost, sk->stream));
  ACE_CUDA(cudaStreamSynchronize(sk->stream));
  for (uint64_t i = 0; i < sk->num_counters; ++i) counters[i] = tmp[i];
  return ACE_OK;
}

ace_status ace_sketch_counters_u32(const AceSketch* sk, uint32_t* counters, int where) {
  if (!sk || !counters) return fail(ACE_E_CONTRACT, "ace_sketch_counters_u32: null argument");
  ACE_FLUSH(sk);
  ACE_CUDA(cudaMemcpyAsync(counters, sk->counters, sk->num_counters * sizeof(uint32_t),
                           where == ACE_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                           sk->stream));
  ACE_CUDA(cudaStreamSynchronize(sk->stream));
  return ACE_OK;
}

// AceSketch::restore (sketch.cpp:132-150).
ace_status ace_sketch_restore(AceSketch* sk, const uint64_t* counters, uint64_t num_counters,
                              uint64_t n, double mean, int saturated) {
  if (!sk) return fail(ACE_E_CONTRACT, "ace_sketch_restore: null sketch");
  ACE_FLUSH(sk);
  if (num_counters != sk->num_counters)
    return fail(ACE_E_CONTRACT, "AceSketch::restore: counter payload size " + std::to_string(num_counters) +
                                    " does not match L * 2^K = " + std::to_string(sk->num_counters));
  std::vector<uint32_t> tmp(num_counters);
  for (uint64_t i = 0; i < num_counters; ++i) {
    if (counters[i] > sk->cap) return fail(ACE_E_CONTRACT, "AceSketch::restore: counter exceeds width");
    tmp[i] = static_cast<uint32_t>(counters[i]);
  }
  ACE_CUDA(cudaMemcpyAsync(sk->counters, tmp.data(), num_counters * sizeof(uint32_t),
                           cudaMemcpyHostToDevice, sk->stream));
  ACE_CUDA(cudaStreamSynchronize(sk->stream));
  DevState s{};
  s.n = n;
  // T = sum of the insert numerators = sum c^2 exactly while nothing has
  // saturated; a saturated 16-bit sketch keeps the rounded mean * n * L
  unsigned __int128 sq = 0;
  for (uint64_t i = 0; i < num_counters; ++i) sq += static_cast<unsigned __int128>(tmp[i]) * tmp[i];
  if (!saturated && (sq >> 64) == 0)
    s.T = static_cast<unsigned long long>(sq);
  else
    s.T = static_cast<unsigned long long>(std::llround(mean * static_cast<double>(n) * sk->fam->d.tables));
  sk->mean_pinned = true;
  sk->pinned_mean = mean;
  s.saturated = saturated ? 1 : 0;
  *sk->hst = s;
  ACE_CUDA(cudaMemcpyAsync(sk->st, sk->hst, sizeof(DevState), cudaMemcpyHostToDevice, sk->stream));
  ACE_CUDA(cudaStreamSynchronize(sk->stream));
  return ACE_OK;
}

const uint32_t* ace_sketch_device_counters(const AceSketch* sk) {
  if (!sk) return nullptr;
  if (flush_point(sk) != ACE_OK) return nullptr;  // counters complete in the sketch's stream order
  return sk->counters;
}

ace_status ace_sketch_set_timing(AceSketch* sk, int enable) {
  if (!sk) return fail(ACE_E_CONTRACT, "ace_sketch_set_timing: null sketch");
  if (enable)
    for (cudaEvent_t& e : sk->ev)
      if (!e) ACE_CUDA(cudaEventCreate(&e));
  sk->timing = enable != 0;
  return ACE_OK;
}

ace_status ace_sketch_timings(const AceSketch* sk, double* ms3) {
  if (!sk || !ms3) return fail(ACE_E_CONTRACT, "ace_sketch_timings: null argument");
  if (sk->stream_timed) {  // the last call was the stream driver
    ms3[0] = sk->stream_ms[0];
    ms3[1] = 0.0;
    ms3[2] = sk->stream_ms[1];
    ms3[3] = 0.0;
    ms3[4] = sk->stream_ms[0];
    return ACE_OK;
  }
  const int pairs[5][2] = {{0, 1}, {1, 2}, {2, 3}, {4, 6}, {6, 5}};
  for (int i = 0; i < 5; ++i) {
    ms3[i] = 0.0;
    const int a = pairs[i][0], b = pairs[i][1];
    if (sk->timing && sk->ev_used[a] && sk->ev_used[b]) {
      float ms = 0.f;
      ACE_CUDA(cudaEventSynchronize(sk->ev[b]));
      ACE_CUDA(cudaEventElapsedTime(&ms, sk->ev[a], sk->ev[b]));
      ms3[i] = ms;
    }
  }
  return ACE_OK;
}

}  // extern "C"
