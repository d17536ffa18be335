// tcgen05 projection kernel for sm_100a (d <= 256): the SRP hash of 128-point
// tiles against every direction on the 5th-generation tensor cores, reading
// the caller's raw fp32 rows straight from HBM (one pass over X).
//
// P = X W^T computed as an error-compensated fp16 split,
//   x~ = x * 2^s(row) = x_hi + x_lo,   w^ = w * 2^14/||w|| = w_hi + w_lo,
//   P~ = x_hi w_hi + x_lo w_hi + x_hi w_lo     (three tcgen05.mma per K16 step),
// accumulated in fp32 in TMEM.  Signs are scale invariant, so sign(P~) equals
// the reference's sign(p) (srp.cpp:78-104) whenever |P~| exceeds the rigorous
// error bound thr(row) = c * ||x~|| * 2^14 + abs; projections inside the bound
// go to a near-tie list and are recomputed as the reference's binary64 fold.
// Buckets are packed MSB-first (srp.cpp:106-113) straight from the
// accumulator columns: one thread owns one point (TMEM lane).
//
// Warp roles (576 threads, one CTA per SM, persistent over point tiles):
//   warp 0      W producer: ring of pre-swizzled W stages (cp.async.bulk)
//   warp 1      TMEM allocator and MMA issuer (one elected lane, TS MMAs with
//               the x split as the TMEM A operand)
//   warps 2-13  epilogue: three warps per TMEM lane quarter, the 32-column
//               groups of each direction tile dealt round-robin; tcgen05.ld
//               -> sign words, near ties
//   warps 14-17 converters, one per lane quarter, one thread per point: the
//               raw fp32 tile arrives by tensor-map TMA (SWIZZLE_128B boxes
//               of 32 columns, OOB rows and columns zero-filled); each thread
//               finds its row's scale, splits into fp16 hi / lo and writes
//               them into a double-buffered TMEM A operand with tcgen05.st,
//               plus the row's error threshold for the epilogue.  Warp 14
//               issues the next tile's TMA as soon as the raw tile is read.
//               One tile behind, the same warps cut the bucket ids from the
//               sign words and store them.
// After the main loop warps 2-17 recheck the listed near ties (shared tail).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>

#include "ace_tc_ptx.cuh"

namespace ace_dev {
using namespace tc;

namespace {

constexpr uint32_t kEpiQ = 4;        // epilogue warps per TMEM lane quarter (one 32-column group each)
constexpr uint32_t kConvW = 2u + 4u * kEpiQ;  // first converter warp
constexpr int kThreads = 32 * (kConvW + 4);   // 22 warps
constexpr uint32_t kMaxWStages = 8;
constexpr uint32_t kRawBox = 16384;  // one raw box: 128 rows x 32 fp32 (SW128)
constexpr uint32_t kConvBar = 10;    // named barrier of the converter warps

// Compile-time instrumentation (-DACE_TC_PROF=1, profiling builds only):
// clock64 cycles per pipeline section summed over CTAs into g_tc_prof
// (read by ace_debug_tc_prof, exported only by such builds).
#ifndef ACE_TC_PROF
#define ACE_TC_PROF 0
#endif
// Experiment switches (profiling builds only; results are then wrong):
// 1 = epilogue skips the sign / near-tie work, 2 = no MMAs issued,
// 4 = packers skip the bucket cut and stores, 8 = W loaded for the first
// point tile only, 64 = near ties not listed
#ifndef ACE_TC_DBG
#define ACE_TC_DBG 0
#endif
#if ACE_TC_PROF
__device__ unsigned long long g_tc_prof[24];
#define TCP_DECL unsigned long long tcp[24] = {0}; long long tcp_t = 0
#define TCP_BEGIN() (tcp_t = clock64())
#define TCP_END(k) (tcp[k] += static_cast<unsigned long long>(clock64() - tcp_t))
#define TCP_FLUSH(cond) \
  if (cond)             \
    for (int k_ = 0; k_ < 24; ++k_) \
      if (tcp[k_]) atomicAdd(&g_tc_prof[k_], tcp[k_])
#else
#define TCP_DECL
#define TCP_BEGIN()
#define TCP_END(k)
#define TCP_FLUSH(cond)
#endif

// Shared memory: the raw fp32 tile (n_raw boxes), then a ring of W stages
// (hi + lo block of one direction tile x 64 K).  TMEM (512 columns): nacc
// fp32 accumulators of tw columns, then n_abuf A operands (hi | lo, 8 columns
// per K16 step each).
struct TcLayout {
  uint32_t n_raw, n_wst, nsteps, acols, nacc, n_abuf, nwords, n_sbuf;
  size_t raw_bytes, sgn_bytes, w_bytes, total;
};

// rows = K * L directions.  Sign words: per point tile, word w of row r at
// sgn[w][r] (one buffer: nwords * 128 u32, rounded to 1 KB); two buffers when
// at least three W stages still fit.
__host__ __device__ inline TcLayout tc_layout(uint64_t dim, uint32_t tw, uint32_t rows) {
  TcLayout L;
  L.n_raw = static_cast<uint32_t>((dim + 31) / 32);
  L.raw_bytes = static_cast<size_t>(L.n_raw) * kRawBox;
  L.nsteps = static_cast<uint32_t>((dim + 15) / 16);
  L.acols = 16u * L.nsteps;
  // a third accumulator where it fits beside two A buffers (d <= 64 at tw = 128)
  L.nacc = (3u * tw + 2u * L.acols <= 512u) ? 3u : 2u;
  L.n_abuf = (L.nacc * tw + 2u * L.acols <= 512u) ? 2u : 1u;
  L.nwords = (rows + 31u) / 32u;
  L.sgn_bytes = (static_cast<size_t>(L.nwords) * kRows * 4u + 1023u) / 1024u * 1024u;
  const size_t room0 = kSmemLimit - 8192 - 1024 - L.raw_bytes;
  const size_t stage = 2u * tw * 128u;
  L.n_sbuf = (room0 >= 2u * L.sgn_bytes + 3u * stage) ? 2u : 1u;
  const size_t room = room0 > L.n_sbuf * L.sgn_bytes ? room0 - L.n_sbuf * L.sgn_bytes : 0;
  size_t st = room / stage;
  if (st > kMaxWStages) st = kMaxWStages;
  L.n_wst = static_cast<uint32_t>(st);
  L.w_bytes = st * stage;
  L.total = L.raw_bytes + L.n_sbuf * L.sgn_bytes + L.w_bytes + 1024;
  return L;
}

// Warp-aggregated counter increments for one table (fused insert, K > 20):
// lanes holding equal buckets are merged over up to three ballot rounds.
__device__ __forceinline__ void insert_bucket_warp(uint32_t* ct, uint32_t bucket, bool valid, uint32_t lane) {
  unsigned rem = __ballot_sync(0xffffffffu, valid);
#pragma unroll
  for (int round = 0; round < 3 && rem; ++round) {
    const int leader = __ffs(rem) - 1;
    const uint32_t bl = __shfl_sync(0xffffffffu, bucket, leader);
    const unsigned eq = __ballot_sync(0xffffffffu, bucket == bl) & rem;
    if (lane == static_cast<uint32_t>(leader)) atomicAdd(&ct[bl], static_cast<uint32_t>(__popc(eq)));
    rem &= ~eq;
  }
  if ((rem >> lane) & 1u) atomicAdd(&ct[bucket], 1u);
}

// Bucket ids are u32, or u16 for the stream driver (K <= 16): element idx of
// the table-major id array.
__device__ __forceinline__ uint32_t id_get(const TcArgs& a, uint64_t idx) {
  return a.ids16 ? static_cast<uint32_t>(__ldcg(reinterpret_cast<const unsigned short*>(a.ids) + idx)) : __ldcg(a.ids + idx);
}
__device__ __forceinline__ void id_put(const TcArgs& a, uint64_t idx, uint32_t v) {
  if (a.ids16)
    reinterpret_cast<unsigned short*>(a.ids)[idx] = static_cast<unsigned short>(v);
  else
    a.ids[idx] = v;
}
// atomic XOR of bits m into id idx (a u16 id through its aligned 32-bit word); the old id
__device__ __forceinline__ uint32_t id_xor(const TcArgs& a, uint64_t idx, uint32_t m) {
  if (!a.ids16) return atomicXor(a.ids + idx, m);
  const uintptr_t p = reinterpret_cast<uintptr_t>(reinterpret_cast<unsigned short*>(a.ids) + idx);
  const uint32_t sh = (p & 2u) ? 16u : 0u;
  return (atomicXor(reinterpret_cast<uint32_t*>(p & ~static_cast<uintptr_t>(3)), m << sh) >> sh) & 0xffffu;
}

// Exact decision of one listed near tie by a group of kG lanes (all lanes of
// the warp call it together; `live` false for idle groups).  The lanes split
// the d products x_i w_i (binary64: exact for fp32 x, one rounding for fp64
// x) and sum them in a tree: p1 and the reference's sequential left fold
// (srp.cpp:78-91) are both within gamma_{d+2} A of the exact value (A = sum
// |x_i w_i|), so |p1| > 2 gamma A decides the reference's sign bit; likewise
// the BASELINE near-tie measure |p| < 1e-6 |x||w| where p1 is clear of its
// threshold.  Otherwise (never seen on the BASELINE data) the group's first
// lane evaluates the reference's fold and the oracle's sequential |x|^2
// themselves.  A wrong fast bit is flipped in the ids (and, with the fused
// insert, the count moves to the corrected bucket).
constexpr uint32_t kG = 8;  // lanes per item
__device__ __forceinline__ void recheck_item(const TcArgs& a, unsigned long long item, bool live, uint32_t gl,
                                             unsigned long long& rr, unsigned long long& ff, unsigned long long& nt) {
  const uint32_t dim = static_cast<uint32_t>(a.dim), K = a.k_bits;
  const double gam = static_cast<double>(dim + 2) * 0x1.0p-53 / (1.0 - static_cast<double>(dim + 2) * 0x1.0p-53);
  const double bound_rel = 2.0 * gam * (1.0 + 4.0 * gam);
  const uint64_t row = item >> 32;
  const uint32_t dir = static_cast<uint32_t>(item & 0xffffffffu);
  const double* w = a.w64 + static_cast<uint64_t>(dir) * dim;
  const uint32_t table = dir / K, bpos = K - 1u - dir % K;
  const uint64_t idx = static_cast<uint64_t>(table) * a.ids_ld + row;
  // the deciding lane's other loads issued up front, beside the row loads
  const bool lead = live && gl == 0;
  const double wn = lead ? __ldg(a.wnorm64 + dir) : 0.0;
  const uint32_t id0 = lead ? id_get(a, idx) : 0u;
  double p = 0.0, ab = 0.0, xx = 0.0;
  if (live) {
    // eight elements per lane per round, all sixteen loads issued before any
    // is used (the rows come from HBM: latency bounds this)
    for (uint32_t k0 = 0; k0 < dim; k0 += 8u * kG) {
      double xv[8], wv[8];
#pragma unroll
      for (uint32_t u = 0; u < 8u; ++u) {
        const uint32_t k = min(k0 + u * kG + gl, dim - 1u);
        xv[u] = a.x_f64 ? static_cast<const double*>(a.x)[row * a.ld + k]
                        : static_cast<double>(static_cast<const float*>(a.x)[row * a.ld + k]);
        wv[u] = __ldg(w + k);
      }
#pragma unroll
      for (uint32_t u = 0; u < 8u; ++u)
        if (k0 + u * kG + gl < dim) {
          const double t = xv[u] * wv[u];
          p += t;
          ab += fabs(t);
          xx += xv[u] * xv[u];
        }
    }
  }
#pragma unroll
  for (uint32_t o = kG / 2; o > 0; o >>= 1) {
    p += __shfl_xor_sync(0xffffffffu, p, o);
    ab += __shfl_xor_sync(0xffffffffu, ab, o);
    xx += __shfl_xor_sync(0xffffffffu, xx, o);
  }
  if (!lead) return;
  const double err = bound_rel * ab + 0x1.0p-1000;
  const double lim = 1e-6 * (sqrt(xx) * wn);
  const bool sign_ok = fabs(p) > err;
  const bool near_sure = fabs(p) + err < lim * (1.0 - 1e-9);
  const bool far_sure = fabs(p) - err > lim * (1.0 + 1e-9);
  uint32_t exact = p >= 0.0 ? 1u : 0u;
  bool near = near_sure;
  if (!sign_ok || !(near_sure || far_sure)) {
    double nx = 0.0;
    const double e = exact_proj_nx(w, a.x, a.x_f64, row, a.ld, dim, &nx);
    exact = e >= 0.0 ? 1u : 0u;
    near = near_tie_1e6(e, nx, wn);
  }
  if (((id0 >> bpos) & 1u) != exact) {
    const uint32_t old = id_xor(a, idx, 1u << bpos);
    if (a.fused_insert) {
      uint32_t* ct = a.counters + (static_cast<uint64_t>(table) << K);
      atomicSub(&ct[old], 1u);
      atomicAdd(&ct[old ^ (1u << bpos)], 1u);
    }
    ++ff;
  }
  if (near) ++nt;
  ++rr;
}

// Bucket packing with a compile-time K (KT = 15, 16: the BASELINE shapes):
// 32 tables span exactly KT sign words, so per group of 32 tables the thread
// loads its row's KT words once and cuts every bucket with constant shifts
// (srp.cpp:106-113, bit 0 = MSB); one store per table, coalesced per table.
template <uint32_t KT, class IdT>
__device__ __forceinline__ void pack_row_k(const uint32_t* sg, uint32_t r, uint32_t nwords, uint32_t tables,
                                           IdT* idp, uint64_t ids_ld, bool valid) {
  constexpr uint32_t kMask = (1u << KT) - 1u;
  for (uint32_t g = 0; g * 32u < tables; ++g) {
    uint32_t w[KT + 1];
#pragma unroll
    for (uint32_t i = 0; i <= KT; ++i) w[i] = sg[min(g * KT + i, nwords - 1u) * kRows + r];
    IdT* p = idp + static_cast<uint64_t>(g) * 32u * ids_ld;
    const uint32_t left = tables - g * 32u;
#pragma unroll
    for (uint32_t u = 0; u < 32u; ++u) {
      const uint32_t s = u * KT, i = s >> 5, sh = s & 31u;
      uint32_t b;
      if (sh + KT <= 32u)
        b = (w[i] >> (32u - sh - KT)) & kMask;
      else
        b = __funnelshift_l(w[i + 1], w[i], sh + KT - 32u) & kMask;
      if (valid && u < left) *p = static_cast<IdT>(b);
      p += ids_ld;
    }
  }
}

template <uint32_t KT>
__global__ void __launch_bounds__(kThreads, 1) hash_tc_kernel(const TcArgs a, const __grid_constant__ CUtensorMap tmx) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bar_wfull[kMaxWStages], bar_wempty[kMaxWStages];
  __shared__ __align__(8) uint64_t bar_rawfull, bar_afull[2], bar_aempty[2], bar_thrfull[2], bar_threempty[2];
  __shared__ __align__(8) uint64_t bar_accfull[3], bar_accempty[3], bar_sfull[2], bar_sempty[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ float thr_sm[2][kRows];    // row thresholds per tile parity (converters -> epilogue)
  __shared__ uint32_t lom_sm[2][4];     // K16 steps with a nonzero x lo part, per A buffer / lane quarter
  __shared__ uint32_t seg_n;            // near ties pushed by this CTA

  const uint32_t TW = a.tw, wblk = a.tw * 128u;  // direction tile width, one W block (hi or lo) in bytes
  const TcLayout L = tc_layout(a.dim, TW, a.k_bits * a.tables);
  // 1 KB aligned (SW128 operands); offset from the __shared__ array itself so
  // the compiler keeps the accesses in the shared state space (LDS / STS)
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* Rsm = base;                // raw fp32 tile [n_raw][128 rows][32] (SW128)
  uint32_t* Ssm = reinterpret_cast<uint32_t*>(base + L.raw_bytes);  // sign words [n_sbuf][nwords][128]
  uint8_t* Wsm = base + L.raw_bytes + L.n_sbuf * L.sgn_bytes;      // [n_wst][hi | lo][tw * 128 B]

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t n_tiles = (a.n + kRows - 1) / kRows;
  const uint64_t my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto tile_of = [&](uint64_t it) -> uint64_t { return blockIdx.x + it * gridDim.x; };
  const uint32_t K = a.k_bits;
  const uint32_t R = a.k_bits * a.tables;  // directions, packed densely in tw-column tiles

  if (threadIdx.x == 0) {
    seg_n = 0;
    for (uint32_t s = 0; s < L.n_wst; ++s) {
      mbar_init(&bar_wfull[s], 1);
      mbar_init(&bar_wempty[s], 1);
    }
    mbar_init(&bar_rawfull, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar_afull[b], 4);      // the four converter warps
      mbar_init(&bar_aempty[b], 1);     // MMA commit after the tile's last MMA
      mbar_init(&bar_thrfull[b], 4);
      mbar_init(&bar_threempty[b], 4u * kEpiQ);  // every epilogue warp reads its rows' thresholds
      mbar_init(&bar_sfull[b], 4u * kEpiQ);  // every epilogue warp, once per point tile
      mbar_init(&bar_sempty[b], 4);     // the four packer (converter) warps
    }
    for (int b = 0; b < 3; ++b) {
      mbar_init(&bar_accfull[b], 1);
      mbar_init(&bar_accempty[b], 4u * kEpiQ);  // every epilogue warp reads its group of each direction tile
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, 512);
  if (warp == kConvW && lane == 0) prefetch_tmap(&tmx);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem_base = tmem_base_sh;
  const unsigned long long seg_cap = a.near_cap / gridDim.x;
  unsigned long long* seg = a.near_list + blockIdx.x * seg_cap;
  const uint32_t a_col0 = L.nacc * TW;  // first TMEM column of the A buffers
  uint32_t dbg_sink = 0;
  (void)dbg_sink;
  TCP_DECL;
  const long long t_kernel = clock64();
  (void)t_kernel;

  if (warp == 0) {
    // ---------------- W producer: per tile, per direction tile j, per K chunk ----------------
    if (lane == 0) {
      uint32_t s = 0, ph = 0;
      for (uint64_t it = 0; it < my_tiles; ++it)
        for (uint32_t j = 0; j < a.ntiles; ++j) {
          const uint32_t bytes = ((min(TW, R - j * TW) + 15u) & ~15u) * 128u;  // rows of the MMA's N
          for (uint32_t kc = 0; kc < a.nkc; ++kc) {
            mbar_wait_sleepy(&bar_wempty[s], ph ^ 1u);
            if ((ACE_TC_DBG & 8) && it > 0) {
              mbar_arrive(&bar_wfull[s]);
              if (++s == L.n_wst) {
                s = 0;
                ph ^= 1u;
              }
              continue;
            }
            mbar_expect_tx(&bar_wfull[s], 2u * bytes);
            const uint8_t* src = reinterpret_cast<const uint8_t*>(a.w16) + (static_cast<uint64_t>(j) * a.nkc + kc) * 2u * wblk;
            uint8_t* dst = Wsm + static_cast<size_t>(s) * 2u * wblk;
            bulk_g2s(dst, src, bytes, &bar_wfull[s]);
            bulk_g2s(dst + wblk, src + wblk, bytes, &bar_wfull[s]);
            if (++s == L.n_wst) {
              s = 0;
              ph ^= 1u;
            }
          }
        }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // The whole warp walks the schedule (operands stay warp-uniform); one
    // elected lane issues one burst per direction tile, waiting for each W
    // stage itself so the tensor queue is refilled without gaps.
    uint32_t s = 0, wph = 0, acc = 0, accph = 0;
    const uint32_t w_base = smem_u32(Wsm);
    for (uint64_t it = 0; it < my_tiles; ++it) {
      const uint32_t b = L.n_abuf == 2u ? static_cast<uint32_t>(it & 1u) : 0u;
      const uint32_t use = static_cast<uint32_t>(L.n_abuf == 2u ? (it >> 1) : it);
      TCP_BEGIN();
      mbar_wait(&bar_afull[b], use & 1u);
      TCP_END(0);
      tc_after();
      // lo x hi MMAs of K16 steps whose x lo parts are all zero in this tile
      // are skipped (they would add exact zeros), e.g. one-hot columns
      const uint32_t lm = lom_sm[b][0] | lom_sm[b][1] | lom_sm[b][2] | lom_sm[b][3];
      const uint32_t ta_hi = tmem_base + a_col0 + b * L.acols, ta_lo = ta_hi + L.acols / 2u;
      for (uint32_t j = 0; j < a.ntiles; ++j) {
        const uint32_t idesc = idesc_f16((min(TW, R - j * TW) + 15u) & ~15u);
        TCP_BEGIN();
        mbar_wait(&bar_accempty[acc], accph ^ 1u);
        TCP_END(1);
        tc_after();
        const uint32_t dt = tmem_base + acc * TW;
        if (elect_one()) {
          uint32_t ss = s, ph = wph;
          for (uint32_t kc = 0; kc < a.nkc; ++kc) {
            TCP_BEGIN();
            mbar_wait(&bar_wfull[ss], ph);
            TCP_END(2);
            const uint32_t b_hi = w_base + ss * 2u * wblk;
            const uint64_t dbh = sw128_desc(b_hi), dbl = sw128_desc(b_hi + wblk);
#pragma unroll
            for (uint32_t kk = 0; kk < 4; ++kk) {
              const uint32_t step = kc * 4u + kk;
              if (step >= L.nsteps) break;
              const uint32_t acol = step * 8u;  // 16 fp16 = 8 TMEM columns
              const uint64_t off = kk * 2u;     // 32 B along K in SW128, >> 4
              if (ACE_TC_DBG & 2) continue;
              mma_f16_ts(dt, ta_hi + acol, dbh + off, idesc, step != 0u);
              if ((lm >> step) & 1u) mma_f16_ts(dt, ta_lo + acol, dbh + off, idesc, 1u);
              mma_f16_ts(dt, ta_hi + acol, dbl + off, idesc, 1u);
            }
            mma_commit(&bar_wempty[ss]);
            if (++ss == L.n_wst) {
              ss = 0;
              ph ^= 1u;
            }
          }
          mma_commit(&bar_accfull[acc]);
        }
        __syncwarp();
        for (uint32_t kc = 0; kc < a.nkc; ++kc)
          if (++s == L.n_wst) {
            s = 0;
            wph ^= 1u;
          }
        if (++acc == L.nacc) {
          acc = 0;
          accph ^= 1u;
        }
      }
      // the A buffer is free once this tile's MMAs have completed
      if (elect_one()) mma_commit(&bar_aempty[b]);
      __syncwarp();
    }
#if ACE_TC_PROF
    tcp[3] += static_cast<unsigned long long>(clock64() - t_kernel);
#endif
    TCP_FLUSH(lane == 0);
  } else if (warp >= kConvW) {
    // ---------------- converters (the last four warps): raw fp32 tile -> TMEM A operand ----------------
    // and, one tile behind, the bucket packers: each thread cuts its row's L
    // bucket ids (MSB-first bit fields of the sign-word stream, srp.cpp:106-113)
    // from the shared sign words and stores them (coalesced per table).
    const uint32_t q = warp & 3u, r = q * 32u + lane;
    const uint32_t sw = r & 7u;  // SW128: 16-byte unit u of row r sits at unit u ^ (r & 7)
    const uint64_t pol = policy_evict_first();
    const uint32_t kmask = (K >= 32u) ? 0xffffffffu : ((1u << K) - 1u);
    auto issue_raw = [&](uint64_t t) {
      mbar_expect_tx(&bar_rawfull, L.n_raw * kRawBox);
      for (uint32_t c = 0; c < L.n_raw; ++c)
        tma_load_2d(Rsm + c * kRawBox, &tmx, static_cast<int32_t>(32u * c), static_cast<int32_t>(t * kRows),
                    &bar_rawfull, pol);
    };
    auto pack = [&](uint64_t itp) {
      const uint32_t sb = L.n_sbuf == 2u ? static_cast<uint32_t>(itp & 1u) : 0u;
      const uint32_t suse = static_cast<uint32_t>(L.n_sbuf == 2u ? (itp >> 1) : itp);
      TCP_BEGIN();
      mbar_wait_sleepy(&bar_sfull[sb], suse & 1u);
      TCP_END(15);
      TCP_BEGIN();
      const uint32_t* sg = Ssm + static_cast<size_t>(sb) * (L.sgn_bytes / 4u);
      const uint64_t row = tile_of(itp) * kRows + r;
      const bool valid = row < a.n;
      if constexpr (ACE_TC_DBG & 4) {
      } else if constexpr (KT != 0) {
        if (a.ids16)
          pack_row_k<KT>(sg, r, L.nwords, a.tables, reinterpret_cast<unsigned short*>(a.ids) + row, a.ids_ld, valid);
        else
          pack_row_k<KT>(sg, r, L.nwords, a.tables, a.ids + row, a.ids_ld, valid);
      } else {
      // eight tables at a time: all sixteen word loads in flight first (a
      // table needs the next word only if it straddles, which then exists)
      for (uint32_t t0 = 0; t0 < a.tables; t0 += 8u) {
        uint32_t bk[8];
#pragma unroll
        for (uint32_t u = 0; u < 8u; ++u) {
          const uint32_t s0 = min(t0 + u, a.tables - 1u) * K, wi = s0 >> 5;
          const uint32_t hi = sg[wi * kRows + r], lo = sg[min(wi + 1u, L.nwords - 1u) * kRows + r];
          const unsigned long long win = (static_cast<unsigned long long>(hi) << 32) | lo;
          bk[u] = static_cast<uint32_t>(win >> (64u - (s0 & 31u) - K)) & kmask;
        }
#pragma unroll
        for (uint32_t u = 0; u < 8u; ++u) {
          const uint32_t tt = t0 + u;
          if (valid && tt < a.tables) id_put(a, static_cast<uint64_t>(tt) * a.ids_ld + row, bk[u]);
          if (a.fused_insert && tt < a.tables)
            insert_bucket_warp(a.counters + (static_cast<uint64_t>(tt) << K), bk[u], valid, lane);
        }
      }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_sempty[sb]);
      TCP_END(14);
    };
    if (warp == kConvW && lane == 0 && my_tiles > 0) issue_raw(tile_of(0));
    const uint32_t lane_base = (q * 32u) << 16;
    for (uint64_t it = 0; it < my_tiles; ++it) {
      const uint64_t t = tile_of(it);
      const uint32_t p = static_cast<uint32_t>(it & 1u);
      const uint32_t b = L.n_abuf == 2u ? p : 0u;
      const uint32_t use = static_cast<uint32_t>(L.n_abuf == 2u ? (it >> 1) : it);
      const bool live = t * kRows + r < a.n;
      TCP_BEGIN();
      mbar_wait_sleepy(&bar_rawfull, static_cast<uint32_t>(it & 1u));
      TCP_END(5);
      TCP_BEGIN();
      // pass 1: max |x| of the row (magnitude bits: NaN > inf > finite)
      uint32_t mb = 0u;
      for (uint32_t c = 0; c < L.n_raw; ++c) {
        const float4* rowp = reinterpret_cast<const float4*>(Rsm + c * kRawBox + r * 128u);
#pragma unroll
        for (uint32_t u = 0; u < 8; ++u) {
          const float4 v = rowp[u ^ sw];
          mb = max(mb, max(max(__float_as_uint(v.x) & 0x7fffffffu, __float_as_uint(v.y) & 0x7fffffffu),
                           max(__float_as_uint(v.z) & 0x7fffffffu, __float_as_uint(v.w) & 0x7fffffffu)));
        }
      }
      const RowScale rs = row_scale(mb, live);
      TCP_END(6);
      TCP_BEGIN();
      mbar_wait_sleepy(&bar_aempty[b], (use & 1u) ^ 1u);
      mbar_wait_sleepy(&bar_threempty[p], (static_cast<uint32_t>(it >> 1) & 1u) ^ 1u);
      TCP_END(7);
      TCP_BEGIN();
      tc_after();
      // pass 2: per K16 step, 16 values -> fp16 hi / lo (packed conversions)
      // -> 8 + 8 TMEM columns
      const uint32_t ta_hi = tmem_base + lane_base + a_col0 + b * L.acols, ta_lo = ta_hi + L.acols / 2u;
      float ss = 0.0f;
      uint32_t lob = 0u;
      for (uint32_t st = 0; st < L.nsteps; ++st) {
        const float4* rowp = reinterpret_cast<const float4*>(Rsm + (st >> 1) * kRawBox + r * 128u);
        const uint32_t u0 = (st & 1u) * 4u;
        float v[16];
#pragma unroll
        for (uint32_t u = 0; u < 4; ++u) {
          const float4 f = rowp[(u0 + u) ^ sw];
          v[4 * u] = f.x;
          v[4 * u + 1] = f.y;
          v[4 * u + 2] = f.z;
          v[4 * u + 3] = f.w;
        }
        uint32_t hw[8], lw[8];
        uint32_t lor = 0u;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float x0 = v[2 * i] * rs.scale, x1 = v[2 * i + 1] * rs.scale;
          ss = fmaf(x0, x0, fmaf(x1, x1, ss));
          const __half2 hh = __floats2half2_rn(x0, x1);  // low half: x0
          const float2 hf = __half22float2(hh);
          const __half2 ll = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
          hw[i] = *reinterpret_cast<const uint32_t*>(&hh);
          lw[i] = *reinterpret_cast<const uint32_t*>(&ll);
          lor |= lw[i];
        }
        if (lor != 0u) lob |= 1u << st;
        tmem_st8(ta_hi + st * 8u, hw);
        tmem_st8(ta_lo + st * 8u, lw);
      }
      TCP_END(8);
      TCP_BEGIN();
      // every converter has read the raw tile: warp kConvW loads the next one
      asm volatile("bar.sync %0, 128;" ::"r"(kConvBar) : "memory");
      if (warp == kConvW && lane == 0 && it + 1 < my_tiles) issue_raw(tile_of(it + 1));
      thr_sm[p][r] = row_threshold(rs, live, ss, a.dim, a.margin_c);
      lob = __reduce_or_sync(0xffffffffu, lob);
      if (lane == 0) lom_sm[b][q] = lob;
      tmem_wait_st();
      tc_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&bar_afull[b]);
        mbar_arrive(&bar_thrfull[p]);
      }
      TCP_END(9);
      if (it > 0) pack(it - 1);
    }
    if (my_tiles > 0) pack(my_tiles - 1);
    TCP_FLUSH(warp == kConvW && lane == 0);
  } else {
    // ---------------- epilogue (warps 2 .. 2 + 4 kEpiQ - 1) ----------------
    // kEpiQ = 4 warps per TMEM lane quarter (q = warp % 4, e = (warp - 2) / 4):
    // warp e reads 32-column group e of every 128-direction tile, i.e. sign
    // word G = 4 j + e.  Per group: sign bits packed MSB-first (one funnel
    // shift per column, four chains) and near ties by one float min over |v|.
    // The sign words go to shared memory (sgn[word][row]), where the
    // converter warps cut the buckets.
    const uint32_t q = warp & 3, e = (warp - 2) >> 2;
    const uint32_t r = q * 32u + lane;
    uint32_t acc = 0, accph = 0;
    for (uint64_t it = 0; it < my_tiles; ++it) {
      const uint64_t t = tile_of(it);
      const uint64_t row = t * kRows + r;
      const bool valid = row < a.n;
      const uint32_t p = static_cast<uint32_t>(it & 1u);
      const uint32_t sb = L.n_sbuf == 2u ? p : 0u;
      const uint32_t suse = static_cast<uint32_t>(L.n_sbuf == 2u ? (it >> 1) : it);
      TCP_BEGIN();
      mbar_wait_sleepy(&bar_thrfull[p], static_cast<uint32_t>(it >> 1) & 1u);
      const float thr = valid ? thr_sm[p][r] : -1.0f;
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_threempty[p]);
      mbar_wait_sleepy(&bar_sempty[sb], (suse & 1u) ^ 1u);  // the packers are done with this buffer
      TCP_END(10);
      uint32_t* sg = Ssm + static_cast<size_t>(sb) * (L.sgn_bytes / 4u);
      const bool zero_row = thr < 0.0f;
      const bool live = !zero_row && valid;
      const uint32_t thr_u = zero_row ? 0u : (isinf(thr) ? 0xffffffffu : (__float_as_uint(thr) << 1));
      for (uint32_t j = 0; j < a.ntiles; ++j) {
        const uint32_t gw = 4u * j + e;  // this warp's sign word (directions 32 gw ..)
        TCP_BEGIN();
        mbar_wait_sleepy(&bar_accfull[acc], accph);
        TCP_END(11);
        TCP_BEGIN();
        tc_after();
        uint32_t v[32];
        ACE_TMEM_LD32(tmem_base + ((q * 32u) << 16) + acc * TW + 32u * e, v);
        tmem_wait_ld();
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_accempty[acc]);  // read: the MMAs may reuse it
        if (!(ACE_TC_DBG & 1) && gw < L.nwords) {
          // near-tie test on |v| as a float min (FMNMX with |.| operands);
          // NaN (non-finite rows, thr = inf) fails `mn > thr`
          uint32_t n4[4] = {0u, 0u, 0u, 0u};
          float m4[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
#pragma unroll
          for (int jj = 0; jj < 8; ++jj)
#pragma unroll
            for (int gq = 0; gq < 4; ++gq) {
              n4[gq] = (n4[gq] << 1) | (v[gq * 8 + jj] >> 31);
              m4[gq] = fminf(m4[gq], fabsf(__uint_as_float(v[gq * 8 + jj])));
            }
          const float mn = fminf(fminf(m4[0], m4[1]), fminf(m4[2], m4[3]));
          // bit (31-jj) = direction 32 gw + jj >= 0
          sg[gw * kRows + r] = zero_row ? 0xffffffffu : ~((n4[0] << 24) | (n4[1] << 16) | (n4[2] << 8) | n4[3]);
          TCP_END(12);
          TCP_BEGIN();
          // columns past R (padding / stale) are masked here, off the hot path
          if (live && !(mn > thr)) {
            const uint32_t ncol = min(32u, R - 32u * gw);
            // only the 8-column chains whose min is inside the bound
            uint32_t nm = 0u;
#pragma unroll
            for (int gq = 0; gq < 4; ++gq)
              if (!(m4[gq] > thr)) {
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) nm |= (((v[gq * 8 + jj] << 1) <= thr_u) ? 1u : 0u) << (gq * 8 + jj);
              }
            if (ncol < 32u) nm &= (1u << ncol) - 1u;
            if (ACE_TC_DBG & 128) {
              dbg_sink += __popc(nm);
            } else if (nm && !(ACE_TC_DBG & 64)) {
              push_near_mask(a.st, seg, seg_cap, &seg_n, a.overflow_rows, nm, row, 32u * gw);
            }
          }
          TCP_END(13);
        }
        if (++acc == L.nacc) {
          acc = 0;
          accph ^= 1u;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_sfull[sb]);
    }
  }

  TCP_FLUSH(warp == 2 && lane == 0);
  // the listed near ties are decided by recheck_near_kernel (next launch,
  // every SM): publish this CTA's list length
  __syncthreads();
  if (threadIdx.x == 0) {
    a.seg_counts[blockIdx.x] = static_cast<uint32_t>(min(static_cast<unsigned long long>(seg_n), seg_cap));
    if (seg_n) atomicAdd(&a.st->near_count, static_cast<unsigned long long>(seg_n));
    if (a.fused_insert && blockIdx.x == 0) atomicAdd(&a.st->n, a.n);
  }
#if ACE_TC_PROF
  if (threadIdx.x == 0) atomicAdd(&g_tc_prof[16], static_cast<unsigned long long>(clock64() - t_kernel));
#endif
  tc_before();
  __syncthreads();
  tc_after();
  if (warp == 1) tmem_dealloc(tmem_base, 512);
}

// Rows that cannot be read by the tensor map directly (fp64 input, stride
// or base not 16-byte aligned): staged as fp32 rows of stride dpad4.
__global__ void stage_f32_kernel(const void* __restrict__ x, int x_f64, uint64_t n, uint64_t ld, uint64_t dim,
                                 uint64_t ld_out, float* __restrict__ out) {
  const uint64_t total = n * ld_out;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t row = i / ld_out, k = i % ld_out;
    float v = 0.0f;
    if (k < dim)
      v = x_f64 ? static_cast<float>(static_cast<const double*>(x)[row * ld + k])
                : static_cast<const float*>(x)[row * ld + k];
    out[i] = v;
  }
}

// The near ties listed by hash_tc_kernel, decided exactly (recheck_item): kG
// lanes per item, blocks dealt over the kernel's list segments (several
// blocks per segment).  Items of rows whose list overflowed are left to the
// second part, which recomputes every bucket of those rows exactly.  Slots
// are reset to ~0 (the list is all ~0 between launches).
__global__ void __launch_bounds__(256) recheck_near_kernel(const TcArgs a, uint32_t nseg) {
  const uint32_t gl = threadIdx.x % kG, grp = threadIdx.x / kG, ngb = blockDim.x / kG;
  const uint32_t P = gridDim.x / nseg;  // blocks per segment
  const uint32_t b = blockIdx.x % nseg, sub = blockIdx.x / nseg;
  const unsigned long long seg_cap = a.near_cap / nseg;
  unsigned long long* seg = a.near_list + b * seg_cap;
  const uint32_t cnt = sub < P ? a.seg_counts[b] : 0u;
  const bool ovf = a.st->near_overflow != 0;
  unsigned long long rr = 0, ff = 0, nt = 0;
  const uint32_t per = P * ngb, rounds = (cnt + per - 1) / per;  // block-uniform (shuffles)
  for (uint32_t rd = 0; rd < rounds; ++rd) {
    const uint32_t i = rd * per + sub * ngb + grp;
    bool live = i < cnt;
    const unsigned long long item = live ? seg[i] : 0ull;
    if (live && ovf) {
      const uint64_t row = item >> 32;
      if ((a.overflow_rows[row >> 5] >> (row & 31)) & 1u) live = false;  // whole row below
    }
    recheck_item(a, item, live, gl, rr, ff, nt);
    if (i < cnt && gl == 0) seg[i] = ~0ull;
  }
  if (ovf) {
    // rows whose near ties overflowed the list: every bucket recomputed exactly
    const uint32_t K = a.k_bits;
    for (uint64_t idx = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < a.n * a.tables;
         idx += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
      const uint64_t row = idx / a.tables;
      const uint32_t table = static_cast<uint32_t>(idx % a.tables);
      if (!((a.overflow_rows[row >> 5] >> (row & 31)) & 1u)) continue;
      uint32_t bucket = 0;
      for (uint32_t bb = 0; bb < K; ++bb) {
        const uint32_t dir = table * K + bb;
        double nx = 0.0;
        const double p = exact_proj_nx(a.w64 + static_cast<uint64_t>(dir) * a.dim, a.x, a.x_f64, row, a.ld, a.dim, &nx);
        bucket = (bucket << 1) | (p >= 0.0 ? 1u : 0u);
        if (near_tie_1e6(p, nx, a.wnorm64[dir])) ++nt;
      }
      const uint64_t ix = static_cast<uint64_t>(table) * a.ids_ld + row;
      const uint32_t old = id_get(a, ix);
      id_put(a, ix, bucket);
      if (a.fused_insert && old != bucket) {
        uint32_t* ct = a.counters + (static_cast<uint64_t>(table) << K);
        atomicSub(&ct[old], 1u);
        atomicAdd(&ct[bucket], 1u);
      }
      rr += K;
    }
  }
  rr = warp_sum_u64(rr);
  ff = warp_sum_u64(ff);
  nt = warp_sum_u64(nt);
  if ((threadIdx.x & 31u) == 0) {
    if (rr) atomicAdd(&a.st->rechecked, rr);
    if (ff) atomicAdd(&a.st->flipped, ff);
    if (nt) atomicAdd(&a.st->near_ties, nt);
  }
  if (ovf) {
    // the last block to finish clears the overflow bitmap and flag, so the
    // next projection launch starts clean without a memset
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(&a.st->ticket_r, 1u) == gridDim.x - 1u;
    }
    __syncthreads();
    if (last) {
      for (uint64_t wd = threadIdx.x; wd < (a.n + 31) / 32; wd += blockDim.x) a.overflow_rows[wd] = 0u;
      if (threadIdx.x == 0) {
        a.st->near_overflow = 0;
        a.st->ticket_r = 0u;
      }
    }
  }
}

// rows whose near ties overflowed the list (the K-streamed path, after its
// own segment recheck): every bucket recomputed exactly
__global__ void recheck_rows_kernel(const TcArgs a) {
  if (!a.st->near_overflow) return;
  const uint32_t K = a.k_bits;
  unsigned long long nt = 0;
  for (uint64_t idx = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < a.n * a.tables;
       idx += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t row = idx / a.tables;
    const uint32_t table = static_cast<uint32_t>(idx % a.tables);
    if (!((a.overflow_rows[row >> 5] >> (row & 31)) & 1u)) continue;
    uint32_t bucket = 0;
    for (uint32_t b = 0; b < K; ++b) {
      const uint32_t dir = table * K + b;
      double nx = 0.0;
      const double p = exact_proj_nx(a.w64 + static_cast<uint64_t>(dir) * a.dim, a.x, a.x_f64, row, a.ld, a.dim, &nx);
      bucket = (bucket << 1) | (p >= 0.0 ? 1u : 0u);
      if (near_tie_1e6(p, nx, a.wnorm64[dir])) ++nt;
    }
    const uint64_t ix = static_cast<uint64_t>(table) * a.ids_ld + row;
    const uint32_t old = id_get(a, ix);
    id_put(a, ix, bucket);
    if (a.fused_insert && old != bucket) {
      uint32_t* ct = a.counters + (static_cast<uint64_t>(table) << K);
      atomicSub(&ct[old], 1u);
      atomicAdd(&ct[bucket], 1u);
    }
    atomicAdd(&a.st->rechecked, static_cast<unsigned long long>(K));
  }
  if (nt) atomicAdd(&a.st->near_ties, nt);
}

// ---- W preparation ------------------------------------------------------------------

// 2^14 / ||w|| per direction: W rows normalised for the fp16 split.
__global__ void dir_norm_kernel(const double* __restrict__ w64, uint64_t dim, uint32_t rows, double* inv) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double s = 0.0;
  for (uint64_t i = 0; i < dim; ++i) s = __dadd_rn(s, __dmul_rn(w64[r * dim + i], w64[r * dim + i]));
  inv[r] = s > 0.0 ? 16384.0 / sqrt(s) : 0.0;
}

// Direction tile j holds directions j*dpt .. j*dpt + dpt - 1 in rows 0..dpt-1
// (dpt = tw: packed densely; dpt = tables-per-tile * K: whole tables per tile,
// the K-streamed kernel), zero rows beyond.
__global__ void pack_w16_kernel(const double* __restrict__ w64, const double* __restrict__ inv, FamilyDev f,
                                uint32_t ntiles, uint32_t nkc, uint32_t tw, uint32_t dpt, uint16_t* w16) {
  const uint64_t total = static_cast<uint64_t>(ntiles) * tw * nkc * kChunk;
  const uint32_t wblk = tw * 128u;
  for (uint64_t idx = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t k = idx % (nkc * kChunk);
    const uint32_t rr = (idx / (nkc * kChunk)) % tw;
    const uint32_t j = static_cast<uint32_t>(idx / (static_cast<uint64_t>(nkc) * kChunk * tw));
    const uint32_t kc = k / kChunk, kk = k % kChunk;
    const uint64_t dir = static_cast<uint64_t>(j) * dpt + rr;
    double w = 0.0;
    if (rr < dpt && dir < f.rows && k < f.dim) w = w64[dir * f.dim + k] * inv[dir];
    const __half hi = __double2half(w);
    const __half lo = __double2half(w - static_cast<double>(__half2float(hi)));
    uint8_t* blk = reinterpret_cast<uint8_t*>(w16) + ((static_cast<uint64_t>(j) * nkc + kc) * 2) * wblk;
    const uint32_t off = rr * 128u + ((((kk >> 3) ^ (rr & 7u)) & 7u) << 4) + ((kk & 7u) << 1);
    *reinterpret_cast<__half*>(blk + off) = hi;
    *reinterpret_cast<__half*>(blk + wblk + off) = lo;
  }
}

__global__ void w32_round_kernel(const double* __restrict__ w64, uint64_t n, float* __restrict__ w32) {
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    w32[i] = static_cast<float>(w64[i]);
}

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

uint64_t dpad4(uint64_t dim) { return (dim + 3) / 4 * 4; }

}  // namespace

int tc_sms() {
  // per device ordinal (a process may drive several GPUs)
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!sms[dev]) cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
  return sms[dev];
}

bool tc_supported(uint64_t dim) { return dim >= 1 && dim <= 8192; }

bool tc_direct_ok(const void* x, int x_f64, uint64_t ld) {
  return !x_f64 && (ld % 4) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
}

size_t tc_stage_bytes(uint64_t n, uint64_t dim) { return static_cast<size_t>(n) * dpad4(dim) * sizeof(float); }

float tc_margin(uint32_t nkc, bool x_f64) {
  // error bound of the fp16x3 split relative to ||x~|| ||w^||:
  // split residuals and the dropped lo x lo term, fp32 accumulation
  // (truncation assumed) per K step, fp64 input rounded to fp32; doubled
  return static_cast<float>(2.0 * (4.0 * 0x1.0p-22 + 0x1.0p-23 * (12.0 * nkc + 16.0) * 1.01 + (x_f64 ? 0x1.0p-23 : 0.0)));
}

cudaError_t tc_prepare_family(const FamilyDev& f, TcFamily* tc) {
  tc->enabled = 0;
  if (!tc_supported(f.dim) || f.k_bits > 128 || !tmap_encoder()) return cudaSuccess;
  const uint32_t nkc = static_cast<uint32_t>((f.dim + kChunk - 1) / kChunk);
  const bool ks = tc_kstream(nkc);
  // 192-direction tiles where two accumulators and two A buffers fit TMEM
  // (d <= 64), else 128; the K-streamed kernel: 256 (whole tables per tile)
  const uint32_t tw = ks ? 256u : 128u;  // the d <= 256 kernel's epilogue reads 4 x 32 columns per tile
  if (!ks && tc_layout(f.dim, tw, f.rows).n_wst < 2) return cudaSuccess;
  tc->nkc = nkc;
  tc->tw = tw;
  const uint32_t tpt = tw / f.k_bits;
  if (ks) {
    if (tpt == 0) return cudaSuccess;
    tc->tpt = tpt;
  }
  const uint32_t dpt = ks ? tpt * f.k_bits : tw;
  tc->ntiles = ks ? (f.tables + tpt - 1) / tpt : (f.rows + tw - 1) / tw;
  const size_t bytes = static_cast<size_t>(tc->ntiles) * nkc * 2 * tw * 128u;
  cudaError_t e = cudaMalloc(&tc->w16, bytes);
  if (e != cudaSuccess) return e;
  double* inv = nullptr;
  if ((e = cudaMalloc(&inv, sizeof(double) * f.rows)) != cudaSuccess) return e;
  dir_norm_kernel<<<(f.rows + 127) / 128, 128>>>(f.w64, f.dim, f.rows, inv);
  pack_w16_kernel<<<1024, 256>>>(f.w64, inv, f, tc->ntiles, nkc, tw, dpt, tc->w16);
  count_launch(2);
  e = cudaDeviceSynchronize();
  cudaFree(inv);
  if (e != cudaSuccess) return e;
  if (ks) {
    if ((e = cudaMalloc(&tc->w32, sizeof(float) * f.rows * f.dim)) != cudaSuccess) return e;
    w32_round_kernel<<<1024, 256>>>(f.w64, static_cast<uint64_t>(f.rows) * f.dim, tc->w32);
    count_launch();
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return e;
    if ((e = tck_prepare(tw)) != cudaSuccess) return e;
  } else {
    // every layout stays within kSmemLimit - 8192 (tc_layout)
    for (const void* fn : {reinterpret_cast<const void*>(hash_tc_kernel<0>), reinterpret_cast<const void*>(hash_tc_kernel<15>),
                           reinterpret_cast<const void*>(hash_tc_kernel<16>)})
      if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSmemLimit - 8192))) != cudaSuccess)
        return e;
  }
  tc->enabled = 1;
  return cudaSuccess;
}

void tc_free_family(TcFamily* tc) {
  cudaFree(tc->w16);
  cudaFree(tc->w32);
  tc->w16 = nullptr;
  tc->w32 = nullptr;
  tc->enabled = 0;
}

cudaError_t launch_hash_tc(const TcArgs& a, void* stage, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  const void* src = a.x;
  uint64_t ld = a.ld;
  if (!tc_direct_ok(a.x, a.x_f64, a.ld)) {
    ld = dpad4(a.dim);
    const uint64_t total = a.n * ld;
    const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, 148ull * 16));
    stage_f32_kernel<<<blocks, 256, 0, s>>>(a.x, a.x_f64, a.n, a.ld, a.dim, ld, static_cast<float*>(stage));
    count_launch();
    src = stage;
  }
  CUtensorMap map;
  const cuuint64_t gdim[2] = {a.dim, a.n};
  const cuuint64_t gstride[1] = {ld * sizeof(float)};
  const cuuint32_t box[2] = {32u, static_cast<cuuint32_t>(kRows)};
  const cuuint32_t es[2] = {1u, 1u};
  const CUresult r = tmap_encoder()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(src), gdim, gstride,
                                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  const uint64_t grid = tc_grid(a.n, a.grid_cap);
  const size_t smem = tc_layout(a.dim, a.tw, a.k_bits * a.tables).total;
  // compile-time K packers for the BASELINE shapes (never with the fused insert, K > 20)
  if (a.k_bits == 15 && !a.fused_insert)
    hash_tc_kernel<15><<<static_cast<unsigned>(grid), kThreads, smem, s>>>(a, map);
  else if (a.k_bits == 16 && !a.fused_insert)
    hash_tc_kernel<16><<<static_cast<unsigned>(grid), kThreads, smem, s>>>(a, map);
  else
    hash_tc_kernel<0><<<static_cast<unsigned>(grid), kThreads, smem, s>>>(a, map);
  count_launch();
  return cudaGetLastError();
}

#if ACE_TC_PROF
extern "C" int ace_debug_tc_prof(unsigned long long* out24, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out24, g_tc_prof, sizeof(unsigned long long) * 24) != cudaSuccess) return -1;
  if (reset) {
    unsigned long long z[24] = {0};
    cudaMemcpyToSymbol(g_tc_prof, z, sizeof(z));
  }
  return 0;
}
#endif

uint32_t tc_grid(uint64_t n, uint32_t cap) {
  const uint64_t sms = cap ? std::min<uint64_t>(cap, static_cast<uint64_t>(tc_sms())) : static_cast<uint64_t>(tc_sms());
  return static_cast<uint32_t>(std::min<uint64_t>((n + kRows - 1) / kRows, sms));
}

cudaError_t launch_recheck_near(const TcArgs& a, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  const uint32_t nseg = tc_grid(a.n, a.grid_cap);
  // eight blocks (256 items) per list segment: one round for the BASELINE
  // shapes' ~40-260 items per segment
  const uint32_t per = std::max<uint32_t>(1u, (8u * static_cast<uint32_t>(tc_sms()) + nseg - 1u) / nseg);
  recheck_near_kernel<<<nseg * per, 256, 0, s>>>(a, nseg);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_recheck(const TcArgs& a, cudaStream_t s) {
  recheck_rows_kernel<<<148, 256, 0, s>>>(a);  // exits at once unless a list segment overflowed
  count_launch(1);
  return cudaGetLastError();
}

}  // namespace ace_dev
