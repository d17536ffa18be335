// tcgen05 projection kernel for sm_100a: the SRP hash of a 128-point tile
// against every direction, on the 5th-generation tensor cores.
//
// P = X W^T computed as an error-compensated fp16 split,
//   x~ = x * 2^s(row) = x_hi + x_lo,   w^ = w * 2^14/||w|| = w_hi + w_lo,
//   P~ = x_hi w_hi + x_lo w_hi + x_hi w_lo     (three tcgen05.mma per K-step),
// accumulated in fp32 in TMEM.  Signs are scale invariant, so sign(P~) equals
// the reference's sign(p) (srp.cpp:78-104) whenever |P~| exceeds the rigorous
// error bound thr(row) = c * ||x~|| * 2^14 + abs; projections inside the bound
// go to a near-tie list and are recomputed as the reference's binary64 fold
// (recheck kernel).  Buckets are packed MSB-first (srp.cpp:106-113) straight
// from the accumulator columns: one thread owns one point (TMEM lane).
//
// Warp roles (384 threads, one CTA per SM, persistent over point tiles):
//   warp 0      producer: cp.async.bulk (TMA engine) of the point tile's A
//               image (fp16 hi | lo, written by convert_x_kernel) and a ring
//               of pre-swizzled W stages
//   warp 1      TMEM allocator; copies A into TMEM (tcgen05.cp) and issues the
//               TS MMAs from one elected lane, one burst per direction tile
//   warps 2-9   epilogue: two warps per TMEM lane quarter on alternate
//               direction tiles; tcgen05.ld -> sign words, near ties, buckets
//   warps 10-11 exact recheck of near ties while the main loop runs; leftovers
//               go to a shared tail after it
// Pipelines (mbarriers): W stages full/empty, A full/empty, two TMEM
// accumulators (192 columns for d <= 128, else 128) full/empty.
// hash_tck_kernel (further down) is the K-streamed variant for d > 256.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "ace_tc.cuh"

namespace ace_dev {

namespace {

constexpr int kRows = 128;                 // points per tile (MMA M)
constexpr int kChunk = 64;                 // K elements per chunk (128 B of fp16)
constexpr int kBlockBytes = kRows * 128;   // one 128 x 64 fp16 block = 16 KB
constexpr int kAccBufs = 3;                // max TMEM accumulators (x 128 columns)
constexpr int kMaxWStages = 12;
#ifndef ACE_TESTWAIT
#define ACE_TESTWAIT 0
#endif
#ifndef ACE_WATCHDOG
#define ACE_WATCHDOG 0
#endif
#ifndef ACE_SLEEPY
#define ACE_SLEEPY 64  // ns back-off of off-critical-path barrier waits (0: spin)
#endif
#ifndef ACE_SPLIT
// epilogue: 1 = both warps of a lane quarter on every direction tile (halves
// of its columns; measured slower: the halves' TMEM loads and barriers cost
// more than the earlier accumulator release gains), 0 = alternate tiles
#define ACE_SPLIT 0
#endif
#ifndef ACE_TILE_BURST
#define ACE_TILE_BURST 0  // MMA issuer: 1 = one elected burst per point tile (measured slower), 0 = per direction tile
#endif
#ifndef ACE_KC_FENCE
#define ACE_KC_FENCE 0
#endif
#ifndef ACE_RW
#define ACE_RW 1  // recheck warps: 0 none (tail only), 1 recheck warps during the main loop
#endif
constexpr int kThreads = ACE_RW ? 384 : 320;  // producer, MMA, 8 epilogue warps, 2 recheck warps
constexpr uint32_t kTail = ACE_RW ? 320 : 256;  // epilogue + recheck threads
constexpr size_t kSmemLimit = 232448;      // 227 KB per CTA
#ifndef ACE_PAIR
#define ACE_PAIR 1
#endif
// CTA pair (cta_group::2): the two CTAs of a cluster run M = 256 MMAs issued
// by the leader; each holds its own 128 points (A, accumulators) and half of
// every W tile (64 directions), so MMA instructions and W bytes per point halve.
constexpr uint32_t kPair = ACE_PAIR;
constexpr uint32_t kCluster = kPair;

struct TcLayout {
  uint32_t nkc, n_abuf, n_wst;
  size_t a_bytes, raw_bytes, w_bytes, total;
};

// Shared memory: one A tile (x, fp16 hi | lo, SW128 image; released as soon as
// tcgen05.cp has moved it into TMEM), with the fused conversion a raw fp32 X
// tile (128 rows, bulk-copied), then a ring of W stages (32 KB each).  TMEM:
// accumulators of 128 columns, then the A operand (hi | lo, dpad columns).
__host__ __device__ inline uint32_t tc_acc_bufs(uint32_t nkc, uint32_t tw = 128) {
  return tw > 128 ? 2u : (nkc <= 2 ? 3u : 2u);
}

__host__ __device__ inline TcLayout tc_layout(uint32_t nkc, uint64_t dim = 0, bool fuse = false, uint32_t tw = 128) {
  TcLayout L;
  L.nkc = nkc;
  L.n_abuf = 1;
  L.a_bytes = static_cast<size_t>(L.n_abuf) * nkc * 2 * kBlockBytes;
  L.raw_bytes = fuse ? (static_cast<size_t>(kRows) * dim * 4 + 1023) / 1024 * 1024 : 0;
  const size_t room = kSmemLimit - 8192 - 1024 - L.a_bytes - L.raw_bytes;  // static smem + align
  const size_t stage = 2u * tw * 128u / kPair;  // a stage: hi + lo of this CTA's share of a W tile
  size_t st = room / stage;
  if (st > kMaxWStages) st = kMaxWStages;
  L.n_wst = static_cast<uint32_t>(st);
  L.w_bytes = static_cast<size_t>(L.n_wst) * stage;
  L.total = L.a_bytes + L.raw_bytes + L.w_bytes + 1024;
  return L;
}

// ---- PTX wrappers --------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity);
// Spin until the phase with `parity` completes.  With ACE_WATCHDOG a wait
// longer than ~2^34 cycles (several seconds, a broken protocol) traps instead
// of hanging the GPU (development builds).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if ACE_WATCHDOG
  if (mbar_try(bar, parity)) return;
  const long long t0 = clock64();
  uint32_t n = 0;
  while (!mbar_try(bar, parity))
    if ((++n & 1023u) == 0 && clock64() - t0 > (1ll << 34)) __trap();
#elif ACE_TESTWAIT
  // non-suspending poll: the waiter sees the phase flip without a wake-up delay
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#else
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#endif
}
// Wait for warps off the critical MMA path: back off between polls so the
// polling does not compete with the tensor pipe for shared memory.
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleepy(uint64_t* bar, uint32_t parity, unsigned long long* acc) {
#if ACE_SLEEPY
  const long long t0 = (acc || ACE_WATCHDOG) ? clock64() : 0;
  uint32_t n = 0;
  while (!mbar_try(bar, parity)) {
    __nanosleep(ACE_SLEEPY);
    if (ACE_WATCHDOG && (++n & 255u) == 0 && clock64() - t0 > (1ll << 34)) __trap();
  }
  if (acc) *acc += static_cast<unsigned long long>(clock64() - t0);
#else
  if (acc) {
    const long long t0 = clock64();
    mbar_wait(bar, parity);
    *acc += static_cast<unsigned long long>(clock64() - t0);
  } else {
    mbar_wait(bar, parity);
  }
#endif
}
// mbar_wait that adds the cycles spent waiting to *acc (instrumentation)
__device__ __forceinline__ void mbar_wait_t(uint64_t* bar, uint32_t parity, unsigned long long* acc) {
  if (acc) {
    const long long t0 = clock64();
    mbar_wait(bar, parity);
    *acc += static_cast<unsigned long long>(clock64() - t0);
  } else {
    mbar_wait(bar, parity);
  }
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "elect.sync _|P, 0xffffffff;\n"
      "selp.u32 %0, 1, 0, P;\n"
      "}\n"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// Fences inside the MMA <-> epilogue pipeline, as the PTX memory model asks
// for thread-synchronised tcgen05 accesses.  (CUTLASS's SM100 pipelines omit
// them; removing them measured no difference here: the ~250 cycles the
// after_thread_sync fence holds the issuing warp are hidden by the queued
// MMAs.)  ACE_TC_FENCES=0 drops them.
#ifndef ACE_TC_FENCES
#define ACE_TC_FENCES 1
#endif
__device__ __forceinline__ void pipe_before() {
  if (ACE_TC_FENCES) tc_before();
}
__device__ __forceinline__ void pipe_after() {
  if (ACE_TC_FENCES) tc_after();
}

// K-major SWIZZLE_128B shared-memory matrix descriptor (sm_100 version 1).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3fff);      // start address
  d |= static_cast<uint64_t>(1) << 16;                     // LBO (unused for SW128 K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;             // SBO: 8-row atom stride
  d |= static_cast<uint64_t>(1) << 46;                     // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;                     // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: A,B fp16 K-major, D fp32, M=128, N=n.
// M = 128 per CTA (256 for the pair)
__device__ __forceinline__ uint32_t idesc_f16(uint32_t n) {
  return (1u << 4) | ((n >> 3) << 17) | (((128u * kPair) >> 4) << 24);
}

__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
#if ACE_PAIR == 2
  // each CTA of the pair: its own shared memory -> its own TMEM, same addresses
  asm volatile("tcgen05.cp.cta_group::2.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc));
#else
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc));
#endif
}
__device__ __forceinline__ void mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
#if ACE_PAIR == 2
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n"
#else
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
#endif
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate));
}
// A and B both from shared memory (K-major SW128 descriptors), one CTA.
__device__ __forceinline__ void mma_f16_ss(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
// Commit: the barrier at this offset in every CTA of the pair gets one arrival
// once all earlier tcgen05 operations of the issuing thread have completed.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
#if ACE_PAIR == 2
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
#else
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
#endif
}
// Arrive on the barrier at the same offset in CTA `rank` of the cluster.
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
  asm volatile(
      "{\n"
      ".reg .b32 ra;\n"
      "mapa.shared::cluster.u32 ra, %0, %1;\n"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(rank)
      : "memory");
}

#define ACE_TMEM_LD32(taddr, v)                                                                    \
  asm volatile(                                                                                    \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"               \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),        \
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),    \
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), \
        "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), \
        "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])                                         \
      : "r"(taddr))

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// byte offset of element (row r, k in [0,64)) in a SW128 K-major block
__device__ __forceinline__ uint32_t sw128_off(uint32_t r, uint32_t k) {
  return r * 128u + ((((k >> 3) ^ (r & 7u)) & 7u) << 4) + ((k & 7u) << 1);
}

__device__ __forceinline__ double exact_proj(const double* __restrict__ w, const void* x, int x_f64,
                                             uint64_t row, uint64_t ld, uint64_t dim) {
  // binary64 left fold, mul then add, from +0.0 (srp.cpp:78-91); operands
  // are loaded 8 ahead so only the add chain is serial
  double acc = 0.0;
  uint64_t i = 0;
  if (x_f64) {
    const double* xr = static_cast<const double*>(x) + row * ld;
    for (; i + 8 <= dim; i += 8) {
      double wv[8], xv[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        wv[k] = w[i + k];
        xv[k] = xr[i + k];
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) acc = __dadd_rn(acc, __dmul_rn(wv[k], xv[k]));
    }
    for (; i < dim; ++i) acc = __dadd_rn(acc, __dmul_rn(w[i], xr[i]));
  } else {
    const float* xr = static_cast<const float*>(x) + row * ld;
    for (; i + 8 <= dim; i += 8) {
      double wv[8];
      float xv[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        wv[k] = w[i + k];
        xv[k] = xr[i + k];
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) acc = __dadd_rn(acc, __dmul_rn(wv[k], static_cast<double>(xv[k])));
    }
    for (; i < dim; ++i) acc = __dadd_rn(acc, __dmul_rn(w[i], static_cast<double>(xr[i])));
  }
  return acc;
}

__device__ __forceinline__ void cp_async_4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

__device__ __forceinline__ unsigned long long warp_sum_u64_tc(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- X conversion pre-pass ------------------------------------------------------

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  return (static_cast<uint32_t>(__half_as_ushort(__float2half_rn(b))) << 16) |
         __half_as_ushort(__float2half_rn(a));
}

// Element k of a row (fp32 or fp64 source), 0 beyond dim.
__device__ __forceinline__ float load_x(const TcArgs& a, uint64_t row, uint64_t k) {
  if (k >= a.dim) return 0.0f;
  if (a.x_f64) return static_cast<float>(static_cast<const double*>(a.x)[row * a.ld + k]);
  return static_cast<const float*>(a.x)[row * a.ld + k];
}

// One row, eight lanes (l8) holding its values v[g][e] = x[32 g + 4 l8 + e]:
// max |x| (NaN > inf > finite as magnitude bits), power-of-two scale to
// [2^14, 2^15), fp16 hi + lo split written into the SW128 K-major image of
// the row's 128-row tile (`tile`: [kc][hi | lo][16 KB]), and the row's error
// threshold thr = c * ||x~|| * 2^14 + abs (-1: exact zero row or padding,
// +inf: recheck every projection).
// Returns this lane's lo-step bits: bit s set iff a lo part it wrote in K16
// step s is nonzero (an x exactly representable in fp16 after scaling, e.g.
// one-hot columns, has a zero lo part and its lo x hi MMAs can be skipped).
template <uint32_t kG>
__device__ __forceinline__ uint32_t convert_row(float (&v)[kG][4], uint32_t l8, bool live, uint32_t groups,
                                                uint32_t nkc, uint64_t dim, float margin_c, uint8_t* tile, uint32_t r,
                                                float* thr_dst) {
  uint32_t mb = 0u, lobits = 0u;
#pragma unroll
  for (uint32_t g = 0; g < kG; ++g)
#pragma unroll
    for (int e = 0; e < 4; ++e) mb = max(mb, __float_as_uint(v[g][e]) & 0x7fffffffu);
  mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, 1));
  mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, 2));
  mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, 4));
  const bool nan = mb > 0x7f800000u;
  const float m = __uint_as_float(nan ? 0x7f800000u : mb);
  const bool zero = (m == 0.0f);
  const bool wild = nan || !(m < 0x1.0p100f) || (!zero && m < 0x1.0p-100f);
  float scale = 0.0f;
  if (live && !zero && !wild) {
    const int e = static_cast<int>((__float_as_uint(m) >> 23) & 0xffu) - 127;
    scale = __uint_as_float(static_cast<uint32_t>(127 + 14 - e) << 23);
  }
  float ss = 0.0f;
#pragma unroll
  for (uint32_t g = 0; g < kG; ++g) {
    if (g >= groups) continue;
    const uint32_t k0 = g * 32u + l8 * 4u;
    const uint32_t kc = k0 / kChunk, kk = k0 % kChunk;
    uint32_t hi[2], lo[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float x0 = v[g][2 * i] * scale, x1 = v[g][2 * i + 1] * scale;
      ss = fmaf(x0, x0, fmaf(x1, x1, ss));
      const float h0 = __half2float(__float2half_rn(x0)), h1 = __half2float(__float2half_rn(x1));
      hi[i] = pack_h2(h0, h1);
      lo[i] = pack_h2(x0 - h0, x1 - h1);
    }
    if ((lo[0] | lo[1]) != 0u) lobits |= 1u << (k0 >> 4);
    uint8_t* blk = tile + kc * 2u * kBlockBytes;
    const uint32_t off = sw128_off(r, kk);
    *reinterpret_cast<uint2*>(blk + off) = make_uint2(hi[0], hi[1]);
    *reinterpret_cast<uint2*>(blk + kBlockBytes + off) = make_uint2(lo[0], lo[1]);
  }
  ss += __shfl_xor_sync(0xffffffffu, ss, 1);
  ss += __shfl_xor_sync(0xffffffffu, ss, 2);
  ss += __shfl_xor_sync(0xffffffffu, ss, 4);
  if (l8 == 0) {
    float thr;
    if (!live || zero) {
      thr = -1.0f;
    } else if (wild) {
      thr = __int_as_float(0x7f800000);
    } else {
      const float nx = sqrtf(ss * (1.0f + static_cast<float>(dim + 4) * 0x1.0p-23f)) * (1.0f + 0x1.0p-20f);
      thr = margin_c * nx * 16384.0f + static_cast<float>(dim) * 0x1.0p-10f;
    }
    *thr_dst = thr;
  }
  return lobits;
}

// Pre-pass: eight lanes per row (four rows per warp, values in registers),
// the SW128 image and thresholds written to global memory.  Lane l8 of a row
// owns K elements 32g + 4*l8 .. +3 (coalesced 128 B per group).  Rows past n
// (tile padding) are written as zeros.
template <uint32_t kG>  // 32-element groups per row held in registers: 2 * nkc rounded up to 2, 4 or 8
__global__ void __launch_bounds__(256) convert_x_kernel(const TcArgs a, uint64_t rows_padded) {
  const uint32_t lane = threadIdx.x & 31, l8 = lane & 7;
  const uint64_t slots = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 3);
  const uint32_t groups = a.nkc * 2;  // 32 K per group, <= 8
  const bool vec4 = !a.x_f64 && (a.ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0);
  for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * (blockDim.x >> 3); base < rows_padded; base += slots) {
    const uint64_t row = base + (threadIdx.x >> 3);
    const bool inb = row < rows_padded;
    const bool live = row < a.n;
    float v[kG][4];
#pragma unroll
    for (uint32_t g = 0; g < kG; ++g) {
      const uint64_t k0 = g * 32u + l8 * 4u;
      v[g][0] = v[g][1] = v[g][2] = v[g][3] = 0.0f;
      if (g < groups && live) {
        if (vec4 && k0 + 3 < a.dim) {
          const float4 u = *reinterpret_cast<const float4*>(static_cast<const float*>(a.x) + row * a.ld + k0);
          v[g][0] = u.x;
          v[g][1] = u.y;
          v[g][2] = u.z;
          v[g][3] = u.w;
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) v[g][e] = load_x(a, row, k0 + e);
        }
      }
    }
    if (!inb) continue;  // (row-uniform per 8-lane group; shuffles stay within the group)
    const uint64_t tile = row / kRows;
    uint32_t lob = convert_row<kG>(v, l8, live, groups, a.nkc, a.dim, a.margin_c,
                                   reinterpret_cast<uint8_t*>(a.x16) + tile * a.nkc * 2u * kBlockBytes,
                                   static_cast<uint32_t>(row % kRows), &a.rowthr[row]);
    // the 4 rows of a warp lie in one point tile (kRows % 4 == 0)
    lob |= __shfl_xor_sync(0xffffffffu, lob, 1);
    lob |= __shfl_xor_sync(0xffffffffu, lob, 2);
    lob |= __shfl_xor_sync(0xffffffffu, lob, 4);
    lob |= __shfl_xor_sync(0xffffffffu, lob, 8);
    lob |= __shfl_xor_sync(0xffffffffu, lob, 16);
    if (a.lomask && lane == 0 && lob) atomicOr(&a.lomask[tile], lob);
  }
}

// Cold path: push the near-tie columns (bit jj of mask = column dir0 + jj)
// into this CTA's list segment; a full segment flags the whole row instead.
__device__ __noinline__ void push_near_mask(DevState* st, unsigned long long* seg, unsigned long long seg_cap,
                                            uint32_t* seg_n, uint32_t* overflow_rows, uint32_t mask, uint64_t row,
                                            uint32_t dir0) {
  while (mask) {
    const uint32_t jj = __ffs(mask) - 1;
    mask &= mask - 1;
    const uint32_t slot = atomicAdd(seg_n, 1u);
    if (slot < seg_cap) {
      seg[slot] = (static_cast<unsigned long long>(row) << 32) | (dir0 + jj);
    } else {
      atomicOr(&overflow_rows[row >> 5], 1u << (row & 31));
      st->near_overflow = 1;
    }
  }
}

// Warp-aggregated counter increments for one table: lanes holding equal
// buckets are merged over up to three ballot rounds, the rest add singly.
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

// Binary64 left fold, mul then add, from +0.0 (srp.cpp:78-91), operands 8
// ahead; gives up (returns false) as soon as *done reaches `until` (the
// epilogue has finished: the shared tail takes the item).  Out of line: cold
// code kept away from the main loop's instruction cache footprint.
__device__ __noinline__ bool exact_proj_until(const double* __restrict__ w, const void* x, int x_f64, uint64_t row,
                                              uint64_t ld, uint32_t dim, const uint32_t* done, uint32_t until,
                                              double* out) {
  double acc = 0.0;
  for (uint32_t k0 = 0; k0 < dim; k0 += 8u) {
    if (*reinterpret_cast<const volatile uint32_t*>(done) >= until) return false;
    double wv[8], xv[8];
#pragma unroll
    for (uint32_t u = 0; u < 8u; ++u) {
      const uint32_t k = min(k0 + u, dim - 1u);
      wv[u] = __ldg(w + k);
      xv[u] = x_f64 ? __ldg(static_cast<const double*>(x) + row * ld + k)
                    : static_cast<double>(__ldg(static_cast<const float*>(x) + row * ld + k));
    }
#pragma unroll
    for (uint32_t u = 0; u < 8u; ++u)
      if (k0 + u < dim) acc = __dadd_rn(acc, __dmul_rn(wv[u], xv[u]));
  }
  *out = acc;
  return true;
}

// Shared tail of the near-tie recheck, run by the kTail epilogue + recheck
// threads (named barrier 9) once the main loop is over: list slots
// [from, cnt) that still hold an item (~0 = already rechecked) are rechecked
// in chunks.  Every MMA has completed by then, so the whole dynamic shared
// memory is free: each chunk's operands (x row and W row, element-major
// [k][item] so the fold reads are conflict-free) are copied global -> shared
// with cp.async (no register staging: all of them in flight at once), then
// each thread folds one item.  Slots are reset to ~0 for the next launch.
__device__ __noinline__ void recheck_tail(const void* x, int x_f64, uint64_t ld, uint32_t dim, const double* w64,
                                          uint32_t* ids, uint64_t n, uint32_t* counters, int fused_insert,
                                          uint32_t K, uint8_t* smem, size_t smem_bytes, unsigned long long* seg,
                                          uint32_t from, uint32_t cnt, uint32_t et, unsigned long long& rr,
                                          unsigned long long& ff) {
  const uint32_t cap_items = min(static_cast<uint32_t>(smem_bytes / (16u * dim + 8u)), kTail);
  unsigned long long* meta = reinterpret_cast<unsigned long long*>(smem);
  double* xs = reinterpret_cast<double*>(smem + 8u * cap_items);
  double* ws = xs + static_cast<size_t>(cap_items) * dim;
  const uint32_t qd = kTail / dim, rd = kTail % dim;
  for (uint32_t c0 = from; c0 < cnt; c0 += cap_items) {
    const uint32_t m = min(cap_items, cnt - c0);
    for (uint32_t i = et; i < m; i += kTail) {
      meta[i] = seg[c0 + i];
      seg[c0 + i] = ~0ull;
    }
    asm volatile("bar.sync 9, %0;" ::"r"(kTail) : "memory");
    const uint32_t total = m * dim;
    uint32_t ci = et / dim, ck = et - (et / dim) * dim;  // (item, k) of element e, advanced incrementally
    for (uint32_t e = et; e < total; e += kTail) {
      const unsigned long long item = meta[ci];
      if (item != ~0ull) {
        const uint64_t row = item >> 32;
        const uint32_t dir = static_cast<uint32_t>(item & 0xffffffffu);
        const size_t slot = static_cast<size_t>(ck) * cap_items + ci;
        if (x_f64)
          cp_async_8(xs + slot, static_cast<const double*>(x) + row * ld + ck);
        else
          cp_async_4(reinterpret_cast<float*>(xs) + slot, static_cast<const float*>(x) + row * ld + ck);
        cp_async_8(ws + slot, w64 + static_cast<uint64_t>(dir) * dim + ck);
      }
      ci += qd;
      ck += rd;
      if (ck >= dim) {
        ck -= dim;
        ++ci;
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    asm volatile("bar.sync 9, %0;" ::"r"(kTail) : "memory");
    if (et < m && meta[et] != ~0ull) {
      // binary64 left fold, mul then add, from +0.0 (srp.cpp:78-91)
      double acc = 0.0;
      const float* xs32 = reinterpret_cast<const float*>(xs);
#pragma unroll 8
      for (uint32_t k = 0; k < dim; ++k) {
        const size_t slot = static_cast<size_t>(k) * cap_items + et;
        const double xv = x_f64 ? xs[slot] : static_cast<double>(xs32[slot]);
        acc = __dadd_rn(acc, __dmul_rn(ws[slot], xv));
      }
      const unsigned long long item = meta[et];
      const uint64_t row = item >> 32;
      const uint32_t dir = static_cast<uint32_t>(item & 0xffffffffu);
      const uint32_t table = dir / K, bpos = K - 1u - dir % K;
      uint32_t* id = &ids[static_cast<uint64_t>(table) * n + row];
      const uint32_t exact = acc >= 0.0 ? 1u : 0u;
      if (((__ldcg(id) >> bpos) & 1u) != exact) {
        const uint32_t old = atomicXor(id, 1u << bpos);
        if (fused_insert) {
          uint32_t* ct = counters + (static_cast<uint64_t>(table) << K);
          atomicSub(&ct[old], 1u);
          atomicAdd(&ct[old ^ (1u << bpos)], 1u);
        }
        ++ff;
      }
      ++rr;
    }
    asm volatile("bar.sync 9, %0;" ::"r"(kTail) : "memory");
  }
}

// ---- the projection kernel ----------------------------------------------------------

// kFuse: X is converted inside the kernel (warps 10-11) from raw fp32 tiles
// the producer bulk-copies, instead of by the convert_x_kernel pre-pass; the
// near-tie recheck is then all done in the shared tail.
template <bool kFuse>
__global__ void __launch_bounds__(kThreads, 1) hash_tc_kernel(const TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bar_wfull[kMaxWStages], bar_wempty[kMaxWStages];
  __shared__ __align__(8) uint64_t bar_afull[2], bar_aempty[2];
  __shared__ __align__(8) uint64_t bar_accfull[kAccBufs], bar_accempty[kAccBufs];
  __shared__ uint32_t tmem_base_sh;
  __shared__ uint32_t lastw[4][2][32];  // epilogue: last sign word of a direction tile, per quarter / parity
  __shared__ uint32_t xw[4][2][2][32];  // split epilogue: last word of each half, per quarter / half / parity
  __shared__ uint32_t seg_n;                        // near ties pushed by this CTA
  __shared__ uint32_t tiles_done;                   // epilogue warps x tiles completed (ids stored)
  __shared__ uint32_t min_next;                     // first list slot the recheck warps left over
  __shared__ unsigned long long blk_rech, blk_flip;
  __shared__ __align__(8) uint64_t bar_rawfull, bar_rawempty, bar_thrfull[2], bar_threempty[2];
  __shared__ float thr_sm[2][kRows];  // fused conversion: row thresholds per tile parity

  TcLayout L = tc_layout(a.nkc, a.dim, kFuse, a.tw);
  const uint32_t TW = a.tw, wblk = a.tw * 128u;  // direction tile width, one W block (hi or lo) in bytes
  if (a.dbg >> 12) L.n_wst = min(L.n_wst, static_cast<uint32_t>(a.dbg >> 12));  // experiment: fewer W stages
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* Asm = base;                               // [n_abuf][nkc][2][16 KB]
  uint8_t* Rsm = base + L.a_bytes;                   // fused: raw fp32 rows [128][dim]
  uint8_t* Wsm = base + L.a_bytes + L.raw_bytes;     // [n_wst][2][16 KB / kPair]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t n_tiles = (a.n + kRows - 1) / kRows;
  const uint32_t K = a.k_bits;
  const uint32_t R = a.k_bits * a.tables;  // directions, packed densely in 128-column tiles
  const uint32_t a_tile_bytes = a.nkc * 2u * kBlockBytes;

  if (threadIdx.x == 0) {
    seg_n = 0;
    tiles_done = 0;
    min_next = (ACE_RW && !kFuse) ? 0xffffffffu : 0u;
    blk_rech = blk_flip = 0;
    // the leader's full barriers also wait for the peer's forwarded arrival,
    // its accumulator-empty barriers for the peer's epilogue warps
    const uint32_t fulls = (kPair == 2 && cluster_ctarank() == 0) ? 2u : 1u;
    for (uint32_t s = 0; s < L.n_wst; ++s) {
      mbar_init(&bar_wfull[s], fulls);
      mbar_init(&bar_wempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar_afull[b], kFuse ? 2u : fulls);  // fused: the two converter warps
      mbar_init(&bar_aempty[b], 1);
      mbar_init(&bar_thrfull[b], 2);
      mbar_init(&bar_threempty[b], 8);
    }
    mbar_init(&bar_rawfull, 1);
    mbar_init(&bar_rawempty, 2);
    for (int b = 0; b < kAccBufs; ++b) {
      mbar_init(&bar_accfull[b], 1);
      mbar_init(&bar_accempty[b], (ACE_SPLIT ? 8 : 4) * kPair);  // epilogue warps per tile, per CTA
    }
    fence_mbar_init();
  }
  if (warp == 1) {
#if ACE_PAIR == 2
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
#else
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
#endif
  }
  tc_before();
  __syncthreads();
  cluster_sync_all();  // remote CTAs may signal our barriers from here on
  tc_after();
  const uint32_t tmem_base = tmem_base_sh;
  // Tile schedule: pair P (of npairs) takes tile groups P, P + npairs, ...;
  // CTA `rank` of the pair takes tile kPair*group + rank.  Every CTA runs the
  // same number of iterations (tiles past the end are skipped by the
  // epilogue) so the pair's shared pipeline stays in lockstep.
  const uint32_t rank = kPair == 2 ? cluster_ctarank() : 0u;
  const uint32_t npairs = gridDim.x / kPair, pair = blockIdx.x / kPair;
  const uint64_t iters = (n_tiles + gridDim.x - 1) / gridDim.x;
  auto tile_of = [&](uint64_t it) -> uint64_t { return (pair + it * npairs) * kPair + rank; };
  // instrumentation (a.prof != null): cycles waiting per barrier kind, per CTA:
  // [0] prod a_empty [1] prod w_empty [2] mma a_full [3] mma acc_empty
  // [4] mma w_full [5] epilogue acc_full (warp 2..5 lane 0 summed) [6] total
  const bool prof = a.prof != nullptr;
  const unsigned long long seg_cap = a.near_cap / gridDim.x;
  unsigned long long pw[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const long long t_start = clock64();
  unsigned long long rr_own = 0, ff_own = 0;  // near ties rechecked / bits flipped by this thread
  unsigned long long g_start = 0;
  if (prof) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_start));

  if (warp == 0) {
    // ---------------- producer: A tile (once per tile) + W stages ----------------
    // A: this CTA's own 128 points.  W: this CTA's share of each direction
    // tile (rows [64 rank, 64 rank + 64) of the hi and lo blocks in pair mode).
    if (lane == 0) {
      uint32_t s = 0, ph = 0;
      const uint32_t share = kBlockBytes / kPair, half = share;  // bytes of one block per CTA
      for (uint64_t it = 0; it < iters; ++it) {
        const uint64_t t = tile_of(it);
        if (kFuse) {
          // raw fp32 rows of the tile (contiguous: ld == dim), converted by warps 10-11
          mbar_wait_sleepy(&bar_rawempty, (static_cast<uint32_t>(it) & 1u) ^ 1u, prof ? &pw[0] : nullptr);
          const uint64_t r0 = t * kRows;
          const uint32_t rows = r0 < a.n ? static_cast<uint32_t>(a.n - r0 < kRows ? a.n - r0 : kRows) : 0u;
          if (rows) {
            const uint32_t bytes = rows * static_cast<uint32_t>(a.dim) * 4u;
            mbar_expect_tx(&bar_rawfull, bytes);
            bulk_g2s(Rsm, static_cast<const float*>(a.x) + r0 * a.dim, bytes, &bar_rawfull);
          } else {
            mbar_arrive(&bar_rawfull);
          }
        } else {
          mbar_wait_sleepy(&bar_aempty[0], (static_cast<uint32_t>(it) & 1u) ^ 1u, prof ? &pw[0] : nullptr);
          const uint64_t tt = t < n_tiles ? t : n_tiles - 1;  // past the end: reload the last tile
          mbar_expect_tx(&bar_afull[0], a_tile_bytes);
          bulk_g2s(Asm, reinterpret_cast<const uint8_t*>(a.x16) + tt * a_tile_bytes, a_tile_bytes, &bar_afull[0]);
        }
        for (uint32_t j = 0; j < a.ntiles; ++j) {
          const uint32_t nmma = kPair == 2 ? 128u : ((min(TW, R - j * TW) + 15u) & ~15u);
          const uint32_t bytes = kPair == 2 ? share : nmma * 128u;
          const uint32_t hblk = kPair == 2 ? half : wblk;  // stage layout: hi block, then lo block
          for (uint32_t kc = 0; kc < a.nkc; ++kc) {
            mbar_wait_sleepy(&bar_wempty[s], ph ^ 1u, prof ? &pw[1] : nullptr);
            if ((a.dbg & 256) && it > 0) {  // experiment: W stages loaded for the first point tile only
              mbar_arrive(&bar_wfull[s]);
            } else {
            mbar_expect_tx(&bar_wfull[s], 2u * bytes);
            const uint8_t* src = reinterpret_cast<const uint8_t*>(a.w16) +
                                 (static_cast<uint64_t>(j) * a.nkc + kc) * 2u * wblk + rank * share;
            uint8_t* dst = Wsm + static_cast<size_t>(s) * 2u * hblk;
            bulk_g2s(dst, src, bytes, &bar_wfull[s]);
            bulk_g2s(dst + hblk, src + wblk, bytes, &bar_wfull[s]);
            }
            if (++s == L.n_wst) {
              s = 0;
              ph ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1 && rank != 0) {
    // ---------------- pair peer: forward stage arrivals to the leader ----------------
    // The leader's MMAs read this CTA's A tile and W shares too: once a local
    // copy has landed, arrive on the leader's barrier at the same offset.
    if (lane == 0) {
      uint32_t s = 0, wph = 0;
      for (uint64_t it = 0; it < iters; ++it) {
        mbar_wait(&bar_afull[0], static_cast<uint32_t>(it) & 1u);
        mbar_arrive_remote(&bar_afull[0], 0);
        for (uint32_t j = 0; j < a.ntiles; ++j)
          for (uint32_t kc = 0; kc < a.nkc; ++kc) {
            mbar_wait(&bar_wfull[s], wph);
            mbar_arrive_remote(&bar_wfull[s], 0);
            if (++s == L.n_wst) {
              s = 0;
              wph ^= 1u;
            }
          }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer: A smem -> TMEM (tcgen05.cp), then TS MMAs ----------------
    // The whole warp walks the schedule (operands stay warp-uniform, so the
    // descriptors live in uniform registers); one elected lane issues.  In
    // pair mode this is the leader, its MMAs and copies cover both CTAs.
    {
      uint32_t s = 0, wph = 0, acc = 0, accph = 0;
      unsigned long long pmi = 0, pmn = 0, pcp = 0;  // instrumentation: MMA-group issue cycles / groups, A copies
      unsigned long long pfence = 0, pwf = 0, pcm = 0;  // instrumentation: W-full waits, commits (issuing lane)
      const long long ploop = clock64();
      const uint32_t nacc = tc_acc_bufs(a.nkc, TW);
      const uint32_t ta_hi = tmem_base + nacc * TW, ta_lo = ta_hi + a.nkc * 32u;  // dpad/2 columns each
      const uint32_t a_base = smem_u32(Asm), w_base = smem_u32(Wsm);
      const uint32_t half = kPair == 2 ? kBlockBytes / kPair : wblk;  // bytes of one W block (hi or lo) per CTA
      // K16 steps past dim hold zero padding: none of their MMAs run
      const uint32_t nsteps = static_cast<uint32_t>((a.dim + 15u) / 16u);
      for (uint64_t it = 0; it < iters; ++it) {
        // lo x hi MMAs of the steps whose x lo parts are all zero in this tile
        // are skipped (the pre-pass sets the bits; they add exact zeros)
        const uint32_t lm = (kPair == 1 && a.lomask && !kFuse) ? __ldcg(a.lomask + min(tile_of(it), n_tiles - 1)) : 0xffffffffu;
        mbar_wait_t(&bar_afull[0], static_cast<uint32_t>(it) & 1u, (prof && lane == 0) ? &pw[2] : nullptr);
        pipe_after();
        const long long pc0 = prof ? clock64() : 0;
        // copies execute in issue order after this CTA's earlier MMAs, so the
        // previous tile's reads of TMEM A are complete before it is replaced
        if (elect_one()) {
          for (uint32_t kc = 0; kc < a.nkc; ++kc) {
            const uint32_t ah = a_base + kc * 2u * kBlockBytes;
#pragma unroll
            for (uint32_t kk = 0; kk < 4; ++kk) {
              // one copy per K16 step and operand; steps whose MMAs are all
              // skipped (past d, or a zero x lo part) are not copied either
              const uint32_t step = kc * 4u + kk;
              if (step >= nsteps) break;
              tmem_cp_128x256b(ta_hi + step * 8u, sw128_desc(ah + kk * 32u));
              if ((lm >> step) & 1u) tmem_cp_128x256b(ta_lo + step * 8u, sw128_desc(ah + kBlockBytes + kk * 32u));
            }
          }
          mma_commit(&bar_aempty[0]);  // shared-memory A free once the copies land
        }
        __syncwarp();
        if (prof) pcp += static_cast<unsigned long long>(clock64() - pc0);
#if ACE_TILE_BURST
        // one elected burst per point tile: the issuing lane waits for the
        // accumulators and W stages itself, no warp-wide syncs in between
        const long long pi0 = prof ? clock64() : 0;
        if (elect_one()) {
          uint32_t ss = s, ph = wph, ac = acc, acph = accph;
          for (uint32_t j = 0; j < a.ntiles; ++j) {
            const uint32_t nmma = kPair == 2 ? 128u : ((min(TW, R - j * TW) + 15u) & ~15u);
            const uint32_t idesc = idesc_f16(nmma);
            mbar_wait(&bar_accempty[ac], acph ^ 1u);
            pipe_after();
            const uint32_t dt = tmem_base + ac * TW;
            for (uint32_t kc = 0; kc < a.nkc; ++kc) {
              mbar_wait(&bar_wfull[ss], ph);
              const uint32_t b_hi = w_base + ss * 2u * half;
              const uint64_t dbh = sw128_desc(b_hi), dbl = sw128_desc(b_hi + half);
#pragma unroll
              for (uint32_t kk = 0; kk < 4; ++kk) {
                const uint32_t step = kc * 4u + kk;
                if (step >= nsteps) break;
                const uint32_t acol = step * 8u;
                const uint64_t off = kk * 2u;
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
            mma_commit(&bar_accfull[ac]);
            if (++ac == nacc) {
              ac = 0;
              acph ^= 1u;
            }
          }
        }
        __syncwarp();
        for (uint32_t j = 0; j < a.ntiles; ++j) {
          for (uint32_t kc = 0; kc < a.nkc; ++kc)
            if (++s == L.n_wst) {
              s = 0;
              wph ^= 1u;
            }
          if (++acc == nacc) {
            acc = 0;
            accph ^= 1u;
          }
        }
        if (prof) {
          pmi += static_cast<unsigned long long>(clock64() - pi0);
          pmn += a.nkc * a.ntiles;
        }
#else
        for (uint32_t j = 0; j < a.ntiles; ++j) {
          const uint32_t nmma = kPair == 2 ? 128u : ((min(TW, R - j * TW) + 15u) & ~15u);
          const uint32_t idesc = idesc_f16(nmma);
          mbar_wait_t(&bar_accempty[acc], accph ^ 1u, (prof && lane == 0) ? &pw[3] : nullptr);
          const long long pf0 = prof ? clock64() : 0;
          pipe_after();
          if (prof) pfence += static_cast<unsigned long long>(clock64() - pf0);
          const uint32_t dt = tmem_base + acc * TW;
          // one elected burst per direction tile: the issuing lane waits for
          // each stage itself (no warp-wide syncs between the MMA groups, so
          // the tensor queue is refilled without gaps)
          const long long pi0 = prof ? clock64() : 0;
          if (elect_one()) {
            uint32_t ss = s, ph = wph;
            for (uint32_t kc = 0; kc < a.nkc; ++kc) {
              const long long pq0 = prof ? clock64() : 0;
              mbar_wait(&bar_wfull[ss], ph);
              if (prof) pwf += static_cast<unsigned long long>(clock64() - pq0);
              const uint32_t b_hi = w_base + ss * 2u * half;
              const uint64_t dbh = sw128_desc(b_hi), dbl = sw128_desc(b_hi + half);
              if (!(a.dbg & 2)) {
#pragma unroll
                for (uint32_t kk = 0; kk < 4; ++kk) {
                  const uint32_t step = kc * 4u + kk;
                  if (step >= nsteps) break;
                  const uint32_t acol = step * 8u;  // 16 fp16 = 8 TMEM columns
                  const uint64_t off = kk * 2u;     // 32 B along K in SW128, >> 4
                  mma_f16_ts(dt, ta_hi + acol, dbh + off, idesc, step != 0u);
                  if ((lm >> step) & 1u) mma_f16_ts(dt, ta_lo + acol, dbh + off, idesc, 1u);
                  mma_f16_ts(dt, ta_hi + acol, dbl + off, idesc, 1u);
                }
              }
              const long long pq1 = prof ? clock64() : 0;
              mma_commit(&bar_wempty[ss]);
              if (prof) pcm += static_cast<unsigned long long>(clock64() - pq1);
              if (++ss == L.n_wst) {
                ss = 0;
                ph ^= 1u;
              }
            }
            const long long pq2 = prof ? clock64() : 0;
            mma_commit(&bar_accfull[acc]);
            if (prof) pcm += static_cast<unsigned long long>(clock64() - pq2);
          }
          __syncwarp();
          for (uint32_t kc = 0; kc < a.nkc; ++kc)
            if (++s == L.n_wst) {
              s = 0;
              wph ^= 1u;
            }
          if (prof) {
            pmi += static_cast<unsigned long long>(clock64() - pi0);
            pmn += a.nkc;
          }
          if (++acc == nacc) {
            acc = 0;
            accph ^= 1u;
          }
        }
#endif
      }
      if (prof && pmn && lane == 0) {
        atomicAdd(&a.prof[20], pmi);
        atomicAdd(&a.prof[21], pmn);
        atomicAdd(&a.prof[22], pcp);
        atomicAdd(&a.prof[23], static_cast<unsigned long long>(clock64() - ploop));
        atomicAdd(&a.prof[24], pw[2] + pw[3] + pw[4]);
        atomicAdd(&a.prof[25], pfence);
      }
      if (prof && pmn) {
        const unsigned long long wf = warp_sum_u64_tc(pwf), cm = warp_sum_u64_tc(pcm);
        if (lane == 0) {
          atomicAdd(&a.prof[26], wf);
          atomicAdd(&a.prof[27], cm);
        }
      }
    }
  } else if (kFuse && warp >= 10) {
    // ---------------- converter warps (10, 11): raw fp32 tile -> A image ----------------
    // Same arithmetic as convert_x_kernel; 8 lanes per row, rows from shared
    // memory.  Hand-offs: raw buffer (producer), A buffer (MMA warp's copy to
    // TMEM), thresholds (epilogue, double-buffered by tile parity).
    const uint32_t l8 = lane & 7, groups = a.nkc * 2u;
    const uint32_t dim = static_cast<uint32_t>(a.dim);
    for (uint64_t it = 0; it < iters; ++it) {
      const uint64_t t = tile_of(it);
      const uint32_t p = static_cast<uint32_t>(it) & 1u;
      mbar_wait_sleepy(&bar_rawfull, p, nullptr);
      mbar_wait_sleepy(&bar_aempty[0], p ^ 1u, nullptr);
      mbar_wait_sleepy(&bar_threempty[p], (static_cast<uint32_t>(it >> 1) & 1u) ^ 1u, nullptr);
      for (uint32_t pass = 0; pass < kRows / 8u; ++pass) {
        const uint32_t r = pass * 8u + (warp - 10u) * 4u + (lane >> 3);
        const bool live = t * kRows + r < a.n;
        float v[8][4];
#pragma unroll
        for (uint32_t g = 0; g < 8; ++g) {
          const uint32_t k0 = g * 32u + l8 * 4u;
          if (g < groups && live && k0 < dim) {  // dim % 4 == 0: whole float4 in range
            const float4 u = *reinterpret_cast<const float4*>(Rsm + (static_cast<size_t>(r) * dim + k0) * 4u);
            v[g][0] = u.x;
            v[g][1] = u.y;
            v[g][2] = u.z;
            v[g][3] = u.w;
          } else {
            v[g][0] = v[g][1] = v[g][2] = v[g][3] = 0.0f;
          }
        }
        (void)convert_row<8>(v, l8, live, groups, a.nkc, a.dim, a.margin_c, Asm, r, &thr_sm[p][r]);
      }
      fence_proxy_async();  // A image (generic stores) -> tcgen05.cp (async proxy)
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&bar_rawempty);
        mbar_arrive(&bar_thrfull[p]);
        mbar_arrive(&bar_afull[0]);
      }
    }
  } else if (warp >= 10) {
    // ---------------- recheck warps (10, 11) ----------------
    // Exact binary64 recheck of near ties while the main loop runs: lane L of
    // recheck warp w takes list slots w*32+L, +64, ... in order, waits until
    // the slot is written and its tile's ids are stored (tiles_done), folds
    // the exact projection, fixes the bit (and, with the fused insert, moves
    // the count) and resets the slot to ~0.  When the epilogue finishes, the
    // lanes stop; the shared tail takes the slots from min_next on.
    const uint32_t total_done = 8u * static_cast<uint32_t>(iters);
    unsigned long long* seg = a.near_list + blockIdx.x * seg_cap;
    uint32_t i = (warp - 10u) * 32u + lane;
    if (!(a.dbg & 32) && !a.ext_recheck) {
      while (true) {
        unsigned long long item = ~0ull;
        while (true) {
          if (*reinterpret_cast<volatile uint32_t*>(&tiles_done) >= total_done) break;
          if (i < seg_cap) item = *reinterpret_cast<volatile unsigned long long*>(seg + i);
          if (item != ~0ull) break;
          __nanosleep(256);
        }
        if (item == ~0ull) break;
        const uint64_t row = item >> 32;
        const uint32_t it = static_cast<uint32_t>(((row >> 7) / kPair - pair) / npairs);  // inverse of tile_of
        while (*reinterpret_cast<volatile uint32_t*>(&tiles_done) < 8u * (it + 1u)) __nanosleep(128);
        __threadfence_block();
        const uint32_t dir = static_cast<uint32_t>(item & 0xffffffffu);
        const uint32_t table = dir / K, bpos = K - 1u - dir % K;
        // binary64 left fold (srp.cpp:78-91), abandoned
        // (slot left for the shared tail) once the epilogue has finished
        double p = 0.0;
        const bool abandoned = !exact_proj_until(a.w64 + static_cast<uint64_t>(dir) * a.dim, a.x, a.x_f64, row, a.ld,
                                                 static_cast<uint32_t>(a.dim), &tiles_done, total_done, &p);
        if (abandoned) break;
        uint32_t* id = &a.ids[static_cast<uint64_t>(table) * a.ids_ld + row];
        const uint32_t exact = p >= 0.0 ? 1u : 0u;
        if (((__ldcg(id) >> bpos) & 1u) != exact) {
          const uint32_t old = atomicXor(id, 1u << bpos);
          if (a.fused_insert) {
            uint32_t* ct = a.counters + (static_cast<uint64_t>(table) << K);
            atomicSub(&ct[old], 1u);
            atomicAdd(&ct[old ^ (1u << bpos)], 1u);
          }
          ++ff_own;
        }
        ++rr_own;
        seg[i] = ~0ull;
        i += 64u;
      }
    }
    atomicMin(&min_next, i);
  } else {
#if ACE_SPLIT
    // ---------------- epilogue (warps 2-9), split direction tiles ----------------
    // Both warps of a TMEM lane quarter (q = warp % 4) work on every direction
    // tile: half h takes columns [h*TW/2, (h+1)*TW/2) in 64-column rounds
    // (two 32-column loads in flight, one for the 96-column half's last
    // round).  Per 32 columns: sign bits packed MSB-first, near ties by one
    // unsigned min over |v| (bits << 1), four independent chains for ILP.  The
    // tile's accumulator is released after half the per-warp work of the
    // whole-tile scheme, so the next MMA into it starts that much sooner.
    // Each half cuts the buckets of the tables ending in its columns; a table
    // straddling the halves needs half 0's last word, a table straddling the
    // previous tile that tile's last word (half 1): both are published in
    // shared memory around one 64-thread pair barrier (1+q) per tile.
    const uint32_t q = warp & 3, h = (warp - 2) >> 2;
    const uint32_t r = q * 32u + lane;
    const uint32_t kmask = (K >= 32u) ? 0xffffffffu : ((1u << K) - 1u);
    const uint32_t nacc = tc_acc_bufs(a.nkc, TW);
    const uint32_t hw = TW / 2u;      // columns per half (64 or 96)
    const uint32_t nwh = hw / 32u;    // sign words per half (2 or 3)
    const uint32_t nwords = TW / 32u;
    uint32_t acc = 0, accph = 0;
    uint64_t g = 0;
    long long pc_ext = 0;
    for (uint64_t it = 0; it < iters; ++it) {
      const uint64_t t = tile_of(it);
      const uint64_t row = t * kRows + r;
      const bool valid = row < a.n;
      float thr;
      if (kFuse) {
        const uint32_t p = static_cast<uint32_t>(it) & 1u;
        mbar_wait_sleepy(&bar_thrfull[p], static_cast<uint32_t>(it >> 1) & 1u, nullptr);
        thr = valid ? thr_sm[p][r] : -1.0f;
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_threempty[p]);
      } else {
        thr = valid ? a.rowthr[row] : -1.0f;
      }
      const bool zero_row = thr < 0.0f;
      const uint32_t thr_u = zero_row ? 0u : (isinf(thr) ? 0xffffffffu : (__float_as_uint(thr) << 1));
      for (uint32_t j = 0; j < a.ntiles; ++j, ++g) {
        const uint32_t used = min(TW, R - j * TW);
        const uint32_t hbase = h * hw;
        const uint32_t hused = used > hbase ? min(hw, used - hbase) : 0u;
        const uint32_t col0 = j * TW + hbase;
        // half 0: the previous tile's last word (half 1 wrote it before the
        // previous pair barrier and rewrites the slot only after this one)
        uint32_t prev = 0u;
        if (h == 0u && g > 0) prev = xw[q][1][(g - 1) & 1u][lane];
        mbar_wait_sleepy(&bar_accfull[acc], accph, (prof && lane == 0) ? &pw[5] : nullptr);
        pipe_after();
        long long pc0 = prof ? clock64() : 0, pc1 = 0, pc2 = 0;
        uint32_t wd0 = 0xffffffffu, wd1 = 0xffffffffu, wd2 = 0xffffffffu;
        if (!(a.dbg & 1)) {
#pragma unroll 1
          for (uint32_t hr = 0; hr < (nwh + 1u) / 2u; ++hr) {
            const uint32_t c0 = 64u * hr;
            if (c0 >= hused) break;
            const bool two = c0 + 32u < hw;  // the round's second 32-column group lies in this half
            uint32_t v[64];
            const uint32_t ta = tmem_base + ((q * 32u) << 16) + acc * TW + hbase + c0;
            ACE_TMEM_LD32(ta, v);
            if (two) ACE_TMEM_LD32(ta + 32u, (v + 32));
            tmem_wait_ld();
            if (prof && hr == 0) pc1 = clock64();
            uint32_t w2[2] = {0xffffffffu, 0xffffffffu};
#pragma unroll
            for (uint32_t g2 = 0; g2 < 2; ++g2) {
              if (g2 == 1u && !two) break;
              const uint32_t cc = c0 + 32u * g2;
              const uint32_t* vv = v + 32 * g2;
              // near-tie test on |v| as a float min (FMNMX3 with |.| operands: half an
              // instruction per column); NaN (non-finite rows, thr = inf) fails `mn > thr`
              uint32_t n4[4] = {0u, 0u, 0u, 0u};
              float m4[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
#pragma unroll
              for (int jj = 0; jj < 8; ++jj)
#pragma unroll
                for (int gq = 0; gq < 4; ++gq) {
                  n4[gq] = (n4[gq] << 1) | (vv[gq * 8 + jj] >> 31);
                  m4[gq] = fminf(m4[gq], fabsf(__uint_as_float(vv[gq * 8 + jj])));
                }
              const uint32_t neg = (n4[0] << 24) | (n4[1] << 16) | (n4[2] << 8) | n4[3];
              const float mn = fminf(fminf(m4[0], m4[1]), fminf(m4[2], m4[3]));
              // columns past `used` (padding / stale) are masked here, off the hot path
              if (!zero_row && valid && !(mn > thr) && cc < hused) {
                const uint32_t ncol = min(32u, hused - cc);
                uint32_t nm = 0u;
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) nm |= (((vv[jj] << 1) <= thr_u) ? 1u : 0u) << jj;
                if (ncol < 32u) nm &= (1u << ncol) - 1u;
                if (nm)
                  push_near_mask(a.st, a.near_list + blockIdx.x * seg_cap, seg_cap, &seg_n, a.overflow_rows, nm, row,
                                 col0 + cc);
              }
              w2[g2] = zero_row ? 0xffffffffu : ~neg;  // bit (31-jj) = column cc+jj >= 0
            }
            if (hr == 0) {
              wd0 = w2[0];
              wd1 = w2[1];
            } else {
              wd2 = w2[0];
            }
          }
        }
        pipe_before();
        __syncwarp();
        if (prof) pc2 = clock64();
        if (lane == 0) {
          if (rank == 0)
            mbar_arrive(&bar_accempty[acc]);
          else
            mbar_arrive_remote(&bar_accempty[acc], 0);  // the leader's MMA reuses our accumulator too
        }
        xw[q][h][g & 1u][lane] = nwh == 2u ? wd1 : wd2;  // this half's last word
        asm volatile("bar.sync %0, 64;" ::"r"(1u + q) : "memory");
        if (prof && lane == 0 && warp == 2) {
          const long long pc3 = clock64();
          atomicAdd(&a.prof[16], static_cast<unsigned long long>(pc1 - pc0));  // TMEM load + wait
          atomicAdd(&a.prof[17], static_cast<unsigned long long>(pc2 - pc1));  // sign / near processing
          atomicAdd(&a.prof[18], static_cast<unsigned long long>(pc3 - pc2));  // arrive + pair barrier
          pc_ext = pc3;
        }
        // buckets of the tables whose last column lies in this half
        const uint32_t tb = j == 0 ? 0u : a.tab_end[j - 1], te = a.tab_end[j];
        const uint32_t tm = min(max((j * TW + hw) / K, tb), te);  // tables ending before half 1
        const uint32_t t0 = h == 0u ? tb : tm, t1 = h == 0u ? tm : te;
        if (t0 < t1) {
          // word stream: the word before this half, then its own words; the
          // first table starts in one of the first two (K <= 32)
          const uint32_t s0 = t0 * K;
          uint32_t w0 = h == 0u ? prev : xw[q][0][g & 1u][lane], w1 = wd0, w2 = wd1, w3 = wd2, w4 = 0u;
          if (static_cast<int>(s0 >> 5) - static_cast<int>(j * nwords + h * nwh) >= 0) {
            w0 = w1; w1 = w2; w2 = w3; w3 = w4;
          }
          uint32_t off = s0 & 31u;
          uint32_t* idp = a.ids + row;
          for (uint32_t tt = t0; tt < t1; ++tt) {
            const unsigned long long win = (static_cast<unsigned long long>(w0) << 32) | w1;
            const uint32_t bucket = static_cast<uint32_t>(win >> (64u - off - K)) & kmask;
            if (valid) idp[static_cast<uint64_t>(tt) * a.ids_ld] = bucket;
            if (a.fused_insert) insert_bucket_warp(a.counters + (static_cast<uint64_t>(tt) << K), bucket, valid, lane);
            off += K;
            if (off >= 32u) {
              off -= 32u;
              w0 = w1; w1 = w2; w2 = w3; w3 = 0u;
            }
          }
        }
        if (prof && lane == 0 && warp == 2) atomicAdd(&a.prof[19], static_cast<unsigned long long>(clock64() - pc_ext));
        if (++acc == nacc) {
          acc = 0;
          accph ^= 1u;
        }
      }
      // this tile's ids (and near-list entries) are written: publish to the
      // recheck warps
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        atomicAdd(&tiles_done, 1u);
      }
    }
#else
    // ---------------- epilogue (warps 2-9) ----------------
    // Two warps per TMEM lane quarter (q = warp % 4) take alternate direction
    // tiles (global tile counter g, owner h = g & 1), all 128 columns each, in
    // two 64-column rounds (two 32-column loads in flight per round).  Per
    // 32 columns: sign bits packed MSB-first (one funnel shift per column),
    // near ties by one unsigned min over |v| (bits << 1), four independent
    // chains for ILP.  The four sign words stay in registers; buckets of the
    // tables ending in the tile are cut from them.  A table straddling the
    // previous tile needs that tile's last word, which the partner warp
    // publishes in shared memory (named barriers 1+q: h=0 -> h=1, 5+q:
    // h=1 -> h=0, one arrive / one sync per tile, strictly alternating).
    const uint32_t q = warp & 3, h = (warp - 2) >> 2;
    const uint32_t r = q * 32u + lane;
    const uint32_t kmask = (K >= 32u) ? 0xffffffffu : ((1u << K) - 1u);
    const uint32_t nacc = tc_acc_bufs(a.nkc, TW);
    const uint32_t nwords = TW / 32u;  // sign words per direction tile (4 or 6)
    const uint64_t g_total = iters * a.ntiles;
    uint32_t acc = 0, accph = 0;
    uint64_t g = 0;
    long long pc_ext = 0;
    for (uint64_t it = 0; it < iters; ++it) {
      const uint64_t t = tile_of(it);
      const uint64_t row = t * kRows + r;
      const bool valid = row < a.n;
      float thr;
      if (kFuse) {
        const uint32_t p = static_cast<uint32_t>(it) & 1u;
        mbar_wait_sleepy(&bar_thrfull[p], static_cast<uint32_t>(it >> 1) & 1u, nullptr);
        thr = valid ? thr_sm[p][r] : -1.0f;
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_threempty[p]);
      } else {
        thr = valid ? a.rowthr[row] : -1.0f;
      }
      const bool zero_row = thr < 0.0f;
      const uint32_t thr_u = zero_row ? 0u : (isinf(thr) ? 0xffffffffu : (__float_as_uint(thr) << 1));
      for (uint32_t j = 0; j < a.ntiles; ++j, ++g) {
        if ((g & 1u) == h) {
          const uint32_t used = min(TW, R - j * TW);
          const uint32_t col0 = j * TW;
          mbar_wait_sleepy(&bar_accfull[acc], accph, (prof && lane == 0) ? &pw[5] : nullptr);
          pipe_after();
          long long pc0 = prof ? clock64() : 0, pc1 = 0, pc2 = 0;
          uint32_t wd0 = 0xffffffffu, wd1 = 0xffffffffu, wd2 = 0xffffffffu, wd3 = 0xffffffffu;
          uint32_t wd4 = 0xffffffffu, wd5 = 0xffffffffu;
          if (!(a.dbg & 1)) {
            // one copy of the 64-column code (small instruction footprint)
#pragma unroll 1
            for (uint32_t hr = 0; hr < nwords / 2u; ++hr) {
              const uint32_t c0 = 64u * hr;
              if (c0 >= used) break;
              uint32_t v[64];
              ACE_TMEM_LD32(tmem_base + ((q * 32u) << 16) + acc * TW + c0, v);
              ACE_TMEM_LD32(tmem_base + ((q * 32u) << 16) + acc * TW + c0 + 32u, (v + 32));
              tmem_wait_ld();
              if (prof && hr == 0) pc1 = clock64();
              uint32_t w2[2];
              if (a.dbg & 16) {  // experiment: TMEM loads only
                w2[0] = v[0] ^ v[63];
                w2[1] = 0u;
              } else {
#pragma unroll
                for (uint32_t g2 = 0; g2 < 2; ++g2) {
                  const uint32_t cc = c0 + 32u * g2;
                  const uint32_t* vv = v + 32 * g2;
                  // near-tie test on |v| as a float min (FMNMX3 with |.| operands: half an
                  // instruction per column); NaN (non-finite rows, thr = inf) fails `mn > thr`
                  uint32_t n4[4] = {0u, 0u, 0u, 0u};
                  float m4[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
#pragma unroll
                  for (int jj = 0; jj < 8; ++jj)
#pragma unroll
                    for (int gq = 0; gq < 4; ++gq) {
                      n4[gq] = (n4[gq] << 1) | (vv[gq * 8 + jj] >> 31);
                      m4[gq] = fminf(m4[gq], fabsf(__uint_as_float(vv[gq * 8 + jj])));
                    }
                  const uint32_t neg = (n4[0] << 24) | (n4[1] << 16) | (n4[2] << 8) | n4[3];
                  const float mn = fminf(fminf(m4[0], m4[1]), fminf(m4[2], m4[3]));
                  // columns past `used` (padding / stale) are masked here, off the hot path
                  if (!zero_row && valid && !(mn > thr) && cc < used) {
                    const uint32_t ncol = min(32u, used - cc);
                    uint32_t nm = 0u;
#pragma unroll
                    for (int jj = 0; jj < 32; ++jj) nm |= (((vv[jj] << 1) <= thr_u) ? 1u : 0u) << jj;
                    if (ncol < 32u) nm &= (1u << ncol) - 1u;
                    if (nm)
                      push_near_mask(a.st, a.near_list + blockIdx.x * seg_cap, seg_cap, &seg_n, a.overflow_rows, nm,
                                     row, col0 + cc);
                  }
                  w2[g2] = zero_row ? 0xffffffffu : ~neg;  // bit (31-jj) = column cc+jj >= 0
                }
              }
              if (hr == 0) {
                wd0 = w2[0];
                wd1 = w2[1];
              } else if (hr == 1) {
                wd2 = w2[0];
                wd3 = w2[1];
              } else {
                wd4 = w2[0];
                wd5 = w2[1];
              }
            }
          }
          pipe_before();
          __syncwarp();
          if (prof) pc2 = clock64();
          if (lane == 0) {
            if (rank == 0)
              mbar_arrive(&bar_accempty[acc]);
            else
              mbar_arrive_remote(&bar_accempty[acc], 0);  // the leader's MMA reuses our accumulator too
          }
          // last word of the previous tile (partner warp), for a straddling table
          uint32_t prev = 0u;
          if (g > 0) {
            asm volatile("bar.sync %0, 64;" ::"r"((h == 1 ? 1u : 5u) + q) : "memory");
            prev = lastw[q][(g - 1) & 1u][lane];
          }
          if (prof && lane == 0 && warp == 2) {
            const long long pc3 = clock64();
            atomicAdd(&a.prof[16], static_cast<unsigned long long>(pc1 - pc0));  // TMEM load + wait
            atomicAdd(&a.prof[17], static_cast<unsigned long long>(pc2 - pc1));  // sign / near processing
            atomicAdd(&a.prof[18], static_cast<unsigned long long>(pc3 - pc2));  // arrive + partner barrier
            pc_ext = pc3;
          }
          // publish this tile's last word for the partner (next tile's owner)
          if (g + 1 < g_total) {
            lastw[q][g & 1u][lane] = nwords == 4u ? wd3 : wd5;
            asm volatile("bar.arrive %0, 64;" ::"r"((h == 0 ? 1u : 5u) + q) : "memory");
          }
          // buckets of the tables whose last column lies in this tile (host
          // precomputed range): bits [t*K, t*K+K) of the big-endian column
          // stream, words nwords*j-1 (prev) .. nwords*j+nwords-1 (wd)
          const uint32_t tb = j == 0 ? 0u : a.tab_end[j - 1], te = a.tab_end[j];
          uint32_t* idp = a.ids + row;
          if (tb < te) {
            // a window over the word stream prev, wd0, wd1, ...: the first
            // table starts in prev or wd0 (it ends in this tile, K <= 32);
            // each table reads the top two words, and the stream moves down
            // a word whenever the bit offset passes 32 (no dynamic indexing)
            const uint32_t s0 = tb * K;
            uint32_t w0 = prev, w1 = wd0, w2 = wd1, w3 = wd2, w4 = wd3, w5 = nwords == 4u ? 0u : wd4,
                     w6 = nwords == 4u ? 0u : wd5;
            if (static_cast<int>(s0 >> 5) - static_cast<int>(nwords * j) >= 0) {
              w0 = w1; w1 = w2; w2 = w3; w3 = w4; w4 = w5; w5 = w6; w6 = 0u;
            }
            uint32_t off = s0 & 31u;
            for (uint32_t tt = tb; tt < te; ++tt) {
              const unsigned long long win = (static_cast<unsigned long long>(w0) << 32) | w1;
              const uint32_t bucket = static_cast<uint32_t>(win >> (64u - off - K)) & kmask;
              if (valid && (!(a.dbg & 128) || bucket == 0xffffffffu)) idp[static_cast<uint64_t>(tt) * a.ids_ld] = bucket;
              if (a.fused_insert) insert_bucket_warp(a.counters + (static_cast<uint64_t>(tt) << K), bucket, valid, lane);
              off += K;
              if (off >= 32u) {
                off -= 32u;
                w0 = w1; w1 = w2; w2 = w3; w3 = w4; w4 = w5; w5 = w6; w6 = 0u;
              }
            }
          }
          if (prof && lane == 0 && warp == 2) atomicAdd(&a.prof[19], static_cast<unsigned long long>(clock64() - pc_ext));
        }
        if (++acc == nacc) {
          acc = 0;
          accph ^= 1u;
        }
      }
      // this tile's ids (and near-list entries) are written: publish to the
      // recheck warps
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        atomicAdd(&tiles_done, 1u);
      }
    }
#endif
  }

  if (warp >= 2) {
    // ---- shared tail: exact recheck (binary64 fold, srp.cpp:78-91) of the
    // list slots the recheck warps did not reach.  Wrong fast bits are flipped
    // in ids and, with the fused insert, the count moves from the old bucket
    // to the corrected one (counters commute).
    asm volatile("bar.sync 9, %0;" ::"r"(kTail) : "memory");  // epilogue done, recheck warps stopped
    if (prof && warp == 2) pw[8] = static_cast<unsigned long long>(clock64() - t_start);
    const uint32_t et = threadIdx.x - 64u;
    const uint32_t cnt = static_cast<uint32_t>(min(static_cast<unsigned long long>(seg_n), seg_cap));
    if (prof && et == 0) {
      atomicAdd(&a.prof[28], static_cast<unsigned long long>(min(min_next, cnt)));  // slots reached by the recheck warps
      atomicAdd(&a.prof[29], static_cast<unsigned long long>(cnt));                 // slots pushed
    }
    if (!(a.dbg & 32) && !a.ext_recheck)
      recheck_tail(a.x, a.x_f64, a.ld, static_cast<uint32_t>(a.dim), a.w64, a.ids, a.ids_ld, a.counters, a.fused_insert,
                   K, base, L.a_bytes + L.w_bytes, a.near_list + blockIdx.x * seg_cap, min(min_next, cnt), cnt, et,
                   rr_own, ff_own);
    rr_own = warp_sum_u64_tc(rr_own);
    ff_own = warp_sum_u64_tc(ff_own);
    if (lane == 0) {
      if (rr_own) atomicAdd(&blk_rech, rr_own);
      if (ff_own) atomicAdd(&blk_flip, ff_own);
    }
    asm volatile("bar.sync 9, %0;" ::"r"(kTail) : "memory");
    if (et == 0) {
      if (blk_rech) atomicAdd(&a.st->rechecked, blk_rech);
      if (blk_flip) atomicAdd(&a.st->flipped, blk_flip);
      if (seg_n) atomicAdd(&a.st->near_count, static_cast<unsigned long long>(seg_n));
      if (a.ext_recheck) a.seg_counts[blockIdx.x] = seg_n;
      if (a.fused_insert && blockIdx.x == 0) atomicAdd(&a.st->n, a.n);
    }
  }

  if (prof) {
    // [6] producer end [7] MMA end [8] epilogue main-loop end (warp 2)
    // [9] epilogue tail end (warp 2), cycles from t_start; [10] min start /
    // [11] max end of %globaltimer (ns) over CTAs
    const unsigned long long dt = static_cast<unsigned long long>(clock64() - t_start);
    if (lane == 0) {
      if (warp == 0) pw[6] = dt;
      if (warp == 1) pw[7] = dt;
      if (warp == 2) pw[9] = dt;
      for (int i = 0; i < 10; ++i)
        if (pw[i]) atomicAdd(&a.prof[i], pw[i]);
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      if (warp == 0) atomicMax(&a.prof[11], g);
      if (warp == 2) {
        atomicMax(&a.prof[12], pw[9]);
        atomicMax(&a.prof[13], pw[8]);
        atomicMax(&a.prof[14], static_cast<unsigned long long>(seg_n));
      }
      if (warp == 0) atomicMin(&a.prof[10], g_start);
    }
  }
  tc_before();
  __syncthreads();
  cluster_sync_all();  // no CTA leaves while its peers may still multicast into it
  tc_after();
  if (warp == 1) {
#if ACE_PAIR == 2
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
#else
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
#endif
  }
}

// ---- K-streamed projection (d > 256) -----------------------------------------------
//
// A point tile no longer fits on chip (d = 4096: 2 MB of fp16 hi + lo), so A
// is streamed in 64-wide K chunks next to the W chunks, one direction tile at
// a time.  Accumulation is chunked: kKsSc K chunks go into a TMEM accumulator
// (double-buffered), the epilogue adds the chunk results into fp32 running
// sums in registers (kTW / 2 columns per thread).  That keeps the rigorous error
// bound at (12 kKsSc + 16 + nchunks / 2) ulp instead of growing with d, so near
// ties stay rare; they are rechecked by recheck_segs_kernel afterwards.

#ifndef ACE_KS_TS
#define ACE_KS_TS 0  // K-streamed MMAs: 1 = A chunks copied into TMEM (TS), 0 = A from shared memory (SS)
#endif
constexpr uint32_t kKsSc = 2;                  // K chunks per accumulation pass
constexpr int kKsThreads = 320;                // producer, MMA, 8 epilogue warps
// Direction tile width kTW (MMA N): 256 (SS MMAs, two 256-column TMEM
// accumulators, ring of two 96 KB slots) or 128 (three 64 KB slots).  A ring
// slot holds one A chunk (hi | lo, 2 x 16 KB) and one W chunk (hi | lo).
template <uint32_t kTW>
struct KsCfg {
  static constexpr uint32_t kSlot = 2u * kBlockBytes + 2u * kTW * 128u;
  static constexpr uint32_t kSlots = kTW == 256 ? 2u : 3u;
  static constexpr uint32_t kCols = kTW / 2u;  // accumulator columns per epilogue warp (two per lane quarter)
  static constexpr uint32_t kWords = kTW / 32u;
};

__host__ __device__ inline uint32_t ks_chunks(uint32_t nkc) { return (nkc + kKsSc - 1) / kKsSc; }
__host__ inline size_t ks_smem_bytes(uint32_t tw) {
  return tw == 256 ? static_cast<size_t>(KsCfg<256>::kSlots) * KsCfg<256>::kSlot + 1024
                   : static_cast<size_t>(KsCfg<128>::kSlots) * KsCfg<128>::kSlot + 1024;
}

template <uint32_t kTW>
__global__ void __launch_bounds__(kKsThreads, 1) hash_tck_kernel(const TcArgs a) {
  using C = KsCfg<kTW>;
  constexpr uint32_t kKsSlot = C::kSlot, kKsSlots = C::kSlots, kCW = C::kCols;
  static_assert(!(ACE_KS_TS && kTW != 128), "TS K-streamed MMAs need 128-direction tiles");
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bar_full[kKsSlots], bar_empty[kKsSlots], bar_accfull[2], bar_accempty[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ uint32_t sgbuf[2][C::kWords][kRows];  // sign words of a direction tile, by tile parity
  __shared__ uint32_t seg_n;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t n_tiles = (a.n + kRows - 1) / kRows;
  const uint32_t K = a.k_bits, nkc = a.nkc, nch = ks_chunks(nkc);
  const uint32_t R = a.k_bits * a.tables;
  if (threadIdx.x == 0) {
    seg_n = 0;
    for (uint32_t i = 0; i < kKsSlots; ++i) {
      mbar_init(&bar_full[i], 1);
      mbar_init(&bar_empty[i], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar_accfull[b], 1);
      mbar_init(&bar_accempty[b], 8);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem_base = tmem_base_sh;
  // work items (point tile t, direction tile j), j fastest: the CTAs running
  // side by side share few point tiles, so A chunks are re-read from L2
  const uint64_t n_items = n_tiles * a.ntiles;
  const uint64_t iters = (n_items + gridDim.x - 1) / gridDim.x;
  const unsigned long long seg_cap = a.near_cap / gridDim.x;
  const uint32_t tpt = a.tpt;  // whole tables per direction tile

  if (warp == 0) {
    // ---- producer: per (tile, direction tile, K chunk) one A chunk + one W chunk
    if (lane == 0) {
      uint32_t s = 0, ph = 0;
      for (uint64_t it = 0; it < iters; ++it) {
        const uint64_t w = min(blockIdx.x + it * gridDim.x, n_items - 1);  // past the end: redo the last item
        const uint64_t tt = w / a.ntiles;
        const uint32_t j = static_cast<uint32_t>(w % a.ntiles);
          for (uint32_t kc = 0; kc < nkc; ++kc) {
            mbar_wait_sleepy(&bar_empty[s], ph ^ 1u, nullptr);
            mbar_expect_tx(&bar_full[s], kKsSlot);
            uint8_t* dst = base + static_cast<size_t>(s) * kKsSlot;
            bulk_g2s(dst, reinterpret_cast<const uint8_t*>(a.x16) + (tt * nkc + kc) * 2u * kBlockBytes,
                     2u * kBlockBytes, &bar_full[s]);
            bulk_g2s(dst + 2u * kBlockBytes,
                     reinterpret_cast<const uint8_t*>(a.w16) + (static_cast<uint64_t>(j) * nkc + kc) * 2u * kTW * 128u,
                     2u * kTW * 128u, &bar_full[s]);
            if (++s == kKsSlots) {
              s = 0;
              ph ^= 1u;
            }
          }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: 12 MMAs per K chunk (SS, or TS with the A chunk copied
    // into a double-buffered TMEM region)
    uint32_t s = 0, ph = 0, ab = 0, abph = 0;
    const uint32_t ta = tmem_base + 256u;  // TS: A buffers [2][hi 32 | lo 32 columns]
    (void)ta;
    const uint32_t idesc = idesc_f16(kTW);
    for (uint64_t it = 0; it < iters; ++it)
        for (uint32_t c = 0; c < nch; ++c) {
          mbar_wait(&bar_accempty[ab], abph ^ 1u);
          pipe_after();
          const uint32_t k0 = c * kKsSc, k1 = min(nkc, k0 + kKsSc);
          const uint32_t dt = tmem_base + ab * kTW;
          if (elect_one()) {
            uint32_t ss = s, pp = ph;
            for (uint32_t kc = k0; kc < k1; ++kc) {
              mbar_wait(&bar_full[ss], pp);
              const uint32_t sa = smem_u32(base + static_cast<size_t>(ss) * kKsSlot);
              const uint64_t dbh = sw128_desc(sa + 2u * kBlockBytes), dbl = sw128_desc(sa + 2u * kBlockBytes + kTW * 128u);
#if ACE_KS_TS
              const uint32_t tb = ta + (kc & 1u) * 64u;
#pragma unroll
              for (uint32_t kk = 0; kk < 4; ++kk) {
                tmem_cp_128x256b(tb + kk * 8u, sw128_desc(sa + kk * 32u));
                tmem_cp_128x256b(tb + 32u + kk * 8u, sw128_desc(sa + kBlockBytes + kk * 32u));
              }
#pragma unroll
              for (uint32_t kk = 0; kk < 4; ++kk) {
                const uint64_t off = kk * 2u;
                mma_f16_ts(dt, tb + kk * 8u, dbh + off, idesc, (kc != k0 || kk != 0u) ? 1u : 0u);
                mma_f16_ts(dt, tb + 32u + kk * 8u, dbh + off, idesc, 1u);
                mma_f16_ts(dt, tb + kk * 8u, dbl + off, idesc, 1u);
              }
#else
              // A read from the slot by the MMAs themselves (no copy into TMEM)
              const uint64_t dah = sw128_desc(sa), dal = sw128_desc(sa + kBlockBytes);
#pragma unroll
              for (uint32_t kk = 0; kk < 4; ++kk) {
                const uint64_t off = kk * 2u;
                mma_f16_ss(dt, dah + off, dbh + off, idesc, (kc != k0 || kk != 0u) ? 1u : 0u);
                mma_f16_ss(dt, dal + off, dbh + off, idesc, 1u);
                mma_f16_ss(dt, dah + off, dbl + off, idesc, 1u);
              }
#endif
              mma_commit(&bar_empty[ss]);
              if (++ss == kKsSlots) {
                ss = 0;
                pp ^= 1u;
              }
            }
            mma_commit(&bar_accfull[ab]);
          }
          __syncwarp();
          for (uint32_t kc = k0; kc < k1; ++kc)
            if (++s == kKsSlots) {
              s = 0;
              ph ^= 1u;
            }
          ab ^= 1u;
          if (ab == 0) abph ^= 1u;
        }
  } else {
    // ---- epilogue (warps 2-9): two warps per lane quarter, kCW columns each
    const uint32_t q = warp & 3, h = (warp - 2) >> 2;
    const uint32_t r = q * 32u + lane;
    const uint32_t kmask = (K >= 32u) ? 0xffffffffu : ((1u << K) - 1u);
    uint32_t ab = 0, abph = 0, par = 0;
    for (uint64_t it = 0; it < iters; ++it, par ^= 1u) {
      const uint64_t w = blockIdx.x + it * gridDim.x;
      const bool live_item = w < n_items;
      const uint64_t t = (live_item ? w : n_items - 1) / a.ntiles;
      const uint32_t j = static_cast<uint32_t>((live_item ? w : n_items - 1) % a.ntiles);
      const uint64_t row = t * kRows + r;
      const bool valid = live_item && row < a.n;
      const float thr = valid ? a.rowthr[row] : -1.0f;
      const bool zero_row = thr < 0.0f;
      const uint32_t t0 = j * tpt, t1 = min(a.tables, t0 + tpt);  // tables of this direction tile
      const uint32_t used = (t1 - t0) * K;
      {
        float acc[kCW];
#pragma unroll
        for (int i = 0; i < static_cast<int>(kCW); ++i) acc[i] = 0.0f;
        for (uint32_t c = 0; c < nch; ++c) {
          mbar_wait_sleepy(&bar_accfull[ab], abph, nullptr);
          pipe_after();
          // kR columns per round (kR / 32 loads in flight; 32 when the
          // running sums take 128 registers)
          constexpr uint32_t kR = kCW > 64u ? 32u : 64u;
#pragma unroll
          for (uint32_t p0 = 0; p0 < kCW; p0 += kR) {
            uint32_t v[kR];
            const uint32_t ta = tmem_base + ((q * 32u) << 16) + ab * kTW + kCW * h + p0;
            ACE_TMEM_LD32(ta, v);
            if constexpr (kR == 64u) ACE_TMEM_LD32(ta + 32u, (v + 32));
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < static_cast<int>(kR); ++i) acc[p0 + i] += __uint_as_float(v[i]);
          }
          pipe_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar_accempty[ab]);
          ab ^= 1u;
          if (ab == 0) abph ^= 1u;
        }
        // sign words and near masks of all columns first (the running sums
        // are dead before the out-of-line pushes: no registers to save)
        uint32_t nms[kCW / 32u];
#pragma unroll
        for (uint32_t g2 = 0; g2 < kCW / 32u; ++g2) {
          uint32_t neg = 0u, nm = 0u;
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const float p = acc[32 * g2 + jj];
            neg = (neg << 1) | (__float_as_uint(p) >> 31);
            nm |= ((!(fabsf(p) > thr)) ? 1u : 0u) << jj;  // NaN projections (wild rows) count as near
          }
          nms[g2] = nm;
          sgbuf[par][(kCW / 32u) * h + g2][r] = zero_row ? 0xffffffffu : ~neg;  // bit (31-jj) = column cc+jj >= 0
        }
#pragma unroll
        for (uint32_t g2 = 0; g2 < kCW / 32u; ++g2) {
          const uint32_t cc = kCW * h + 32u * g2;
          uint32_t nm = nms[g2];
          if (cc < used && !zero_row && valid) {
            if (used - cc < 32u) nm &= (1u << (used - cc)) - 1u;
            if (nm)
              push_near_mask(a.st, a.near_list + blockIdx.x * seg_cap, seg_cap, &seg_n, a.overflow_rows, nm, row,
                             t0 * K + cc);
          }
        }
        asm volatile("bar.sync %0, 64;" ::"r"(1u + q) : "memory");  // the quarter's two warps
        uint32_t* idp = a.ids + row;
        for (uint32_t tt = t0 + h; tt < t1; tt += 2) {
          const uint32_t s0 = (tt - t0) * K;  // whole tables: no straddling
          const uint32_t wi = s0 >> 5, off = s0 & 31u;
          const uint32_t hi = sgbuf[par][wi][r];
          const uint32_t lo = wi + 1u < C::kWords ? sgbuf[par][wi + 1][r] : 0u;
          const unsigned long long win = (static_cast<unsigned long long>(hi) << 32) | lo;
          const uint32_t bucket = static_cast<uint32_t>(win >> (64u - off - K)) & kmask;
          if (valid) idp[static_cast<uint64_t>(tt) * a.ids_ld] = bucket;
        }
      }
    }
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (threadIdx.x == 0) {
    a.seg_counts[blockIdx.x] = seg_n;
    if (seg_n) atomicAdd(&a.st->near_count, static_cast<unsigned long long>(seg_n));
  }
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
}

// Conversion for the K-streamed path: one warp per row, any d.  With fp32
// rows of 16-byte multiples the row is read as float4 (held in registers for
// both passes when d <= 4096).
__device__ __forceinline__ void wide_store(const TcArgs& a, uint64_t tile, uint32_t r, uint32_t k, float x0, float x1,
                                           float x2, float x3, float& ss) {
  ss = fmaf(x0, x0, fmaf(x1, x1, fmaf(x2, x2, fmaf(x3, x3, ss))));
  const float h0 = __half2float(__float2half_rn(x0)), h1 = __half2float(__float2half_rn(x1));
  const float h2 = __half2float(__float2half_rn(x2)), h3 = __half2float(__float2half_rn(x3));
  uint8_t* blk = reinterpret_cast<uint8_t*>(a.x16) + ((tile * a.nkc + k / kChunk) * 2u) * kBlockBytes;
  const uint32_t off = sw128_off(r, k % kChunk);
  *reinterpret_cast<uint2*>(blk + off) = make_uint2(pack_h2(h0, h1), pack_h2(h2, h3));
  *reinterpret_cast<uint2*>(blk + kBlockBytes + off) = make_uint2(pack_h2(x0 - h0, x1 - h1), pack_h2(x2 - h2, x3 - h3));
}

__global__ void __launch_bounds__(256) convert_x_wide_kernel(const TcArgs a, uint64_t rows_padded) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  const uint32_t dpad = a.nkc * kChunk;
  const bool vec = !a.x_f64 && (a.dim % 4 == 0) && (a.ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0) &&
                   dpad <= 4096;
  for (uint64_t row = static_cast<uint64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows_padded;
       row += warps) {
    const bool live = row < a.n;
    const uint64_t tile = row / kRows;
    const uint32_t r = static_cast<uint32_t>(row % kRows);
    if (vec) {
      // lane owns float4 groups lane, lane + 32, ... (k = 4 * group)
      float4 v[32];
      uint32_t mb = 0u;
      const float4* xr = reinterpret_cast<const float4*>(static_cast<const float*>(a.x) + row * a.ld);
#pragma unroll
      for (uint32_t i = 0; i < 32; ++i) {
        const uint32_t g = lane + 32u * i;
        v[i] = (live && 4u * g < a.dim) ? xr[g] : make_float4(0.f, 0.f, 0.f, 0.f);
        mb = max(mb, max(max(__float_as_uint(v[i].x) & 0x7fffffffu, __float_as_uint(v[i].y) & 0x7fffffffu),
                         max(__float_as_uint(v[i].z) & 0x7fffffffu, __float_as_uint(v[i].w) & 0x7fffffffu)));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, o));
      const bool nan = mb > 0x7f800000u;
      const float m = __uint_as_float(nan ? 0x7f800000u : mb);
      const bool zero = (m == 0.0f);
      const bool wild = nan || !(m < 0x1.0p100f) || (!zero && m < 0x1.0p-100f);
      float scale = 0.0f;
      if (live && !zero && !wild) {
        const int e = static_cast<int>((__float_as_uint(m) >> 23) & 0xffu) - 127;
        scale = __uint_as_float(static_cast<uint32_t>(127 + 14 - e) << 23);
      }
      float ss = 0.0f;
#pragma unroll
      for (uint32_t i = 0; i < 32; ++i) {
        const uint32_t k = 4u * (lane + 32u * i);
        if (k < dpad)
          wide_store(a, tile, r, k, v[i].x * scale, v[i].y * scale, v[i].z * scale, v[i].w * scale, ss);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) {
        float thr;
        if (!live || zero) {
          thr = -1.0f;
        } else if (wild) {
          thr = __int_as_float(0x7f800000);
        } else {
          const float nx = sqrtf(ss * (1.0f + static_cast<float>(a.dim + 4) * 0x1.0p-23f)) * (1.0f + 0x1.0p-20f);
          thr = a.margin_c * nx * 16384.0f + static_cast<float>(a.dim) * 0x1.0p-10f;
        }
        a.rowthr[row] = thr;
      }
      continue;
    }
    uint32_t mb = 0u;
    if (live)
      for (uint32_t k = lane; k < a.dim; k += 32u) mb = max(mb, __float_as_uint(load_x(a, row, k)) & 0x7fffffffu);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, o));
    const bool nan = mb > 0x7f800000u;
    const float m = __uint_as_float(nan ? 0x7f800000u : mb);
    const bool zero = (m == 0.0f);
    const bool wild = nan || !(m < 0x1.0p100f) || (!zero && m < 0x1.0p-100f);
    float scale = 0.0f;
    if (live && !zero && !wild) {
      const int e = static_cast<int>((__float_as_uint(m) >> 23) & 0xffu) - 127;
      scale = __uint_as_float(static_cast<uint32_t>(127 + 14 - e) << 23);
    }
    float ss = 0.0f;
    for (uint32_t k = 4u * lane; k < dpad; k += 128u) {
      float xv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) xv[e] = (live ? load_x(a, row, k + e) : 0.0f) * scale;
      wide_store(a, tile, r, k, xv[0], xv[1], xv[2], xv[3], ss);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) {
      float thr;
      if (!live || zero) {
        thr = -1.0f;
      } else if (wild) {
        thr = __int_as_float(0x7f800000);
      } else {
        const float nx = sqrtf(ss * (1.0f + static_cast<float>(a.dim + 4) * 0x1.0p-23f)) * (1.0f + 0x1.0p-20f);
        thr = a.margin_c * nx * 16384.0f + static_cast<float>(a.dim) * 0x1.0p-10f;
      }
      a.rowthr[row] = thr;
    }
  }
}

__global__ void w32_round_kernel(const double* __restrict__ w64, uint64_t n, float* __restrict__ w32) {
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    w32[i] = static_cast<float>(w64[i]);
}

// Near ties of the K-streamed kernel, one warp per list item, kKsRbPerSeg
// blocks per CTA segment.  Stage 1: p1 = sum x_i w32_i in binary64 (the
// products of two fp32 values are exact), w32 = w rounded to fp32, and
// A = sum |x_i w32_i|.  |p1 - sum x_i w_i| <= 2^-24 (1 + 2^-23) A + gamma_d A
// and the reference's left fold is within gamma_d sum |x_i w_i| of the exact
// value, so |p1| above the sum of both decides the reference's sign.
// Stage 2 (rare): the reference's sequential binary64 fold (srp.cpp:78-91).
constexpr uint32_t kKsRbPerSeg = 8;

__global__ void __launch_bounds__(256) recheck_segs_kernel(const TcArgs a, uint32_t grid) {
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const unsigned long long seg_cap = a.near_cap / grid;
  const uint32_t K = a.k_bits;
  const uint32_t dim = static_cast<uint32_t>(a.dim);
  const double gam = static_cast<double>(dim + 2) * 0x1.0p-53 / (1.0 - static_cast<double>(dim + 2) * 0x1.0p-53);
  const double bound_rel = (0x1.0p-24 * (1.0 + 0x1.0p-22) + 3.0 * gam) * (1.0 + 4.0 * gam);
  const bool vec = !a.x_f64 && (dim % 4 == 0) && (a.ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0);
  unsigned long long rr = 0, ff = 0;
  const uint32_t b = blockIdx.x / kKsRbPerSeg, sub = blockIdx.x % kKsRbPerSeg;
  if (b < grid) {
    unsigned long long* seg = a.near_list + b * seg_cap;
    const uint32_t cnt = static_cast<uint32_t>(min(static_cast<unsigned long long>(a.seg_counts[b]), seg_cap));
    const uint32_t stride = kKsRbPerSeg * (blockDim.x >> 5);
    for (uint32_t i = sub * (blockDim.x >> 5) + wib; i < cnt; i += stride) {
      const unsigned long long item = seg[i];
      const uint64_t row = item >> 32;
      const uint32_t dir = static_cast<uint32_t>(item & 0xffffffffu);
      const float* w = a.w32 + static_cast<uint64_t>(dir) * dim;
      double p = 0.0, ab = 0.0;
      if (vec) {
        const float4* xr = reinterpret_cast<const float4*>(static_cast<const float*>(a.x) + row * a.ld);
        const float4* wr = reinterpret_cast<const float4*>(w);
#pragma unroll 4
        for (uint32_t k = lane; k < dim / 4u; k += 32u) {
          const float4 xv = xr[k], wv = __ldg(wr + k);
          const double t0 = static_cast<double>(xv.x) * wv.x, t1 = static_cast<double>(xv.y) * wv.y;
          const double t2 = static_cast<double>(xv.z) * wv.z, t3 = static_cast<double>(xv.w) * wv.w;
          p += (t0 + t1) + (t2 + t3);
          ab += (fabs(t0) + fabs(t1)) + (fabs(t2) + fabs(t3));
        }
      } else {
        for (uint32_t k = lane; k < dim; k += 32u) {
          const double xv = a.x_f64 ? static_cast<const double*>(a.x)[row * a.ld + k]
                                    : static_cast<double>(static_cast<const float*>(a.x)[row * a.ld + k]);
          const double t = xv * static_cast<double>(__ldg(w + k));  // x fp64 input: products rounded (in gam)
          p += t;
          ab += fabs(t);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        p += __shfl_xor_sync(0xffffffffu, p, o);
        ab += __shfl_xor_sync(0xffffffffu, ab, o);
      }
      int bit;
      if (fabs(p) > bound_rel * ab + 0x1.0p-1000) {
        bit = p >= 0.0 ? 1 : 0;
      } else {
        double e = 0.0;
        if (lane == 0) e = exact_proj(a.w64 + static_cast<uint64_t>(dir) * dim, a.x, a.x_f64, row, a.ld, dim);
        e = __shfl_sync(0xffffffffu, e, 0);
        bit = e >= 0.0 ? 1 : 0;
      }
      if (lane == 0) {
        const uint32_t table = dir / K, bpos = K - 1u - dir % K;
        uint32_t* id = &a.ids[static_cast<uint64_t>(table) * a.ids_ld + row];
        if (static_cast<int>((*id >> bpos) & 1u) != bit) {
          atomicXor(id, 1u << bpos);
          ++ff;
        }
        ++rr;
        seg[i] = ~0ull;  // the list is all ~0 between launches
      }
    }
  }
  if (lane == 0) {
    if (rr) atomicAdd(&a.st->rechecked, rr);
    if (ff) atomicAdd(&a.st->flipped, ff);
  }
}

// ---- near-tie recheck ------------------------------------------------------------

// rows whose near ties overflowed the list: every bucket recomputed exactly
__global__ void recheck_rows_kernel(const TcArgs a, const double* __restrict__ w64) {
  if (!a.st->near_overflow) return;
  const uint32_t K = a.k_bits;
  for (uint64_t idx = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < a.n * a.tables;
       idx += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t row = idx / a.tables;
    const uint32_t table = static_cast<uint32_t>(idx % a.tables);
    if (!((a.overflow_rows[row >> 5] >> (row & 31)) & 1u)) continue;
    uint32_t bucket = 0;
    for (uint32_t b = 0; b < K; ++b) {
      const double p = exact_proj(w64 + (static_cast<uint64_t>(table) * K + b) * a.dim, a.x, a.x_f64, row,
                                  a.ld, a.dim);
      bucket = (bucket << 1) | (p >= 0.0 ? 1u : 0u);
    }
    uint32_t* id = &a.ids[static_cast<uint64_t>(table) * a.ids_ld + row];
    const uint32_t old = *id;
    *id = bucket;
    if (a.fused_insert && old != bucket) {
      uint32_t* ct = a.counters + (static_cast<uint64_t>(table) << K);
      atomicSub(&ct[old], 1u);
      atomicAdd(&ct[bucket], 1u);
    }
    atomicAdd(&a.st->rechecked, static_cast<unsigned long long>(K));
  }
}

// ---- W preparation ------------------------------------------------------------------

__global__ void dir_norm_kernel(const double* __restrict__ w64, uint64_t dim, uint32_t rows, double* inv) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double s = 0.0;
  for (uint64_t i = 0; i < dim; ++i) s += w64[r * dim + i] * w64[r * dim + i];
  inv[r] = s > 0.0 ? 16384.0 / sqrt(s) : 0.0;
}

// Direction tile j holds directions j*dpt .. j*dpt + dpt - 1 in rows 0..dpt-1
// (dpt = tw: packed densely; dpt = tables-per-tile * K: whole tables per tile,
// the K-streamed kernel), zero rows beyond.
__global__ void pack_w16_kernel(const double* __restrict__ w64, const double* __restrict__ inv,
                                FamilyDev f, uint32_t ntiles, uint32_t nkc, uint32_t tw, uint32_t dpt, uint16_t* w16) {
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

}  // namespace

bool tc_supported(uint64_t dim) { return dim >= 1 && dim <= 8192; }
bool tc_kstream(uint32_t nkc) { return nkc > 4; }
// The in-kernel conversion needs whole 16-byte rows and room for a raw tile
// next to the A image and at least two W stages.
bool tc_fuse_ok_dim(uint64_t dim, uint32_t nkc) {
  return kPair == 1 && dim % 4 == 0 && nkc <= 2 && tc_layout(nkc, dim, true).n_wst >= 2;
}

void tc_fill_tables(TcArgs* a) {
  for (uint32_t j = 0; j < a->ntiles && j < 64; ++j) {
    const uint32_t end_col = std::min((j + 1) * a->tw, a->k_bits * a->tables);
    a->tab_end[j] = static_cast<uint16_t>(std::min(end_col / a->k_bits, a->tables));
  }
}

size_t tc_smem_bytes(uint32_t nkc) { return tc_layout(nkc).total; }

cudaError_t tc_prepare_family(const FamilyDev& f, TcFamily* tc) {
  tc->enabled = 0;
  if (!tc_supported(f.dim) || f.k_bits > 128) return cudaSuccess;
  const uint32_t nkc = static_cast<uint32_t>((f.dim + kChunk - 1) / kChunk);
  // 192-direction tiles (MMA N = 192, two accumulators) for d <= 128: a third
  // fewer MMA instructions and epilogue hand-offs than 128-direction tiles
  static int tw_env = -1;
  if (tw_env < 0) {
    const char* e = getenv("ACE_TW");
    tw_env = e ? atoi(e) : 192;
  }
  const uint32_t tw = (kPair == 1 && nkc <= 2 && tw_env == 192) ? 192u : 128u;
  const TcLayout L = tc_layout(nkc, 0, false, tw);
  if ((!tc_kstream(nkc) && L.n_wst < 2) || (tc_kstream(nkc) && kPair != 1)) return cudaSuccess;
  tc->nkc = nkc;
  tc->tw = tw;
  // K-streamed kernel: whole tables per direction tile (no table straddles
  // two tiles, so (point tile, direction tile) items are independent)
  // 256-direction tiles (SS MMAs with N = 256) unless ACE_KS_TW=128
  static int kstw_env = -1;
  if (kstw_env < 0) {
    const char* e = getenv("ACE_KS_TW");
    kstw_env = e ? atoi(e) : 256;
  }
  const uint32_t ktw = (ACE_KS_TS || kstw_env == 128) ? 128u : 256u;
  const uint32_t wtw = tc_kstream(nkc) ? ktw : tw;  // W tile rows
  const uint32_t tpt = wtw / f.k_bits;
  if (tc_kstream(nkc)) {
    tc->tw = wtw;
    tc->tpt = tpt;
  }
  const uint32_t dpt = tc_kstream(nkc) ? tpt * f.k_bits : tw;
  tc->ntiles = tc_kstream(nkc) ? (f.tables + tpt - 1) / tpt : (f.rows + tw - 1) / tw;
  if (tc->ntiles > 64 && !tc_kstream(nkc)) return cudaSuccess;  // TcArgs::tab_end
  const size_t bytes = static_cast<size_t>(tc->ntiles) * nkc * 2 * wtw * 128u;
  cudaError_t e = cudaMalloc(&tc->w16, bytes);
  if (e != cudaSuccess) return e;
  double* inv = nullptr;
  if ((e = cudaMalloc(&inv, sizeof(double) * f.rows)) != cudaSuccess) return e;
  dir_norm_kernel<<<(f.rows + 127) / 128, 128>>>(f.w64, f.dim, f.rows, inv);
  pack_w16_kernel<<<1024, 256>>>(f.w64, inv, f, tc->ntiles, nkc, wtw, dpt, tc->w16);
  count_launch(2);
  e = cudaDeviceSynchronize();
  cudaFree(inv);
  if (e != cudaSuccess) return e;
  e = cudaMalloc(&tc->w32, sizeof(float) * f.rows * f.dim);
  if (e != cudaSuccess) return e;
  w32_round_kernel<<<1024, 256>>>(f.w64, static_cast<uint64_t>(f.rows) * f.dim, tc->w32);
  count_launch();
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return e;
  if (tc_kstream(nkc)) {
    e = wtw == 256 ? cudaFuncSetAttribute(hash_tck_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(ks_smem_bytes(256)))
                   : cudaFuncSetAttribute(hash_tck_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(ks_smem_bytes(128)));
    if (e != cudaSuccess) return e;
    tc->enabled = 1;
    return cudaSuccess;
  }
  e = cudaFuncSetAttribute(hash_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(L.total));
  if (e != cudaSuccess) return e;
  if (tw == 128 && tc_fuse_ok_dim(f.dim, tc->nkc)) {
    e = cudaFuncSetAttribute(hash_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(tc_layout(tc->nkc, f.dim, true).total));
    if (e != cudaSuccess) return e;
  }
  tc->enabled = 1;
  return cudaSuccess;
}

void tc_free_family(TcFamily* tc) {
  if (tc->w16) cudaFree(tc->w16);
  tc->w16 = nullptr;
  if (tc->w32) cudaFree(tc->w32);
  tc->w32 = nullptr;
  tc->enabled = 0;
}

cudaError_t launch_hash_tc(const TcArgs& a, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const uint64_t tiles = (a.n + kRows - 1) / kRows;
  uint64_t grid = tiles < static_cast<uint64_t>(sms) ? tiles : static_cast<uint64_t>(sms);
  grid = (grid + kCluster - 1) / kCluster * kCluster;
  if (grid > static_cast<uint64_t>(sms)) grid = static_cast<uint64_t>(sms) / kCluster * kCluster;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = tc_layout(a.nkc, a.dim, a.fuse_convert != 0, a.tw).total;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = a.fuse_convert ? cudaLaunchKernelEx(&cfg, hash_tc_kernel<true>, a)
                                 : cudaLaunchKernelEx(&cfg, hash_tc_kernel<false>, a);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_convert_x(const TcArgs& a, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const uint64_t rows = (a.n + kRows - 1) / kRows * kRows;
  uint64_t blocks = (rows + 31) / 32;  // 32 rows per 256-thread block
  if (blocks > static_cast<uint64_t>(sms) * 16) blocks = static_cast<uint64_t>(sms) * 16;
  const uint32_t groups = a.nkc * 2u;
  if (groups <= 2)
    convert_x_kernel<2><<<static_cast<unsigned>(blocks), 256, 0, s>>>(a, rows);
  else if (groups <= 4)
    convert_x_kernel<4><<<static_cast<unsigned>(blocks), 256, 0, s>>>(a, rows);
  else
    convert_x_kernel<8><<<static_cast<unsigned>(blocks), 256, 0, s>>>(a, rows);
  count_launch();
  return cudaGetLastError();
}

static int tc_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

uint32_t tck_grid(uint64_t n) {
  const uint64_t tiles = (n + kRows - 1) / kRows;
  return static_cast<uint32_t>(tiles < static_cast<uint64_t>(tc_sms()) ? tiles : tc_sms());
}

cudaError_t launch_convert_x_wide(const TcArgs& a, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  const uint64_t rows = (a.n + kRows - 1) / kRows * kRows;
  uint64_t blocks = (rows + 7) / 8;  // 8 rows (warps) per block
  if (blocks > static_cast<uint64_t>(tc_sms()) * 16) blocks = static_cast<uint64_t>(tc_sms()) * 16;
  convert_x_wide_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(a, rows);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_hash_tck(const TcArgs& a, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  if (a.tw == 256)
    hash_tck_kernel<256><<<tck_grid(a.n), kKsThreads, ks_smem_bytes(256), s>>>(a);
  else
    hash_tck_kernel<128><<<tck_grid(a.n), kKsThreads, ks_smem_bytes(128), s>>>(a);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_recheck_segs(const TcArgs& a, cudaStream_t s) {
  if (a.n == 0) return cudaSuccess;
  const uint32_t grid = tck_grid(a.n);
  recheck_segs_kernel<<<grid * kKsRbPerSeg, 256, 0, s>>>(a, grid);
  count_launch();
  return cudaGetLastError();
}

// The chunk results are added in fp32 registers with round-to-nearest (the
// epilogue's FADD): each partial sum is bounded by ||x~|| ||w^|| (Cauchy-
// Schwarz over the chunks), so each add errs by at most 2^-24 of it, half the
// 2^-23 allowed for each (truncating) tensor-core accumulation step.
float tck_margin(uint32_t nkc, bool x_f64) {
  return static_cast<float>(2.0 * (4.0 * 0x1.0p-22 +
                                   (0x1.0p-23 * (12.0 * kKsSc + 16.0) + 0x1.0p-24 * ks_chunks(nkc)) * 1.01 +
                                   (x_f64 ? 0x1.0p-23 : 0.0)));
}

cudaError_t launch_recheck(const TcArgs& a, const double* w64, cudaStream_t s) {
  recheck_rows_kernel<<<148, 256, 0, s>>>(a, w64);  // exits at once unless a list segment overflowed
  count_launch(1);
  return cudaGetLastError();
}

}  // namespace ace_dev
