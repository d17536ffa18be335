// PTX wrappers shared by the tcgen05 projection kernels (ace_hash_tc.cu,
// ace_hash_tck.cu): mbarriers, bulk / tensor-map TMA copies, tcgen05 MMA,
// TMEM load / store / copy, shared-memory matrix descriptors, and the exact
// binary64 fold of the reference (srp.cpp:78-91) used by the rechecks.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ace_tc.cuh"

namespace ace_dev {
namespace tc {

constexpr int kRows = 128;                // points per tile (MMA M)
constexpr int kChunk = 64;                // K elements per W chunk (128 B of fp16)
constexpr int kBlockBytes = kRows * 128;  // one 128 x 64 fp16 SW128 block = 16 KB
constexpr size_t kSmemLimit = 232448;     // 227 KB dynamic + static per CTA

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
// Spin until the phase with `parity` completes (critical-path waits).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Waits off the critical MMA path back off between polls so the polling does
// not compete with the busy warps for issue slots.  (A try_wait suspend-time
// hint instead of the back-off measured slower: 145.7 vs 137.3 us per
// 262,144-row cfg-5 hashing launch.)
__device__ __forceinline__ void mbar_wait_sleepy(uint64_t* bar, uint32_t parity) {
  while (!mbar_try(bar, parity)) __nanosleep(64);
}

// 1-D bulk copy global -> shared (TMA engine), completion on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// 2-D tensor-map TMA load of one box (coordinates c0 innermost), completion
// on an mbarrier; the L2 policy marks the streamed rows evict-first.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
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
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t base, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols));
}

// K-major SWIZZLE_128B shared-memory matrix descriptor (sm_100 version 1).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3fff);  // start address
  d |= static_cast<uint64_t>(1) << 16;                 // LBO (unused for SW128 K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;         // SBO: 8-row atom stride
  d |= static_cast<uint64_t>(1) << 46;                 // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;                 // SWIZZLE_128B
  return d;
}
// kind::f16 instruction descriptor: A, B fp16 K-major, D fp32, M = 128, N = n.
__device__ __forceinline__ uint32_t idesc_f16(uint32_t n) { return (1u << 4) | ((n >> 3) << 17) | ((128u >> 4) << 24); }

// D (TMEM) += A (TMEM) * B (shared), one CTA.
__device__ __forceinline__ void mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate));
}
// D (TMEM) += A (shared) * B (shared), one CTA.
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
// The mbarrier gets one arrival once all earlier tcgen05 operations of the
// issuing thread have completed.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
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
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// 8 consecutive 32-bit TMEM columns of this thread's lane (the warp's lane
// quarter is encoded in taddr bits 16..).
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
      "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
      : "memory");
}

// byte offset of element (row r, k in [0,64)) in a SW128 K-major fp16 block
__device__ __forceinline__ uint32_t sw128_off(uint32_t r, uint32_t k) {
  return r * 128u + ((((k >> 3) ^ (r & 7u)) & 7u) << 4) + ((k & 7u) << 1);
}

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  return (static_cast<uint32_t>(__half_as_ushort(__float2half_rn(b))) << 16) | __half_as_ushort(__float2half_rn(a));
}

// Row scale of the fp16 split: a power of two taking max |x| to [2^14, 2^15)
// (exact), or 0 for rows that go entirely to the exact path (zero rows,
// non-finite values, magnitudes outside [2^-100, 2^100]).  mb = max of the
// magnitude bits (NaN > inf > finite).
struct RowScale {
  float scale;
  bool zero, wild;
};
__device__ __forceinline__ RowScale row_scale(uint32_t mb, bool live) {
  const bool nan = mb > 0x7f800000u;
  const float m = __uint_as_float(nan ? 0x7f800000u : mb);
  RowScale s;
  s.zero = (m == 0.0f);
  s.wild = nan || !(m < 0x1.0p100f) || (!s.zero && m < 0x1.0p-100f);
  s.scale = 0.0f;
  if (live && !s.zero && !s.wild) {
    const int e = static_cast<int>((__float_as_uint(m) >> 23) & 0xffu) - 127;
    s.scale = __uint_as_float(static_cast<uint32_t>(127 + 14 - e) << 23);
  }
  return s;
}
// Error threshold of a row's fast projections from the sum of squares of the
// scaled row: -1 = exact zero row or padding (every bit 1,
// srp.cpp:103), +inf = recheck every projection.
__device__ __forceinline__ float row_threshold(const RowScale& s, bool live, float ss, uint64_t dim, float margin_c) {
  if (!live || s.zero) return -1.0f;
  if (s.wild) return __int_as_float(0x7f800000);
  const float nx = sqrtf(ss * (1.0f + static_cast<float>(dim + 4) * 0x1.0p-23f)) * (1.0f + 0x1.0p-20f);
  return margin_c * nx * 16384.0f + static_cast<float>(dim) * 0x1.0p-10f;
}

// The reference's projection: binary64 left fold, mul then add, from +0.0
// (srp.cpp:78-91); operands loaded 8 ahead so only the add chain is serial.
__device__ __forceinline__ double exact_proj(const double* __restrict__ w, const void* x, int x_f64, uint64_t row,
                                             uint64_t ld, uint64_t dim) {
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

// The exact fold plus the sequential binary64 sum of squares of the row
// (the oracle's |x| for the near-tie measure |p| < 1e-6 |x| |w|).
__device__ __forceinline__ double exact_proj_nx(const double* __restrict__ w, const void* x, int x_f64, uint64_t row,
                                                uint64_t ld, uint64_t dim, double* nx_out) {
  double acc = 0.0, nx = 0.0;
  for (uint64_t i = 0; i < dim; ++i) {
    const double xv = x_f64 ? static_cast<const double*>(x)[row * ld + i]
                            : static_cast<double>(static_cast<const float*>(x)[row * ld + i]);
    acc = __dadd_rn(acc, __dmul_rn(w[i], xv));
    nx = __dadd_rn(nx, __dmul_rn(xv, xv));
  }
  *nx_out = nx;
  return acc;
}
// BASELINE.json near-tie predicate, evaluated as the oracle does
// (oracle/ace_oracle.c ora_near_tie): |p| < 1e-6 * (sqrt(nx) * |w|).
__device__ __forceinline__ bool near_tie_1e6(double p, double nx, double wn) {
  return fabs(p) < __dmul_rn(1e-6, __dmul_rn(__dsqrt_rn(nx), wn));
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Cold path: push the near-tie columns (bit jj of mask = direction dir0 + jj)
// into this CTA's list segment; a full segment flags the whole row for the
// exact recompute instead (recheck_rows_kernel).
__device__ __forceinline__ void push_near_mask(DevState* st, unsigned long long* seg, unsigned long long seg_cap,
                                                   uint32_t* seg_n, uint32_t* overflow_rows, uint32_t mask,
                                                   uint64_t row, uint32_t dir0) {
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

}  // namespace tc
}  // namespace ace_dev
