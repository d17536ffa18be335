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
// Warp roles (256 threads, one CTA per SM, persistent over point tiles):
//   warp 0      W producer: cp.async.bulk of pre-swizzled W blocks (TMA engine)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-3   X converters: fp32 rows -> scaled fp16 hi/lo, SW128 K-major smem
//   warps 4-7   epilogue: tcgen05.ld accumulators -> signs, near ties, buckets
// Pipelines (mbarriers): W stages full/empty, A buffers full/empty,
// 4 TMEM accumulator buffers of 128 columns full/empty.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ace_tc.cuh"

namespace ace_dev {

namespace {

constexpr int kRows = 128;                 // points per tile (MMA M)
constexpr int kChunk = 64;                 // K elements per chunk (128 B of fp16)
constexpr int kBlockBytes = kRows * 128;   // one 128 x 64 fp16 block = 16 KB
constexpr int kAccBufs = 4;                // TMEM accumulators (4 x 128 columns)
constexpr int kMaxWStages = 4;
constexpr int kThreads = 256;
constexpr size_t kSmemLimit = 232448;      // 227 KB per CTA

struct TcLayout {
  uint32_t nkc, n_abuf, n_wst;
  size_t a_bytes, w_bytes, total;
};

__host__ __device__ inline TcLayout tc_layout(uint32_t nkc) {
  TcLayout L;
  L.nkc = nkc;
  L.n_abuf = nkc <= 2 ? 2 : 1;
  L.a_bytes = static_cast<size_t>(L.n_abuf) * nkc * 2 * kBlockBytes;
  const size_t room = kSmemLimit - 2048 - 1024 - L.a_bytes;  // static smem + align slack
  size_t st = room / (2 * kBlockBytes);
  if (st > kMaxWStages) st = kMaxWStages;
  L.n_wst = static_cast<uint32_t>(st);
  L.w_bytes = static_cast<size_t>(L.n_wst) * 2 * kBlockBytes;
  L.total = L.a_bytes + L.w_bytes + 1024;
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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

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
__device__ __forceinline__ uint32_t idesc_f16(uint32_t n) {
  return (1u << 4) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
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
  double acc = 0.0;
  if (x_f64) {
    const double* xr = static_cast<const double*>(x) + row * ld;
    for (uint64_t i = 0; i < dim; ++i) acc = __dadd_rn(acc, __dmul_rn(w[i], xr[i]));
  } else {
    const float* xr = static_cast<const float*>(x) + row * ld;
    for (uint64_t i = 0; i < dim; ++i) acc = __dadd_rn(acc, __dmul_rn(w[i], static_cast<double>(xr[i])));
  }
  return acc;
}

// ---- the kernel ----------------------------------------------------------------

__global__ void __launch_bounds__(kThreads, 1) hash_tc_kernel(const TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bar_wfull[kMaxWStages], bar_wempty[kMaxWStages];
  __shared__ __align__(8) uint64_t bar_afull[2], bar_aempty[2];
  __shared__ __align__(8) uint64_t bar_accfull[kAccBufs], bar_accempty[kAccBufs];
  __shared__ float rowthr[2][kRows];
  __shared__ uint32_t tmem_base_sh;

  const TcLayout L = tc_layout(a.nkc);
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* A = base;                  // [n_abuf][nkc][2][16 KB]
  uint8_t* Wsm = base + L.a_bytes;    // [n_wst][2][16 KB]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t n_tiles = (a.n + kRows - 1) / kRows;
  const uint32_t K = a.k_bits;

  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < L.n_wst; ++s) {
      mbar_init(&bar_wfull[s], 1);
      mbar_init(&bar_wempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar_afull[b], 2);   // two converter warps
      mbar_init(&bar_aempty[b], 5);  // MMA commit + four epilogue warps
    }
    for (int b = 0; b < kAccBufs; ++b) {
      mbar_init(&bar_accfull[b], 1);
      mbar_init(&bar_accempty[b], 4);
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

  if (warp == 0) {
    // ---------------- W producer ----------------
    if (lane == 0) {
      uint32_t s = 0, ph = 0;
      for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        for (uint32_t j = 0; j < a.ntiles; ++j) {
          const uint32_t tables_here = min(a.tpt, a.tables - j * a.tpt);
          const uint32_t nmma = (tables_here * K + 15u) & ~15u;
          const uint32_t bytes = nmma * 128u;
          for (uint32_t kc = 0; kc < a.nkc; ++kc) {
            mbar_wait(&bar_wempty[s], ph ^ 1u);
            mbar_expect_tx(&bar_wfull[s], 2u * bytes);
            const uint16_t* src = a.w16 + (static_cast<uint64_t>(j) * a.nkc + kc) * 2u * (kBlockBytes / 2);
            uint8_t* dst = Wsm + static_cast<size_t>(s) * 2 * kBlockBytes;
            bulk_g2s(dst, src, bytes, &bar_wfull[s]);
            bulk_g2s(dst + kBlockBytes, src + kBlockBytes / 2, bytes, &bar_wfull[s]);
            if (++s == L.n_wst) {
              s = 0;
              ph ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      uint32_t s = 0, wph = 0, acc = 0, accph = 0, it = 0;
      for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
        const uint32_t buf = it % L.n_abuf, use = it / L.n_abuf;
        mbar_wait(&bar_afull[buf], use & 1u);
        tc_after();
        const uint8_t* Ab = A + static_cast<size_t>(buf) * a.nkc * 2 * kBlockBytes;
        for (uint32_t j = 0; j < a.ntiles; ++j) {
          const uint32_t tables_here = min(a.tpt, a.tables - j * a.tpt);
          const uint32_t nmma = (tables_here * K + 15u) & ~15u;
          const uint32_t idesc = idesc_f16(nmma);
          mbar_wait(&bar_accempty[acc], accph ^ 1u);
          tc_after();
          const uint32_t dt = tmem_base + acc * 128u;
          for (uint32_t kc = 0; kc < a.nkc; ++kc) {
            mbar_wait(&bar_wfull[s], wph);
            tc_after();
            const uint32_t a_hi = smem_u32(Ab + (static_cast<size_t>(kc) * 2 + 0) * kBlockBytes);
            const uint32_t a_lo = smem_u32(Ab + (static_cast<size_t>(kc) * 2 + 1) * kBlockBytes);
            const uint32_t b_hi = smem_u32(Wsm + static_cast<size_t>(s) * 2 * kBlockBytes);
            const uint32_t b_lo = b_hi + kBlockBytes;
#pragma unroll
            for (uint32_t kk = 0; kk < 4; ++kk) {
              const uint32_t off = kk * 32u;  // 16 fp16 along K
              mma_f16(dt, sw128_desc(a_hi + off), sw128_desc(b_hi + off), idesc, (kc | kk) != 0u);
              mma_f16(dt, sw128_desc(a_lo + off), sw128_desc(b_hi + off), idesc, 1u);
              mma_f16(dt, sw128_desc(a_hi + off), sw128_desc(b_lo + off), idesc, 1u);
            }
            mma_commit(&bar_wempty[s]);
            if (++s == L.n_wst) {
              s = 0;
              wph ^= 1u;
            }
          }
          mma_commit(&bar_accfull[acc]);
          if (++acc == kAccBufs) {
            acc = 0;
            accph ^= 1u;
          }
        }
        mma_commit(&bar_aempty[buf]);
      }
    }
    __syncwarp();
  } else if (warp < 4) {
    // ---------------- X converters ----------------
    const uint32_t cw = warp - 2;
    uint32_t it = 0;
    const uint32_t groups = (a.nkc * kChunk + 127) / 128;  // 128 K per lane-group pass
    for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
      const uint32_t buf = it % L.n_abuf, use = it / L.n_abuf;
      mbar_wait(&bar_aempty[buf], (use & 1u) ^ 1u);
      uint8_t* Ab = A + static_cast<size_t>(buf) * a.nkc * 2 * kBlockBytes;
      for (uint32_t r = cw; r < kRows; r += 2) {
        const uint64_t row = t * kRows + r;
        const bool live = row < a.n;
        float v[2][4];
        float m = 0.0f;
#pragma unroll
        for (uint32_t g = 0; g < 2; ++g)
#pragma unroll
          for (uint32_t e = 0; e < 4; ++e) {
            const uint64_t k = g * 128u + lane * 4u + e;
            float val = 0.0f;
            if (live && g < groups && k < a.dim) {
              if (a.x_f64)
                val = static_cast<float>(static_cast<const double*>(a.x)[row * a.ld + k]);
              else
                val = static_cast<const float*>(a.x)[row * a.ld + k];
            }
            v[g][e] = val;
            m = fmaxf(m, fabsf(val));
            if (val != val) m = __int_as_float(0x7f800000);  // NaN -> force exact path
          }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        const bool zero = (m == 0.0f);
        const bool wild = !(m < 0x1.0p100f) || (!zero && m < 0x1.0p-100f);
        float scale = 1.0f;
        if (!zero && !wild) {
          const int e = static_cast<int>((__float_as_uint(m) >> 23) & 0xffu) - 127;
          scale = __uint_as_float(static_cast<uint32_t>(127 + 14 - e) << 23);
        }
        float ss = 0.0f;
#pragma unroll
        for (uint32_t g = 0; g < 2; ++g) {
          if (g >= groups) break;
          const uint32_t k0 = g * 128u + lane * 4u;  // 4 consecutive K
          const uint32_t kc = k0 / kChunk, kk = k0 % kChunk;
          __half hi[4], lo[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float xs = wild ? 0.0f : v[g][e] * scale;
            ss = fmaf(xs, xs, ss);
            hi[e] = __float2half_rn(xs);
            lo[e] = __float2half_rn(xs - __half2float(hi[e]));
          }
          if (kc < a.nkc) {
            uint8_t* blk = Ab + static_cast<size_t>(kc) * 2 * kBlockBytes;
            const uint32_t off = sw128_off(r, kk);
            uint2 ph, pl;
            ph.x = (static_cast<uint32_t>(__half_as_ushort(hi[1])) << 16) | __half_as_ushort(hi[0]);
            ph.y = (static_cast<uint32_t>(__half_as_ushort(hi[3])) << 16) | __half_as_ushort(hi[2]);
            pl.x = (static_cast<uint32_t>(__half_as_ushort(lo[1])) << 16) | __half_as_ushort(lo[0]);
            pl.y = (static_cast<uint32_t>(__half_as_ushort(lo[3])) << 16) | __half_as_ushort(lo[2]);
            *reinterpret_cast<uint2*>(blk + off) = ph;
            *reinterpret_cast<uint2*>(blk + kBlockBytes + off) = pl;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        if (lane == 0) {
          float thr;
          if (!live || zero) {
            thr = -1.0f;  // exact zeros: every projection is +-0, bit 1
          } else if (wild) {
            thr = __int_as_float(0x7f800000);  // recheck every projection exactly
          } else {
            const float nx = sqrtf(ss * (1.0f + static_cast<float>(a.dim + 4) * 0x1.0p-23f)) * (1.0f + 0x1.0p-20f);
            thr = a.margin_c * nx * 16384.0f + static_cast<float>(a.dim) * 0x1.0p-10f;
          }
          rowthr[buf][r] = thr;
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_afull[buf]);
    }
  } else {
    // ---------------- epilogue ----------------
    const uint32_t q = warp - 4;  // TMEM lane quarter
    const uint32_t r = q * 32u + lane;
    uint32_t it = 0, acc = 0, accph = 0;
    for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
      const uint32_t buf = it % L.n_abuf, use = it / L.n_abuf;
      mbar_wait(&bar_afull[buf], use & 1u);
      const float thr = rowthr[buf][r];
      const uint64_t row = t * kRows + r;
      const bool valid = row < a.n;
      for (uint32_t j = 0; j < a.ntiles; ++j) {
        const uint32_t tables_here = min(a.tpt, a.tables - j * a.tpt);
        const uint32_t used = tables_here * K;
        const uint32_t table0 = j * a.tpt;
        mbar_wait(&bar_accfull[acc], accph);
        tc_after();
        uint32_t bucket = 0, b = 0, tt = 0;
        for (uint32_t c0 = 0; c0 < used; c0 += 32) {
          uint32_t v[32];
          ACE_TMEM_LD32(tmem_base + ((q * 32u) << 16) + acc * 128u + c0, v);
          tmem_wait_ld();
          const uint32_t ncol = min(32u, used - c0);
          bool anynear = false;
#pragma unroll
          for (uint32_t jj = 0; jj < 32; ++jj) {
            if (jj < ncol) {
              const float f = __uint_as_float(v[jj]);
              bucket = (bucket << 1) | (f >= 0.0f ? 1u : 0u);
              anynear |= !(fabsf(f) > thr);
              if (++b == K) {
                if (valid) a.ids[static_cast<uint64_t>(table0 + tt) * a.n + row] = bucket;
                ++tt;
                b = 0;
                bucket = 0;
              }
            }
          }
          if (anynear && valid) {
#pragma unroll
            for (uint32_t jj = 0; jj < 32; ++jj) {
              const float f = __uint_as_float(v[jj]);
              if (jj < ncol && !(fabsf(f) > thr)) {
                const uint32_t dir = table0 * K + c0 + jj;
                const unsigned long long slot = atomicAdd(&a.st->near_count, 1ull);
                if (slot < a.near_cap) {
                  a.near_list[slot] = (static_cast<unsigned long long>(row) << 32) | dir;
                } else {
                  atomicOr(&a.overflow_rows[row >> 5], 1u << (row & 31));
                  a.st->near_overflow = 1;
                }
              }
            }
          }
        }
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_accempty[acc]);
        if (++acc == kAccBufs) {
          acc = 0;
          accph ^= 1u;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_aempty[buf]);
    }
  }

  tc_before();
  __syncthreads();
  tc_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
}

// ---- near-tie recheck ------------------------------------------------------------

__global__ void recheck_list_kernel(const TcArgs a, const double* __restrict__ w64) {
  __shared__ unsigned long long blk_r, blk_f;
  if (threadIdx.x == 0) blk_r = blk_f = 0;
  __syncthreads();
  const unsigned long long cnt = min(a.st->near_count, a.near_cap);
  const uint32_t K = a.k_bits;
  unsigned long long rr = 0, ff = 0;
  for (unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt;
       i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    const unsigned long long item = a.near_list[i];
    const uint64_t row = item >> 32;
    const uint32_t dir = static_cast<uint32_t>(item & 0xffffffffu);
    const uint32_t table = dir / K, bpos = K - 1u - dir % K;
    const double p = exact_proj(w64 + static_cast<uint64_t>(dir) * a.dim, a.x, a.x_f64, row, a.ld, a.dim);
    uint32_t* id = &a.ids[static_cast<uint64_t>(table) * a.n + row];
    const uint32_t fast = (*id >> bpos) & 1u;
    const uint32_t exact = p >= 0.0 ? 1u : 0u;
    if (fast != exact) {
      atomicXor(id, 1u << bpos);
      ++ff;
    }
    ++rr;
  }
  if (rr) atomicAdd(&blk_r, rr);
  if (ff) atomicAdd(&blk_f, ff);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (blk_r) atomicAdd(&a.st->rechecked, blk_r);
    if (blk_f) atomicAdd(&a.st->flipped, blk_f);
  }
}

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
    a.ids[static_cast<uint64_t>(table) * a.n + row] = bucket;
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

__global__ void pack_w16_kernel(const double* __restrict__ w64, const double* __restrict__ inv,
                                FamilyDev f, uint32_t nkc, uint16_t* w16) {
  const uint64_t total = static_cast<uint64_t>(f.ntiles) * kRows * nkc * kChunk;
  for (uint64_t idx = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t k = idx % (nkc * kChunk);
    const uint32_t rr = (idx / (nkc * kChunk)) % kRows;
    const uint32_t j = static_cast<uint32_t>(idx / (static_cast<uint64_t>(nkc) * kChunk * kRows));
    const uint32_t kc = k / kChunk, kk = k % kChunk;
    const uint32_t table = j * f.tpt + rr / f.k_bits;
    double w = 0.0;
    if (rr < f.tpt * f.k_bits && table < f.tables && k < f.dim) {
      const uint64_t dir = static_cast<uint64_t>(table) * f.k_bits + rr % f.k_bits;
      w = w64[dir * f.dim + k] * inv[dir];
    }
    const __half hi = __double2half(w);
    const __half lo = __double2half(w - static_cast<double>(__half2float(hi)));
    uint8_t* blk = reinterpret_cast<uint8_t*>(w16) + ((static_cast<uint64_t>(j) * nkc + kc) * 2) * kBlockBytes;
    const uint32_t off = rr * 128u + ((((kk >> 3) ^ (rr & 7u)) & 7u) << 4) + ((kk & 7u) << 1);
    *reinterpret_cast<__half*>(blk + off) = hi;
    *reinterpret_cast<__half*>(blk + kBlockBytes + off) = lo;
  }
}

}  // namespace

bool tc_supported(uint64_t dim) { return dim >= 1 && dim <= 256; }

size_t tc_smem_bytes(uint32_t nkc) { return tc_layout(nkc).total; }

cudaError_t tc_prepare_family(const FamilyDev& f, TcFamily* tc) {
  tc->enabled = 0;
  if (!tc_supported(f.dim) || f.k_bits > 128) return cudaSuccess;
  const uint32_t nkc = static_cast<uint32_t>((f.dim + kChunk - 1) / kChunk);
  const TcLayout L = tc_layout(nkc);
  if (L.n_wst < 2) return cudaSuccess;
  tc->nkc = nkc;
  const size_t bytes = static_cast<size_t>(f.ntiles) * nkc * 2 * kBlockBytes;
  cudaError_t e = cudaMalloc(&tc->w16, bytes);
  if (e != cudaSuccess) return e;
  double* inv = nullptr;
  if ((e = cudaMalloc(&inv, sizeof(double) * f.rows)) != cudaSuccess) return e;
  dir_norm_kernel<<<(f.rows + 127) / 128, 128>>>(f.w64, f.dim, f.rows, inv);
  pack_w16_kernel<<<1024, 256>>>(f.w64, inv, f, nkc, tc->w16);
  count_launch(2);
  e = cudaDeviceSynchronize();
  cudaFree(inv);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(hash_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(L.total));
  if (e != cudaSuccess) return e;
  tc->enabled = 1;
  return cudaSuccess;
}

void tc_free_family(TcFamily* tc) {
  if (tc->w16) cudaFree(tc->w16);
  tc->w16 = nullptr;
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
  const unsigned grid = static_cast<unsigned>(tiles < static_cast<uint64_t>(sms) ? tiles : sms);
  hash_tc_kernel<<<grid, kThreads, tc_layout(a.nkc).total, s>>>(a);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_recheck(const TcArgs& a, const double* w64, cudaStream_t s) {
  recheck_list_kernel<<<592, 256, 0, s>>>(a, w64);
  recheck_rows_kernel<<<592, 256, 0, s>>>(a, w64);
  count_launch(2);
  return cudaGetLastError();
}

}  // namespace ace_dev
