// K-streamed tcgen05 projection for d > 256 (BASELINE config 4: d = 4096).
// Same split and exactness argument as ace_hash_tc.cu; a point tile no longer
// fits on chip, so converted A chunks and W chunks stream through a ring of
// shared-memory slots and both MMA operands come from shared memory.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ace_tc_ptx.cuh"

namespace ace_dev {
using namespace tc;

namespace {

// ---- K-streamed projection (d > 256) -----------------------------------------------
//
// A point tile no longer fits on chip (d = 4096: 2 MB of fp16 hi + lo), so A
// is streamed in 64-wide K chunks next to the W chunks, one direction tile at
// a time.  Accumulation is chunked: kKsSc K chunks go into a TMEM accumulator
// (double-buffered), the epilogue adds the chunk results into fp32 running
// sums in registers (kTW / 2 columns per thread).  That keeps the rigorous error
// bound at (12 kKsSc + 16 + nchunks / 2) ulp instead of growing with d, so near
// ties stay rare; they are rechecked by recheck_segs_kernel afterwards.

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
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bar_full[kKsSlots], bar_empty[kKsSlots], bar_accfull[2], bar_accempty[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ uint32_t sgbuf[2][C::kWords][kRows];  // sign words of a direction tile, by tile parity
  __shared__ uint32_t seg_n;
  // 1 KB aligned (SW128 operands); offset from the __shared__ array itself so
  // the compiler keeps the accesses in the shared state space (LDS / STS)
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t n_tiles = (a.n + kRows - 1) / kRows;
  const uint32_t K = a.k_bits, nkc = a.nkc, nch = ks_chunks(nkc);
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
    tmem_alloc(&tmem_base_sh, 512);
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
            mbar_wait_sleepy(&bar_empty[s], ph ^ 1u);
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
    // ---- MMA issuer: 12 MMAs per K chunk, A and B from the shared-memory slot
    uint32_t s = 0, ph = 0, ab = 0, abph = 0;
    const uint32_t idesc = idesc_f16(kTW);
    for (uint64_t it = 0; it < iters; ++it)
        for (uint32_t c = 0; c < nch; ++c) {
          mbar_wait(&bar_accempty[ab], abph ^ 1u);
          tc_after();
          const uint32_t k0 = c * kKsSc, k1 = min(nkc, k0 + kKsSc);
          const uint32_t dt = tmem_base + ab * kTW;
          if (elect_one()) {
            uint32_t ss = s, pp = ph;
            for (uint32_t kc = k0; kc < k1; ++kc) {
              mbar_wait(&bar_full[ss], pp);
              const uint32_t sa = smem_u32(base + static_cast<size_t>(ss) * kKsSlot);
              const uint64_t dbh = sw128_desc(sa + 2u * kBlockBytes), dbl = sw128_desc(sa + 2u * kBlockBytes + kTW * 128u);
              // A read from the slot by the MMAs themselves (no copy into TMEM)
              const uint64_t dah = sw128_desc(sa), dal = sw128_desc(sa + kBlockBytes);
#pragma unroll
              for (uint32_t kk = 0; kk < 4; ++kk) {
                const uint64_t off = kk * 2u;
                mma_f16_ss(dt, dah + off, dbh + off, idesc, (kc != k0 || kk != 0u) ? 1u : 0u);
                mma_f16_ss(dt, dal + off, dbh + off, idesc, 1u);
                mma_f16_ss(dt, dah + off, dbl + off, idesc, 1u);
              }
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
          mbar_wait_sleepy(&bar_accfull[ab], abph);
          tc_after();
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
          tc_before();
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
  if (warp == 1) tmem_dealloc(tmem_base, 512);
}

// Conversion for the K-streamed path: one warp per row, any d.  With fp32
// rows of 16-byte multiples the row is read as float4 (held in registers for
// both passes when d <= 4096).
// Element k of a row (fp32 or fp64 source), 0 beyond dim.
__device__ __forceinline__ float load_x(const TcArgs& a, uint64_t row, uint64_t k) {
  if (k >= a.dim) return 0.0f;
  if (a.x_f64) return static_cast<float>(static_cast<const double*>(a.x)[row * a.ld + k]);
  return static_cast<const float*>(a.x)[row * a.ld + k];
}

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
  unsigned long long rr = 0, ff = 0, nt = 0;
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
      double p = 0.0, ab = 0.0, xx = 0.0;
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
          xx += (static_cast<double>(xv.x) * xv.x + static_cast<double>(xv.y) * xv.y) +
                (static_cast<double>(xv.z) * xv.z + static_cast<double>(xv.w) * xv.w);
        }
      } else {
        for (uint32_t k = lane; k < dim; k += 32u) {
          const double xv = a.x_f64 ? static_cast<const double*>(a.x)[row * a.ld + k]
                                    : static_cast<double>(static_cast<const float*>(a.x)[row * a.ld + k]);
          const double t = xv * static_cast<double>(__ldg(w + k));  // x fp64 input: products rounded (in gam)
          p += t;
          ab += fabs(t);
          xx += xv * xv;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        p += __shfl_xor_sync(0xffffffffu, p, o);
        ab += __shfl_xor_sync(0xffffffffu, ab, o);
        xx += __shfl_xor_sync(0xffffffffu, xx, o);
      }
      // sign and the near-tie measure from p1 where the bound decides them,
      // else from the reference's fold (and the oracle's sequential |x|^2)
      const double err = bound_rel * ab + 0x1.0p-1000;
      const double lim = 1e-6 * (sqrt(xx) * a.wnorm64[dir]);
      const bool sign_ok = fabs(p) > err;
      const bool near_sure = fabs(p) + err < lim * (1.0 - 1e-9);
      const bool far_sure = fabs(p) - err > lim * (1.0 + 1e-9);
      int bit = p >= 0.0 ? 1 : 0;
      bool near = near_sure;
      if (!sign_ok || !(near_sure || far_sure)) {
        double e = 0.0, nx = 0.0;
        if (lane == 0) e = exact_proj_nx(a.w64 + static_cast<uint64_t>(dir) * dim, a.x, a.x_f64, row, a.ld, dim, &nx);
        e = __shfl_sync(0xffffffffu, e, 0);
        nx = __shfl_sync(0xffffffffu, nx, 0);
        bit = e >= 0.0 ? 1 : 0;
        near = near_tie_1e6(e, nx, a.wnorm64[dir]);
      }
      if (lane == 0) {
        nt += near ? 1u : 0u;
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
    if (nt) atomicAdd(&a.st->near_ties, nt);
  }
}
}  // namespace

bool tc_kstream(uint32_t nkc) { return nkc > 4; }

uint32_t tck_grid(uint64_t n) {
  const uint64_t tiles = (n + kRows - 1) / kRows;
  return static_cast<uint32_t>(tiles < static_cast<uint64_t>(tc_sms()) ? tiles : tc_sms());
}

cudaError_t tck_prepare(uint32_t tw) {
  return tw == 256 ? cudaFuncSetAttribute(hash_tck_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(ks_smem_bytes(256)))
                   : cudaFuncSetAttribute(hash_tck_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(ks_smem_bytes(128)));
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

}  // namespace ace_dev
