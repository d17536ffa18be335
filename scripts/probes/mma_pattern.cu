// tcgen05.mma issue-pattern microbenchmark (dev tool): M=128, N=128, K=16
// kind::f16 TS MMAs (A in TMEM) issued by one elected thread, with the
// projection kernel's pattern switched on feature by feature:
//   bit 0: tcgen05.commit to an mbarrier after every 12 MMAs
//   bit 1: accumulator rotates over 3 TMEM buffers every 24 MMAs (first MMA
//          of a buffer overwrites)
//   bit 2: A columns / hi-lo operands vary like the kernel's fp16x3 split
//   bit 3: B descriptor rotates over 4 shared-memory stages (32 KB apart)
//   bit 4: random operand data instead of zeros
//   bit 5: stage ring: the MMA warp waits on a full barrier per 12 MMAs and
//          commits an empty barrier; a producer warp re-arms (4 stages)
//   bit 6: the producer also bulk-copies 32 KB from global into the stage
//   bit 7: whole warp walks the MMA loop (elect + __syncwarp), as the kernel
//   bit 8: warps 4-7 drain accumulators with tcgen05.ld 32x32b.x32 (all 128
//          lanes) the whole time, as the epilogue does; reports LDTM B/cycle
//   bit 9: with bit 8, the loads use 32x32b.x64 (64 registers per load)
//   bit 10: with bit 8, 16x256b.x8 shape instead
// Prints cycles per MMA for each mode.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3fff) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
               "r"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                   smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}

__global__ void mma_pattern(int n_tiles, int mode, const uint8_t* gsrc, unsigned long long* out) {
  __shared__ volatile int done;
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar, cbar, full[4], empty[4];
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  uint32_t seed = 0x9e3779b9u * (threadIdx.x + 1);
  for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x) {
    seed = seed * 1664525u + 1013904223u;
    // fp16 pairs with exponents in a sane range when random
    reinterpret_cast<uint32_t*>(sm)[i] = (mode & 16) ? ((seed & 0x3bff3bffu) | 0x20002000u) : 0u;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&cbar)));
    for (int i = 0; i < 4; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    done = 0;
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tbase;
  const uint32_t idesc = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
  // A (hi | lo) in TMEM columns 384..511 (as in the kernel: after 3 accumulators)
  if ((mode & 16) && threadIdx.x < 32) {
    for (int kk = 0; kk < 16; ++kk)
      asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(t + 384u + kk * 8u),
                   "l"(sw128_desc(smem_u32(sm) + (kk & 3) * 32u + (kk >> 2) * 16384u)));
  }
  long long t0 = 0, t1 = 0;
  if ((mode & 32) && threadIdx.x == 32) {
    uint32_t s = 0, ph = 0;
    for (int g = 0; g < n_tiles * 2; ++g) {
      while (!mbar_try(&empty[s], ph ^ 1u)) __nanosleep(64);
      if (mode & 64) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(32768));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(sm + 32768u * s)), "l"(gsrc + (static_cast<size_t>(g % 64) << 15)), "r"(32768),
                     "r"(smem_u32(&full[s])) : "memory");
      } else {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])));
      }
      if (++s == 4) { s = 0; ph ^= 1u; }
    }
  }
  if (threadIdx.x < 32) {
    t0 = clock64();
    uint32_t pred = 0;
    asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(pred));
    if ((mode & 128) || pred) {
      uint32_t s = 0, ph = 0;
      for (int tile = 0; tile < n_tiles; ++tile) {
        const uint32_t acc = (mode & 2) ? static_cast<uint32_t>(tile % 3) : 0u;
        const uint32_t dt = t + acc * 128u;
        for (uint32_t kc = 0; kc < 2; ++kc) {
          if (mode & 32) mbar_wait(&full[s], ph);
          uint32_t e = 1;
          if (mode & 128) asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(e));
          const uint32_t bs = (mode & 8) ? s : 0u;
          const uint64_t dbh = sw128_desc(smem_u32(sm) + 32768u * bs), dbl = sw128_desc(smem_u32(sm) + 32768u * bs + 16384u);
          if (e)
          for (uint32_t kk = 0; kk < 4; ++kk) {
            const uint32_t acol = (mode & 4) ? (kc * 4u + kk) * 8u : 0u;
            const uint32_t ahi = t + 384u + acol, alo = (mode & 4) ? ahi + 64u : ahi;
            const uint64_t off = (mode & 4) ? kk * 2u : 0u;
            const uint32_t first = (mode & 2) && kc == 0 && kk == 0;
            mma_ts(dt, ahi, dbh + off, idesc, first ? 0u : 1u);
            mma_ts(dt, alo, dbh + off, idesc, 1u);
            mma_ts(dt, ahi, (mode & 4) ? dbl + off : dbh + off, idesc, 1u);
          }
          if ((mode & 1) && e)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&cbar)));
          if ((mode & 32) && e)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&empty[s])));
          if (mode & 128) __syncwarp();
          s = (s + 1) & 3u;
          if (s == 0) ph ^= 1u;
        }
      }
      if (!(mode & 128) || pred)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    __syncwarp();
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)));
    t1 = clock64();
    if (threadIdx.x == 0) {
      atomicAdd(out, static_cast<unsigned long long>(t1 - t0));
      done = 1;
    }
  }
  if ((mode & 256) && threadIdx.x >= 128) {
    const uint32_t lane_base = ((threadIdx.x / 32) & 3u) * 32u;
    uint32_t acc = 0;
    unsigned long long bytes = 0;
    const long long s0 = clock64();
    uint32_t col = 0;
    while (!done) {
      const uint32_t addr = t + (lane_base << 16) + col;
      uint32_t r[64];
      if (mode & 1024) {
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                     "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                       "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                       "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                       "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                       "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                     : "r"(addr));
        for (int i = 32; i < 64; ++i) r[i] = 0;
        bytes += 16 * 32 * 4;  // per warp: 16 lanes x 64 cols... counted as 32 regs x 32 threads x 4 B
        bytes += 0;
      } else {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                     "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                       "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                       "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                       "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                       "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                     : "r"(addr));
        if (mode & 512) {
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                       "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                       : "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]),
                         "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]),
                         "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]),
                         "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]),
                         "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
                       : "r"(addr + 32u));
          bytes += 32 * 32 * 4;
        } else {
          for (int i = 32; i < 64; ++i) r[i] = 0;
        }
        bytes += 32 * 32 * 4;
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      #pragma unroll
      for (int i = 0; i < 64; ++i) acc += r[i];
      col = (col + 64u) % 384u;
    }
    const long long s1 = clock64();
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(out + 1, bytes);
      atomicAdd(out + 2, static_cast<unsigned long long>(s1 - s0));
    }
    if (acc == 0x12345678u) out[3] = acc;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(512));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(mma_pattern, cudaFuncAttributeMaxDynamicSharedMemorySize, 130 * 1024);
  unsigned long long* d;
  cudaMalloc(&d, 32);
  uint8_t* src;
  cudaMalloc(&src, 64 << 15);
  cudaMemset(src, 0, 64 << 15);
  const int n_tiles = 2000;  // x 24 MMAs
  int modes[32], nm = 0;
  if (getenv("MODES")) {
    for (char* p = getenv("MODES"); *p && nm < 32;) {
      modes[nm++] = static_cast<int>(strtol(p, &p, 0));
      while (*p == ',') ++p;
    }
  } else {
    const int def[] = {31, 31 | 256, 31 | 256 | 512, 31 | 256 | 1024, 31 | 32 | 64 | 128, 31 | 32 | 64 | 128 | 256,
                       31 | 32 | 64 | 128 | 256 | 512};
    for (int m : def) modes[nm++] = m;
  }
  for (int mi = 0; mi < nm; ++mi) {
    const int mode = modes[mi];
    double per = 0, ldb = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(d, 0, 32);
      mma_pattern<<<sms, (mode & 256) ? 256 : 128, 130 * 1024>>>(n_tiles, mode, src, d);
      cudaDeviceSynchronize();
      unsigned long long h[4] = {0, 0, 0, 0};
      cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
      per = static_cast<double>(h[0]) / sms / (n_tiles * 24.0);
      ldb = h[2] ? static_cast<double>(h[1]) / (static_cast<double>(h[2]) / 4.0) : 0.0;  // per SM: 4 warps
    }
    printf("mode %4d: %.1f cycles/MMA, LDTM %.1f B/cycle/SM\n", mode, per, ldb);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fprintf(stderr, "%s\n", cudaGetErrorString(e));
  return 0;
}
