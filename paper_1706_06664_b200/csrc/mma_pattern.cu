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
// Prints cycles per MMA for each mode.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

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
    if (threadIdx.x == 0) atomicAdd(out, static_cast<unsigned long long>(t1 - t0));
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
  cudaMalloc(&d, 8);
  uint8_t* src;
  cudaMalloc(&src, 64 << 15);
  cudaMemset(src, 0, 64 << 15);
  const int n_tiles = 2000;  // x 24 MMAs
  for (int mode : {0, 16, 15, 31, 15 | 32, 31 | 32, 15 | 32 | 64 | 128, 31 | 32 | 64 | 128, 0, 31}) {
    double per = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(d, 0, 8);
      mma_pattern<<<sms, 128, 130 * 1024>>>(n_tiles, mode, src, d);
      cudaDeviceSynchronize();
      unsigned long long cyc = 0;
      cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
      per = static_cast<double>(cyc) / sms / (n_tiles * 24.0);
    }
    printf("mode %2d: %.1f cycles/MMA\n", mode, per);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fprintf(stderr, "%s\n", cudaGetErrorString(e));
  return 0;
}
