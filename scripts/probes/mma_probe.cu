// tcgen05.mma issue-rate microbenchmark (kind::f16, fp32 accumulate, M=128,
// cta_group::1): back-to-back MMAs from one elected thread, operands in shared
// memory (SS) or A in TMEM (TS), N = 64/128/256.  One CTA per SM, all SMs.
// Prints cycles per MMA and the implied dense TFLOP/s.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3fff) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

__global__ void mma_rate(int n_mma, uint32_t n, int ts, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tbase;
  const uint32_t idesc = (1u << 4) | ((n >> 3) << 17) | ((128u >> 4) << 24);
  const uint64_t da = sw128_desc(smem_u32(sm)), db = sw128_desc(smem_u32(sm + 32768));
  long long t0 = 0, t1 = 0;
  if (threadIdx.x < 32) {
    t0 = clock64();
    uint32_t pred = 0;
    asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(pred));
    if (pred) {
      for (int i = 0; i < n_mma; ++i) {
        if (ts)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(t),
                       "r"(t + 256u), "l"(db), "r"(idesc), "r"(1));
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(t),
                       "l"(da), "l"(db), "r"(idesc), "r"(1));
      }
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
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int n_mma = 20000;
  printf("{");
  int first = 1;
  for (int ts = 0; ts < 2; ++ts)
    for (uint32_t n : {64u, 128u, 256u}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(d, 0, 8);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        mma_rate<<<sms, 128, 100 * 1024>>>(n_mma, n, ts, d);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        unsigned long long cyc = 0;
        cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
        if (rep == 1) {
          const double per = static_cast<double>(cyc) / sms / n_mma;
          const double tf = 2.0 * 128 * n * 16 * n_mma * sms / (ms * 1e-3) / 1e12;
          printf("%s\"%s_N%u\": {\"cycles_per_mma\": %.1f, \"tflops\": %.0f}", first ? "" : ", ", ts ? "TS" : "SS", n, per, tf);
          first = 0;
        }
      }
    }
  printf("}\n");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fprintf(stderr, "%s\n", cudaGetErrorString(e));
  return 0;
}
