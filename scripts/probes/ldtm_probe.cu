// TMEM read throughput probe: W warps (4 or 8, lane quarters w % 4) each issue
// R rounds of tcgen05.ld (x32 or x64 columns of 32-bit, 32 lanes) + wait::ld;
// reports bytes per cycle per SM.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ldtm_probe ldtm_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int X>
__device__ __forceinline__ void ld(uint32_t taddr, uint32_t* v);
template <>
__device__ __forceinline__ void ld<32>(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

template <int W, int NLD>
__global__ void probe(unsigned long long* out, int rounds) {
  __shared__ uint32_t base_sh;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&base_sh)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = base_sh + (((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  uint32_t acc = 0;
  const long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    uint32_t v[32 * NLD];
#pragma unroll
    for (int k = 0; k < NLD; ++k) ld<32>(base + ((r * 32 * NLD + 32 * k) & 127), v + 32 * k);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int k = 0; k < 32 * NLD; ++k) acc ^= v[k];
  }
  const long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = acc;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base_sh), "r"(512));
}

template <int W, int NLD>
void run(unsigned long long* d, int rounds) {
  probe<W, NLD><<<148, W * 32>>>(d, rounds);
  cudaDeviceSynchronize();
  unsigned long long h[296];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < 148; ++i) cyc += h[2 * i];
  cyc /= 148;
  const double bytes = (double)W * rounds * NLD * 32 * 32 * 4;
  printf("warps %d, %d x32 loads in flight: %.1f B/cycle/SM (%.0f cycles per round)\n", W, NLD, bytes / cyc,
         cyc / rounds);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 296 * 8);
  const int R = 4096;
  run<4, 1>(d, R);
  run<4, 2>(d, R);
  run<4, 4>(d, R);
  run<8, 1>(d, R);
  run<8, 2>(d, R);
  run<8, 4>(d, R);
  run<16, 2>(d, R);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
