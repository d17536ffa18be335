// Bucket-packing probe: 4 warps x 32 rows cut L K-bit fields from sign words
// in shared memory and store them table-major (stride ld).  Variants: store
// to global (table-major stride), store to shared, no store.  Cycles per table.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void pack_probe(uint32_t* ids, uint64_t ld, uint32_t tables, uint32_t K, int reps, unsigned long long* out) {
  __shared__ uint32_t sg[32 * 128];
  __shared__ uint32_t st[32 * 128];
  const uint32_t r = threadIdx.x;
  for (int i = r; i < 32 * 128; i += blockDim.x) sg[i] = i * 2654435761u;
  __syncthreads();
  const uint32_t nwords = (tables * K + 31) / 32;
  const uint32_t kmask = (1u << K) - 1u;
  uint32_t acc = 0;
  const long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    const uint64_t row = (uint64_t)blockIdx.x * 128 + r + (uint64_t)rep * 128 * gridDim.x;
    uint32_t* idp = ids + (row % ld);
    for (uint32_t t0b = 0; t0b < tables; t0b += 8) {
      uint32_t bk[8];
#pragma unroll
      for (uint32_t u = 0; u < 8; ++u) {
        const uint32_t s0 = min(t0b + u, tables - 1) * K, wi = s0 >> 5;
        const uint32_t hi = sg[wi * 128 + r], lo = sg[min(wi + 1, nwords - 1) * 128 + r];
        const unsigned long long win = ((unsigned long long)hi << 32) | lo;
        bk[u] = (uint32_t)(win >> (64 - (s0 & 31) - K)) & kmask;
      }
#pragma unroll
      for (uint32_t u = 0; u < 8; ++u) {
        const uint32_t tt = t0b + u;
        if (tt < tables) {
          if (MODE == 0) idp[(uint64_t)tt * ld] = bk[u];
          else if (MODE == 1) st[(tt & 31) * 128 + r] = bk[u];
          else acc ^= bk[u];
        }
      }
    }
  }
  const long long t1 = clock64();
  if (MODE == 1) acc ^= st[r];
  if (r == 0) { out[blockIdx.x * 2] = t1 - t0; out[blockIdx.x * 2 + 1] = acc; }
}

int main() {
  const uint64_t ld = 131072;  // cfg 5 group stride
  const uint32_t L = 50, K = 15;
  uint32_t* ids; cudaMalloc(&ids, sizeof(uint32_t) * ld * L);
  unsigned long long* d; cudaMalloc(&d, 148 * 16);
  unsigned long long h[296];
  const int reps = 64;
  auto rep = [&](const char* nm) {
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double c = 0; for (int i = 0; i < 148; ++i) c += h[2 * i]; c /= 148;
    printf("%-14s %.1f cycles per table per warp (%s)\n", nm, c / reps / L, cudaGetErrorString(cudaGetLastError()));
  };
  for (uint64_t l2 : {131072ull, 16384ull, 1024ull, 512ull}) {
    printf("ld %llu\n", (unsigned long long)l2);
    pack_probe<0><<<148, 128>>>(ids, l2, L, K, reps, d); rep("global store");
    pack_probe<0><<<148, 128>>>(ids, l2, L, K, reps, d); rep("global store");
  }
  pack_probe<1><<<148, 128>>>(ids, ld, L, K, reps, d); rep("shared store");
  pack_probe<2><<<148, 128>>>(ids, ld, L, K, reps, d); rep("no store");
  return 0;
}
