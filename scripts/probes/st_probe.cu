// Store throughput probe: W warps per SM each issue N coalesced global stores
// (32-bit or 128-bit per lane) to rows far apart; cycles per store instruction.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int VEC>
__global__ void st_probe(uint32_t* buf, uint64_t ld, int n, unsigned long long* out) {
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    uint32_t* p = buf + ((uint64_t)(i * 37 + w * 7 + blockIdx.x * 3) % 64) * ld + (blockIdx.x * 32 + w) * 128;
    if (VEC == 1) p[lane] = i;
    else reinterpret_cast<uint4*>(p)[lane] = make_uint4(i, i, i, i);
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
int main() {
  const uint64_t ld = 1 << 22;
  uint32_t* b; cudaMalloc(&b, 64 * ld * 4);
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  unsigned long long h[148];
  for (int warps : {1, 4, 8, 16}) for (int vec : {1, 4}) {
    const int n = 4096;
    if (vec == 1) st_probe<1><<<148, warps * 32>>>(b, ld, n, d); else st_probe<4><<<148, warps * 32>>>(b, ld, n, d);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
    printf("warps %2d vec %d: %.1f cycles per store per warp, %.1f B/cycle/SM\n", warps, vec, c / n, warps * n * 128.0 * vec / c);
  }
  return 0;
}
