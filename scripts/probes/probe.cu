// Roofline denominators MEASURED_PEAKS.json does not carry (it has HBM copy
// and cuBLAS bf16): FP32 FFMA, FP64 DFMA, and L2 atomic throughput of
// red.add.u32 at the ACE counter-array sizes.  Prints one JSON object.
// Usage: ace_probe   (one GPU; ~2 s)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <vector>

#define CK(x)                                                               \
  do {                                                                      \
    cudaError_t e = (x);                                                    \
    if (e != cudaSuccess) {                                                 \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));               \
      return 1;                                                             \
    }                                                                       \
  } while (0)

template <typename T>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
    x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
      x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
    }
  }
  if (x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == (T)1.2345) out[0] = x0;
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

// each thread issues `per` red.add to pseudo-random counters in [0, num)
__global__ void red_random(uint32_t* c, uint32_t num, int per, uint32_t salt) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < per; ++i) {
    const uint32_t idx = hash32(t * 2654435761u + i * 40503u + salt) % num;
    atomicAdd(&c[idx], 1u);  // result unused -> RED
  }
}

// same, as gathers (the score pass)
__global__ void gather_random(const uint32_t* c, uint32_t num, int per, uint32_t salt, uint32_t* out) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t s = 0;
  for (int i = 0; i < per; ++i) s += c[hash32(t * 2654435761u + i * 40503u + salt) % num];
  if (s == 0xdeadbeef) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float ms = 0;
  float* fo;
  double* dout;
  CK(cudaMalloc(&fo, 64));
  CK(cudaMalloc(&dout, 64));
  const int blocks = sms * 8, threads = 256, iters = 2048;
  fma_loop<float><<<blocks, threads>>>(fo, 16, 1.0001f, 0.5f);
  CK(cudaEventRecord(a));
  fma_loop<float><<<blocks, threads>>>(fo, iters, 1.0001f, 0.5f);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  CK(cudaEventElapsedTime(&ms, a, b));
  const double fp32_tf = 2.0 * 8 * 16 * (double)iters * blocks * threads / (ms * 1e-3) / 1e12;
  fma_loop<double><<<blocks, threads>>>(dout, 16, 1.0001, 0.5);
  CK(cudaEventRecord(a));
  fma_loop<double><<<blocks, threads>>>(dout, iters / 4, 1.0001, 0.5);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  CK(cudaEventElapsedTime(&ms, a, b));
  const double fp64_tf = 2.0 * 8 * 16 * (double)(iters / 4) * blocks * threads / (ms * 1e-3) / 1e12;

  printf("{\"sms\": %d, \"clock_mhz\": %d, \"fp32_ffma_tflops\": %.2f, \"fp64_dfma_tflops\": %.2f", sms,
         clk / 1000, fp32_tf, fp64_tf);
  const uint64_t sizes[3] = {6553600ull, 26214400ull, 67108864ull};
  uint32_t *c, *o;
  CK(cudaMalloc(&c, sizes[2]));
  CK(cudaMalloc(&o, 64));
  printf(", \"l2_red_u32_gops\": {");
  for (int s = 0; s < 3; ++s) {
    const uint32_t num = sizes[s] / 4;
    CK(cudaMemset(c, 0, sizes[s]));
    const int per = 64, rb = sms * 16, rt = 256;
    red_random<<<rb, rt>>>(c, num, per, 1);
    CK(cudaEventRecord(a));
    red_random<<<rb, rt>>>(c, num, per, 2);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms, a, b));
    const double ops = (double)rb * rt * per;
    printf("%s\"%llu\": %.1f", s ? ", " : "", (unsigned long long)sizes[s], ops / (ms * 1e-3) / 1e9);
  }
  printf("}, \"l2_gather_u32_gops\": {");
  for (int s = 0; s < 3; ++s) {
    const uint32_t num = sizes[s] / 4;
    const int per = 64, rb = sms * 16, rt = 256;
    gather_random<<<rb, rt>>>(c, num, per, 1, o);
    CK(cudaEventRecord(a));
    gather_random<<<rb, rt>>>(c, num, per, 3, o);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms, a, b));
    const double ops = (double)rb * rt * per;
    printf("%s\"%llu\": %.1f", s ? ", " : "", (unsigned long long)sizes[s], ops / (ms * 1e-3) / 1e9);
  }
  printf("}}\n");
  return 0;
}
