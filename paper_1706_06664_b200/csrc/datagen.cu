// Synthetic workload generation (test/bench input, not the ACE hot path).
// Host: pthreads over row ranges.  Device: one thread per row.  Both evaluate
// datagen_core.h, compiled without FMA contraction (nvcc --fmad=false,
// -Xcompiler -ffp-contract=off) so the rows are bit-identical.
#include <cuda_runtime.h>
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "datagen_core.h"

namespace {

struct HostJob {
  const dg_params* p;
  uint64_t row0, row1;
  float* out;
  uint8_t* labels;
};

void* host_worker(void* arg) {
  HostJob* j = static_cast<HostJob*>(arg);
  const uint64_t d = j->p->dim;
  for (uint64_t r = j->row0; r < j->row1; ++r) {
    const int l = dg_row(j->p, r, j->out + (r - j->row0) * d);
    if (j->labels) j->labels[r - j->row0] = (uint8_t)l;
  }
  return nullptr;
}

double* make_basis_host(uint64_t seed) {
  double* b = static_cast<double*>(malloc(sizeof(double) * 32 * 4096));
  for (uint64_t r = 0; r < 32; ++r)
    for (uint64_t k = 0; k < 4096; ++k) b[r * 4096 + k] = dg_basis_entry(seed, r, k);
  return b;
}

__global__ void device_rows(dg_params p, uint64_t row0, uint64_t nrows,
                            float* __restrict__ out, uint8_t* __restrict__ labels) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  const int l = dg_row(&p, row0 + i, out + i * p.dim);
  if (labels) labels[i] = (uint8_t)l;
}

}  // namespace

extern "C" {

uint64_t ace_datagen_dim(int cfg) { return dg_dim(cfg); }

// Rows [row0, row0+nrows) of configuration cfg into out (nrows x dim floats,
// row-major) and labels (nrows bytes, may be NULL).  Returns 0 on success.
int ace_datagen_host(int cfg, uint64_t seed, uint64_t row0, uint64_t nrows,
                     float* out, uint8_t* labels, int threads) {
  if (dg_dim(cfg) == 0) return -1;
  double* basis = cfg == 4 ? make_basis_host(seed) : nullptr;
  dg_params p;
  dg_init(&p, cfg, seed, basis);
  if (threads < 1) threads = 1;
  if ((uint64_t)threads > nrows) threads = nrows ? (int)nrows : 1;
  pthread_t* tid = static_cast<pthread_t*>(malloc(sizeof(pthread_t) * threads));
  HostJob* jobs = static_cast<HostJob*>(malloc(sizeof(HostJob) * threads));
  const uint64_t chunk = (nrows + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const uint64_t a = t * chunk, b = a + chunk < nrows ? a + chunk : nrows;
    jobs[t] = HostJob{&p, row0 + (a < nrows ? a : nrows), row0 + b,
                      out + (a < nrows ? a : nrows) * p.dim,
                      labels ? labels + (a < nrows ? a : nrows) : nullptr};
    pthread_create(&tid[t], nullptr, host_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], nullptr);
  free(tid);
  free(jobs);
  free(basis);
  return 0;
}

// Same rows generated on the device into d_out / d_labels (device pointers).
int ace_datagen_device(int cfg, uint64_t seed, uint64_t row0, uint64_t nrows,
                       float* d_out, uint8_t* d_labels, void* stream) {
  if (dg_dim(cfg) == 0) return -1;
  double* d_basis = nullptr;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cfg == 4) {
    double* h = make_basis_host(seed);
    if (cudaMalloc(&d_basis, sizeof(double) * 32 * 4096) != cudaSuccess) {
      free(h);
      return -2;
    }
    cudaMemcpy(d_basis, h, sizeof(double) * 32 * 4096, cudaMemcpyHostToDevice);
    free(h);
  }
  dg_params p;
  dg_init(&p, cfg, seed, d_basis);
  const unsigned threads = 128;
  const uint64_t blocks = (nrows + threads - 1) / threads;
  if (blocks) device_rows<<<(unsigned)blocks, threads, 0, s>>>(p, row0, nrows, d_out, d_labels);
  cudaError_t e = cudaStreamSynchronize(s);
  if (d_basis) cudaFree(d_basis);
  return e == cudaSuccess ? 0 : -3;
}

}  // extern "C"
