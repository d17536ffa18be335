/* C entry points of libace.so (the host side of the drop-in) for non-C++
 * hosts such as the Python mirror.  The C++ API is include/ace/ *.hpp. */
#ifndef ACE_HOST_H
#define ACE_HOST_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* W (K*L rows of dim binary64, row t*K+b) exactly as SrpFamily's constructor
 * generates it (reference srp.cpp:36-48, rng.hpp:10-58; glibc libm).  0 ok. */
int ace_generate_directions(uint64_t seed, uint64_t dim, uint32_t k_bits, uint32_t num_tables, double* w);

/* ace::io::load_dataset (reference io.cpp:89-182).  has_label selects
 * label_column (0-based, negative from the end).  On 0: *values is a malloc'd
 * rows x cols binary64 matrix, *labels a malloc'd rows-byte 0/1 vector (or
 * NULL without a label column); free both with ace_free.  Errors: ACE_E_DATA
 * (the reference's DataError; message from ace_host_last_error) or
 * ACE_E_CONTRACT. */
int ace_load_dataset_csv(const char* path, int has_label, int label_column, double** values, uint64_t* rows,
                         uint64_t* cols, uint8_t** labels);
const char* ace_host_last_error(void);

/* Noise terms of the noisy hash variant for ticks tick0 .. tick0+count-1
 * (reference srp.cpp:97-101): noise_scale * NormalStream(mix_seed(noise_seed,
 * tick)).next() with glibc libm, as the reference draws them; input to
 * ace_family_buckets_noisy.  0 ok. */
int ace_noise_terms(uint64_t noise_seed, uint64_t tick0, uint64_t count, double noise_scale, double* out);
void ace_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
