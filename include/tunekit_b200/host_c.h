/* tunekit_b200/host_c.h -- C-linkage helpers of libtunekit_b200.so. */
#ifndef TUNEKIT_B200_HOST_C_H
#define TUNEKIT_B200_HOST_C_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* generate_synthetic_kernel_space (generators.hpp) over a space whose
 * parameter i takes the values 0..radix[i]-1: rank-indexed means and ok flags.
 * profile: "smooth" | "ridged" | "rugged".  0 = ok, 1 = invalid argument. */
int tk_host_generate_synthetic(uint32_t dims, const uint32_t* radix, double fail_fraction,
                               const char* profile, uint64_t seed, double* fitness, uint8_t* ok);

#ifdef __cplusplus
}
#endif
#endif
