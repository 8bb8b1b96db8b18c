/* Seeded, counter-based generator for the BASELINE Dyson matrices
 *   A(E) = (E + i eta) I - H - Sigma^R.
 * The reference ships no Dyson generator (SURVEY.md finding 5); this is the one
 * spec both the GPU path and the oracle consume. Every entry is a pure function of
 * (seed, layer, offset, entry, component), so host and device produce identical
 * bytes in parallel. Restated independently in oracle/dyson_oracle.py.
 *
 *   u(seed,a,off,k,c) = (mix64(mix64(seed) ^ ctr) >> 11) * 2^-52 - 1   in [-1, 1)
 *   ctr               = (a << 40) | ((off + 8) << 36) | (2k + c),  k = col*b + row
 *   H_aa[i][j]        = 0.5 * (X[i][j] + conj(X[j][i])),   X = u(.., a, 0, ..)
 *   H_a,a+1           = 0.5 * u(.., a, +1, ..)    H_a+1,a = H_a,a+1^dagger
 *   H_a,a+2           = 0.2 * u(.., a, +2, ..)    H_a+2,a = H_a,a+2^dagger
 * (offsets > 2 use 0.2 as well). Sigma^R = sigma_a I per layer.
 */
#ifndef BBSI_DYSON_GEN_H
#define BBSI_DYSON_GEN_H
#include <stdint.h>

#ifdef __CUDACC__
#define BBSI_HD __host__ __device__ __forceinline__
#else
#define BBSI_HD static inline
#endif

BBSI_HD uint64_t bbsi_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

BBSI_HD double bbsi_uniform(uint64_t seedmix, int a, int off, long long k, int c) {
  uint64_t ctr = ((uint64_t)a << 40) | ((uint64_t)(off + 8) << 36) | (uint64_t)(2 * k + c);
  uint64_t x = bbsi_mix64(seedmix ^ ctr);
  return (double)(x >> 11) * (1.0 / 4503599627370496.0) - 1.0; /* 2^-52 */
}

BBSI_HD double bbsi_coupling_scale(int off) { return off == 1 ? 0.5 : 0.2; }

/* Entry (i, j) of H block (a, a+off), b x b blocks; re/im via *re, *im. */
BBSI_HD void bbsi_h_entry(uint64_t seedmix, int b, int a, int off, int i, int j, double* re, double* im) {
  if (off == 0) {
    double xr = bbsi_uniform(seedmix, a, 0, (long long)j * b + i, 0);
    double xi = bbsi_uniform(seedmix, a, 0, (long long)j * b + i, 1);
    double yr = bbsi_uniform(seedmix, a, 0, (long long)i * b + j, 0);
    double yi = bbsi_uniform(seedmix, a, 0, (long long)i * b + j, 1);
    *re = 0.5 * (xr + yr);
    *im = 0.5 * (xi - yi);
  } else if (off > 0) {
    double s = bbsi_coupling_scale(off);
    *re = s * bbsi_uniform(seedmix, a, off, (long long)j * b + i, 0);
    *im = s * bbsi_uniform(seedmix, a, off, (long long)j * b + i, 1);
  } else {
    /* H_{a, a+off} = (H_{a+off, a})^dagger: entry (i, j) = conj(H_{a+off,a}[j][i]) */
    int o = -off;
    double s = bbsi_coupling_scale(o);
    *re = s * bbsi_uniform(seedmix, a + off, o, (long long)i * b + j, 0);
    *im = -(s * bbsi_uniform(seedmix, a + off, o, (long long)i * b + j, 1));
  }
}

#endif
