/*
 * stategen.c -- seeded synthetic state vectors (input generation only).
 *
 * Shared input infrastructure for both the CUDA path's callers and the
 * oracle's tests.  It contains none of the method's arithmetic (no gate, no
 * address map, no gather): it only fills k1 with seeded values.
 *
 * Counter-based: entry j's value is a pure function of (seed, j), so any
 * entry can be regenerated on its own (full-size parity samples, M = 32) and
 * the result does not depend on the number of threads.
 *
 *   key   = splitmix64(seed)
 *   u1(j) = ((splitmix64(key + 2j)     >> 11) + 1) * 2^-53   in (0, 1]
 *   u2(j) = ( splitmix64(key + 2j + 1) >> 11     ) * 2^-53   in [0, 1)
 *   gauss: r = sqrt(-2 ln u1), re = r cos(2 pi u2), im = r sin(2 pi u2)
 *          (Box-Muller: i.i.d. standard-normal real and imaginary parts)
 *   polar: re = u1 cos(2 pi u2), im = u1 sin(2 pi u2)
 *          (magnitude ~U(0,1], phase ~U(0, 2 pi))
 *
 * Normalisation (input recipe): the float64 sum of re^2 + im^2 is
 * accumulated per block of 2^16 entries, and the block sums are added in
 * block order, so the scale 1/sqrt(sum) is bit-reproducible; the stored
 * value is (float)(re * scale) for complex64, re * scale for complex128.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#define GEN_BLOCK ((uint64_t)1 << 16)

static inline uint64_t splitmix64(uint64_t z)
{
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static inline void gen_entry(uint64_t key, int mode, uint64_t j, double *re, double *im)
{
    const double two_pi = 6.283185307179586476925286766559;
    double u1 = (double)((splitmix64(key + 2 * j) >> 11) + 1) * 0x1.0p-53;
    double u2 = (double)(splitmix64(key + 2 * j + 1) >> 11) * 0x1.0p-53;
    double r = (mode == 0) ? sqrt(-2.0 * log(u1)) : u1;
    *re = r * cos(two_pi * u2);
    *im = r * sin(two_pi * u2);
}

/* float64 sum of |z_j|^2 over [0, N) in fixed block order. */
double gen_sumsq(uint64_t seed, int32_t mode, uint64_t N)
{
    uint64_t key = splitmix64(seed);
    uint64_t nblk = (N + GEN_BLOCK - 1) / GEN_BLOCK;
    double *part = (double *)malloc(nblk * sizeof(double));
    if (!part) return -1.0;
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < (int64_t)nblk; ++b) {
        uint64_t lo = (uint64_t)b * GEN_BLOCK;
        uint64_t hi = lo + GEN_BLOCK < N ? lo + GEN_BLOCK : N;
        double s = 0.0;
        for (uint64_t j = lo; j < hi; ++j) {
            double re, im;
            gen_entry(key, mode, j, &re, &im);
            s += re * re + im * im;
        }
        part[b] = s;
    }
    double total = 0.0;
    for (uint64_t b = 0; b < nblk; ++b) total += part[b];
    free(part);
    return total;
}

/* Fill entries [start, start+count) with scale * z_j.  elem_bytes 8 -> two
 * float32 per entry (complex64), 16 -> two float64 (complex128).          */
void gen_fill(uint64_t seed, int32_t mode, double scale, int32_t elem_bytes,
              uint64_t start, uint64_t count, void *out)
{
    uint64_t key = splitmix64(seed);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < (int64_t)count; ++r) {
        double re, im;
        gen_entry(key, mode, start + (uint64_t)r, &re, &im);
        if (elem_bytes == 8) {
            float *o = (float *)out + 2 * r;
            o[0] = (float)(re * scale);
            o[1] = (float)(im * scale);
        } else {
            double *o = (double *)out + 2 * r;
            o[0] = re * scale;
            o[1] = im * scale;
        }
    }
}

/* Index-tagged state (a constructed test input): the real part's bits hold
 * j and the imaginary part's bits hold ~j, so every entry is distinct and
 * NaN / denormal bit patterns are exercised.                              */
void gen_tagged(int32_t elem_bytes, uint64_t start, uint64_t count, void *out)
{
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < (int64_t)count; ++r) {
        uint64_t j = start + (uint64_t)r;
        if (elem_bytes == 8) {
            uint32_t *o = (uint32_t *)out + 2 * r;
            o[0] = (uint32_t)j;
            o[1] = ~(uint32_t)j;
        } else {
            uint64_t *o = (uint64_t *)out + 2 * r;
            o[0] = j;
            o[1] = ~j;
        }
    }
}
