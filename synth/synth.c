/*
 * synth/synth.c -- seeded, counter-based synthetic input generators.
 *
 * Shared by the tests (oracle side and CUDA side get the same bytes) and by
 * bench.py.  Holds none of the FCFS arithmetic: only random numbers and the
 * value recipes of BASELINE.json's configs.
 *
 * Every element is a pure function of (seed, global index), so any sub-range
 * (a rank's batch slice or row strip) is bit-identical to slicing the whole.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

static inline uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* h(seed, i): counter-based 64-bit hash */
static inline uint64_t h64(uint64_t seed, uint64_t i) { return splitmix64(splitmix64(seed) ^ (i * 0xD1B54A32D192ED03ull)); }

uint64_t synth_hash(uint64_t seed, uint64_t i) { return h64(seed, i); }

/* uniform [0,1) on the fp32 grid k * 2^-24 */
void synth_uniform_f32(uint64_t seed, int64_t off, int64_t n, float *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = (float)((double)(h64(seed, (uint64_t)(off + i)) >> 40) * 0x1p-24);
}

/* uniform [0,1) on the fp16 grid k * 2^-11 (exact in fp16), returned as fp32 */
void synth_uniform_f16grid(uint64_t seed, int64_t off, int64_t n, float *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = (float)((double)(h64(seed, (uint64_t)(off + i)) >> 53) * 0x1p-11);
}

/* N(0,1) by Box-Muller in double from two counter draws, rounded to fp32 */
void synth_normal_f32(uint64_t seed, int64_t off, int64_t n, float *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        uint64_t k = (uint64_t)(off + i);
        double u1 = ((double)(h64(seed, 2 * k) >> 11) + 1.0) * 0x1p-53; /* (0,1] */
        double u2 = (double)(h64(seed, 2 * k + 1) >> 11) * 0x1p-53;     /* [0,1) */
        out[i] = (float)(sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
    }
}

/* Smooth random field on an N x N image (config 5):
 *   v(y,x) = sum_{k<16} (1/16) sin(2 pi (fx_k x + fy_k y)/N + phi_k) + 0.01 U[0,1)
 * fx_k, fy_k in [1,64], phi_k in [0, 2 pi) drawn from the seed; rows
 * [r0, r1) of a W-wide image are produced (angle addition per (row, col)). */
void synth_field_f32(uint64_t seed, int64_t N, int64_t W, int64_t r0, int64_t r1, float *out) {
    int fx[16], fy[16];
    double phi[16];
    for (int k = 0; k < 16; ++k) {
        fx[k] = 1 + (int)(h64(seed ^ 0xF1E1Dull, 3 * k) % 64);
        fy[k] = 1 + (int)(h64(seed ^ 0xF1E1Dull, 3 * k + 1) % 64);
        phi[k] = (double)(h64(seed ^ 0xF1E1Dull, 3 * k + 2) >> 11) * 0x1p-53 * 6.283185307179586;
    }
    const double tw = 6.283185307179586 / (double)N;
    double *sa = (double *)malloc(sizeof(double) * 16 * (size_t)W);
    double *ca = (double *)malloc(sizeof(double) * 16 * (size_t)W);
    if (!sa || !ca) { free(sa); free(ca); return; }
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < W; ++x)
        for (int k = 0; k < 16; ++k) {
            double a = tw * (double)((fx[k] * x) % N);
            sa[k * W + x] = sin(a);
            ca[k * W + x] = cos(a);
        }
#pragma omp parallel for schedule(static)
    for (int64_t r = r0; r < r1; ++r) {
        double sb[16], cb[16];
        for (int k = 0; k < 16; ++k) {
            double b = tw * (double)((fy[k] * r) % N) + phi[k];
            sb[k] = sin(b);
            cb[k] = cos(b);
        }
        for (int64_t x = 0; x < W; ++x) {
            double acc = 0.0;
            for (int k = 0; k < 16; ++k) acc += (sa[k * W + x] * cb[k] + ca[k * W + x] * sb[k]) * (1.0 / 16.0);
            double u = (double)(h64(seed, (uint64_t)(r * W + x)) >> 40) * 0x1p-24;
            out[(r - r0) * W + x] = (float)(acc + 0.01 * u);
        }
    }
    free(sa);
    free(ca);
}
