/*
 * coolchic_synth.h — the seeded synthetic image shared by every arm (product,
 * reference checker, port checker, bench).  BASELINE.json configs: "sum of 8
 * random 2-D sinusoids, freq 1-32 cycles/image, plus N(0,0.02) noise,
 * clamped"; SURVEY.md 8(d) fixes the draw order:
 *   v_c(y,x) = 0.5 + sum_{j<8} a_j sin(2 pi (fx_j x/W + fy_j y/H) + phi_j)
 *              + 0.02 N(0,1),  clamped to [0,1]
 *   fx, fy ~ U[1,32]; phi ~ U[0, 2 pi); a ~ U[0.03, 0.08]
 * All draws use the reference's counter RNG (mathutil.hpp:18-44) keyed by
 * (seed, channel, component).  Evaluated in double on the host; tests always
 * hand the SAME buffer to every implementation, so compiler differences in
 * the generator can never leak into a parity comparison.
 */
#ifndef COOLCHIC_SYNTH_H
#define COOLCHIC_SYNTH_H

#include <math.h>
#include <stddef.h>
#include <stdint.h>

static inline uint64_t ccs_splitmix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
static inline uint64_t ccs_hash_combine(uint64_t a, uint64_t b) {
    return ccs_splitmix64(a ^ (b + 0x9e3779b97f4a7c15ull));
}
static inline double ccs_unit(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }
static inline double ccs_gauss(uint64_t stream, uint64_t index) {
    const uint64_t h = ccs_splitmix64(stream + index);
    const double u1 = ((double)(h >> 40) + 1.0) * 0x1.0p-24;
    const double u2 = (double)((h >> 16) & 0xffffffu) * 0x1.0p-24;
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

static inline void ccs_make_image(int h, int w, uint64_t seed, float* out) {
    const double two_pi = 6.283185307179586;
    for (int c = 0; c < 3; ++c) {
        double fx[8], fy[8], ph[8], am[8];
        const uint64_t cs = ccs_hash_combine(ccs_hash_combine(seed, 0x5157u), (uint64_t)c);
        for (int j = 0; j < 8; ++j) {
            const uint64_t js = ccs_hash_combine(cs, (uint64_t)j);
            fx[j] = 1.0 + 31.0 * ccs_unit(ccs_splitmix64(js + 0));
            fy[j] = 1.0 + 31.0 * ccs_unit(ccs_splitmix64(js + 1));
            ph[j] = two_pi * ccs_unit(ccs_splitmix64(js + 2));
            am[j] = 0.03 + 0.05 * ccs_unit(ccs_splitmix64(js + 3));
        }
        const uint64_t ns = ccs_hash_combine(cs, 0x401u);
        float* plane = out + (size_t)c * (size_t)h * (size_t)w;
        for (int y = 0; y < h; ++y) {
            for (int x = 0; x < w; ++x) {
                double v = 0.5;
                for (int j = 0; j < 8; ++j)
                    v += am[j] * sin(two_pi * (fx[j] * x / w + fy[j] * y / h) + ph[j]);
                v += 0.02 * ccs_gauss(ns, (uint64_t)y * (uint64_t)w + (uint64_t)x);
                v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
                plane[(size_t)y * w + x] = (float)v;
            }
        }
    }
}

#endif /* COOLCHIC_SYNTH_H */
