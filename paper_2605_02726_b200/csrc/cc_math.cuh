// cc_math.cuh — device restatements of the reference numerics that parity
// depends on.  Every function follows mathutil.hpp / layers.hpp line by line;
// no MUFU approximations (__expf etc.) and no --use_fast_math anywhere, so the
// polynomials evaluate exactly as on the CPU (up to FMA contraction, which the
// reference build also enables: proj/CMakeLists.txt:13 -ffp-contract=fast).
#pragma once

#include <stdint.h>

namespace ccb {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;
constexpr float kSigmaMinF = 0.06f;        // layers.hpp:591
constexpr float kSigmaMaxF = 256.0f;       // layers.hpp:592
constexpr float kProbFloorF = 1.0f / 65536.0f;  // layers.hpp:593
constexpr float kInvSqrt2F = 0.7071067811865476f;  // layers.hpp:594
constexpr float kLog2EF = 1.4426950408889634f;     // mathutil.hpp:100
constexpr float kLn2F = 0.6931471805599453f;       // layers.hpp:628

// mathutil.hpp:20-29
__host__ __device__ inline uint64_t splitmix64(uint64_t z) {
    z += kGolden;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t hash_combine(uint64_t a, uint64_t b) {
    return splitmix64(a ^ (b + kGolden));
}
// mathutil.hpp:32
__host__ __device__ inline double unit_from_bits(uint64_t h) {
    return double(h >> 11) * 0x1.0p-53;
}
// mathutil.hpp:35-40 — Box-Muller in double, one draw per (stream, index).
__device__ inline float counter_gauss(uint64_t stream, uint64_t index) {
    const uint64_t h = splitmix64(stream + index);
    const double u1 = (double(h >> 40) + 1.0) * 0x1.0p-24;
    const double u2 = double((h >> 16) & 0xffffffu) * 0x1.0p-24;
    return float(sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
}
// mathutil.hpp:42-44 (contracted the way the reference build contracts it)
__host__ __device__ inline float counter_uniform(uint64_t stream, uint64_t index, float lo,
                                                 float hi) {
    return fmaf(hi - lo, float(unit_from_bits(splitmix64(stream + index))), lo);
}

// std::max / std::min with the reference's argument order (NaN behaviour kept).
__host__ __device__ __forceinline__ float std_max(float a, float b) { return (a < b) ? b : a; }
__host__ __device__ __forceinline__ float std_min(float a, float b) { return (b < a) ? b : a; }

// mathutil.hpp:55-71
__device__ __forceinline__ float cc_exp(float x) {
    const float kLn2 = 0.69314718055994531f;
    const float kInvLn2 = 1.44269504088896341f;
    x = std_min(88.0f, std_max(-87.0f, x));
    // z = x*log2(e) feeds two add/subs; the reference build (-ffp-contract=fast)
    // fuses both into FMAs, so the restatement spells them out.
    const float nf = floorf(fmaf(x, kInvLn2, 0.5f));
    const float t = fmaf(x, kInvLn2, -nf) * kLn2;
    float p = 0.0013888889f;
    p = fmaf(t, p, 0.008333334f);
    p = fmaf(t, p, 0.041666668f);
    p = fmaf(t, p, 0.16666667f);
    p = fmaf(t, p, 0.5f);
    p = fmaf(t, p, 1.0f);
    p = fmaf(t, p, 1.0f);
    const float s = __int_as_float((int(nf) + 127) << 23);
    return p * s;
}

// mathutil.hpp:73-86
__device__ __forceinline__ float cc_log(float x) {
    const uint32_t bits = __float_as_uint(x);
    int e = int(bits >> 23) - 127;
    float m = __uint_as_float((bits & 0x007fffffu) | 0x3f800000u);
    if (m > 1.41421356f) {
        m *= 0.5f;
        ++e;
    }
    const float s = (m - 1.0f) / (m + 1.0f);
    const float s2 = s * s;
    float p = 0.11111111f;
    p = fmaf(s2, p, 0.14285715f);
    p = fmaf(s2, p, 0.2f);
    p = fmaf(s2, p, 0.33333333f);
    p = fmaf(s2, p, 1.0f);
    return fmaf(2.0f * s, p, float(e) * 0.69314718f);
}

// mathutil.hpp:88-94
__device__ __forceinline__ float cc_tanh(float x) {
    float ax = fabsf(x);
    ax = std_min(ax, 9.0f);
    const float t = cc_exp(-2.0f * ax);
    const float r = (1.0f - t) / (1.0f + t);
    return x < 0.0f ? -r : r;
}

// layers.hpp:546-547
__device__ __forceinline__ float softround_denom(float temp) {
    return 2.0f * cc_tanh(1.0f / (2.0f * temp));
}

// e / n for small non-negative ints (e < 2^22, n >= 1) without an integer
// division (tile index splits in the stencil kernels): (e + 0.5) / n is at
// least 0.5/n away from an integer, far above the fp32 rounding error.
struct FDiv {
    float inv;
    int n;
    __device__ __forceinline__ explicit FDiv(int n_) : inv(1.0f / float(n_)), n(n_) {}
    __device__ __forceinline__ int div(int e) const { return int((float(e) + 0.5f) * inv); }
};

// e / n for 0 <= e < 2^31, 1 <= n < 2^31: m = ceil(2^63 / n), e / n =
// (m * 2e) >> 64 — the rounding error e * (m - 2^63/n) / 2^63 < 2^-32 stays
// below the 1/n gap to the next integer, so the quotient is exact.
struct FDivU {
    unsigned long long m;
    __device__ __forceinline__ explicit FDivU(int n) {
        const unsigned long long t = 1ull << 63;
        m = t / (unsigned long long)n + (t % (unsigned long long)n != 0 ? 1ull : 0ull);
    }
    __device__ __forceinline__ int div(int e) const {
        return int(__umul64hi(m, 2ull * (unsigned long long)e));
    }
};

// Asynchronous 4-byte global -> shared copy (LDGSTS): window staging keeps
// every load of a tile in flight at once instead of load/wait/store.
__device__ __forceinline__ void cp_async4(float* smem, const float* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
// Packed fp32 FMA (sm_100 FFMA2): lane-wise d = a * b + c, each lane an IEEE
// fmaf (round-to-nearest, no flush), i.e. bit-identical to two fmaf calls.
// A float2 built from one scalar folds into FFMA2's broadcast operand form.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    unsigned long long ua, ub, uc, ud;
    asm("mov.b64 %0, {%1, %2};" : "=l"(ua) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(ub) : "f"(b.x), "f"(b.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(uc) : "f"(c.x), "f"(c.y));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(ud) : "l"(ua), "l"(ub), "l"(uc));
    float2 d;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(ud));
    return d;
}
__device__ __forceinline__ float2 ffma2(float2 a, float b, float2 c) { return ffma2(a, make_float2(b, b), c); }

// Programmatic dependent launch (PDL): a kernel launched with the
// programmatic-serialization attribute may start while its predecessor in
// the stream drains; it reads only long-settled data (plan, parameters,
// forward activations) before pdl_wait(), which blocks until the
// predecessor grid has completed and its writes are visible.  pdl_trigger()
// then lets the successor's CTAs be scheduled.  Both are no-ops for a
// kernel launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// Laplace sigma head (entropy_model.hpp:260, layers.hpp:591-592).
__device__ __forceinline__ float sigma_from_raw(float raw1) {
    return std_min(kSigmaMaxF, std_max(kSigmaMinF, cc_exp(raw1)));
}

}  // namespace ccb
