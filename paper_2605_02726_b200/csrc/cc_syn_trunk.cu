// cc_syn_trunk.cu — synthesis trunk backward (conv1x1 c1 -> ReLU -> conv1x1
// c2, plus the linear stabilizer): synthesize_backward's trunk part
// (synthesis.hpp:216-233; conv1x1_backward layers.hpp:216-250).
//
// Per tile of 128 pixels, 256 threads (persistent CTAs, 2 per SM):
//   phase A  two threads per pixel, each owning half of the F hidden units:
//            recompute pre-activations (bias, then z in channel order),
//            h1 = relu, dh1 = (c2ᵀ·dt) ⊙ relu'(h1), and dz = stabᵀ·dx̂ + c1ᵀ·dh1
//            with FFMA2 (pairs of hidden units / pairs of z channels); h1,
//            dh1, z, dt, dx̂ are written FEATURE-MAJOR to shared memory;
//   phase B  the weight gradients [dh1 | dt | dx̂] x [z|1, h1|1, z] as 4x4
//            register micro-tiles over the pixel axis, each job split in
//            NPART pixel ranges so that every thread owns ~one unit; the
//            accumulators stay in registers across all tiles of the CTA and
//            are summed (ranges in fixed order, fp64) once at the end.
// Deterministic: fixed thread->work mapping, no atomics.
//
// PART selects the work: 0 both phases (one launch); 1 the data path only
// (dz, the input of the upsampling backward: on the critical chain); 2 the
// weight gradients only (h1, dh1 recomputed, phase B, partial rows: an
// off-critical-path launch beside the upsampling backward).  1 + 2 compute
// exactly what 0 does.
#include <cuda_runtime.h>

#include "cc_kernels.h"
#include "cc_math.cuh"
#include "cc_reduce.cuh"
#include "cc_tile.cuh"

namespace ccb {

namespace {

constexpr int T = kSynTile;   // pixels per tile (128)
constexpr int NT = 2 * T;     // threads per CTA
constexpr int LT = T + 4;     // feature-major row stride (floats)
constexpr int kLZ = kMaxLevels;

template <int FP>
struct TB {
    static_assert(T == 128 && FP % 4 == 0, "tile mapping");
    static constexpr int FQ = FP / 4;  // hidden units per phase-A thread (a pixel pair)
    static constexpr int U = FQ < 4 ? FQ : 4;  // hidden units per weight load
    static_assert(FQ % U == 0, "hidden-unit chunks");
    static constexpr int RZ = 12;      // z 0..7, ones at 8
    static constexpr int RH = FP + 4;  // h1, ones at FP
    static constexpr int O_Z = 0;
    static constexpr int O_H = O_Z + RZ * LT;
    static constexpr int O_DH = O_H + RH * LT;
    static constexpr int O_DT = O_DH + FP * LT;
    static constexpr int O_DX = O_DT + 4 * LT;
    static constexpr int O_DZ = O_DX + 4 * LT;   // quarters 1..3: partial dz
    static constexpr int O_Z2 = O_DZ + 3 * kLZ * LT; // next tile's z / dt / dx̂ (cp.async)
    static constexpr int O_DT2 = O_Z2 + RZ * LT;
    static constexpr int O_DX2 = O_DT2 + 4 * LT;
    static constexpr int ACT = O_DX2 + 4 * LT;
    static constexpr int J1 = (FP / 4) * 3;      // dh1 x [z|1]
    static constexpr int J2 = FP / 4 + 1;        // dt x [h1|1]
    static constexpr int J3 = 2;                 // dx̂ x z (stabilizer)
    static constexpr int NJ = J1 + J2 + J3;
    static constexpr int NPART = NT / NJ > 8 ? 8 : (NT / NJ < 1 ? 1 : NT / NJ);
    static constexpr int PS = 4 * ((T / 4 + NPART - 1) / NPART);  // pixels per range
    static constexpr int NU = NJ * NPART;
    static constexpr int MAXU = (NU + NT - 1) / NT;
    static_assert(NU * 16 <= ACT, "epilogue staging fits");
};

template <int FP>
struct alignas(16) TBSmem {
    using K = TB<FP>;
    alignas(16) float W1T[kLZ][FP];  // c1.w as [k][f]: pre-activation pairs (f, f+1)
    alignas(16) float W1[FP][kLZ];   // c1.w as [f][k]: dz pairs (k, k+1)
    alignas(16) float c1b[FP];
    alignas(16) float c2w[3][FP];
    alignas(16) float st[3][kLZ];
    alignas(16) float act[K::ACT];
};

__device__ __forceinline__ void cp_async16_zfill(float* smem, const float* gmem, int bytes) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async4_zfill(float* smem, const float* gmem, bool full) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(full ? 4 : 0) : "memory");
}

// Asynchronous load of tile t's inputs into feature-major rows: z planes
// 0..7 (zero past L), dt 0..2, dx̂ 0..2; zero past the last pixel.  16-byte
// copies when every plane is 16-byte aligned (Plan::zvec).  Always commits
// one cp.async group.
__device__ __forceinline__ void issue_tile(const Plan& P, const float* __restrict__ dt_in, int64_t t,
                                           float* bZ, float* bDT, float* bDX, int tid) {
    const int64_t np = P.npix, p0 = t * T;
    const bool vec = P.zvec != 0;  // npix and every z-plane offset are multiples of 4
    for (int c = tid; c < 14 * (T / 4); c += NT) {
        const int row = c / (T / 4), q = c % (T / 4);
        const int64_t p = p0 + 4 * q;
        const float* src;
        float* dst;
        bool ok;
        if (row < kLZ) {
            src = P.z + (row < P.L ? P.zpix[row] : 0) + p;
            dst = bZ + row * LT + 4 * q;
            ok = row < P.L;
        } else if (row < kLZ + 3) {
            src = dt_in + int64_t(row - kLZ) * np + p;
            dst = bDT + (row - kLZ) * LT + 4 * q;
            ok = true;
        } else {
            src = P.syn_dx + int64_t(row - kLZ - 3) * np + p;
            dst = bDX + (row - kLZ - 3) * LT + 4 * q;
            ok = true;
        }
        const int64_t left = np - p;
        const int n = ok ? (left >= 4 ? 4 : (left > 0 ? int(left) : 0)) : 0;
        if (vec) {
            cp_async16_zfill(dst, n > 0 ? src : P.z, 4 * n);
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) cp_async4_zfill(dst + i, i < n ? src + i : P.z, i < n);
        }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}

template <int FP, int PART>
__global__ void __launch_bounds__(NT, 2) k_syn_trunk_bwd2(const Plan* __restrict__ pp) {
    constexpr bool kDz = PART != 2, kDw = PART != 1;
    using K = TB<FP>;
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    const float* __restrict__ dt_in = P.syn_dt;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TBSmem<FP>& sm = *reinterpret_cast<TBSmem<FP>*>(smem_raw);
    const int tid = threadIdx.x;
    const int L = P.L, F = P.syn_F;
    const bool has_stab = P.off_sstab >= 0;
    for (int e = tid; e < FP * kLZ; e += NT) {
        const int f = e / kLZ, k = e - f * kLZ;
        const float w = (f < F && k < L) ? P.params[P.off_c1w + f * L + k] : 0.0f;
        sm.W1[f][k] = w;
        sm.W1T[k][f] = w;
    }
    for (int e = tid; e < FP; e += NT) sm.c1b[e] = e < F ? P.params[P.off_c1b + e] : 0.0f;
    for (int e = tid; e < 3 * FP; e += NT) {
        const int co = e / FP, f = e - co * FP;
        sm.c2w[co][f] = f < F ? P.params[P.off_c2w + co * F + f] : 0.0f;
    }
    for (int e = tid; e < 3 * kLZ; e += NT) {
        const int co = e / kLZ, k = e - co * kLZ;
        sm.st[co][k] = (has_stab && k < L) ? P.params[P.off_sstab + co * L + k] : 0.0f;
    }
    for (int e = tid; e < K::ACT; e += NT) sm.act[e] = 0.0f;
    __syncthreads();

    float* sZ = sm.act + K::O_Z;
    float* sDT = sm.act + K::O_DT;
    float* sDX = sm.act + K::O_DX;
    float* nZ = sm.act + K::O_Z2;
    float* nDT = sm.act + K::O_DT2;
    float* nDX = sm.act + K::O_DX2;
    float* const sH = sm.act + K::O_H;
    float* const sDH = sm.act + K::O_DH;
    float* const sDZ = sm.act + K::O_DZ;

    double uacc[K::MAXU][16];  // fp64 across tiles (large images: millions of pixels)
#pragma unroll
    for (int m = 0; m < K::MAXU; ++m)
#pragma unroll
        for (int e = 0; e < 16; ++e) uacc[m][e] = 0.0;

    const int64_t np = P.npix;
    const int64_t ntiles = (np + T - 1) / T;
    pdl_wait();  // dt / dx of the posts kernel (weights above were staged before)
    pdl_trigger();
    if (blockIdx.x < ntiles) issue_tile(P, dt_in, blockIdx.x, sZ, sDT, sDX, tid);
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        // the next tile's inputs land in the other buffers while this one computes
        if (t + gridDim.x < ntiles)
            issue_tile(P, dt_in, t + gridDim.x, nZ, nDT, nDX, tid);
        else
            asm volatile("cp.async.commit_group;\n" ::: "memory");
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        __syncthreads();
        // ---- phase A: thread = pixel pair (FFMA2 lanes) x a quarter of the
        // hidden units; weights are broadcast operands ----
        const int pq = tid & 63, qt = tid >> 6, px0 = 2 * pq;
        const int64_t p0 = t * T + px0;
        const bool v0 = p0 < np, v1 = p0 + 1 < np;
        float2 z[kLZ], dt[3];
#pragma unroll
        for (int k = 0; k < kLZ; ++k) z[k] = *reinterpret_cast<const float2*>(sZ + k * LT + px0);
#pragma unroll
        for (int co = 0; co < 3; ++co) dt[co] = *reinterpret_cast<const float2*>(sDT + co * LT + px0);
        // dz starts with the stabilizer term (synthesis.hpp:220), then c1 (:232)
        float2 dz[kLZ];
#pragma unroll
        for (int k = 0; k < kLZ; ++k) dz[k] = make_float2(0.0f, 0.0f);
        if (kDz && qt == 0 && has_stab) {
            float2 dx[3];
#pragma unroll
            for (int co = 0; co < 3; ++co) dx[co] = *reinterpret_cast<const float2*>(sDX + co * LT + px0);
#pragma unroll
            for (int k = 0; k < kLZ; ++k) {
                float2 a = make_float2(0.0f, 0.0f);
#pragma unroll
                for (int co = 0; co < 3; ++co) a = ffma2(dx[co], sm.st[co][k], a);
                dz[k] = a;
            }
        }
        const int f0 = qt * K::FQ;
#pragma unroll 1
        for (int fc = 0; fc < K::FQ; fc += K::U) {
            const int f = f0 + fc;
            float2 a[K::U];
#pragma unroll
            for (int u = 0; u < K::U; ++u) a[u] = make_float2(sm.c1b[f + u], sm.c1b[f + u]);
#pragma unroll
            for (int k = 0; k < kLZ; ++k) {
                float w[K::U];
                if constexpr (K::U == 4) {
                    const float4 w4 = *reinterpret_cast<const float4*>(&sm.W1T[k][f]);
                    w[0] = w4.x; w[1] = w4.y; w[2] = w4.z; w[3] = w4.w;
                } else {
#pragma unroll
                    for (int u = 0; u < K::U; ++u) w[u] = sm.W1T[k][f + u];
                }
#pragma unroll
                for (int u = 0; u < K::U; ++u) a[u] = ffma2(z[k], w[u], a[u]);
            }
#pragma unroll
            for (int u = 0; u < K::U; ++u) {
                const float2 h = make_float2(a[u].x > 0.0f ? a[u].x : 0.0f, a[u].y > 0.0f ? a[u].y : 0.0f);
                float2 d = make_float2(0.0f, 0.0f);
#pragma unroll
                for (int co = 0; co < 3; ++co) d = ffma2(dt[co], sm.c2w[co][f + u], d);
                d.x = h.x > 0.0f ? d.x : 0.0f;
                d.y = h.y > 0.0f ? d.y : 0.0f;
                if (kDz) {
#pragma unroll
                    for (int kq = 0; kq < kLZ / 4; ++kq) {
                        const float4 w4 = *reinterpret_cast<const float4*>(&sm.W1[f + u][4 * kq]);
                        dz[4 * kq + 0] = ffma2(d, w4.x, dz[4 * kq + 0]);
                        dz[4 * kq + 1] = ffma2(d, w4.y, dz[4 * kq + 1]);
                        dz[4 * kq + 2] = ffma2(d, w4.z, dz[4 * kq + 2]);
                        dz[4 * kq + 3] = ffma2(d, w4.w, dz[4 * kq + 3]);
                    }
                }
                if (kDw) {
                    *reinterpret_cast<float2*>(sH + (f + u) * LT + px0) = make_float2(v0 ? h.x : 0.0f, v1 ? h.y : 0.0f);
                    *reinterpret_cast<float2*>(sDH + (f + u) * LT + px0) = d;
                }
            }
        }
        if (qt == 0) {
            if (kDw) *reinterpret_cast<float2*>(sZ + kLZ * LT + px0) = make_float2(v0 ? 1.0f : 0.0f, v1 ? 1.0f : 0.0f);
        } else {
            if (kDw && qt == 1)
                *reinterpret_cast<float2*>(sH + FP * LT + px0) = make_float2(v0 ? 1.0f : 0.0f, v1 ? 1.0f : 0.0f);
            if (kDz)
#pragma unroll
                for (int k = 0; k < kLZ; ++k)
                    *reinterpret_cast<float2*>(sDZ + ((qt - 1) * kLZ + k) * LT + px0) = dz[k];
        }
        __syncthreads();
        if (kDz && qt == 0 && v0) {  // quarters summed in order
#pragma unroll
            for (int k = 0; k < kLZ; ++k) {
                if (k >= L) continue;
                float2 v = dz[k];
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const float2 o = *reinterpret_cast<const float2*>(sDZ + (q * kLZ + k) * LT + px0);
                    v.x += o.x;
                    v.y += o.y;
                }
                float* dst = P.dz + P.zpix[k] + p0;
                if (P.zvec) {
                    *reinterpret_cast<float2*>(dst) = v;
                } else {
                    dst[0] = v.x;
                    if (v1) dst[1] = v.y;
                }
            }
        }
        // ---- phase B: weight gradients ----
#pragma unroll
        for (int m = 0; m < (kDw ? K::MAXU : 0); ++m) {
            const int u = tid + m * NT;
            if (u < K::NU) {
                const int j = u / K::NPART, s = u - j * K::NPART;
                const int i0 = s * K::PS, i1 = min(i0 + K::PS, T);
                const float* A;
                const float* B;
                if (j < K::J1) {
                    A = sDH + 4 * (j / 3) * LT;
                    B = sZ + 4 * (j % 3) * LT;
                } else if (j < K::J1 + K::J2) {
                    A = sDT;
                    B = sH + 4 * (j - K::J1) * LT;
                } else {
                    A = sDX;
                    B = sZ + 4 * (j - K::J1 - K::J2) * LT;
                }
                if (i0 < i1) dw_tile4x4<LT>(A, B, i0, i1, uacc[m]);
            }
        }
        __syncthreads();
        float* x = sZ; sZ = nZ; nZ = x;
        x = sDT; sDT = nDT; nDT = x;
        x = sDX; sDX = nDX; nDX = x;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    if (!kDw) return;
    __syncthreads();

    // ---- epilogue: stage the units, sum ranges in order, one row per CTA ----
    static_assert(K::NU * 16 * 2 <= K::ACT, "fp64 staging fits in the activation buffers");
    double* stage = reinterpret_cast<double*>(sm.act);
#pragma unroll
    for (int m = 0; m < K::MAXU; ++m) {
        const int u = tid + m * NT;
        if (u < K::NU)
#pragma unroll
            for (int e = 0; e < 16; ++e) stage[u * 16 + e] = uacc[m][e];
    }
    __syncthreads();
    const PartialRegion& R = P.region[P.reg_syn_trunk];
    const PartialRow row(P, R, blockIdx.x);
    for (int e = tid; e < R.count; e += NT) {
        const int pidx = R.param_off + e;
        int job = -1, q = 0;
        if (pidx >= P.off_c1w && pidx < P.off_c1w + F * L) {
            const int r = pidx - P.off_c1w, f = r / L, k = r - f * L;
            job = (f / 4) * 3 + k / 4;
            q = (f % 4) * 4 + k % 4;
        } else if (pidx >= P.off_c1b && pidx < P.off_c1b + F) {
            const int f = pidx - P.off_c1b;
            job = (f / 4) * 3 + 2;
            q = (f % 4) * 4;
        } else if (pidx >= P.off_c2w && pidx < P.off_c2w + 3 * F) {
            const int r = pidx - P.off_c2w, co = r / F, f = r - co * F;
            job = K::J1 + f / 4;
            q = co * 4 + f % 4;
        } else if (pidx >= P.off_c2b && pidx < P.off_c2b + 3) {
            job = K::J1 + FP / 4;
            q = (pidx - P.off_c2b) * 4;
        } else if (has_stab && pidx >= P.off_sstab && pidx < P.off_sstab + 3 * L) {
            const int r = pidx - P.off_sstab, co = r / L, k = r - co * L;
            job = K::J1 + K::J2 + k / 4;
            q = co * 4 + k % 4;
        }
        double v = 0.0;
        if (job >= 0)
            for (int s = 0; s < K::NPART; ++s) v += stage[(job * K::NPART + s) * 16 + q];
        row[e] = v;
    }
}

template <int FP>
size_t tb_smem() {
    return sizeof(TBSmem<FP>);
}

template <int FP>
void launch_t(const LaunchCtx& L, int part) {
    const dim3 g(L.syn_blocks, 1, L.batch), b(NT);
    if (part == 1) launch_pdl(k_syn_trunk_bwd2<FP, 1>, g, b, tb_smem<FP>(), L.stream, 's', L.plan);
    else if (part == 2) launch_pdl(k_syn_trunk_bwd2<FP, 2>, g, b, tb_smem<FP>(), L.stream, 's', L.plan);
    else launch_pdl(k_syn_trunk_bwd2<FP, 0>, g, b, tb_smem<FP>(), L.stream, 's', L.plan);
}

template <int FP>
void configure_t() {
    const int sm = int(tb_smem<FP>());
    cudaFuncSetAttribute(k_syn_trunk_bwd2<FP, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_syn_trunk_bwd2<FP, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_syn_trunk_bwd2<FP, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
}

}  // namespace

int syn_padded_hidden(int F) {
    if (F <= 8) return 8;
    if (F <= 16) return 16;
    if (F <= 48) return 48;
    if (F <= 64) return 64;
    return -1;
}

size_t syn_trunk_smem(int FP) {
    switch (FP) {
        case 8: return tb_smem<8>();
        case 16: return tb_smem<16>();
        case 48: return tb_smem<48>();
        default: return tb_smem<64>();
    }
}

int syn_trunk_blocks_per_sm(int FP) {  // __launch_bounds__(256, 2)
    const int b = int((227 * 1024) / (syn_trunk_smem(FP) + 1024));
    return b < 1 ? 1 : (b > 2 ? 2 : b);
}

void syn_configure(int FP) {
    switch (FP) {
        case 8: configure_t<8>(); break;
        case 16: configure_t<16>(); break;
        case 48: configure_t<48>(); break;
        default: configure_t<64>(); break;
    }
}

void launch_syn_backward(const LaunchCtx& L, int part) {
    const Plan& H = *L.host;
    switch (syn_padded_hidden(H.syn_F)) {
        case 8: launch_t<8>(L, part); break;
        case 16: launch_t<16>(L, part); break;
        case 48: launch_t<48>(L, part); break;
        default: launch_t<64>(L, part); break;
    }
}

}  // namespace ccb
