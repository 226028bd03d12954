// cc_syn.cu — synthesis forward + MSE + backward.
//
// Replaces synthesize_forward / synthesize_backward (synthesis.hpp:191-233),
// conv1x1_* (layers.hpp:196-250), conv3x3_* (layers.hpp:257-343), mse_*
// (layers.hpp:643-657) and the straight-through clamp (layers.hpp:661-664,
// synthesis.hpp:215).  Three kernels per iteration:
//
//   k_syn_trunk_fwd   per pixel: z -> relu(c1) -> c2 = t, and the linear
//                     stabilizer term s = stab·z (3 + 3 planes); the F-wide
//                     hidden layer never leaves registers (663 MAC/px HOP)
//   k_syn_post        per 16x16 tile, in shared memory on replicate-clamped
//                     halos: residual 3x3 posts forward, clamp, MSE (fp64,
//                     owned pixels), dx̂, posts backward (transposed conv by
//                     gather), post weight gradients -> dt
//   k_syn_trunk_bwd2  (cc_syn_trunk.cu) recompute h1, dh1, dz and the
//                     c1/c2/stab weight gradients
#include <cuda_runtime.h>

#include "cc_kernels.h"
#include "cc_math.cuh"
#include "cc_reduce.cuh"

namespace ccb {

namespace {

constexpr int kLZ = kMaxLevels;  // z vector padded to 8 channels
// kSynTile (pixels per trunk-backward tile) lives in cc_plan.h


__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// ---------------------------------------------------------------- trunk fwd
__global__ void __launch_bounds__(256) k_syn_trunk_fwd(const Plan* __restrict__ pp) {
    const Plan& P = *pp;
    __shared__ float c1w[64 * kLZ], c1b[64], c2w[3 * 64], c2b[4], st[3 * kLZ];
    const int L = P.L, F = P.syn_F;
    for (int e = threadIdx.x; e < 64 * kLZ; e += blockDim.x) {
        const int f = e / kLZ, k = e - f * kLZ;
        c1w[e] = (f < F && k < L) ? P.params[P.off_c1w + f * L + k] : 0.0f;
    }
    for (int e = threadIdx.x; e < 64; e += blockDim.x) c1b[e] = e < F ? P.params[P.off_c1b + e] : 0.0f;
    for (int e = threadIdx.x; e < 3 * 64; e += blockDim.x) {
        const int co = e / 64, f = e - co * 64;
        c2w[e] = f < F ? P.params[P.off_c2w + co * F + f] : 0.0f;
    }
    if (threadIdx.x < 4) c2b[threadIdx.x] = threadIdx.x < 3 ? P.params[P.off_c2b + threadIdx.x] : 0.0f;
    if (threadIdx.x < 3 * kLZ) {
        const int co = threadIdx.x / kLZ, k = threadIdx.x - co * kLZ;
        st[threadIdx.x] = (P.off_sstab >= 0 && k < L) ? P.params[P.off_sstab + co * L + k] : 0.0f;
    }
    __syncthreads();
    const int64_t np = P.npix;
    for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < np;
         p += int64_t(gridDim.x) * blockDim.x) {
        float zv[kLZ];
#pragma unroll
        for (int k = 0; k < kLZ; ++k) zv[k] = k < L ? P.z[int64_t(k) * np + p] : 0.0f;
        float t0 = c2b[0], t1 = c2b[1], t2 = c2b[2];
        for (int f = 0; f < F; ++f) {
            float acc = c1b[f];
#pragma unroll
            for (int k = 0; k < kLZ; ++k) acc = fmaf(zv[k], c1w[f * kLZ + k], acc);
            const float h = acc > 0.0f ? acc : 0.0f;
            t0 = fmaf(c2w[f], h, t0);
            t1 = fmaf(c2w[64 + f], h, t1);
            t2 = fmaf(c2w[128 + f], h, t2);
        }
        P.syn_t[p] = t0;
        P.syn_t[np + p] = t1;
        P.syn_t[2 * np + p] = t2;
        // stabilizer s = stab·z (synthesis.hpp:211; zero padding is exact)
#pragma unroll
        for (int co = 0; co < 3; ++co) {
            float a = 0.0f;
#pragma unroll
            for (int k = 0; k < kLZ; ++k) a = fmaf(st[co * kLZ + k], zv[k], a);
            P.syn_sz[co * np + p] = a;
        }
    }
}

// ------------------------------------------------- fused posts + MSE (NP posts)
// On replicate-clamped windows W_h (the 16x16 tile grown by h, cut at the
// image border):
//   p_0 = t on W_2NP,  p_i = p_{i-1} + conv_i(p_{i-1}) on W_{2NP-i}
//   x̂ = clamp01(p_NP + s) on W_NP, dx̂ = 2(x̂ - x)/(3HW)        (encoder.hpp:256-260)
//   d_i = d_{i+1} + conv_iᵀ(d_{i+1}) on W_i, d_NP = dx̂           (synthesis.hpp:222-228)
// so dt = d_0 on the tile.  MSE and the post weight gradients sum over OWNED
// pixels only.
constexpr int kPT = 16;

template <int NP>
struct PostSmem {
    static constexpr int PW = kPT + 4 * NP;   // p_0 window edge
    static constexpr int DW = kPT + 2 * NP;   // d_NP window edge
    float p[NP + 1][3][PW * PW];
    float d[NP + 1][3][DW * DW];
    float sz[3][DW * DW];   // stabilizer term on W_NP
    float img[3][DW * DW];  // target on W_NP
    double red[8];
};

struct PWin {
    int r0, r1, c0, c1;  // inclusive, clamped
    __device__ __forceinline__ int w() const { return c1 - c0 + 1; }
    __device__ __forceinline__ int n() const { return (r1 - r0 + 1) * (c1 - c0 + 1); }
};

template <int NP>
__global__ void __launch_bounds__(256, 2) k_syn_post(const Plan* __restrict__ pp, int with_grad) {
    const Plan& P = *pp;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PostSmem<NP>& sm = *reinterpret_cast<PostSmem<NP>*>(smem_raw);
    __shared__ float w[2][81], bb[2][3];
    const int H = P.H, W = P.W;
    const int64_t np = P.npix;
    for (int i = 0; i < NP; ++i) {
        if (threadIdx.x < 81) w[i][threadIdx.x] = P.params[P.off_pw[i] + threadIdx.x];
        if (threadIdx.x < 3) bb[i][threadIdx.x] = P.params[P.off_pb[i] + threadIdx.x];
    }
    const float s = float(2.0 / double(3 * np));
    float wacc[2][10];
#pragma unroll
    for (int k = 0; k < 10; ++k) wacc[0][k] = wacc[1][k] = 0.0f;
    double mse = 0.0;
    const int tiles_x = (W + kPT - 1) / kPT;
    const int ntiles = tiles_x * ((H + kPT - 1) / kPT);
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int y0 = (tile / tiles_x) * kPT, x0 = (tile % tiles_x) * kPT;
        auto win = [&](int h) {
            return PWin{max(y0 - h, 0), min(y0 + kPT - 1 + h, H - 1), max(x0 - h, 0),
                        min(x0 + kPT - 1 + h, W - 1)};
        };
        __syncthreads();
        {  // stage p_0 = t on W_2NP, and s, x on W_NP (all loads in flight)
            const PWin a = win(2 * NP);
            const FDiv fa(a.w());
            for (int e = threadIdx.x; e < a.n(); e += 256) {
                const int q_ = fa.div(e);
                const int64_t p = int64_t(a.r0 + q_) * W + (a.c0 + (e - q_ * a.w()));
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) cp_async4(&sm.p[0][ch][e], P.syn_t + ch * np + p);
            }
            const PWin b = win(NP);
            const FDiv fb(b.w());
            for (int e = threadIdx.x; e < b.n(); e += 256) {
                const int q_ = fb.div(e);
                const int64_t p = int64_t(b.r0 + q_) * W + (b.c0 + (e - q_ * b.w()));
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    cp_async4(&sm.sz[ch][e], P.syn_sz + ch * np + p);
                    cp_async4(&sm.img[ch][e], P.image + ch * np + p);
                }
            }
        }
        cp_async_wait_all();
        __syncthreads();
        // forward posts: conv3x3_forward (layers.hpp:257-300) + residual (synthesis.hpp:207)
#pragma unroll
        for (int i = 1; i <= NP; ++i) {
            const PWin a = win(2 * NP - i + 1), b = win(2 * NP - i);
            const int aw = a.w();
            for (int e = threadIdx.x; e < b.n(); e += 256) {
                const int q_ = FDiv(b.w()).div(e);
                const int r = b.r0 + q_, c = b.c0 + (e - q_ * b.w());
                const int rm = max(r - 1, 0) - a.r0, r0 = r - a.r0, rp = min(r + 1, H - 1) - a.r0;
                const int cm = max(c - 1, 0) - a.c0, c0 = c - a.c0, cp = min(c + 1, W - 1) - a.c0;
                float x[3][9];
#pragma unroll
                for (int ci = 0; ci < 3; ++ci) {
                    const float* xs = sm.p[i - 1][ci];
                    x[ci][0] = xs[rm * aw + cm]; x[ci][1] = xs[rm * aw + c0]; x[ci][2] = xs[rm * aw + cp];
                    x[ci][3] = xs[r0 * aw + cm]; x[ci][4] = xs[r0 * aw + c0]; x[ci][5] = xs[r0 * aw + cp];
                    x[ci][6] = xs[rp * aw + cm]; x[ci][7] = xs[rp * aw + c0]; x[ci][8] = xs[rp * aw + cp];
                }
#pragma unroll
                for (int co = 0; co < 3; ++co) {
                    float v = bb[i - 1][co];
#pragma unroll
                    for (int ci = 0; ci < 3; ++ci) {
                        const float* k = w[i - 1] + (co * 3 + ci) * 9;
                        v += k[0] * x[ci][0] + k[1] * x[ci][1] + k[2] * x[ci][2] + k[3] * x[ci][3] +
                             k[4] * x[ci][4] + k[5] * x[ci][5] + k[6] * x[ci][6] + k[7] * x[ci][7] +
                             k[8] * x[ci][8];
                    }
                    sm.p[i][co][e] = v + x[co][4];
                }
            }
            __syncthreads();
        }
        {  // x̂, MSE (owned), dx̂ on W_NP  (synthesis.hpp:210-212, layers.hpp:643-657)
            const PWin a = win(NP);
            for (int e = threadIdx.x; e < a.n(); e += 256) {
                const int q_ = FDiv(a.w()).div(e);
                const int r = a.r0 + q_, c = a.c0 + (e - q_ * a.w());
                const int64_t p = int64_t(r) * W + c;
                const bool own = r >= y0 && r < y0 + kPT && c >= x0 && c < x0 + kPT;
#pragma unroll
                for (int co = 0; co < 3; ++co) {
                    float x = sm.p[NP][co][e] + sm.sz[co][e];
                    x = std_min(1.0f, std_max(0.0f, x));
                    const float tgt = sm.img[co][e];
                    if (own) {
                        const double dd = double(x) - double(tgt);
                        mse += dd * dd;
                    }
                    const float g = s * (x - tgt);
                    sm.d[NP][co][e] = g;
                    if (own && with_grad) P.syn_dx[co * np + p] = g;
                }
            }
        }
        if (!with_grad) continue;
        __syncthreads();
        // backward posts: transposed conv by gather (layers.hpp:302-343)
#pragma unroll
        for (int i = NP - 1; i >= 0; --i) {
            const PWin a = win(i + 1), b = win(i);
            const int aw = a.w();
            for (int e = threadIdx.x; e < b.n(); e += 256) {
                const int q_ = FDiv(b.w()).div(e);
                const int r = b.r0 + q_, c = b.c0 + (e - q_ * b.w());
                const int ra = r - a.r0, ca = c - a.c0;
                float sum[3] = {0.0f, 0.0f, 0.0f};
                if (r >= 1 && r <= H - 2 && c >= 1 && c <= W - 2) {
                    // interior: the exact flipped-kernel correlation
#pragma unroll
                    for (int co = 0; co < 3; ++co) {
                        const float* g = sm.d[i + 1][co];
                        float gv[9];
#pragma unroll
                        for (int q = 0; q < 9; ++q)
                            gv[q] = g[(ra - (q / 3 - 1)) * aw + (ca - (q % 3 - 1))];
#pragma unroll
                        for (int ci = 0; ci < 3; ++ci) {
                            const float* k = w[i] + (co * 3 + ci) * 9;
#pragma unroll
                            for (int q = 0; q < 9; ++q) sum[ci] = fmaf(k[q], gv[q], sum[ci]);
                        }
                    }
                } else {
                    // border: every (r', tap) with clamp(r' + dr) == r
                    int rr[3], dr[3], cc[3], dc[3];
                    int nr = 0, nc = 0;
                    for (int q = r - 1; q <= r + 1; ++q) {
                        if (q < 0 || q >= H) continue;
                        for (int d = -1; d <= 1; ++d)
                            if (clampi(q + d, 0, H - 1) == r && nr < 3) { rr[nr] = q - a.r0; dr[nr] = d; ++nr; }
                    }
                    for (int q = c - 1; q <= c + 1; ++q) {
                        if (q < 0 || q >= W) continue;
                        for (int d = -1; d <= 1; ++d)
                            if (clampi(q + d, 0, W - 1) == c && nc < 3) { cc[nc] = q - a.c0; dc[nc] = d; ++nc; }
                    }
                    for (int co = 0; co < 3; ++co) {
                        const float* g = sm.d[i + 1][co];
                        for (int u = 0; u < nr; ++u)
                            for (int v = 0; v < nc; ++v) {
                                const float gv = g[rr[u] * aw + cc[v]];
                                const int tap = (dr[u] + 1) * 3 + (dc[v] + 1);
#pragma unroll
                                for (int ci = 0; ci < 3; ++ci) sum[ci] += w[i][(co * 3 + ci) * 9 + tap] * gv;
                            }
                    }
                }
#pragma unroll
                for (int ci = 0; ci < 3; ++ci) {
                    const float dv = sum[ci] + sm.d[i + 1][ci][ra * aw + ca];  // residual path
                    sm.d[i][ci][e] = dv;
                    if (i == 0) P.syn_dt[ci * np + int64_t(r) * W + c] = dv;
                }
            }
            __syncthreads();
        }
        if (NP == 0) {  // dt = dx̂
            const PWin a = win(0);
            for (int e = threadIdx.x; e < a.n(); e += 256) {
                const int q_ = FDiv(a.w()).div(e);
                const int r = a.r0 + q_, c = a.c0 + (e - q_ * a.w());
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) P.syn_dt[ch * np + int64_t(r) * W + c] = sm.d[0][ch][e];
            }
        }
        // post weight gradients over OWNED pixels: thread (column c, slot s)
        // walks the 16 rows of column c for pairs s and s+16 of the NP*9
        // (post, co, ci) pairs: 9 tap sums each (+ the bias sum, used when
        // ci == 0).  A warp reads 16 consecutive columns: no bank conflicts.
        if constexpr (NP > 0) {
            const int cc = threadIdx.x % kPT, slot = threadIdx.x / kPT;
            const int c = x0 + cc;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int pair = slot + 16 * h;
                if (pair >= NP * 9 || c >= W) continue;
                const int i = pair / 9, co = (pair % 9) / 3, ci = pair % 3;
                const PWin a = win(i + 1), x = win(2 * NP - i);
                const int aw = a.w(), xw = x.w();
                const float* g = sm.d[i + 1][co];
                const float* xs = sm.p[i][ci];
                const int cm = max(c - 1, 0) - x.c0, c0 = c - x.c0, cp = min(c + 1, W - 1) - x.c0;
                const int rend = min(kPT, H - y0);
                for (int rr = 0; rr < rend; ++rr) {
                    const int r = y0 + rr;
                    const int rm = max(r - 1, 0) - x.r0, r0 = r - x.r0, rp = min(r + 1, H - 1) - x.r0;
                    const float gv = g[(r - a.r0) * aw + (c - a.c0)];
                    float* wa = wacc[h];
                    wa[0] = fmaf(gv, xs[rm * xw + cm], wa[0]);
                    wa[1] = fmaf(gv, xs[rm * xw + c0], wa[1]);
                    wa[2] = fmaf(gv, xs[rm * xw + cp], wa[2]);
                    wa[3] = fmaf(gv, xs[r0 * xw + cm], wa[3]);
                    wa[4] = fmaf(gv, xs[r0 * xw + c0], wa[4]);
                    wa[5] = fmaf(gv, xs[r0 * xw + cp], wa[5]);
                    wa[6] = fmaf(gv, xs[rp * xw + cm], wa[6]);
                    wa[7] = fmaf(gv, xs[rp * xw + c0], wa[7]);
                    wa[8] = fmaf(gv, xs[rp * xw + cp], wa[8]);
                    wa[9] += gv;
                }
            }
        }
    }
    // fixed-order reductions: MSE partial + per-post weight-gradient partial rows
    const double mtot = block_sum(mse, sm.red);
    if (threadIdx.x == 0) P.mse_part[blockIdx.x] = mtot;
    if constexpr (NP > 0) {
        if (!with_grad) return;
        __syncthreads();
        float* scratch = &sm.p[0][0][0];  // [pair][column][10]
        {
            const int cc = threadIdx.x % kPT, slot = threadIdx.x / kPT;
            for (int h = 0; h < 2; ++h) {
                const int pair = slot + 16 * h;
                if (pair < NP * 9)
                    for (int k = 0; k < 10; ++k) scratch[(pair * kPT + cc) * 10 + k] = wacc[h][k];
            }
        }
        __syncthreads();
        for (int i = 0; i < NP; ++i) {
            const PartialRegion& R = P.region[P.reg_post[i]];
            double* row = P.partials + R.base + int64_t(blockIdx.x) * R.count;
            for (int e = threadIdx.x; e < R.count; e += blockDim.x) {
                const int pidx = R.param_off + e;
                double v = 0.0;
                int pair = -1, k = 0;
                if (pidx >= P.off_pw[i] && pidx < P.off_pw[i] + 81) {
                    const int q = pidx - P.off_pw[i];  // (co*3 + ci)*9 + tap
                    pair = i * 9 + q / 9;
                    k = q % 9;
                } else if (pidx >= P.off_pb[i] && pidx < P.off_pb[i] + 3) {
                    pair = i * 9 + (pidx - P.off_pb[i]) * 3;  // (co, ci = 0) carries the bias
                    k = 9;
                }
                if (pair >= 0)
                    for (int gq = 0; gq < kPT; ++gq) v += double(scratch[(pair * kPT + gq) * 10 + k]);
                row[e] = v;
            }
        }
    }
}

}  // namespace

void syn_post_configure() {
    cudaFuncSetAttribute(k_syn_post<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(PostSmem<0>)));
    cudaFuncSetAttribute(k_syn_post<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(PostSmem<1>)));
    cudaFuncSetAttribute(k_syn_post<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(PostSmem<2>)));
}

int syn_post_tiles(int H, int W) { return ((H + kPT - 1) / kPT) * ((W + kPT - 1) / kPT); }

void launch_syn_forward(const LaunchCtx& L, bool backward) {
    const Plan& H = *L.host;
    k_syn_trunk_fwd<<<L.pix_blocks, 256, 0, L.stream>>>(L.plan);
    const int g = H.n_mse_part;
    const int wg = backward ? 1 : 0;
    switch (H.posts) {
        case 0: k_syn_post<0><<<g, 256, sizeof(PostSmem<0>), L.stream>>>(L.plan, wg); break;
        case 1: k_syn_post<1><<<g, 256, sizeof(PostSmem<1>), L.stream>>>(L.plan, wg); break;
        default: k_syn_post<2><<<g, 256, sizeof(PostSmem<2>), L.stream>>>(L.plan, wg); break;
    }
}

}  // namespace ccb
