// cc_syn_post.cu — the synthesis "posts" (residual 3x3 convs), x̂, MSE and
// their backward: synthesis.hpp:202-228, conv3x3_forward/backward
// (layers.hpp:257-343), mse_forward/backward (layers.hpp:643-657), clamp01
// (layers.hpp:661-664).
//
// One CTA (256 threads) walks 32x16-pixel tiles.  Everything lives in
// shared memory on a VIRTUAL window: the tile grown by 2·NP pixels, where a
// position outside the image holds the replicate-padded value (the clamped
// in-image position), so every 3x3 stencil reads its neighbours directly:
//   p_0 = t on W_2NP (loaded clamped),
//   p_i = p_{i-1} + b_i + conv_i(p_{i-1}) on W_{2NP-i}  (then re-clamped),
//   x̂ = clamp01(p_NP + s), dx̂ = 2(x̂ - x)/(3HW) on W_NP (0 outside the image),
//   d_i = d_{i+1} + conv_iᵀ(d_{i+1}) on W_i, where the transposed stencil is
//   computed in virtual space and the ring outside the image is folded back
//   onto the edge (the adjoint of the clamp), dt = d_0 on the tile.
// Convolutions run as register strips: a thread owns one column and RS rows,
// keeps the (RS+2)x3 neighbourhood of every channel in registers and the 27
// weights of one output channel at a time (loads : FMAs ≈ 1 : 10).
// MSE (fp64) and the post weight gradients sum over OWNED pixels only; the
// weight gradients stay in registers across tiles and are reduced in a fixed
// order once per CTA.  No atomics.
#include <cuda_runtime.h>

#include <type_traits>

#include "cc_kernels.h"
#include "cc_math.cuh"
#include "cc_reduce.cuh"

namespace ccb {

namespace {

constexpr int TW = 32, TH = 16;  // owned tile (columns x rows)
constexpr int NT = 256;

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

template <int NP>
struct PC {
    static constexpr int H4 = 2 * NP;          // halo of p_0
    static constexpr int PW = TW + 2 * H4;     // virtual window pitch
    static constexpr int PH = TH + 2 * H4;
    static constexpr int PL = PW * PH;         // floats per plane
    static constexpr int NPL = NP > 0 ? NP : 1;
};

template <int NP>
struct alignas(16) PostSmem2 {
    using C = PC<NP>;
    float p[NP + 1][3][C::PL];   // p_0 .. p_NP
    float d[NP + 1][3][C::PL];   // d_0 .. d_NP (d_NP = dx̂)
    float sz[3][C::PL];
    float img[3][C::PL];
    float wf[C::NPL][3 * 27];    // forward weights  [co][ci][tap]
    float wb[C::NPL][3 * 27];    // transposed       [ci][co][flipped tap]
    float2 wfp[C::NPL][27];      // (co 0, co 1) pairs of wf per [ci][tap]: FFMA2 operands
    float2 wbp[C::NPL][27];      // the same for wb
    float bias[C::NPL][4];
    double red[NT / 32];
};

// out[co] over window W_h (virtual coords) from the 3 planes `in`:
//   out = (bias) + sum_{ci,tap} wk[co][ci][tap] * in[ci][v + off(tap)] + in[co][v]
// `wk` is [co][27] in shared memory, `wkp` its (co 0, co 1) pairs per
// [ci][tap]: output channels 0 and 1 are the two FFMA2 lanes (the input value
// the broadcast operand), channel 2 a plain FMA — the per-channel order of
// the terms (ci, then tap) is unchanged.  One thread = one column x RS rows.
template <int NP, int h>
__device__ __forceinline__ void conv_pass(const float* __restrict__ in, float* __restrict__ out,
                                          const float* __restrict__ wk, const float2* __restrict__ wkp,
                                          const float* __restrict__ bias, int tid) {
    using C = PC<NP>;
    constexpr int w = TW + 2 * h, hh = TH + 2 * h;
    constexpr int NS = (NT / w) < hh ? (NT / w) : hh;
    constexpr int RS = (hh + NS - 1) / NS;
    if (tid >= w * NS) return;
    const int vc = C::H4 - h + tid % w;
    const int ra = C::H4 - h + (tid / w) * RS;
    const int rb = min(ra + RS, C::H4 - h + hh);
    if (ra >= rb) return;
    float x[3][RS + 2][3];
#pragma unroll
    for (int ci = 0; ci < 3; ++ci)
#pragma unroll
        for (int rr = 0; rr < RS + 2; ++rr)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc)
                x[ci][rr][cc] = (ra - 1 + rr <= rb) ? in[ci * C::PL + (ra - 1 + rr) * C::PW + vc - 1 + cc] : 0.0f;
    float2 v01[RS];
    float v2[RS];
    {
        const float b0 = bias ? bias[0] : 0.0f, b1 = bias ? bias[1] : 0.0f, b2 = bias ? bias[2] : 0.0f;
#pragma unroll
        for (int rr = 0; rr < RS; ++rr) {
            v01[rr] = make_float2(b0, b1);
            v2[rr] = b2;
        }
    }
#pragma unroll
    for (int ci = 0; ci < 3; ++ci) {
        float2 wp[9];
        float w2[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            wp[q] = wkp[ci * 9 + q];
            w2[q] = wk[2 * 27 + ci * 9 + q];
        }
#pragma unroll
        for (int rr = 0; rr < RS; ++rr)
#pragma unroll
            for (int q = 0; q < 9; ++q) {
                const float xv = x[ci][rr + q / 3][q % 3];
                v01[rr] = ffma2(wp[q], make_float2(xv, xv), v01[rr]);
                v2[rr] = fmaf(w2[q], xv, v2[rr]);
            }
    }
#pragma unroll
    for (int rr = 0; rr < RS; ++rr)
        if (ra + rr < rb) {
            float* o = out + (ra + rr) * C::PW + vc;
            o[0] = v01[rr].x + x[0][rr + 1][1];
            o[C::PL] = v01[rr].y + x[1][rr + 1][1];
            o[2 * C::PL] = v2[rr] + x[2][rr + 1][1];
        }
}

template <int NP>
__global__ void __launch_bounds__(NT, 2) k_syn_post2(const Plan* __restrict__ pp, int with_grad) {
    using C = PC<NP>;
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PostSmem2<NP>& sm = *reinterpret_cast<PostSmem2<NP>*>(smem_raw);
    const int tid = threadIdx.x;
    const int H = P.H, W = P.W;
    const int64_t np = P.npix;
    for (int i = 0; i < NP; ++i) {
        for (int e = tid; e < 81; e += NT) {
            const float v = P.params[P.off_pw[i] + e];  // w[co][ci][tap]
            const int co = e / 27, ci = (e / 9) % 3, q = e % 9;
            sm.wf[i][e] = v;
            sm.wb[i][ci * 27 + co * 9 + (8 - q)] = v;
            // FFMA2 pairs: wf as [ci][tap] (co 0 | co 1), wb as [co][flipped tap] (ci 0 | ci 1)
            if (co < 2) reinterpret_cast<float*>(&sm.wfp[i][ci * 9 + q])[co] = v;
            if (ci < 2) reinterpret_cast<float*>(&sm.wbp[i][co * 9 + (8 - q)])[ci] = v;
        }
        if (tid < 4) sm.bias[i][tid] = tid < 3 ? P.params[P.off_pb[i] + tid] : 0.0f;
    }
    const float s = float(2.0 / double(3 * P.npix_global));  // layers.hpp:655 (whole image)
    const int own_lo = P.pix_own_lo, own_hi = P.pix_own_hi;  // row bands: loss rows
    // post weight-gradient accumulators: thread (column wc, slot ws) owns the
    // (post, co, ci) pairs ws, ws+8, ws+16: 9 taps + the bias sum (ci == 0)
    const int wc = tid % TW, ws = tid / TW;
    float wacc[3][10];
#pragma unroll
    for (int hq = 0; hq < 3; ++hq)
#pragma unroll
        for (int k = 0; k < 10; ++k) wacc[hq][k] = 0.0f;
    double mse = 0.0;
    const int tiles_x = (W + TW - 1) / TW;
    const int ntiles = tiles_x * ((H + TH - 1) / TH);
    // large images: every 16 tiles the fp32 per-thread dW sums move into an
    // fp64 per-thread slot (their fp32 chains stay <= 256 terms long)
    double* flush = P.post_scratch ? P.post_scratch + (int64_t(blockIdx.x) * NT + tid) * 30 : nullptr;
    int tcount = 0;
    pdl_wait();  // t, s of the trunk forward (weights above were staged before)
    pdl_trigger();
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        if (flush && NP > 0 && with_grad && ++tcount % 16 == 0) {
#pragma unroll
            for (int hq = 0; hq < 3; ++hq)
#pragma unroll
                for (int k = 0; k < 10; ++k) {
                    flush[hq * 10 + k] += double(wacc[hq][k]);
                    wacc[hq][k] = 0.0f;
                }
        }
        const int y0 = (tile / tiles_x) * TH, x0 = (tile % tiles_x) * TW;
        const int gy0 = y0 - C::H4, gx0 = x0 - C::H4;  // global coords of virtual (0,0)
        const bool border = gy0 < 0 || gx0 < 0 || gy0 + C::PH > H || gx0 + C::PW > W;
        __syncthreads();
        // ---- stage p_0 = t (W_2NP) and s, x (W_NP), replicate-clamped ----
        for (int e = tid; e < C::PL; e += NT) {
            const int vr = e / C::PW, vc = e % C::PW;
            const int64_t p = int64_t(clampi(gy0 + vr, 0, H - 1)) * W + clampi(gx0 + vc, 0, W - 1);
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) cp_async4(&sm.p[0][ch][e], P.syn_t + ch * np + p);
            const bool in_np = vr >= C::H4 - NP && vr < C::H4 + TH + NP && vc >= C::H4 - NP && vc < C::H4 + TW + NP;
            if (in_np) {
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    cp_async4(&sm.sz[ch][e], P.syn_sz + ch * np + p);
                    cp_async4(&sm.img[ch][e], P.image + ch * np + p);
                }
            }
        }
        cp_async_wait_all();
        __syncthreads();
        // ---- forward posts ----
        if constexpr (NP >= 1) {
            conv_pass<NP, 2 * NP - 1>(sm.p[0][0], sm.p[1][0], sm.wf[0], sm.wfp[0], sm.bias[0], tid);
            __syncthreads();
            if (border) {  // re-clamp p_1 outside the image
                constexpr int h = 2 * NP - 1;
                for (int e = tid; e < C::PL; e += NT) {
                    const int vr = e / C::PW, vc = e % C::PW;
                    if (vr < C::H4 - h || vr >= C::H4 + TH + h || vc < C::H4 - h || vc >= C::H4 + TW + h) continue;
                    const int gr = gy0 + vr, gc = gx0 + vc;
                    if (gr >= 0 && gr < H && gc >= 0 && gc < W) continue;
                    const int src = (clampi(gr, 0, H - 1) - gy0) * C::PW + (clampi(gc, 0, W - 1) - gx0);
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) sm.p[1][ch][e] = sm.p[1][ch][src];
                }
                __syncthreads();
            }
        }
        if constexpr (NP >= 2) {
            conv_pass<NP, 2 * NP - 2>(sm.p[1][0], sm.p[2][0], sm.wf[1], sm.wfp[1], sm.bias[1], tid);
            __syncthreads();
            // p_2 is only read on W_NP by the x̂ pass and in-image by dW: no re-clamp
        }
        // ---- x̂, MSE (owned), dx̂ on W_NP; d_NP = 0 outside the image (the
        // transposed stencils of border tiles read it one ring further out) ----
        {
            for (int v = tid; v < C::PL; v += NT) {
                const int vr = v / C::PW, vc = v % C::PW;
                const int gr = gy0 + vr, gc = gx0 + vc;
                if (vr < C::H4 - NP || vr >= C::H4 + TH + NP || vc < C::H4 - NP || vc >= C::H4 + TW + NP) {
#pragma unroll
                    for (int co = 0; co < 3; ++co) sm.d[NP][co][v] = 0.0f;
                    continue;
                }
                const bool inimg = gr >= 0 && gr < H && gc >= 0 && gc < W;
                const bool loss = inimg && gr >= own_lo && gr < own_hi;  // band-owned pixel
                const bool own = gr >= y0 && gr < y0 + TH && gc >= x0 && gc < x0 + TW && inimg;
#pragma unroll
                for (int co = 0; co < 3; ++co) {
                    float xh = sm.p[NP][co][v] + sm.sz[co][v];
                    xh = std_min(1.0f, std_max(0.0f, xh));
                    const float tgt = sm.img[co][v];
                    if (own && loss) {
                        const double dd = double(xh) - double(tgt);
                        mse += dd * dd;
                    }
                    const float g = loss ? s * (xh - tgt) : 0.0f;
                    sm.d[NP][co][v] = g;
                    if (own && with_grad) P.syn_dx[co * np + int64_t(gr) * W + gc] = g;
                }
            }
        }
        if (!with_grad) continue;
        __syncthreads();
        // ---- backward posts: d_i = d_{i+1} + conv_iᵀ(d_{i+1}) ----
        auto back = [&](auto hconst, int i) {
            constexpr int hi = decltype(hconst)::value;  // window of d_i
            if (!border) {
                conv_pass<NP, hi>(sm.d[i + 1][0], sm.d[i][0], sm.wb[i], sm.wbp[i], nullptr, tid);
                __syncthreads();
                return;
            }
            // border tile: compute on W_{i+1} (covers the ring outside the
            // image next to W_i), fold the ring onto the edge, zero it
            conv_pass<NP, hi + 1>(sm.d[i + 1][0], sm.d[i][0], sm.wb[i], sm.wbp[i], nullptr, tid);
            __syncthreads();
            constexpr int w = TW + 2 * hi, hh = TH + 2 * hi;
            float acc[3][3];
            int cnt = 0;
            for (int e = tid; e < w * hh; e += NT, ++cnt) {
                const int vr = C::H4 - hi + e / w, vc = C::H4 - hi + e % w;
                const int gr = gy0 + vr, gc = gx0 + vc;
                float a[3] = {0.0f, 0.0f, 0.0f};
                if (gr >= 0 && gr < H && gc >= 0 && gc < W && (gr == 0 || gr == H - 1 || gc == 0 || gc == W - 1)) {
                    for (int dr = -1; dr <= 1; ++dr)
                        for (int dc = -1; dc <= 1; ++dc) {
                            if (dr == 0 && dc == 0) continue;
                            const int qr = gr + dr, qc = gc + dc;
                            const bool pre = (qr < 0 || qr >= H || qc < 0 || qc >= W) &&
                                             clampi(qr, 0, H - 1) == gr && clampi(qc, 0, W - 1) == gc;
                            if (!pre) continue;
                            const int v = (qr - gy0) * C::PW + (qc - gx0);
#pragma unroll
                            for (int ch = 0; ch < 3; ++ch) a[ch] += sm.d[i][ch][v];
                        }
                }
                if (cnt < 3)
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) acc[cnt][ch] = a[ch];
            }
            __syncthreads();
            cnt = 0;
            for (int e = tid; e < w * hh; e += NT, ++cnt) {
                const int vr = C::H4 - hi + e / w, vc = C::H4 - hi + e % w;
                const int gr = gy0 + vr, gc = gx0 + vc;
                const int v = vr * C::PW + vc;
                if (cnt < 3 && gr >= 0 && gr < H && gc >= 0 && gc < W)
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) sm.d[i][ch][v] += acc[cnt][ch];
            }
            // zero the virtual positions outside the image on W_{i+1}
            constexpr int w1 = TW + 2 * (hi + 1), h1 = TH + 2 * (hi + 1);
            for (int e = tid; e < w1 * h1; e += NT) {
                const int vr = C::H4 - hi - 1 + e / w1, vc = C::H4 - hi - 1 + e % w1;
                const int gr = gy0 + vr, gc = gx0 + vc;
                if (gr >= 0 && gr < H && gc >= 0 && gc < W) continue;
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) sm.d[i][ch][vr * C::PW + vc] = 0.0f;
            }
            __syncthreads();
        };
        if constexpr (NP >= 2) back(std::integral_constant<int, 1>{}, 1);
        if constexpr (NP >= 1) back(std::integral_constant<int, 0>{}, 0);
        // dt = d_0 on the owned pixels
        for (int e = tid; e < TW * TH; e += NT) {
            const int rr = e / TW, cc = e % TW;
            const int gr = y0 + rr, gc = x0 + cc;
            if (gr >= H || gc >= W) continue;
            const int v = (C::H4 + rr) * C::PW + (C::H4 + cc);
#pragma unroll
            for (int ch = 0; ch < 3; ++ch)
                P.syn_dt[ch * np + int64_t(gr) * W + gc] = NP > 0 ? sm.d[0][ch][v] : sm.d[NP][ch][v];
        }
        // ---- post weight gradients over OWNED pixels (virtual clamped p_i) ----
        if constexpr (NP > 0) {
            const int gc = x0 + wc;
            if (gc < W) {
                const int rend = min(TH, H - y0);
#pragma unroll
                for (int hq = 0; hq < 3; ++hq) {
                    const int pair = ws + 8 * hq;
                    if (pair >= NP * 9) continue;
                    const int i = pair / 9, co = (pair % 9) / 3, ci = pair % 3;
                    const float* g = sm.d[i + 1][co];
                    const float* xs = sm.p[i][ci];
                    const int vc = C::H4 + wc;
                    float x0r[3], x1r[3];
#pragma unroll
                    for (int cc = 0; cc < 3; ++cc) {
                        x0r[cc] = xs[(C::H4 - 1) * C::PW + vc - 1 + cc];
                        x1r[cc] = xs[C::H4 * C::PW + vc - 1 + cc];
                    }
                    float* wa = wacc[hq];
                    for (int rr = 0; rr < rend; ++rr) {
                        const int vr = C::H4 + rr;
                        float x2r[3];
#pragma unroll
                        for (int cc = 0; cc < 3; ++cc) x2r[cc] = xs[(vr + 1) * C::PW + vc - 1 + cc];
                        const float gv = g[vr * C::PW + vc];
#pragma unroll
                        for (int cc = 0; cc < 3; ++cc) {
                            wa[cc] = fmaf(gv, x0r[cc], wa[cc]);
                            wa[3 + cc] = fmaf(gv, x1r[cc], wa[3 + cc]);
                            wa[6 + cc] = fmaf(gv, x2r[cc], wa[6 + cc]);
                        }
                        wa[9] += gv;
#pragma unroll
                        for (int cc = 0; cc < 3; ++cc) {
                            x0r[cc] = x1r[cc];
                            x1r[cc] = x2r[cc];
                        }
                    }
                }
            }
        }
    }
    // ---- fixed-order reductions ----
    const double mtot = block_sum(mse, sm.red);
    if (tid == 0) P.mse_part[blockIdx.x] = mtot;
    if constexpr (NP > 0) {
        if (!with_grad) return;
        __syncthreads();
        static_assert(sizeof(double) * NP * 9 * TW * 10 <= sizeof(float) * 2 * (NP + 1) * 3 * C::PL,
                      "fp64 scratch fits in the p / d planes");
        double* scratch = reinterpret_cast<double*>(&sm.p[0][0][0]);  // [pair][column][10]
#pragma unroll
        for (int hq = 0; hq < 3; ++hq) {
            const int pair = ws + 8 * hq;
            if (pair < NP * 9)
#pragma unroll
                for (int k = 0; k < 10; ++k)
                    scratch[(pair * TW + wc) * 10 + k] =
                        double(wacc[hq][k]) + (flush ? flush[hq * 10 + k] : 0.0);
        }
        __syncthreads();
        for (int i = 0; i < NP; ++i) {
            const PartialRegion& R = P.region[P.reg_post[i]];
            const PartialRow row(P, R, blockIdx.x);
            for (int e = tid; e < R.count; e += NT) {
                const int pidx = R.param_off + e;
                int pair = -1, k = 0;
                if (pidx >= P.off_pw[i] && pidx < P.off_pw[i] + 81) {
                    const int q = pidx - P.off_pw[i];  // (co*3 + ci)*9 + tap
                    pair = i * 9 + q / 9;
                    k = q % 9;
                } else if (pidx >= P.off_pb[i] && pidx < P.off_pb[i] + 3) {
                    pair = i * 9 + (pidx - P.off_pb[i]) * 3;  // (co, ci = 0) carries the bias
                    k = 9;
                }
                double v = 0.0;
                if (pair >= 0)
                    for (int c = 0; c < TW; ++c) v += scratch[(pair * TW + c) * 10 + k];
                row[e] = v;
            }
        }
    }
}

}  // namespace

void syn_post_configure() {
    cudaFuncSetAttribute(k_syn_post2<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(PostSmem2<0>)));
    cudaFuncSetAttribute(k_syn_post2<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(PostSmem2<1>)));
    cudaFuncSetAttribute(k_syn_post2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(PostSmem2<2>)));
}

int syn_post_tiles(int H, int W) { return ((H + TH - 1) / TH) * ((W + TW - 1) / TW); }

void launch_syn_post(const LaunchCtx& L, bool backward) {
    const Plan& H = *L.host;
    if (H.post_scratch && backward) {
        if (L.batch != 1) throw_config("batched launches need images below the posts' fp64 flush-slot size");
        cuda_check(cudaMemsetAsync(H.post_scratch, 0, sizeof(double) * size_t(H.n_mse_part) * NT * 30, L.stream),
                   "cudaMemsetAsync");
    }
    const int g = H.n_mse_part;
    const int wg = backward ? 1 : 0;
    switch (H.posts) {
        case 0: launch_pdl(k_syn_post2<0>, dim3(g, 1, L.batch), dim3(NT), sizeof(PostSmem2<0>), L.stream, 's', L.plan, wg); break;
        case 1: launch_pdl(k_syn_post2<1>, dim3(g, 1, L.batch), dim3(NT), sizeof(PostSmem2<1>), L.stream, 's', L.plan, wg); break;
        default: launch_pdl(k_syn_post2<2>, dim3(g, 1, L.batch), dim3(NT), sizeof(PostSmem2<2>), L.stream, 's', L.plan, wg); break;
    }
}

}  // namespace ccb
