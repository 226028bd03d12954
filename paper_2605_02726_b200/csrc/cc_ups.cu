// cc_ups.cu — learned 2x upsampling chain, forward and backward.
//
// Replaces upsample_forward / upsample_backward (synthesis.hpp:55-139) built
// from tconv2x_rows/cols (layers.hpp:353-460) and conv3x3_sym
// (layers.hpp:467-515).  Main grid k >= 1 is lifted through stages
// j = k-1 .. 0 (stage parameters ups[j] are shared by every grid passing
// through it).  All grids that are at stage j run in ONE launch per sub-op
// (blockIdx.y = grid), so the chain costs 3 launches per stage regardless of
// the number of grids.  The backward is written as deterministic GATHERS over
// the replicate-clamped index maps (the reference scatters with +=), and the
// tap gradients dk4 / dr3 are per-CTA fp64 partials reduced in fixed order.
#include <cuda_runtime.h>

#include "cc_kernels.h"
#include "cc_math.cuh"
#include "cc_reduce.cuh"

namespace ccb {

namespace {

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Polyphase tap table of the symmetric x2 transposed conv (layers.hpp:346-351):
// output t reads inputs idx[0..3] with taps tap[0..3].
__device__ __forceinline__ void tconv_map(int t, int last, int (&idx)[4], int (&tap)[4]) {
    const int u = t >> 1;
    if ((t & 1) == 0) {
        idx[0] = u >= 2 ? u - 2 : 0;
        idx[1] = u >= 1 ? u - 1 : 0;
        idx[2] = u;
        idx[3] = u < last ? u + 1 : last;
        tap[0] = 0; tap[1] = 2; tap[2] = 3; tap[3] = 1;
    } else {
        idx[0] = u >= 1 ? u - 1 : 0;
        idx[1] = u;
        idx[2] = u < last ? u + 1 : last;
        idx[3] = u + 2 < last ? u + 2 : last;
        tap[0] = 1; tap[1] = 3; tap[2] = 2; tap[3] = 0;
    }
}

__device__ __forceinline__ const float* stage_in(const Plan& P, const UpsStage& s) {
    return s.in_is_pad ? P.yhat_pad + s.in_off : P.ups_buf + s.in_off;
}
__device__ __forceinline__ float* stage_out(const Plan& P, const UpsStage& s) {
    return s.out_is_z ? P.z + s.out_off : P.ups_buf + s.out_off;
}
__device__ __forceinline__ const float* stage_dout(const Plan& P, const UpsStage& s) {
    return s.dout_is_z ? P.dz + s.dout_off : P.ups_grad + s.dout_off;
}
__device__ __forceinline__ float* stage_din(const Plan& P, const UpsStage& s) {
    return s.din_is_lat ? P.dups + s.din_off : P.ups_grad + s.din_off;
}

// ---------------------------------------------------------------- forward
// tconv2x_rows_forward (layers.hpp:353-376): rowtmp[u][t], u < rows_in.
__global__ void k_ups_rows_fwd(const Plan* __restrict__ pp, int j) {
    const Plan& P = *pp;
    const UpsStage& s = P.ups[j][blockIdx.y];
    const float* k4 = P.params + P.off_tconv[j];
    const float k0 = k4[0], k1 = k4[1], k2 = k4[2], k3 = k4[3];
    const float* in = stage_in(P, s);
    float* out = P.ups_buf + s.row_off;
    const int64_t n = int64_t(s.rows_in) * s.cols_out;
    const int last = s.cols_in - 1;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int r = int(e / s.cols_out), t = int(e - int64_t(r) * s.cols_out);
        const float* xi = in + int64_t(r) * s.in_stride;
        const int u = t >> 1;
        float y;
        if ((t & 1) == 0) {
            const int a = u >= 2 ? u - 2 : 0, b = u >= 1 ? u - 1 : 0, d = u < last ? u + 1 : last;
            y = k0 * xi[a] + k2 * xi[b] + k3 * xi[u] + k1 * xi[d];
        } else {
            const int a = u >= 1 ? u - 1 : 0, b = u < last ? u + 1 : last;
            const int d = u + 2 < last ? u + 2 : last;
            y = k1 * xi[a] + k3 * xi[u] + k2 * xi[b] + k0 * xi[d];
        }
        out[e] = y;
    }
}

// tconv2x_cols_forward (layers.hpp:407-429): coltmp[t][c], t < rows_out.
__global__ void k_ups_cols_fwd(const Plan* __restrict__ pp, int j) {
    const Plan& P = *pp;
    const UpsStage& s = P.ups[j][blockIdx.y];
    const float* k4 = P.params + P.off_tconv[j];
    const float* in = P.ups_buf + s.row_off;
    float* out = P.ups_buf + s.col_off;
    const int w = s.cols_out;
    const int64_t n = int64_t(s.rows_out) * w;
    const int last = s.rows_in - 1;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int t = int(e / w), c = int(e - int64_t(t) * w);
        int idx[4], tap[4];
        tconv_map(t, last, idx, tap);
        out[e] = k4[tap[0]] * in[int64_t(idx[0]) * w + c] + k4[tap[1]] * in[int64_t(idx[1]) * w + c] +
                 k4[tap[2]] * in[int64_t(idx[2]) * w + c] + k4[tap[3]] * in[int64_t(idx[3]) * w + c];
    }
}

// conv3x3_sym_forward (layers.hpp:467-483), replicate padding.
__global__ void k_ups_refine_fwd(const Plan* __restrict__ pp, int j) {
    const Plan& P = *pp;
    const UpsStage& s = P.ups[j][blockIdx.y];
    const float* r3 = P.params + P.off_refine[j];
    const float kc = r3[0], ke = r3[1], ko = r3[2];
    const float* in = P.ups_buf + s.col_off;
    float* out = stage_out(P, s);
    const int h = s.rows_out, w = s.cols_out;
    const int64_t n = int64_t(h) * w;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int r = int(e / w), c = int(e - int64_t(r) * w);
        const int rm = r > 0 ? r - 1 : 0, rp = r < h - 1 ? r + 1 : h - 1;
        const int cm = c > 0 ? c - 1 : 0, cp = c < w - 1 ? c + 1 : w - 1;
        const float* x0 = in + int64_t(rm) * w;
        const float* x1 = in + int64_t(r) * w;
        const float* x2 = in + int64_t(rp) * w;
        out[e] = kc * x1[c] + ke * (x0[c] + x2[c] + x1[cm] + x1[cp]) +
                 ko * (x0[cm] + x0[cp] + x2[cm] + x2[cp]);
    }
}

// z plane 0 is main grid 0 itself (synthesis.hpp:62-64).
__global__ void k_copy_z0(const Plan* __restrict__ pp) {
    const Plan& P = *pp;
    const GridGeom& g = P.g[P.main_gi[0]];
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < P.npix;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int r = int(e / P.W), c = int(e - int64_t(r) * P.W);
        P.z[e] = P.yhat_pad[g.pad_base + int64_t(r) * g.stride + c];
    }
}

// --------------------------------------------------------------- backward
// (r', d) pairs with clamp(r' + d, 0, n-1) == r, d in {-1, 0, 1}, r' in [0, n).
__device__ __forceinline__ int nbr_pairs(int r, int n, int (&rr)[4], int (&dd)[4]) {
    int k = 0;
    for (int rp = r - 1; rp <= r + 1; ++rp) {
        if (rp < 0 || rp >= n) continue;
        for (int d = -1; d <= 1; ++d)
            if (clampi(rp + d, 0, n - 1) == r && k < 4) {
                rr[k] = rp;
                dd[k] = d;
                ++k;
            }
    }
    return k;
}

// conv3x3_sym_backward (layers.hpp:486-515): dcol by gather, dr3 partials.
__global__ void k_ups_refine_bwd(const Plan* __restrict__ pp, int j) {
    const Plan& P = *pp;
    const UpsStage& s = P.ups[j][blockIdx.y];
    const float* r3 = P.params + P.off_refine[j];
    const float kc = r3[0], ke = r3[1], ko = r3[2];
    const float* x = P.ups_buf + s.col_off;
    const float* dout = stage_dout(P, s);
    float* dcol = P.ups_grad + s.col_off;
    const int h = s.rows_out, w = s.cols_out;
    const int64_t n = int64_t(h) * w;
    double acc[3] = {0.0, 0.0, 0.0};
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int r = int(e / w), c = int(e - int64_t(r) * w);
        // dr3 partials, as written by the forward-direction loop
        const int rm = r > 0 ? r - 1 : 0, rp = r < h - 1 ? r + 1 : h - 1;
        const int cm = c > 0 ? c - 1 : 0, cp = c < w - 1 ? c + 1 : w - 1;
        const float* x0 = x + int64_t(rm) * w;
        const float* x1 = x + int64_t(r) * w;
        const float* x2 = x + int64_t(rp) * w;
        const float g = dout[e];
        acc[0] += double(g) * double(x1[c]);
        acc[1] += double(g) * double(x0[c] + x2[c] + x1[cm] + x1[cp]);
        acc[2] += double(g) * double(x0[cm] + x0[cp] + x2[cm] + x2[cp]);
        // dcol gather
        int rr[4], dr[4], cc[4], dc[4];
        const int nr = nbr_pairs(r, h, rr, dr), nc = nbr_pairs(c, w, cc, dc);
        float sum = 0.0f;
        for (int a = 0; a < nr; ++a)
            for (int b = 0; b < nc; ++b) {
                const int cls = (dr[a] != 0) + (dc[b] != 0);
                const float kw = cls == 0 ? kc : (cls == 1 ? ke : ko);
                sum += kw * dout[int64_t(rr[a]) * w + cc[b]];
            }
        dcol[e] = sum;
    }
    __shared__ double sbuf[3 * 8];
    __shared__ double tot[3];
    block_sum_vec<3>(acc, sbuf, tot);
    __syncthreads();
    const PartialRegion& R = P.region[P.reg_ups_ref[j]];
    const int row = blockIdx.y * gridDim.x + blockIdx.x;
    if (threadIdx.x < 3) P.partials[R.base + int64_t(row) * R.count + threadIdx.x] = tot[threadIdx.x];
}

// tconv2x_cols_backward (layers.hpp:432-460): drow by gather over the column
// (row-index) map, dk4 partials from rowtmp.
__global__ void k_ups_cols_bwd(const Plan* __restrict__ pp, int j) {
    const Plan& P = *pp;
    const UpsStage& s = P.ups[j][blockIdx.y];
    const float* k4 = P.params + P.off_tconv[j];
    const float* rowtmp = P.ups_buf + s.row_off;
    const float* dcol = P.ups_grad + s.col_off;
    float* drow = P.ups_grad + s.row_off;
    const int w = s.cols_out, hin = s.rows_in, hout = s.rows_out;
    const int last = hin - 1;
    const int64_t nA = int64_t(hin) * w, nB = int64_t(hout) * w;
    const int64_t n = nA > nB ? nA : nB;
    const int vmax = (hout - 1) >> 1;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
         e += int64_t(gridDim.x) * blockDim.x) {
        if (e < nB) {  // dk4 from output row t
            const int t = int(e / w), c = int(e - int64_t(t) * w);
            int idx[4], tap[4];
            tconv_map(t, last, idx, tap);
            const double g = double(dcol[e]);
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[tap[q]] += g * double(rowtmp[int64_t(idx[q]) * w + c]);
        }
        if (e < nA) {  // drow[u][c]
            const int u = int(e / w), c = int(e - int64_t(u) * w);
            float sum = 0.0f;
            const int v0 = u - 2 < 0 ? 0 : u - 2, v1 = u + 2 > vmax ? vmax : u + 2;
            for (int v = v0; v <= v1; ++v)
                for (int par = 0; par < 2; ++par) {
                    const int t = 2 * v + par;
                    if (t >= hout) continue;
                    int idx[4], tap[4];
                    tconv_map(t, last, idx, tap);
                    const float g = dcol[int64_t(t) * w + c];
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (idx[q] == u) sum += k4[tap[q]] * g;
                }
            drow[e] = sum;
        }
    }
    __shared__ double sbuf[4 * 8];
    __shared__ double tot[4];
    block_sum_vec<4>(acc, sbuf, tot);
    __syncthreads();
    const PartialRegion& R = P.region[P.reg_ups_cols[j]];
    const int row = blockIdx.y * gridDim.x + blockIdx.x;
    if (threadIdx.x < 4) P.partials[R.base + int64_t(row) * R.count + threadIdx.x] = tot[threadIdx.x];
}

// tconv2x_rows_backward (layers.hpp:378-405): din by gather, dk4 partials from
// the stage input.
__global__ void k_ups_rows_bwd(const Plan* __restrict__ pp, int j, int write_din) {
    const Plan& P = *pp;
    const UpsStage& s = P.ups[j][blockIdx.y];
    const float* k4 = P.params + P.off_tconv[j];
    const float* in = stage_in(P, s);
    const float* drow = P.ups_grad + s.row_off;
    float* din = stage_din(P, s);
    const int win = s.cols_in, wout = s.cols_out, h = s.rows_in;
    const int last = win - 1;
    const int64_t nA = int64_t(h) * win, nB = int64_t(h) * wout;
    const int64_t n = nA > nB ? nA : nB;
    const int vmax = (wout - 1) >> 1;
    const bool wd = write_din || !s.din_is_lat;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
         e += int64_t(gridDim.x) * blockDim.x) {
        if (e < nB) {
            const int r = int(e / wout), t = int(e - int64_t(r) * wout);
            int idx[4], tap[4];
            tconv_map(t, last, idx, tap);
            const double g = double(drow[e]);
            const float* xi = in + int64_t(r) * s.in_stride;
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[tap[q]] += g * double(xi[idx[q]]);
        }
        if (wd && e < nA) {
            const int r = int(e / win), u = int(e - int64_t(r) * win);
            const float* go = drow + int64_t(r) * wout;
            float sum = 0.0f;
            const int v0 = u - 2 < 0 ? 0 : u - 2, v1 = u + 2 > vmax ? vmax : u + 2;
            for (int v = v0; v <= v1; ++v)
                for (int par = 0; par < 2; ++par) {
                    const int t = 2 * v + par;
                    if (t >= wout) continue;
                    int idx[4], tap[4];
                    tconv_map(t, last, idx, tap);
                    const float g = go[t];
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (idx[q] == u) sum += k4[tap[q]] * g;
                }
            // main-grid targets are flat unpadded (dups); intermediate ones too
            din[e] = sum;
        }
    }
    __shared__ double sbuf[4 * 8];
    __shared__ double tot[4];
    block_sum_vec<4>(acc, sbuf, tot);
    __syncthreads();
    const PartialRegion& R = P.region[P.reg_ups_rows[j]];
    const int row = blockIdx.y * gridDim.x + blockIdx.x;
    if (threadIdx.x < 4) P.partials[R.base + int64_t(row) * R.count + threadIdx.x] = tot[threadIdx.x];
}

}  // namespace

void launch_ups_forward(const LaunchCtx& L) {
    const Plan& H = *L.host;
    k_copy_z0<<<L.pix_blocks, 256, 0, L.stream>>>(L.plan);
    for (int j = H.L - 2; j >= 0; --j) {
        if (H.ups_n[j] == 0) continue;
        const dim3 grid(L.red_blocks, H.ups_n[j]);
        k_ups_rows_fwd<<<grid, 256, 0, L.stream>>>(L.plan, j);
        k_ups_cols_fwd<<<grid, 256, 0, L.stream>>>(L.plan, j);
        k_ups_refine_fwd<<<grid, 256, 0, L.stream>>>(L.plan, j);
    }
}

void launch_ups_backward(const LaunchCtx& L, bool latent_grads) {
    const Plan& H = *L.host;
    for (int j = 0; j <= H.L - 2; ++j) {
        if (H.ups_n[j] == 0) continue;
        const dim3 grid(L.red_blocks, H.ups_n[j]);
        k_ups_refine_bwd<<<grid, 256, 0, L.stream>>>(L.plan, j);
        k_ups_cols_bwd<<<grid, 256, 0, L.stream>>>(L.plan, j);
        k_ups_rows_bwd<<<grid, 256, 0, L.stream>>>(L.plan, j, latent_grads ? 1 : 0);
    }
}

}  // namespace ccb
