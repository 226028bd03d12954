// cc_soap.cu — SOAP for the NN parameters (EncoderConfig::use_soap, the
// reference default, config.hpp:107): soap_step (optim.hpp:189-250) with the
// cyclic Jacobi eigendecomposition (optim.hpp:60-106) on the device.
//
// One CTA per parameter tensor (viewed as rows x cols, MatView::of,
// tensor.hpp:74-78).  State in HBM per tensor (fp64): the preconditioner EMAs
// L = EMA(G Gᵀ) and R = EMA(Gᵀ G) and their eigenbases QL, QR; the first
// moment (original space) and second moment (rotated space) reuse the Adam
// buffers nn_m / nn_v (fp32, as SoapState::m1 / v2), the step counter nn_t.
// Every 10th step warp 0 re-diagonalises L while warp 1 does R: the same
// cyclic (p, q) rotation order as the reference, one rotation at a time, the
// k-loops of a rotation spread over the lanes; a non-finite sweep keeps the
// previous basis (optim.hpp:210-217).  Products keep the reference's
// per-element summation order.
#include <cuda_runtime.h>

#include "cc_kernels.h"
#include "cc_math.cuh"

namespace ccb {

namespace {

constexpr int kThreads = 128;

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// jacobi_eigen (optim.hpp:60-106), one warp: a (n x n, destroyed), q receives
// the eigenvectors as columns.  Returns false on a non-finite sweep.
__device__ bool jacobi_warp(double* a, double* q, int n) {
    const int lane = threadIdx.x & 31;
    for (int e = lane; e < n * n; e += 32) q[e] = (e / n == e % n) ? 1.0 : 0.0;
    __syncwarp();
    if (n == 1) return isfinite(a[0]);
    for (int sweep = 0; sweep < 32; ++sweep) {
        double off = 0.0, diag = 0.0;
        for (int i = lane; i < n; i += 32) {
            diag += fabs(a[i * n + i]);
            for (int j = i + 1; j < n; ++j) off += fabs(a[i * n + j]);
        }
        off = warp_sum_d(off);
        diag = warp_sum_d(diag);
        if (!isfinite(off) || !isfinite(diag)) return false;
        if (off <= 1e-14 * (diag + 1e-300)) return true;
        for (int p = 0; p < n - 1; ++p) {
            for (int r = p + 1; r < n; ++r) {
                const double apq = a[p * n + r];
                if (apq == 0.0) continue;  // uniform across the warp
                const double app = a[p * n + p];
                const double aqq = a[r * n + r];
                const double theta = (aqq - app) / (2.0 * apq);
                const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(fma(theta, theta, 1.0)));
                const double c = 1.0 / sqrt(fma(t, t, 1.0));
                const double s = t * c;
                __syncwarp();
                for (int k = lane; k < n; k += 32) {
                    const double akp = a[k * n + p], akq = a[k * n + r];
                    a[k * n + p] = c * akp - s * akq;
                    a[k * n + r] = s * akp + c * akq;
                }
                __syncwarp();
                for (int k = lane; k < n; k += 32) {
                    const double apk = a[p * n + k], aqk = a[r * n + k];
                    a[p * n + k] = c * apk - s * aqk;
                    a[r * n + k] = s * apk + c * aqk;
                    const double qkp = q[k * n + p], qkq = q[k * n + r];
                    q[k * n + p] = c * qkp - s * qkq;
                    q[k * n + r] = s * qkp + c * qkq;
                }
                __syncwarp();
            }
        }
    }
    return true;
}

// out[i][j] = sum_kk a[kk][i] * b[kk][j]   (matmul_atb: Aᵀ B; a is K x R, b is K x C)
__device__ void mm_atb(const double* a, const double* b, double* out, int K, int R, int C) {
    for (int e = threadIdx.x; e < R * C; e += blockDim.x) {
        const int i = e / C, j = e - (e / C) * C;
        double acc = 0.0;
        for (int kk = 0; kk < K; ++kk) acc = fma(a[kk * R + i], b[kk * C + j], acc);
        out[e] = acc;
    }
}
// out[i][j] = sum_kk a[i][kk] * b[kk][j]   (matmul_ab; a is R x K, b is K x C)
__device__ void mm_ab(const double* a, const double* b, double* out, int R, int K, int C) {
    for (int e = threadIdx.x; e < R * C; e += blockDim.x) {
        const int i = e / C, j = e - (e / C) * C;
        double acc = 0.0;
        for (int kk = 0; kk < K; ++kk) acc = fma(a[i * K + kk], b[kk * C + j], acc);
        out[e] = acc;
    }
}
// out[i][j] = sum_kk a[i][kk] * b[j][kk]   (matmul_abt; a is R x K, b is C x K)
__device__ void mm_abt(const double* a, const double* b, double* out, int R, int K, int C) {
    for (int e = threadIdx.x; e < R * C; e += blockDim.x) {
        const int i = e / C, j = e - (e / C) * C;
        double acc = 0.0;
        for (int kk = 0; kk < K; ++kk) acc = fma(a[i * K + kk], b[j * K + kk], acc);
        out[e] = acc;
    }
}

__global__ void __launch_bounds__(kThreads) k_soap_step(const Plan* __restrict__ pp, int do_step,
                                                        int count_iter, int log_rec) {
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    const int* __restrict__ tensor_ok = P.tensor_ok;
    double* __restrict__ cost_log = log_rec ? P.rec : nullptr;
    const int ti = blockIdx.x;
    DevScalars* s = P.scal;
    if (count_iter && ti == 0 && threadIdx.x == 0 && s->cost_ok) s->global_iter += 1;
    if (cost_log && ti == 0 && threadIdx.x == 0) {
        double* rec = cost_log + 4 * s->sched_pos;
        rec[0] = s->cost;
        rec[1] = s->mse;
        rec[2] = s->bits;
        rec[3] = double(s->global_iter);
        s->sched_pos += 1;
    }
    if (!(do_step && s->cost_ok)) return;
    if (!tensor_ok[ti]) {  // soap_step returns false before t += 1 (optim.hpp:192)
        if (threadIdx.x == 0) atomicAdd(&s->skipped, 1);
        return;
    }
    const int R = P.tensor_rows[ti], C = P.tensor_cols[ti], n = R * C;
    const int off = P.tensor_off[ti];
    const int64_t t = P.nn_t[ti] + 1;
    double* L = P.soap + P.soap_off[ti];
    double* Rm = L + R * R;
    double* QL = Rm + C * C;
    double* QR = QL + R * R;
    const int D2 = P.soap_dmax * P.soap_dmax, NM = P.soap_nmax;
    extern __shared__ __align__(16) double sd[];
    double* gd = sd;                 // NM each
    double* t1 = gd + NM;
    double* gp = t1 + NM;
    double* m1d = gp + NM;
    double* v2d = m1d + NM;
    double* m1p = v2d + NM;
    double* aL = m1p + NM;           // D2 each
    double* qL = aL + D2;
    double* aR = qL + D2;
    double* qR = aR + D2;

    for (int e = threadIdx.x; e < n; e += blockDim.x) gd[e] = double(P.grads[off + e]);
    __syncthreads();
    // preconditioner EMAs (optim.hpp:197-208)
    const double bs = 0.95;
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
        const int i = e / R, j = e - (e / R) * R;
        double acc = 0.0;
        for (int k = 0; k < C; ++k) acc = fma(gd[i * C + k], gd[j * C + k], acc);
        const double v = fma(bs, L[e], (1.0 - bs) * acc);
        L[e] = v;
        aL[e] = v;
    }
    for (int e = threadIdx.x; e < C * C; e += blockDim.x) {
        const int i = e / C, j = e - (e / C) * C;
        double acc = 0.0;
        for (int k = 0; k < R; ++k) acc = fma(gd[k * C + i], gd[k * C + j], acc);
        const double v = fma(bs, Rm[e], (1.0 - bs) * acc);
        Rm[e] = v;
        aR[e] = v;
    }
    __syncthreads();
    if ((t - 1) % 10 == 0) {  // eigenbasis refresh (optim.hpp:210-217)
        const int w = threadIdx.x >> 5;
        if (w == 0) {
            const bool ok = jacobi_warp(aL, qL, R);
            if (!ok)
                for (int e = threadIdx.x; e < R * R; e += 32) qL[e] = QL[e];
        } else if (w == 1) {
            const bool ok = jacobi_warp(aR, qR, C);
            if (!ok)
                for (int e = (threadIdx.x & 31); e < C * C; e += 32) qR[e] = QR[e];
        }
        __syncthreads();
        for (int e = threadIdx.x; e < R * R; e += blockDim.x) QL[e] = qL[e];
        for (int e = threadIdx.x; e < C * C; e += blockDim.x) QR[e] = qR[e];
    } else {
        for (int e = threadIdx.x; e < R * R; e += blockDim.x) qL[e] = QL[e];
        for (int e = threadIdx.x; e < C * C; e += blockDim.x) qR[e] = QR[e];
    }
    __syncthreads();
    // Gp = QLᵀ G QR
    mm_atb(qL, gd, t1, R, R, C);
    __syncthreads();
    mm_ab(t1, qR, gp, R, C, C);
    __syncthreads();
    const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
    const double bc1 = 1.0 - pow(b1, double(t)), bc2 = 1.0 - pow(b2, double(t));
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const double mt = b1 * double(P.nn_m[off + e]) + (1.0 - b1) * gd[e];
        P.nn_m[off + e] = float(mt);
        m1d[e] = mt;
        const double vt = b2 * double(P.nn_v[off + e]) + (1.0 - b2) * gp[e] * gp[e];
        P.nn_v[off + e] = float(vt);
        v2d[e] = vt;
    }
    __syncthreads();
    // m1 into the rotated space, inner Adam, rotate back (optim.hpp:234-246)
    mm_atb(qL, m1d, t1, R, R, C);
    __syncthreads();
    mm_ab(t1, qR, m1p, R, C, C);
    __syncthreads();
    for (int e = threadIdx.x; e < n; e += blockDim.x) m1p[e] = (m1p[e] / bc1) / (sqrt(v2d[e] / bc2) + eps);
    __syncthreads();
    mm_ab(qL, m1p, t1, R, R, C);
    __syncthreads();
    mm_abt(t1, qR, gp, R, C, C);  // gp <- update
    __syncthreads();
    const double lr = s->lr;
    for (int e = threadIdx.x; e < n; e += blockDim.x)
        P.params[off + e] = float(double(P.params[off + e]) - lr * gp[e]);
    if (threadIdx.x == 0) P.nn_t[ti] = t;
}

__global__ void k_soap_reset(const Plan* __restrict__ pp) {
    const Plan& P = pp[blockIdx.z];  // batched launches: one plan per image
    const int ti = blockIdx.x;
    const int R = P.tensor_rows[ti], C = P.tensor_cols[ti];
    double* L = P.soap + P.soap_off[ti];
    double* Rm = L + R * R;
    double* QL = Rm + C * C;
    double* QR = QL + R * R;
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
        L[e] = 0.0;
        QL[e] = (e / R == e % R) ? 1.0 : 0.0;
    }
    for (int e = threadIdx.x; e < C * C; e += blockDim.x) {
        Rm[e] = 0.0;
        QR[e] = (e / C == e % C) ? 1.0 : 0.0;
    }
}

}  // namespace

size_t soap_smem(const Plan& H) {
    return sizeof(double) * (6 * size_t(H.soap_nmax) + 4 * size_t(H.soap_dmax) * H.soap_dmax);
}

void soap_configure(const Plan& H) {
    cudaFuncSetAttribute(k_soap_step, cudaFuncAttributeMaxDynamicSharedMemorySize, int(soap_smem(H)));
}

void launch_soap_apply(const LaunchCtx& L, bool do_step, bool count_iter, bool log_rec) {
    const Plan& H = *L.host;
    k_soap_step<<<dim3(H.n_tensors, 1, L.batch), kThreads, soap_smem(H), L.stream>>>(
        L.plan, do_step ? 1 : 0, count_iter ? 1 : 0, log_rec ? 1 : 0);
}

void launch_soap_reset(const LaunchCtx& L) {
    k_soap_reset<<<dim3(L.host->n_tensors, 1, L.batch), 128, 0, L.stream>>>(L.plan);
}

}  // namespace ccb
