// cc_reduce.cuh — deterministic block reductions (fixed shuffle tree, then a
// fixed-order sum over warps).  No float atomics anywhere in the library: the
// reference promises bit-determinism in (image, lambda, config, seed)
// (tests/test_encoder.cpp:27-54) and so does this port.
#pragma once

#include "cc_plan.h"

namespace ccb {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Sum of `v` over the block; the result is valid in thread 0 only.
// `sbuf` needs blockDim.x / 32 doubles.  Must be called by every thread.
// A CTA's partial row of a PartialRegion.  Storage is PARAMETER-major
// (row b of parameter e at base + e * nblocks + b), so k_nn_reduce reads the
// rows of one parameter contiguously; the writers index it like a row.
struct PartialRow {
    double* p;
    int64_t stride;
    __device__ __forceinline__ PartialRow(const Plan& P, const PartialRegion& R, int64_t b)
        : p(P.partials + R.base + b), stride(R.nblocks) {}
    __device__ __forceinline__ double& operator[](int64_t e) const { return p[e * stride]; }
};

__device__ __forceinline__ double block_sum(double v, double* sbuf) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sbuf[warp] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        for (int i = 0; i < nw; ++i) r += sbuf[i];
    }
    return r;
}

// Reduce NV per-thread values; thread 0 gets the block totals in out[0..NV).
template <int NV>
__device__ __forceinline__ void block_sum_vec(double (&v)[NV], double* sbuf /* NV * nwarps */,
                                              double* out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
    __syncthreads();
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) sbuf[k * nw + warp] = v[k];
    }
    __syncthreads();
    if (threadIdx.x < NV) {
        double r = 0.0;
        for (int i = 0; i < nw; ++i) r += sbuf[threadIdx.x * nw + i];
        out[threadIdx.x] = r;
    }
}

}  // namespace ccb
