// On-device image metrics (reference metrics.cpp:8-23): the squared
// error of two framebuffers summed in double, deterministically (fixed per-block partials,
// then one block in fixed order), for PSNR = 10 log10(1 / MSE).
#include "gscg_common.cuh"
#include "gscg_kernels.h"

namespace gscg {

namespace {
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

__device__ double block_sum(double v) {
    __shared__ double s_w[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    if (lane == 0) s_w[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (warp == 0) {
        t = lane < static_cast<int>(blockDim.x >> 5) ? s_w[lane] : 0.0;
        t = warp_sum(t);
    }
    return t;  // valid in thread 0
}
}  // namespace

__global__ void __launch_bounds__(kSseThreads)
k_sse_partial(const float* a, const float* b, uint64_t n, double* partial) {
    double acc = 0.0;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double d = static_cast<double>(a[i]) - static_cast<double>(b[i]);
        acc += d * d;
    }
    const double t = block_sum(acc);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

__global__ void __launch_bounds__(kSseThreads)
k_sse_final(const double* partial, uint32_t blocks, double* out) {
    double acc = 0.0;
    for (uint32_t i = threadIdx.x; i < blocks; i += blockDim.x) acc += partial[i];
    const double t = block_sum(acc);
    if (threadIdx.x == 0) *out = t;
}

}  // namespace gscg
