// transforms.cu — K7: preprocessing for the paper's extensions (reading R17).
//
//  * angular similarity: rows normalised to unit l2 norm before hashing;
//  * maximum inner product search (App. B): data rows P(v) = (sqrt(kappa^2 -
//    ||v||^2), v), queries Q(u) = (0, u), kappa = max_i ||v_i||; FastLSH then hashes the (n+1)-dim
//    rows as usual.
// One warp per row: fp32 sum of squares with lane-strided terms and a fixed butterfly reduction,
// IEEE sqrt/division. Bound: HBM (one read, one write of the row).
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"

namespace fastlsh {
namespace {

__device__ __forceinline__ float row_sumsq(const float* row, int n, int lane) {
    float s = 0.f;
    for (int d = lane; d < n; d += 32) s = fmaf(row[d], row[d], s);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

__global__ void normalize_kernel(const float* __restrict__ X, long long N, int n, float* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long r = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < N; r += warps) {
        const float* row = X + r * n;
        const float nrm = __fsqrt_rn(row_sumsq(row, n, lane));
        float* o = out + r * n;
        for (int d = lane; d < n; d += 32) o[d] = nrm > 0.f ? __fdiv_rn(row[d], nrm) : 0.f;
    }
}

__global__ void max_norm_kernel(const float* __restrict__ X, long long N, int n, float* __restrict__ kappa) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    float best = 0.f;
    for (long long r = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < N; r += warps)
        best = fmaxf(best, __fsqrt_rn(row_sumsq(X + r * n, n, lane)));
    // non-negative floats order like their bit patterns
    if (lane == 0) atomicMax(reinterpret_cast<int*>(kappa), __float_as_int(best));
}

__global__ void mips_kernel(const float* __restrict__ X, long long N, int n, const float* __restrict__ kappa,
                            int is_query, float* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    const float k2 = is_query ? 0.f : __fmul_rn(*kappa, *kappa);
    for (long long r = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < N; r += warps) {
        const float* row = X + r * n;
        float* o = out + r * (long long)(n + 1);
        float head = 0.f;
        if (!is_query) head = __fsqrt_rn(fmaxf(__fsub_rn(k2, row_sumsq(row, n, lane)), 0.f));
        if (lane == 0) o[0] = head;
        for (int d = lane; d < n; d += 32) o[d + 1] = row[d];
    }
}

int grid_for(long long N) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long want = (N + 7) / 8;
    return (int)(want < (long long)sms * 8 ? (want > 0 ? want : 1) : (long long)sms * 8);
}

}  // namespace

fastlsh_status launch_normalize(const float* X, long long N, int n, float* out, cudaStream_t s) {
    normalize_kernel<<<grid_for(N), 256, 0, s>>>(X, N, n, out);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? FASTLSH_OK : set_cuda_error(e);
}

fastlsh_status launch_max_norm(const float* X, long long N, int n, float* kappa, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(kappa, 0, sizeof(float), s);
    if (e != cudaSuccess) return set_cuda_error(e);
    if (N > 0) max_norm_kernel<<<grid_for(N), 256, 0, s>>>(X, N, n, kappa);
    e = cudaGetLastError();
    return e == cudaSuccess ? FASTLSH_OK : set_cuda_error(e);
}

fastlsh_status launch_mips(const float* X, long long N, int n, const float* kappa, int is_query, float* out,
                           cudaStream_t s) {
    mips_kernel<<<grid_for(N), 256, 0, s>>>(X, N, n, kappa, is_query, out);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? FASTLSH_OK : set_cuda_error(e);
}

}  // namespace fastlsh
