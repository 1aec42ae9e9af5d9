// generic.cu — K0: the generic fallback hashing kernel, for params no specialised kernel can pack
// (n > 4400: a 4-row stage no longer fits in shared memory for K1 / K1r; m > 32768 slots per hash).
//
// h_i(v) = floor((a_i . S_i(v) + b_i) / w)   (Eq. 5), straight from global memory:
// a CTA takes one row at a time, its threads take hashes, and every sampled coordinate is an
// L1/L2-cached __ldg of the row (the row is reused by all k hashes). The projection follows the
// paper's slot order (p = x[i0] a0, then fma) and the epilogue is K1r's (__fadd_rn, IEEE / w or an
// exact * 1/w for power-of-two w, floor toward -inf, INT32_MIN + counters). Correctness path only:
// no shared-memory staging, no bank scheduling.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "internal.h"

namespace fastlsh {
namespace {

__global__ void __launch_bounds__(256) generic_kernel(const float* __restrict__ X, long long N, int n, int m, int k,
                                                      const int32_t* __restrict__ idx, const float* __restrict__ a,
                                                      const float* __restrict__ b, float w, int32_t* __restrict__ codes,
                                                      float* __restrict__ proj, unsigned long long* flags) {
    const float inv_w = 1.0f / w;
    const bool w_pow2 = (__float_as_uint(w) & 0x007fffffu) == 0 && isfinite(inv_w) && inv_w != 0.0f;
    for (long long r = blockIdx.x; r < N; r += gridDim.x) {
        const float* xr = X + r * (long long)n;
        for (int h = threadIdx.x; h < k; h += blockDim.x) {
            const int32_t* id = idx + (long long)h * m;
            const float* co = a + (long long)h * m;
            float p = __fmul_rn(__ldg(xr + __ldg(id)), __ldg(co));
            for (int j = 1; j < m; ++j) p = __fmaf_rn(__ldg(xr + __ldg(id + j)), __ldg(co + j), p);
            if (proj) {
                proj[r * k + h] = p;
                continue;
            }
            const float num = __fadd_rn(p, __ldg(b + h));
            const float q = w_pow2 ? __fmul_rn(num, inv_w) : __fdiv_rn(num, w);
            int c = __float2int_rd(q);
            if (!(fabsf(q) < 2147483648.0f)) {
                c = INT_MIN;
                atomicAdd(flags + (isfinite(q) ? 1 : 0), 1ull);
            }
            codes[r * k + h] = c;
        }
    }
}

}  // namespace

fastlsh_status launch_generic(const fastlsh_params* p, const DeviceCopy& d, const float* X, int64_t N, int32_t* codes,
                              float* proj, cudaStream_t stream) {
    if (!d.j_idx || !d.j_a) return FASTLSH_ESTATE;
    int dev = 0, sms = 148;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return set_cuda_error(e);
    const long long grid = N < (long long)sms * 8 ? N : (long long)sms * 8;
    generic_kernel<<<(unsigned)grid, 256, 0, stream>>>(X, N, p->n, p->m, p->k, d.j_idx, d.j_a, d.b, p->w, codes, proj,
                                                      d.flags);
    e = cudaGetLastError();
    return e == cudaSuccess ? FASTLSH_OK : set_cuda_error(e);
}

}  // namespace fastlsh
