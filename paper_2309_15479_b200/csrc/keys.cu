// keys.cu — K3: compound bucket keys (§3.2).
//
// key_l(v) = (r[l][0] + sum_{j<K} r[l][j+1] * u32(code[v][l*K+j])) mod (2^61 - 1), exactly
// (reading R9). A CTA takes 32 rows; for each slice of tables it stages the rows' codes
// into shared memory with coalesced loads, one thread per (row, table) folds the K codes with
// 64x64->128-bit products and Mersenne reduction, and the [table][row] keys are written as
// contiguous 256-byte runs per table (table-major output for the NCCL all-gather).
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"

namespace fastlsh {
namespace {

constexpr uint64_t P61 = (1ull << 61) - 1;
constexpr int kKeyRows = 32;
constexpr int kKeyThreads = 256;
constexpr int kCodeSmemInts = 8192;  // 32 KB of staged codes per slice

__device__ __forceinline__ uint64_t mulmod61(uint64_t r, uint32_t c) {
    const uint64_t lo = r * (uint64_t)c;
    const uint64_t hi = __umul64hi(r, (uint64_t)c);  // < 2^29 since r < 2^61
    uint64_t x = (lo & P61) + (lo >> 61) + (hi << 3);
    if (x >= P61) x -= P61;
    return x;
}

__global__ void __launch_bounds__(kKeyThreads) keys_kernel(const uint64_t* __restrict__ rmul,
                                                           const int32_t* __restrict__ codes,
                                                           long long N, int k, int L, int K,
                                                           uint64_t* __restrict__ out, long long ldk) {
    extern __shared__ __align__(16) unsigned char ksmem[];
    uint64_t* s_r = reinterpret_cast<uint64_t*>(ksmem);
    int32_t* s_c = reinterpret_cast<int32_t*>(s_r + L * (K + 1));
    for (int i = threadIdx.x; i < L * (K + 1); i += blockDim.x) s_r[i] = rmul[i];
    const int slice_ints = max(kCodeSmemInts, kKeyRows * K);
    const int TL = max(1, min(L, slice_ints / (kKeyRows * K)));  // tables per slice
    for (long long v0 = (long long)blockIdx.x * kKeyRows; v0 < N; v0 += (long long)gridDim.x * kKeyRows) {
        const int rows = (int)min((long long)kKeyRows, N - v0);
        for (int l0 = 0; l0 < L; l0 += TL) {
            const int tl = min(TL, L - l0);
            const int cols = tl * K;
            __syncthreads();
            for (int i = threadIdx.x; i < rows * cols; i += blockDim.x) {
                const int r = i / cols, c = i - r * cols;
                s_c[r * cols + c] = codes[(v0 + r) * k + l0 * K + c];
            }
            __syncthreads();
            for (int i = threadIdx.x; i < tl * kKeyRows; i += blockDim.x) {
                const int l = i / kKeyRows, r = i - l * kKeyRows;
                if (r >= rows) continue;
                const uint64_t* rl = s_r + (l0 + l) * (K + 1);
                uint64_t acc = rl[0];
                const int32_t* cr = s_c + r * cols + l * K;
                for (int j = 0; j < K; ++j) {
                    acc += mulmod61(rl[j + 1], (uint32_t)cr[j]);
                    if (acc >= P61) acc -= P61;
                }
                out[(long long)(l0 + l) * ldk + v0 + r] = acc;
            }
        }
    }
}

}  // namespace

fastlsh_status launch_build_keys(const fastlsh_keys* keys, const uint64_t* dev_r,
                                 const int32_t* codes, int64_t N, int32_t k, uint64_t* out,
                                 int64_t ldk, cudaStream_t stream) {
    const int L = keys->L, K = keys->K;
    const size_t smem = (size_t)L * (K + 1) * 8 + (size_t)(K * kKeyRows > kCodeSmemInts ? K * kKeyRows : kCodeSmemInts) * 4;
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(keys_kernel),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_cuda_error(e);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    long long blocks = (N + kKeyRows - 1) / kKeyRows;
    const long long cap = (long long)sms * 4;
    if (blocks > cap) blocks = cap;
    keys_kernel<<<(unsigned)blocks, kKeyThreads, smem, stream>>>(dev_r, codes, N, k, L, K, out, ldk);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e);
    return FASTLSH_OK;
}

}  // namespace fastlsh
