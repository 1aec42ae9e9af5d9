// keys.cu — K3: compound bucket keys (§3.2).
//
// key_l(v) = (r[l][0] + sum_{j<K} r[l][j+1] * u32(code[v][l*K+j])) mod (2^61 - 1), exactly
// (reading R9).
//
// A CTA takes 32 rows. Warp w handles rows w, w+8, ...; its lanes take consecutive tables of a
// row, so a warp's loads cover one contiguous run of the row's codes (coalesced). Each term
// r * u32(c) < 2^93 is accumulated exactly in 128 bits (K <= 2^30 terms cannot overflow) and
// reduced mod 2^61-1 once. Keys go through shared memory so that the [table][row] output is
// written as contiguous 256-byte runs per table (table-major, ready for the NCCL all-gather).
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"

namespace fastlsh {
namespace {

constexpr uint64_t P61 = (1ull << 61) - 1;
constexpr int kKeyRows = 32;
constexpr int kKeyThreads = 256;
constexpr int kTablesPerTile = 256;  // 64 KB of staged keys per tile

__device__ __forceinline__ uint64_t reduce128(uint64_t hi, uint64_t lo) {
    // hi*2^64 + lo with 2^64 = 8 * 2^61 == 8 (mod 2^61 - 1); hi < 2^40 here
    uint64_t x = (lo & P61) + (lo >> 61) + (hi << 3);
    x = (x & P61) + (x >> 61);
    return x >= P61 ? x - P61 : x;
}

__global__ void __launch_bounds__(kKeyThreads) keys_kernel(const uint64_t* __restrict__ rmul,
                                                           const int32_t* __restrict__ codes,
                                                           long long N, int k, int L, int K,
                                                           uint64_t* __restrict__ out, long long ldk,
                                                           int TL) {
    extern __shared__ __align__(16) unsigned char ksmem[];
    uint64_t* s_r = reinterpret_cast<uint64_t*>(ksmem);        // [L][K+1]
    uint64_t* s_key = s_r + L * (K + 1);                        // [TL][kKeyRows]
    for (int i = threadIdx.x; i < L * (K + 1); i += blockDim.x) s_r[i] = rmul[i];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (long long t = blockIdx.x; t < ((N + kKeyRows - 1) / kKeyRows) * ((L + TL - 1) / TL); t += gridDim.x) {
        const long long v0 = (t / ((L + TL - 1) / TL)) * kKeyRows;
        const int l0 = (int)(t % ((L + TL - 1) / TL)) * TL;
        const int l1 = min(L, l0 + TL);
        const int rows = (int)min((long long)kKeyRows, N - v0);
        __syncthreads();  // s_r ready / previous tile's keys written out
        for (int rr = warp; rr < rows; rr += nw) {
            const int32_t* crow = codes + (v0 + rr) * (long long)k;
            for (int l = l0 + lane; l < l1; l += 32) {
                const uint64_t* rl = s_r + l * (K + 1);
                const int32_t* c = crow + l * K;
                uint64_t lo = rl[0], hi = 0;
                for (int j = 0; j < K; ++j) {
                    const uint64_t r = rl[j + 1];
                    const uint64_t u = (uint32_t)__ldg(c + j);
                    const uint64_t plo = r * u;
                    const uint64_t phi = __umul64hi(r, u);
                    lo += plo;
                    hi += phi + (lo < plo ? 1 : 0);
                }
                s_key[(l - l0) * kKeyRows + rr] = reduce128(hi, lo);
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < (l1 - l0) * kKeyRows; i += blockDim.x) {
            const int l = i / kKeyRows, rr = i - l * kKeyRows;
            if (rr < rows) out[(long long)(l0 + l) * ldk + v0 + rr] = s_key[i];
        }
    }
}

}  // namespace

fastlsh_status launch_build_keys(const fastlsh_keys* keys, const uint64_t* dev_r,
                                 const int32_t* codes, int64_t N, int32_t k, uint64_t* out,
                                 int64_t ldk, cudaStream_t stream) {
    const int L = keys->L, K = keys->K;
    const int TL = L < kTablesPerTile ? L : kTablesPerTile;  // tables per tile
    const size_t smem = (size_t)L * (K + 1) * 8 + (size_t)TL * kKeyRows * 8;
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(keys_kernel),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_cuda_error(e);
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(keys_kernel),
                                                      kKeyThreads, smem);
    if (e != cudaSuccess) return set_cuda_error(e);
    if (per_sm < 1) return FASTLSH_EUNSUPPORTED;
    long long blocks = ((N + kKeyRows - 1) / kKeyRows) * ((L + TL - 1) / TL);
    const long long cap = (long long)sms * per_sm;
    if (blocks > cap) blocks = cap;
    keys_kernel<<<(unsigned)blocks, kKeyThreads, smem, stream>>>(dev_r, codes, N, k, L, K, out, ldk, TL);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e);
    return FASTLSH_OK;
}

}  // namespace fastlsh
