// query.cu — K6: LSH query with exact re-ranking (§3.2; SURVEY.md §8(f)2;
// DESIGN.md reading R16).
//
// For a query u with keys H_l(u) (computed by K1 + K3 like any row), the candidates are the
// distinct points stored in the L buckets H_l(u) of the canonical tables (K5); they are re-ranked
// by their exact squared l2 distance and the top-k by (distance, id) is returned.
//
// One CTA per query (grid-stride over queries): threads binary-search the L buckets; warps walk
// the buckets 32 entries at a time, keep the first occurrence of every candidate with a
// test-and-set in the CTA's visited bitmap (N bits in global memory, cleared again after the
// query), and score fresh candidates one at a time with the whole warp (coalesced row read,
// query in shared memory, four independent partial sums per lane so four loads are in flight,
// fixed-order reduction); each warp keeps a sorted top-k list that thread 0 merges at the end.
// Work per query: the bucket searches plus one row read per distinct candidate — bound by
// HBM/L2 reads of candidate rows (C1: 10^4 queries x 2,106 candidates x 3,840 B in 38 ms).
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "internal.h"

namespace fastlsh {
namespace {

constexpr int kQWarps = 8;
constexpr int kMaxTopk = 32;

__device__ __forceinline__ bool less_pair(float da, int ia, float db, int ib) {
    return da < db || (da == db && ia < ib);
}

__global__ void __launch_bounds__(kQWarps * 32) query_kernel(const float* __restrict__ X, long long N, int n,
                                                            const uint64_t* __restrict__ sk,
                                                            const uint32_t* __restrict__ ids, int L,
                                                            const float* __restrict__ Q,
                                                            const uint64_t* __restrict__ qkeys, long long nq,
                                                            long long ldq, int topk, int32_t* __restrict__ out_ids,
                                                            float* __restrict__ out_dist,
                                                            long long* __restrict__ out_ncand,
                                                            uint32_t* __restrict__ bitmaps, long long words) {
    extern __shared__ __align__(16) unsigned char qsm[];
    float* squery = reinterpret_cast<float*>(qsm);                          // [n]
    long long* bs = reinterpret_cast<long long*>(squery + ((n + 3) & ~3));  // [L] bucket begin
    long long* be = bs + L;                                                 // [L] bucket end
    __shared__ float wd[kQWarps][kMaxTopk];
    __shared__ int wi[kQWarps][kMaxTopk];
    __shared__ int wcnt[kQWarps];
    __shared__ unsigned long long ncand;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t* bm = bitmaps + (long long)blockIdx.x * words;

    for (long long q = blockIdx.x; q < nq; q += gridDim.x) {
        for (int d = tid; d < n; d += blockDim.x) squery[d] = Q[q * n + d];
        if (tid < kQWarps) wcnt[tid] = 0;
        if (tid == 0) ncand = 0;
        for (int l = tid; l < L; l += blockDim.x) {  // bucket H_l(q): [lower_bound, upper_bound)
            const uint64_t key = qkeys[(long long)l * ldq + q];
            const uint64_t* kl = sk + (long long)l * N;
            long long lo = 0, hi = N;
            while (lo < hi) {
                const long long mid = (lo + hi) >> 1;
                if (kl[mid] < key) lo = mid + 1; else hi = mid;
            }
            long long lo2 = lo, hi2 = N;
            while (lo2 < hi2) {
                const long long mid = (lo2 + hi2) >> 1;
                if (kl[mid] <= key) lo2 = mid + 1; else hi2 = mid;
            }
            bs[l] = lo;
            be[l] = lo2;
        }
        __syncthreads();
        for (int l = warp; l < L; l += kQWarps) {
            const uint32_t* il = ids + (long long)l * N;
            for (long long j0 = bs[l]; j0 < be[l]; j0 += 32) {
                const long long j = j0 + lane;
                uint32_t c = 0;
                bool fresh = false;
                if (j < be[l]) {
                    c = il[j];
                    const uint32_t bit = 1u << (c & 31);
                    fresh = (atomicOr(bm + (c >> 5), bit) & bit) == 0;
                }
                unsigned todo = __ballot_sync(0xffffffffu, fresh);
                if (lane == 0 && todo) atomicAdd(&ncand, (unsigned long long)__popc(todo));
                while (todo) {
                    const int src = __ffs(todo) - 1;
                    todo &= todo - 1;
                    const uint32_t cc = __shfl_sync(0xffffffffu, c, src);
                    const float* row = X + (long long)cc * n;
                    // four independent partial sums (dims d, d+32, d+64, d+96 of each 128-block)
                    // keep four row loads in flight per lane; fixed combination order
                    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
                    int d = lane;
                    for (; d + 96 < n; d += 128) {
                        const float x0 = __ldg(row + d), x1 = __ldg(row + d + 32);
                        const float x2 = __ldg(row + d + 64), x3 = __ldg(row + d + 96);
                        const float d0 = x0 - squery[d], d1 = x1 - squery[d + 32];
                        const float d2 = x2 - squery[d + 64], d3 = x3 - squery[d + 96];
                        a0 = fmaf(d0, d0, a0);
                        a1 = fmaf(d1, d1, a1);
                        a2 = fmaf(d2, d2, a2);
                        a3 = fmaf(d3, d3, a3);
                    }
                    for (; d < n; d += 32) {
                        const float df = __ldg(row + d) - squery[d];
                        a0 = fmaf(df, df, a0);
                    }
                    float acc = (a0 + a1) + (a2 + a3);
#pragma unroll
                    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                    if (lane == 0) {  // insert into this warp's sorted top-k list
                        int cnt = wcnt[warp];
                        const int id = (int)cc;
                        if (cnt < topk || less_pair(acc, id, wd[warp][cnt - 1], wi[warp][cnt - 1])) {
                            int p = cnt < topk ? cnt : topk - 1;
                            while (p > 0 && less_pair(acc, id, wd[warp][p - 1], wi[warp][p - 1])) {
                                wd[warp][p] = wd[warp][p - 1];
                                wi[warp][p] = wi[warp][p - 1];
                                --p;
                            }
                            wd[warp][p] = acc;
                            wi[warp][p] = id;
                            if (cnt < topk) wcnt[warp] = cnt + 1;
                        }
                    }
                    __syncwarp();
                }
            }
        }
        __syncthreads();
        if (tid == 0) {  // merge the warps' sorted lists
            int head[kQWarps];
            for (int w = 0; w < kQWarps; ++w) head[w] = 0;
            for (int r = 0; r < topk; ++r) {
                int bw = -1;
                for (int w = 0; w < kQWarps; ++w)
                    if (head[w] < wcnt[w] &&
                        (bw < 0 || less_pair(wd[w][head[w]], wi[w][head[w]], wd[bw][head[bw]], wi[bw][head[bw]])))
                        bw = w;
                if (bw < 0) {
                    out_ids[q * topk + r] = -1;
                    out_dist[q * topk + r] = __int_as_float(0x7f800000);  // +inf
                } else {
                    out_ids[q * topk + r] = wi[bw][head[bw]];
                    out_dist[q * topk + r] = wd[bw][head[bw]];
                    ++head[bw];
                }
            }
            out_ncand[q] = (long long)ncand;
        }
        // clear this query's bits (every word touched holds only this query's candidates)
        for (int l = warp; l < L; l += kQWarps) {
            const uint32_t* il = ids + (long long)l * N;
            for (long long j = bs[l] + lane; j < be[l]; j += 32) bm[il[j] >> 5] = 0u;
        }
        __syncthreads();
    }
}

}  // namespace

size_t query_workspace_bytes(long long N, int grid) { return (size_t)grid * (size_t)((N + 31) / 32) * 4; }

int query_grid(long long nq) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long g = (long long)sms * 4;
    return (int)(nq < g ? (nq > 0 ? nq : 1) : g);
}

fastlsh_status launch_query(const float* X, long long N, int n, const uint64_t* sk, const uint32_t* ids, int L,
                            const float* Q, const uint64_t* qkeys, long long nq, long long ldq, int topk,
                            int32_t* out_ids, float* out_dist, long long* out_ncand, void* ws, cudaStream_t stream) {
    const int grid = query_grid(nq);
    const long long words = (N + 31) / 32;
    cudaError_t e = cudaMemsetAsync(ws, 0, query_workspace_bytes(N, grid), stream);
    if (e != cudaSuccess) return set_cuda_error(e);
    const size_t smem = (size_t)((n + 3) & ~3) * 4 + (size_t)L * 16;
    if (smem > 227 * 1024) return FASTLSH_EUNSUPPORTED;
    if (fastlsh_status so = smem_optin_once(reinterpret_cast<const void*>(query_kernel)); so != FASTLSH_OK) return so;
    query_kernel<<<grid, kQWarps * 32, smem, stream>>>(X, N, n, sk, ids, L, Q, qkeys, nq, ldq, topk, out_ids, out_dist,
                                                      out_ncand, static_cast<uint32_t*>(ws), words);
    e = cudaGetLastError();
    return e == cudaSuccess ? FASTLSH_OK : set_cuda_error(e);
}

}  // namespace fastlsh
