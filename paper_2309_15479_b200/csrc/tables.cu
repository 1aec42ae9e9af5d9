// tables.cu — K5: bucket tables from compound keys (§3.2).
//
// Table l holds the pairs (key_l(v), v) of all rows v. The library builds it in the canonical
// bulk form of DESIGN.md reading R15: keys ascending, ids ascending inside a bucket (equal keys),
// plus the first position of every bucket. That is a stable sort of (key, id) by key, done as an
// LSD radix sort with 8-bit digits (keys < 2^61: 8 passes), independently per table:
//   pass p: (1) per-tile digit histograms, (2) per-table exclusive scan over (digit, tile),
//           (3) stable scatter: inside a tile, warps take consecutive runs of 32 elements, rank
//               equal digits with __match_any_sync and keep warp-private running counts; warps'
//               counts are prefixed in shared memory, so the order of equal digits is the input
//               order (stability, which makes the row id the tie-break).
// Then one CTA per table marks bucket starts (key differs from its predecessor) and compacts
// their positions with a block scan. Bound: HBM (per pass each element is read twice and written
// once: 8 B key + 4 B id).
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"

namespace fastlsh {
namespace {

constexpr int kRadixBits = 8;
constexpr int kBins = 1 << kRadixBits;
constexpr int kPasses = 8;            // 61-bit keys
constexpr int kSortWarps = 8;
constexpr int kItems = 16;            // rounds of 32 elements per warp
constexpr int kTile = kSortWarps * kItems * 32;  // 4096 elements per CTA tile

__device__ __forceinline__ uint32_t digit_of(uint64_t k, int shift) { return (uint32_t)(k >> shift) & (kBins - 1); }

// hist[l][d][t] = number of elements of tile t of table l with digit d
__global__ void __launch_bounds__(256) radix_hist(const uint64_t* __restrict__ keys, long long ldk, long long N,
                                                  int T, int shift, uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[kBins];
    const int l = blockIdx.y, t = blockIdx.x;
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const uint64_t* kl = keys + (long long)l * ldk;
    const long long e0 = (long long)t * kTile;
    const long long e1 = min(N, e0 + kTile);
    for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) atomicAdd(&h[digit_of(kl[e], shift)], 1u);
    __syncthreads();
    uint32_t* hl = hist + (size_t)l * kBins * T;
    for (int d = threadIdx.x; d < kBins; d += blockDim.x) hl[(size_t)d * T + t] = h[d];
}

// in-place exclusive scan of hist[l][*][*] (digit-major) for every table: one CTA per table
__global__ void __launch_bounds__(1024) radix_scan(uint32_t* __restrict__ hist, int T) {
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t carry;
    uint32_t* hl = hist + (size_t)blockIdx.x * kBins * T;
    const long long total = (long long)kBins * T;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (long long base = 0; base < total; base += blockDim.x) {
        const long long i = base + threadIdx.x;
        const uint32_t v = i < total ? hl[i] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t s = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            warp_sums[lane] = s;  // inclusive prefix of warp totals
        }
        __syncthreads();
        const uint32_t before = carry + (warp ? warp_sums[warp - 1] : 0u) + x - v;
        if (i < total) hl[i] = before;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = before + v;
        __syncthreads();
    }
}

// stable scatter of one tile; ids_in == nullptr means ids are the row indices (first pass)
__global__ void __launch_bounds__(kSortWarps * 32) radix_scatter(const uint64_t* __restrict__ keys_in, long long ldk_in,
                                                               const uint32_t* __restrict__ ids_in,
                                                               uint64_t* __restrict__ keys_out,
                                                               uint32_t* __restrict__ ids_out, long long N, int T,
                                                               int shift, const uint32_t* __restrict__ offs) {
    __shared__ uint32_t wcnt[kSortWarps][kBins];
    const int l = blockIdx.y, t = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kSortWarps * kBins; i += blockDim.x) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    const uint64_t* kl = keys_in + (long long)l * ldk_in;
    const uint32_t* il = ids_in ? ids_in + (long long)l * N : nullptr;
    const long long w0 = (long long)t * kTile + (long long)warp * kItems * 32;
    uint64_t k[kItems];
    uint32_t id[kItems], loc[kItems];
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const long long e = w0 + r * 32 + lane;
        const bool live = e < N;
        k[r] = live ? kl[e] : 0ull;
        id[r] = live ? (il ? il[e] : (uint32_t)e) : 0u;
        const uint32_t d = digit_of(k[r], shift);
        // dead lanes (past N) are the last ones of the tile, after every live element: their
        // digit ranks do not disturb live ones; they are masked out of the counts below
        const unsigned live_mask = __ballot_sync(0xffffffffu, live);
        const unsigned peers = __match_any_sync(0xffffffffu, live ? d : 0xffffffffu) & live_mask;
        const uint32_t before = wcnt[warp][d & (kBins - 1)];
        __syncwarp();
        loc[r] = before + __popc(peers & ((1u << lane) - 1u));
        if (live && (peers & ((1u << lane) - 1u)) == 0) wcnt[warp][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // exclusive prefix over warps, per digit
    for (int d = threadIdx.x; d < kBins; d += blockDim.x) {
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) {
            const uint32_t c = wcnt[w][d];
            wcnt[w][d] = s;
            s += c;
        }
    }
    __syncthreads();
    const uint32_t* ol = offs + (size_t)l * kBins * T;
    uint64_t* ko = keys_out + (long long)l * N;
    uint32_t* io = ids_out + (long long)l * N;
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const long long e = w0 + r * 32 + lane;
        if (e >= N) continue;
        const uint32_t d = digit_of(k[r], shift);
        const uint32_t pos = ol[(size_t)d * T + t] + wcnt[warp][d] + loc[r];
        ko[pos] = k[r];
        io[pos] = id[r];
    }
}

// bucket starts of every table: positions j with j == 0 or key[j] != key[j-1], then N
__global__ void __launch_bounds__(1024) bucket_starts(const uint64_t* __restrict__ sk, long long N,
                                                     uint32_t* __restrict__ starts, long long* __restrict__ nbuckets) {
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t carry;
    const int l = blockIdx.x;
    const uint64_t* kl = sk + (long long)l * N;
    uint32_t* sl = starts + (long long)l * (N + 1);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (long long base = 0; base < N; base += blockDim.x) {
        const long long j = base + threadIdx.x;
        const uint32_t f = (j < N && (j == 0 || kl[j] != kl[j - 1])) ? 1u : 0u;
        uint32_t x = f;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t s = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            warp_sums[lane] = s;
        }
        __syncthreads();
        const uint32_t idx = carry + (warp ? warp_sums[warp - 1] : 0u) + x - f;
        if (f) sl[idx] = (uint32_t)j;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = idx + f;
        __syncthreads();
    }
    const uint32_t nb = carry;
    for (long long j = nb + threadIdx.x; j <= N; j += blockDim.x) sl[j] = (uint32_t)N;  // sentinel + fill
    if (threadIdx.x == 0) nbuckets[l] = nb;
}

}  // namespace

size_t tables_workspace_bytes(int L, long long N) {
    const long long T = (N + kTile - 1) / kTile;
    return (size_t)L * N * 12 + (size_t)L * kBins * T * 4 + 256;
}

fastlsh_status launch_build_tables(const uint64_t* keys, int L, long long N, long long ldk, uint64_t* sorted_keys,
                                   uint32_t* ids, uint32_t* starts, long long* nbuckets, void* ws,
                                   cudaStream_t stream) {
    const int T = (int)((N + kTile - 1) / kTile);
    unsigned char* w = static_cast<unsigned char*>(ws);
    uint64_t* alt_k = reinterpret_cast<uint64_t*>(w);
    uint32_t* alt_i = reinterpret_cast<uint32_t*>(alt_k + (size_t)L * N);
    uintptr_t hp = reinterpret_cast<uintptr_t>(alt_i + (size_t)L * N);
    hp = (hp + 255) & ~(uintptr_t)255;
    uint32_t* hist = reinterpret_cast<uint32_t*>(hp);
    const dim3 grid(T, L);
    for (int p = 0; p < kPasses; ++p) {
        const int shift = p * kRadixBits;
        // pass 0 reads the caller's keys (ids = row indices); then ping-pong so the last pass
        // (odd) lands in the output arrays
        const uint64_t* kin = p == 0 ? keys : (p % 2 ? alt_k : sorted_keys);
        const long long ldin = p == 0 ? ldk : N;
        const uint32_t* iin = p == 0 ? nullptr : (p % 2 ? alt_i : ids);
        uint64_t* kout = p % 2 ? sorted_keys : alt_k;
        uint32_t* iout = p % 2 ? ids : alt_i;
        radix_hist<<<grid, 256, 0, stream>>>(kin, ldin, N, T, shift, hist);
        radix_scan<<<L, 1024, 0, stream>>>(hist, T);
        radix_scatter<<<grid, kSortWarps * 32, 0, stream>>>(kin, ldin, iin, kout, iout, N, T, shift, hist);
    }
    bucket_starts<<<L, 1024, 0, stream>>>(sorted_keys, N, starts, nbuckets);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? FASTLSH_OK : set_cuda_error(e);
}

}  // namespace fastlsh
