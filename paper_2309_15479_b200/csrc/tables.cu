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
//               The tile is reordered by digit in shared memory first, so global writes are
//               contiguous runs per digit.
// Then bucket starts (key differs from its predecessor): per-tile flag counts, a per-table scan
// over tiles, and per-tile block-scanned writes. Bound: HBM (per pass each element is read twice
// and written once: 8 B key + 4 B id).
// Tables of N <= kMsdMaxN rows take the MSD form instead: ONE global pass of the same machinery on
// the top digit (bits 53-60) splits each table into 256 segments (~N/256 entries), then one CTA
// per segment finishes it with the 7 remaining stable LSD passes over bits 0-55 (segment_sort),
// ping-ponging between the workspace and the output inside its segment — a few tens of KB per
// CTA, so the intermediate passes stay in L2 and HBM sees about one read and one write per pass
// of the whole table instead of eight.
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

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

// in-place exclusive scan of `per_table` consecutive values per table: one CTA per table
__device__ __forceinline__ void scan_rows(uint32_t* __restrict__ hl, long long total) {
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t carry;
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

// hist[l][*][*] (digit-major, kBins * T values per table)
__global__ void __launch_bounds__(1024) radix_scan(uint32_t* __restrict__ hist, int T) {
    scan_rows(hist + (size_t)blockIdx.x * kBins * T, (long long)kBins * T);
}

// cnt[l][*] (T values per table)
__global__ void __launch_bounds__(1024) radix_scan_rows(uint32_t* __restrict__ cnt, int T) {
    scan_rows(cnt + (size_t)blockIdx.x * T, (long long)T);
}

// stable scatter of one tile; ids_in == nullptr means ids are the row indices (first pass).
// The tile is first reordered by digit in shared memory (stable), then written out so that
// consecutive threads write consecutive entries of each digit's run (coalesced stores).
__global__ void __launch_bounds__(kSortWarps * 32, 3) radix_scatter(const uint64_t* __restrict__ keys_in, long long ldk_in,
                                                               const uint32_t* __restrict__ ids_in,
                                                               uint64_t* __restrict__ keys_out,
                                                               uint32_t* __restrict__ ids_out, long long N, int T,
                                                               int shift, const uint32_t* __restrict__ offs) {
    __shared__ uint32_t wcnt[kSortWarps][kBins];
    __shared__ uint32_t dstart[kBins];  // tile-local first position of each digit
    __shared__ uint32_t gbase[kBins];   // global position of the digit's first element of this tile
    extern __shared__ __align__(16) unsigned char tile_smem[];  // dynamic: the tile in digit order
    uint64_t* sk = reinterpret_cast<uint64_t*>(tile_smem);
    uint32_t* si = reinterpret_cast<uint32_t*>(sk + kTile);
    const int l = blockIdx.y, t = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kSortWarps * kBins; i += blockDim.x) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    const uint64_t* kl = keys_in + (long long)l * ldk_in;
    const uint32_t* il = ids_in ? ids_in + (long long)l * N : nullptr;
    const long long tile0 = (long long)t * kTile;
    const long long w0 = tile0 + (long long)warp * kItems * 32;
    uint64_t k[kItems];
    uint32_t id[kItems], loc[kItems];
#pragma unroll
    for (int r = 0; r < kItems; ++r) {  // all loads first: kItems independent loads in flight
        const long long e = w0 + r * 32 + lane;
        const bool live = e < N;
        k[r] = live ? __ldg(kl + e) : 0ull;
        id[r] = live ? (il ? __ldg(il + e) : (uint32_t)e) : 0u;
    }
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const long long e = w0 + r * 32 + lane;
        const bool live = e < N;
        const uint32_t d = digit_of(k[r], shift);
        // dead lanes (past N) are the tile's last elements: masked out of every count
        const unsigned live_mask = __ballot_sync(0xffffffffu, live);
        const unsigned peers = __match_any_sync(0xffffffffu, live ? d : 0xffffffffu) & live_mask;
        const uint32_t before = wcnt[warp][d];
        __syncwarp();
        loc[r] = before + __popc(peers & ((1u << lane) - 1u));
        if (live && (peers & ((1u << lane) - 1u)) == 0) wcnt[warp][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // per digit: exclusive prefix over warps, and the tile total
    uint32_t total = 0;
    const int d_mine = threadIdx.x;  // blockDim.x == kBins
    {
        uint32_t sacc = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) {
            const uint32_t c = wcnt[w][d_mine];
            wcnt[w][d_mine] = sacc;
            sacc += c;
        }
        total = sacc;
    }
    // exclusive scan of the digit totals across the block (256 threads = 8 warps)
    {
        __shared__ uint32_t wsum[kSortWarps];
        uint32_t x = total;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        uint32_t base = 0;
        for (int w = 0; w < warp; ++w) base += wsum[w];
        dstart[d_mine] = base + x - total;
        gbase[d_mine] = offs[((size_t)l * kBins + d_mine) * T + t] - (base + x - total);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const long long e = w0 + r * 32 + lane;
        if (e >= N) continue;
        const uint32_t d = digit_of(k[r], shift);
        const uint32_t p = dstart[d] + wcnt[warp][d] + loc[r];
        sk[p] = k[r];
        si[p] = id[r];
    }
    __syncthreads();
    const int live_n = (int)min((long long)kTile, N - tile0);
    uint64_t* ko = keys_out + (long long)l * N;
    uint32_t* io = ids_out + (long long)l * N;
    for (int j = threadIdx.x; j < live_n; j += blockDim.x) {
        const uint64_t kk = sk[j];
        const uint32_t pos = gbase[digit_of(kk, shift)] + (uint32_t)j;
        ko[pos] = kk;
        io[pos] = si[j];
    }
}

// MSD form, second level: table l's top-digit segment d = [hist[l][d][0], hist[l][d+1][0]) (the
// scanned level-1 histogram) is sorted by the CTA (d, l) with 7 stable LSD passes over bits 0-55
// (bits 53-55 are equal inside a segment: harmless). Pass p reads ping (p even: the workspace
// alt_*, else the output) and writes pong; each pass walks the segment in tiles of kTile elements
// in order, ranks a tile like radix_scatter (warps take consecutive runs, __match_any_sync, warp
// counts prefixed in shared memory) and carries per-digit running offsets across tiles, so equal
// digits keep their order (stability: the row id stays the tie-break). The next pass's histogram
// is counted while scattering. Plain (not read-only-path) loads: the CTA rereads what it wrote,
// ordered by __syncthreads.
constexpr long long kMsdMaxN = 1ll << 22;
constexpr int kMsdShift = 53;      // level 1: bits 53-60 of the 61-bit keys
constexpr int kSegPasses = 7;      // level 2: bits 0-55
__global__ void __launch_bounds__(kSortWarps * 32, 3) segment_sort(uint64_t* __restrict__ alt_k, uint32_t* __restrict__ alt_i,
                                                              uint64_t* __restrict__ out_k, uint32_t* __restrict__ out_i,
                                                              long long N, int T, const uint32_t* __restrict__ hist) {
    __shared__ uint32_t hcnt[kBins];  // histogram of the current pass's digit (next pass's while scattering)
    __shared__ uint32_t base[kBins];  // running output offset of each digit
    __shared__ uint32_t wcnt[kSortWarps][kBins];
    __shared__ uint32_t wsum[kSortWarps];
    const int d0 = blockIdx.x, l = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t* hl = hist + (size_t)l * kBins * T;
    const long long s0 = hl[(size_t)d0 * T];
    const long long s1 = d0 + 1 < kBins ? (long long)hl[(size_t)(d0 + 1) * T] : N;
    const int len = (int)(s1 - s0);
    if (len <= 0) return;
    uint64_t* ak = alt_k + (long long)l * N + s0;
    uint32_t* ai = alt_i + (long long)l * N + s0;
    uint64_t* ok = out_k + (long long)l * N + s0;
    uint32_t* oi = out_i + (long long)l * N + s0;
    if (len == 1) {
        if (tid == 0) {
            ok[0] = ak[0];
            oi[0] = ai[0];
        }
        return;
    }
    if (len <= kTile) {
        // the common case (segments average N/256 entries): the whole segment is one tile, kept in
        // shared memory; each pass loads it into registers, ranks it (the tile's digit totals are the
        // segment's histogram: no separate count) and scatters it back in place
        extern __shared__ __align__(16) unsigned char seg_smem[];
        uint64_t* bk = reinterpret_cast<uint64_t*>(seg_smem);
        uint32_t* bi = reinterpret_cast<uint32_t*>(bk + kTile);
        for (int e = tid; e < len; e += blockDim.x) {
            bk[e] = ak[e];
            bi[e] = ai[e];
        }
        const int w0 = warp * kItems * 32;
        for (int p = 0; p < kSegPasses; ++p) {
            const int shift = p * kRadixBits;
            for (int w = 0; w < kSortWarps; ++w) wcnt[w][tid] = 0;
            __syncthreads();
            uint64_t k[kItems];
            uint32_t id[kItems], loc[kItems];
#pragma unroll
            for (int r = 0; r < kItems; ++r) {
                const int e = w0 + r * 32 + lane;
                const bool live = e < len;
                k[r] = live ? bk[e] : 0ull;
                id[r] = live ? bi[e] : 0u;
            }
#pragma unroll
            for (int r = 0; r < kItems; ++r) {
                const bool live = w0 + r * 32 + lane < len;
                const uint32_t d = digit_of(k[r], shift);
                const unsigned live_mask = __ballot_sync(0xffffffffu, live);
                const unsigned peers = __match_any_sync(0xffffffffu, live ? d : 0xffffffffu) & live_mask;
                const uint32_t before = wcnt[warp][d];
                __syncwarp();
                loc[r] = before + __popc(peers & ((1u << lane) - 1u));
                if (live && (peers & ((1u << lane) - 1u)) == 0) wcnt[warp][d] = before + __popc(peers);
                __syncwarp();
            }
            __syncthreads();
            uint32_t tot = 0;  // digit tid: exclusive prefix over warps, segment total
#pragma unroll
            for (int w = 0; w < kSortWarps; ++w) {
                const uint32_t c = wcnt[w][tid];
                wcnt[w][tid] = tot;
                tot += c;
            }
            uint32_t x = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) wsum[warp] = x;
            __syncthreads();
            uint32_t b = 0;
            for (int w = 0; w < warp; ++w) b += wsum[w];
            base[tid] = b + x - tot;
            __syncthreads();
#pragma unroll
            for (int r = 0; r < kItems; ++r) {
                if (w0 + r * 32 + lane >= len) continue;
                const uint32_t d = digit_of(k[r], shift);
                const uint32_t pos = base[d] + wcnt[warp][d] + loc[r];
                bk[pos] = k[r];
                bi[pos] = id[r];
            }
            __syncthreads();
        }
        for (int e = tid; e < len; e += blockDim.x) {
            ok[e] = bk[e];
            oi[e] = bi[e];
        }
        return;
    }
    hcnt[tid] = 0;  // blockDim.x == kBins
    __syncthreads();
    for (int e = tid; e < len; e += blockDim.x) atomicAdd(&hcnt[digit_of(ak[e], 0)], 1u);
    __syncthreads();
    for (int p = 0; p < kSegPasses; ++p) {
        const int shift = p * kRadixBits;
        const uint64_t* sk = (p & 1) ? ok : ak;
        const uint32_t* si = (p & 1) ? oi : ai;
        uint64_t* dk = (p & 1) ? ak : ok;
        uint32_t* di = (p & 1) ? ai : oi;
        {   // base = exclusive scan of hcnt; hcnt restarts for the next pass
            const uint32_t v = hcnt[tid];
            uint32_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) wsum[warp] = x;
            __syncthreads();
            uint32_t b = 0;
            for (int w = 0; w < warp; ++w) b += wsum[w];
            base[tid] = b + x - v;
            hcnt[tid] = 0;
        }
        for (int t0 = 0; t0 < len; t0 += kTile) {
            for (int w = 0; w < kSortWarps; ++w) wcnt[w][tid] = 0;
            __syncthreads();
            const int w0 = t0 + warp * kItems * 32;
            uint64_t k[kItems];
            uint32_t id[kItems], loc[kItems];
#pragma unroll
            for (int r = 0; r < kItems; ++r) {
                const int e = w0 + r * 32 + lane;
                const bool live = e < len;
                k[r] = live ? sk[e] : 0ull;
                id[r] = live ? si[e] : 0u;
            }
#pragma unroll
            for (int r = 0; r < kItems; ++r) {
                const bool live = w0 + r * 32 + lane < len;
                const uint32_t d = digit_of(k[r], shift);
                const unsigned live_mask = __ballot_sync(0xffffffffu, live);
                const unsigned peers = __match_any_sync(0xffffffffu, live ? d : 0xffffffffu) & live_mask;
                const uint32_t before = wcnt[warp][d];
                __syncwarp();
                loc[r] = before + __popc(peers & ((1u << lane) - 1u));
                if (live && (peers & ((1u << lane) - 1u)) == 0) wcnt[warp][d] = before + __popc(peers);
                __syncwarp();
            }
            __syncthreads();
            uint32_t tot = 0;  // this thread's digit (tid): exclusive prefix over warps, tile total
#pragma unroll
            for (int w = 0; w < kSortWarps; ++w) {
                const uint32_t c = wcnt[w][tid];
                wcnt[w][tid] = tot;
                tot += c;
            }
            __syncthreads();
#pragma unroll
            for (int r = 0; r < kItems; ++r) {
                if (w0 + r * 32 + lane >= len) continue;
                const uint32_t d = digit_of(k[r], shift);
                const uint32_t pos = base[d] + wcnt[warp][d] + loc[r];
                dk[pos] = k[r];
                di[pos] = id[r];
                if (p + 1 < kSegPasses) atomicAdd(&hcnt[digit_of(k[r], shift + kRadixBits)], 1u);
            }
            __syncthreads();
            base[tid] += tot;
        }
        __syncthreads();  // this pass's global writes are visible to the CTA before the next pass reads
    }
}

// bucket starts of every table: positions j with j == 0 or key[j] != key[j-1], then N.
// (1) per-tile flag counts, (2) per-table exclusive scan over tiles (radix_scan with one "bin"),
// (3) per tile: block scan of the flags, positions written at the tile's offset.
__device__ __forceinline__ uint32_t is_start(const uint64_t* kl, long long j) {
    return (j == 0 || kl[j] != kl[j - 1]) ? 1u : 0u;
}

__global__ void __launch_bounds__(256) bucket_count(const uint64_t* __restrict__ sk, long long N, int T,
                                                   uint32_t* __restrict__ cnt) {
    __shared__ uint32_t tot;
    const int l = blockIdx.y, t = blockIdx.x;
    const uint64_t* kl = sk + (long long)l * N;
    if (threadIdx.x == 0) tot = 0;
    __syncthreads();
    uint32_t c = 0;
    const long long e0 = (long long)t * kTile, e1 = min(N, e0 + kTile);
    for (long long j = e0 + threadIdx.x; j < e1; j += blockDim.x) c += is_start(kl, j);
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&tot, c);
    __syncthreads();
    if (threadIdx.x == 0) cnt[(size_t)l * T + t] = tot;
}

__global__ void __launch_bounds__(256) bucket_write(const uint64_t* __restrict__ sk, long long N, int T,
                                                   const uint32_t* __restrict__ cnt_scanned,
                                                   const uint32_t* __restrict__ cnt_raw,
                                                   uint32_t* __restrict__ starts, long long* __restrict__ nbuckets) {
    __shared__ uint32_t wsum[8];
    const int l = blockIdx.y, t = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t* kl = sk + (long long)l * N;
    uint32_t* sl = starts + (long long)l * (N + 1);
    __shared__ uint64_t tk[kTile + 1];  // tk[0] = key before the tile
    const long long e0 = (long long)t * kTile;
    uint32_t base = cnt_scanned[(size_t)l * T + t];
    for (int i = threadIdx.x; i <= kTile; i += blockDim.x) {
        const long long j = e0 - 1 + i;
        tk[i] = (j >= 0 && j < N) ? kl[j] : 0ull;
    }
    __syncthreads();
    // flags with a coalesced mapping (thread i: entries i, i + 256, ...) into bytes, then each
    // thread takes 16 consecutive flags with one 16-byte load: local count, block scan, write
    __shared__ __align__(16) uint8_t tf[kTile];
    for (int i = threadIdx.x; i < kTile; i += blockDim.x) {
        const long long j = e0 + i;
        tf[i] = (j < N && (j == 0 || tk[i + 1] != tk[i])) ? 1 : 0;
    }
    __syncthreads();
    const long long j0 = e0 + (long long)threadIdx.x * (kTile / 256);
    const uint4 fw = reinterpret_cast<const uint4*>(tf)[threadIdx.x];
    const uint32_t fwords[4] = {fw.x, fw.y, fw.z, fw.w};
    uint32_t f[kTile / 256], c = 0;
#pragma unroll
    for (int i = 0; i < kTile / 256; ++i) {
        f[i] = (fwords[i >> 2] >> (8 * (i & 3))) & 0xffu;
        c += f[i];
    }
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    uint32_t local = 0;  // this thread's first slot inside the tile's run of bucket starts
    for (int w = 0; w < warp; ++w) local += wsum[w];
    local += x - c;
    uint32_t tile_n = 0;
    for (int w = 0; w < 8; ++w) tile_n += wsum[w];
    // positions go to shared memory first (tk is free again), then out with coalesced stores
    __syncthreads();
    uint32_t* tpos = reinterpret_cast<uint32_t*>(tk);
#pragma unroll
    for (int i = 0; i < kTile / 256; ++i)
        if (f[i]) tpos[local++] = (uint32_t)(j0 + i);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < tile_n; i += blockDim.x) sl[base + i] = tpos[i];
    if (t == T - 1 && threadIdx.x == 0) {
        const uint32_t nb = cnt_scanned[(size_t)l * T + t] + cnt_raw[(size_t)l * T + t];
        nbuckets[l] = nb;
    }
}

// bucket_start[l][nb .. N] = N (sentinel and fill)
__global__ void bucket_fill(long long N, uint32_t* __restrict__ starts, const long long* __restrict__ nbuckets) {
    const int l = blockIdx.y;
    const long long nb = nbuckets[l];
    uint32_t* sl = starts + (long long)l * (N + 1);
    for (long long j = nb + (long long)blockIdx.x * blockDim.x + threadIdx.x; j <= N; j += (long long)gridDim.x * blockDim.x)
        sl[j] = (uint32_t)N;
}

}  // namespace

size_t tables_workspace_bytes(int L, long long N) {
    const long long T = (N + kTile - 1) / kTile;
    return (size_t)L * N * 12 + (size_t)L * kBins * T * 4 + (size_t)2 * L * T * 4 + 512;
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
    {   // the dynamic shared-memory opt-in once per device (not per call)
        int dev = 0;
        cudaError_t ae = cudaGetDevice(&dev);
        if (ae != cudaSuccess) return set_cuda_error(ae);
        if (dev < 0 || dev >= kMaxDevices) return FASTLSH_EUNSUPPORTED;
        static bool attr_set[kMaxDevices] = {};
        static std::mutex mu;
        std::lock_guard<std::mutex> g(mu);
        if (!attr_set[dev]) {
            ae = cudaFuncSetAttribute(reinterpret_cast<const void*>(radix_scatter),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kTile * 12);
            if (ae != cudaSuccess) return set_cuda_error(ae);
            attr_set[dev] = true;
        }
    }
    if (N <= kMsdMaxN) {
        // MSD form: one global pass on the top digit into the workspace, then per-segment sorts
        radix_hist<<<grid, 256, 0, stream>>>(keys, ldk, N, T, kMsdShift, hist);
        radix_scan<<<L, 1024, 0, stream>>>(hist, T);
        radix_scatter<<<grid, kSortWarps * 32, kTile * 12, stream>>>(keys, ldk, nullptr, alt_k, alt_i, N, T, kMsdShift,
                                                                     hist);
        // one tile of (key, id) in dynamic shared memory (segments <= kTile are sorted there; larger
        // ones ping-pong through L2, where the 3 CTAs per SM this size allows keep them resident)
        if (fastlsh_status so = smem_optin_once(reinterpret_cast<const void*>(segment_sort)); so != FASTLSH_OK) return so;
        segment_sort<<<dim3(kBins, L), kSortWarps * 32, kTile * 12, stream>>>(alt_k, alt_i, sorted_keys, ids, N, T, hist);
    }
    for (int p = 0; p < kPasses && N > kMsdMaxN; ++p) {
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
        radix_scatter<<<grid, kSortWarps * 32, kTile * 12, stream>>>(kin, ldin, iin, kout, iout, N, T, shift, hist);
    }
    uint32_t* cnt = hist + (size_t)L * kBins * T;     // [L][T] flag counts (scanned in place)
    uint32_t* cnt_raw = cnt + (size_t)L * T;           // [L][T] copy before the scan
    bucket_count<<<grid, 256, 0, stream>>>(sorted_keys, N, T, cnt);
    cudaMemcpyAsync(cnt_raw, cnt, (size_t)L * T * 4, cudaMemcpyDeviceToDevice, stream);
    radix_scan_rows<<<L, 1024, 0, stream>>>(cnt, T);
    bucket_write<<<grid, 256, 0, stream>>>(sorted_keys, N, T, cnt, cnt_raw, starts, nbuckets);
    bucket_fill<<<dim3(64, L), 256, 0, stream>>>(N, starts, nbuckets);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? FASTLSH_OK : set_cuda_error(e);
}

}  // namespace fastlsh
