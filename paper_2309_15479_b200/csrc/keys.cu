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
#include <cstdlib>
#include <mutex>
#include <utility>
#include <vector>

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


// Fast path (K <= 16): a warp owns a group of TPW consecutive tables (lane % TPW = table, its
// K+1 multipliers in registers as three 21-bit limbs r = r2*2^42 + r1*2^21 + r0) and RPW =
// 32 / TPW rows at a time (lane / TPW), over a block of RB rows. Per term, three IMAD.WIDE.U32
// accumulate limb*u32(c) (< 2^53) into 64-bit sums S0, S1, S2 (K <= 2^10 terms cannot
// overflow); then
//   key = (r_0 + S0 + S1*2^21 + S2*2^42) mod (2^61-1),
// where x*2^j mod (2^61-1) is a 61-bit rotation — all exact. HBM streaming: the codes of B row
// steps are loaded before any of them is reduced (addresses clamped into the valid range, so
// the loads are unconditional and ptxas issues them back to back: B*K*4 bytes in flight per
// lane). TPW is chosen so that few lanes idle (C1, L = 50: TPW = 10, 30 of 32 lanes busy). The
// keys of a (group, row block) go through shared memory so each table's RB rows leave as one
// contiguous run.
constexpr int kKeySlots = 32 * 33 + 64;  // per warp: TPW * (RB + 1) u64 keys

// row steps per load batch (measured on C1/C4, K = 10: 2 -> 0.72 ms, 3 -> 0.60 ms, 4 -> 0.64 ms;
// more rows per batch means more bytes in flight but more registers, hence fewer warps; K = 16
// on C3: the 8M-row microbenchmark has 1 -> 2.07 ms, 2 -> 2.16 ms, 3 -> 2.41 ms, but the chunked
// 2e8-row bench build 2 -> 45.5 ms vs 1 -> 51.8 ms: 2 is kept)
#ifndef FASTLSH_KEYS_B10
#define FASTLSH_KEYS_B10 3
#endif
#ifndef FASTLSH_KEYS_B16
#define FASTLSH_KEYS_B16 2
#endif
__host__ __device__ constexpr int keys_batch(int K) {
    return K <= 5 ? 8 : K <= 10 ? FASTLSH_KEYS_B10 : FASTLSH_KEYS_B16;
}

__device__ __forceinline__ uint64_t mod61(uint64_t x) {  // x < 2^64 -> x mod (2^61 - 1)
    x = (x & P61) + (x >> 61);
    return x >= P61 ? x - P61 : x;
}
__device__ __forceinline__ uint64_t rotl61(uint64_t x, int j) {  // x < 2^61: x * 2^j mod (2^61 - 1)
    return ((x << j) & P61) | (x >> (61 - j));
}

struct KeysShape {
    int TPW, RPW, RB;
};

inline KeysShape keys_shape(int L, int K) {
    // lanes busy = TPW * RPW of 32, table slots used = L / (groups * TPW): maximise the product
    // (ties: larger TPW, fewer multiplier reloads)
    const int B = keys_batch(K);
    KeysShape best{1, 32, 32};
    double best_eff = -1;
    for (int tpw = 32; tpw >= 1; --tpw) {
        const int rpw = 32 / tpw;
        const int groups = (L + tpw - 1) / tpw;
        const int step = rpw * B;
        const int rb = step * ((32 + step - 1) / step);
        const double eff = (double)(tpw * rpw) / 32.0 * (double)L / (double)(groups * tpw);
        if (tpw * (rb + 1) <= kKeySlots && eff > best_eff + 1e-9) {
            best_eff = eff;
            best = KeysShape{tpw, rpw, rb};
        }
    }
    return best;
}

template <int K, int V>
__device__ __forceinline__ void load_codes(const int32_t* c, uint32_t (&u)[K]) {
    if (K % 4 == 0 && V == 4) {  // 16-byte aligned runs: 128-bit loads
#pragma unroll
        for (int j = 0; j < K; j += 4) {
            const int4 q = __ldg(reinterpret_cast<const int4*>(c + j));
            u[j] = q.x; u[j + 1] = q.y; u[j + 2] = q.z; u[j + 3] = q.w;
        }
    } else if (K % 2 == 0 && V >= 2) {  // 8-byte aligned runs: 64-bit loads
#pragma unroll
        for (int j = 0; j < K; j += 2) {
            const int2 q = __ldg(reinterpret_cast<const int2*>(c + j));
            u[j] = q.x; u[j + 1] = q.y;
        }
    } else {
#pragma unroll
        for (int j = 0; j < K; ++j) u[j] = (uint32_t)__ldg(c + j);
    }
}

#ifndef FASTLSH_KEYS_MINB
#define FASTLSH_KEYS_MINB 1
#endif
template <int K, int V>
__global__ void __launch_bounds__(128, FASTLSH_KEYS_MINB) keys_kernel_fast(const uint64_t* __restrict__ rmul,
                                                        const int32_t* __restrict__ codes, long long N,
                                                        int k, int L, uint64_t* __restrict__ out,
                                                        long long ldk, int TPW, int RB) {
    constexpr int B = keys_batch(K);
    __shared__ uint64_t s_key[4][kKeySlots];  // [warp][table * (RB + 1) + row]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int RPW = 32 / TPW;
    const bool lane_busy = lane < TPW * RPW;
    const int tl = lane % TPW, rsub = lane / TPW;
    const int groups = (L + TPW - 1) / TPW;
    const long long rblocks = (N + RB - 1) / RB;
    const long long items = rblocks * groups;
    uint64_t* sk = s_key[warp];
    for (long long it = (long long)blockIdx.x * 4 + warp; it < items; it += (long long)gridDim.x * 4) {
        const int g = (int)(it % groups);
        const long long v0 = (it / groups) * RB;
        const int l = g * TPW + tl;
        const bool live_l = lane_busy && l < L;
        const int lc = l < L ? l : L - 1;  // clamped: loads stay in range, results are dropped
        uint32_t r0[K], r1[K], r2[K];
        const uint64_t rc = rmul[(size_t)lc * (K + 1)];
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const uint64_t r = rmul[(size_t)lc * (K + 1) + j + 1];
            r0[j] = (uint32_t)(r & 0x1fffff);
            r1[j] = (uint32_t)((r >> 21) & 0x1fffff);
            r2[j] = (uint32_t)(r >> 42);
        }
        const int rows = (int)min((long long)RB, N - v0);
        for (int rb = 0; rb < RB; rb += RPW * B) {
            uint32_t u[B][K];
#pragma unroll
            for (int bb = 0; bb < B; ++bb) {
                const int rr = rb + bb * RPW + rsub;
                const int rcl = rr < rows ? rr : rows - 1;
                load_codes<K, V>(codes + (v0 + rcl) * (long long)k + lc * K, u[bb]);
            }
#pragma unroll
            for (int bb = 0; bb < B; ++bb) {
                const int rr = rb + bb * RPW + rsub;
                uint64_t s0 = 0, s1 = 0, s2 = 0;
#pragma unroll
                for (int j = 0; j < K; ++j) {
                    s0 += (uint64_t)r0[j] * u[bb][j];
                    s1 += (uint64_t)r1[j] * u[bb][j];
                    s2 += (uint64_t)r2[j] * u[bb][j];
                }
                const uint64_t key = mod61(rc + mod61(s0) + rotl61(mod61(s1), 21) + rotl61(mod61(s2), 42));
                if (live_l && rr < rows) sk[tl * (RB + 1) + rr] = key;
            }
        }
        __syncwarp();
        for (int t = 0; t < TPW; ++t) {
            const int lt = g * TPW + t;
            if (lt >= L) break;
            for (int r = lane; r < rows; r += 32) out[(long long)lt * ldk + v0 + r] = sk[t * (RB + 1) + r];
        }
        __syncwarp();
    }
}

typedef void (*FastKeysFn)(const uint64_t*, const int32_t*, long long, int, int, uint64_t*, long long, int, int);
// vector width V of the per-(row, table) code runs: 4 when every run is 16-byte aligned, 2 when
// 8-byte aligned, else 1
FastKeysFn fast_keys_for(int K, int V) {
    switch (K) {
#define FASTLSH_KCASE(X) \
    case X: return V == 4 && X % 4 == 0 ? keys_kernel_fast<X, 4> : V >= 2 && X % 2 == 0 ? keys_kernel_fast<X, 2> : keys_kernel_fast<X, 1>;
        FASTLSH_KCASE(1) FASTLSH_KCASE(2) FASTLSH_KCASE(3) FASTLSH_KCASE(4) FASTLSH_KCASE(5) FASTLSH_KCASE(6)
        FASTLSH_KCASE(7) FASTLSH_KCASE(8) FASTLSH_KCASE(9) FASTLSH_KCASE(10) FASTLSH_KCASE(11) FASTLSH_KCASE(12)
        FASTLSH_KCASE(13) FASTLSH_KCASE(14) FASTLSH_KCASE(15) FASTLSH_KCASE(16)
#undef FASTLSH_KCASE
        default: return nullptr;
    }
}

// TMA-staged path (K <= 16, k % 4 == 0, codes 16-byte aligned): a persistent CTA of 512 threads
// streams blocks of RB consecutive code rows — one bulk copy of RB*k*4 contiguous bytes per block
// into a 3-stage shared-memory ring (complete_tx on an mbarrier) — so tens of KB per SM are in
// flight without costing registers (the register-batched kernel above reached ~4 TB/s on C1).
// Thread (t, j) owns table t (its K multipliers held in registers as 21-bit limbs, loaded once) and
// rows j, j + TPT, ... of every block (TPT = threads per table): per term one shared-memory code
// load and three IMAD.WIDE.U32, the exact limb combination of keys_kernel_fast.
constexpr int kTKThreads = 512;
constexpr int kTKStages = 3;

template <int K>
__global__ void __launch_bounds__(kTKThreads, 1) keys_kernel_tma(const uint64_t* __restrict__ rmul,
                                                             const int32_t* __restrict__ codes, long long N,
                                                             int k, int L, uint64_t* __restrict__ out,
                                                             long long ldk, int RB) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int stage_words = RB * k;
    int32_t* stage = reinterpret_cast<int32_t*>(sm);
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(stage + kTKStages * stage_words);
    const int tid = threadIdx.x;
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(bars);
    if (tid == 0) {
        for (int s = 0; s < kTKStages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8u * s) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int TPT = blockDim.x / L;             // threads per table (>= 1: L <= blockDim)
    const int t = tid / TPT, j = tid - t * TPT;
    const bool live = t < L;
    uint32_t r0[K], r1[K], r2[K];
    uint64_t rc = 0;
    if (live) {
        rc = rmul[(size_t)t * (K + 1)];
#pragma unroll
        for (int jj = 0; jj < K; ++jj) {
            const uint64_t r = rmul[(size_t)t * (K + 1) + jj + 1];
            r0[jj] = (uint32_t)(r & 0x1fffff);
            r1[jj] = (uint32_t)((r >> 21) & 0x1fffff);
            r2[jj] = (uint32_t)(r >> 42);
        }
    }
    const long long nblocks = (N + RB - 1) / RB;
    const long long my = blockIdx.x < nblocks ? (nblocks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    auto issue = [&](long long i) {  // thread 0: block blockIdx.x + i*gridDim.x into stage i % kTKStages
        const long long b = blockIdx.x + i * gridDim.x;
        const long long rows = min((long long)RB, N - b * RB);
        const uint32_t bytes = (uint32_t)(rows * k * 4);
        const uint32_t bar = bar0 + 8u * (uint32_t)(i % kTKStages);
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(stage + (i % kTKStages) * stage_words);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                     "l"(codes + b * RB * (long long)k), "r"(bytes), "r"(bar)
                     : "memory");
    };
    if (tid == 0)
        for (long long i = 0; i < kTKStages && i < my; ++i) issue(i);
    for (long long i = 0; i < my; ++i) {
        const long long b = blockIdx.x + i * gridDim.x;
        const int rows = (int)min((long long)RB, N - b * RB);
        const uint32_t bar = bar0 + 8u * (uint32_t)(i % kTKStages), parity = (uint32_t)((i / kTKStages) & 1);
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "TK_WAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra TK_WAIT_%=;\n}" ::"r"(bar),
            "r"(parity)
            : "memory");
        const int32_t* st = stage + (i % kTKStages) * stage_words;
        if (live) {
            for (int r = j; r < rows; r += TPT) {
                const int32_t* cc = st + r * k + t * K;
                uint64_t s0 = 0, s1 = 0, s2 = 0;
#pragma unroll
                for (int jj = 0; jj < K; ++jj) {
                    const uint32_t c = (uint32_t)cc[jj];
                    s0 += (uint64_t)r0[jj] * c;
                    s1 += (uint64_t)r1[jj] * c;
                    s2 += (uint64_t)r2[jj] * c;
                }
                out[(long long)t * ldk + b * RB + r] =
                    mod61(rc + mod61(s0) + rotl61(mod61(s1), 21) + rotl61(mod61(s2), 42));
            }
        }
        __syncthreads();  // every thread is done with this stage
        if (tid == 0 && i + kTKStages < my) issue(i + kTKStages);
    }
}

typedef void (*TmaKeysFn)(const uint64_t*, const int32_t*, long long, int, int, uint64_t*, long long, int);
TmaKeysFn tma_keys_for(int K) {
    switch (K) {
#define FASTLSH_TKCASE(X) \
    case X: return keys_kernel_tma<X>;
        FASTLSH_TKCASE(1) FASTLSH_TKCASE(2) FASTLSH_TKCASE(3) FASTLSH_TKCASE(4) FASTLSH_TKCASE(5) FASTLSH_TKCASE(6)
        FASTLSH_TKCASE(7) FASTLSH_TKCASE(8) FASTLSH_TKCASE(9) FASTLSH_TKCASE(10) FASTLSH_TKCASE(11) FASTLSH_TKCASE(12)
        FASTLSH_TKCASE(13) FASTLSH_TKCASE(14) FASTLSH_TKCASE(15) FASTLSH_TKCASE(16)
#undef FASTLSH_TKCASE
        default: return nullptr;
    }
}

}  // namespace

fastlsh_status launch_build_keys(const fastlsh_keys* keys, const uint64_t* dev_r,
                                 const int32_t* codes, int64_t N, int32_t k, uint64_t* out,
                                 int64_t ldk, cudaStream_t stream) {
    const int L = keys->L, K = keys->K;
    const uintptr_t base = reinterpret_cast<uintptr_t>(codes);
    const int vec = (k % 4 == 0 && K % 4 == 0 && base % 16 == 0) ? 4 : (k % 2 == 0 && K % 2 == 0 && base % 8 == 0) ? 2 : 1;
    // TMA-staged path: rows 16-byte multiples, codes 16-byte aligned, every table owns >= 1 thread
    // (k % 32 == 0 puts every staged row on the same banks, so the lanes of one table read one bank:
    // C3, k = 256, measured 7.7 vs 2.3 ms — those shapes keep the register-batched kernel)
    static const bool no_tma = std::getenv("FASTLSH_KEYS_NO_TMA") != nullptr;  // experiment knob, read once
    TmaKeysFn tk = (k % 4 == 0 && k % 32 != 0 && base % 16 == 0 && L <= kTKThreads && !no_tma)
                       ? tma_keys_for(K) : nullptr;
    if (tk) {
        int RB = (int)((56 * 1024) / ((long long)k * 4)) & ~7;  // ~56 KB per stage, multiple of 8 rows
        if (RB > 64) RB = 64;
        const size_t smem = (size_t)kTKStages * RB * k * 4 + kTKStages * 8;
        if (RB >= 8 && smem <= 227 * 1024) {
            int dev = 0;
            cudaError_t e = cudaGetDevice(&dev);
            if (e != cudaSuccess || dev < 0 || dev >= kMaxDevices) return e != cudaSuccess ? set_cuda_error(e) : FASTLSH_EUNSUPPORTED;
            // per device: SM count once, and the dynamic shared-memory opt-in once per kernel at the
            // device maximum (every later launch needs <= that), instead of one attribute call per launch
            static int sms_of[kMaxDevices] = {};
            static std::mutex mu;
            static std::vector<std::pair<const void*, int>> attr_done;
            {
                std::lock_guard<std::mutex> g(mu);
                if (!sms_of[dev]) {
                    int sms = 0;
                    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
                    if (e != cudaSuccess) return set_cuda_error(e);
                    sms_of[dev] = sms;
                }
                const void* fn = reinterpret_cast<const void*>(tk);
                bool done = false;
                for (auto& d : attr_done) done |= d.first == fn && d.second == dev;
                if (!done) {
                    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
                    if (e != cudaSuccess) return set_cuda_error(e);
                    attr_done.push_back({fn, dev});
                }
            }
            const int sms = sms_of[dev];
            long long blocks = (N + RB - 1) / RB;
            if (blocks > sms) blocks = sms;
            tk<<<(unsigned)blocks, kTKThreads, smem, stream>>>(dev_r, codes, N, k, L, out, ldk, RB);
            e = cudaGetLastError();
            return e == cudaSuccess ? FASTLSH_OK : set_cuda_error(e);
        }
    }
    if (FastKeysFn fk = fast_keys_for(K, vec)) {  // K <= 16: register-resident limbs (above)
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const KeysShape sh = keys_shape(L, K);
        const long long items = ((N + sh.RB - 1) / sh.RB) * ((L + sh.TPW - 1) / sh.TPW);
        long long blocks = (items + 3) / 4;
        const long long cap = (long long)sms * 16;
        if (blocks > cap) blocks = cap;
        fk<<<(unsigned)blocks, 128, 0, stream>>>(dev_r, codes, N, k, L, out, ldk, sh.TPW, sh.RB);
        cudaError_t e = cudaGetLastError();
        return e == cudaSuccess ? FASTLSH_OK : set_cuda_error(e);
    }
    const int TL = L < kTablesPerTile ? L : kTablesPerTile;  // tables per tile
    const size_t smem = (size_t)L * (K + 1) * 8 + (size_t)TL * kKeyRows * 8;
    int dev = 0, sms = 0, per_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess || dev < 0 || dev >= kMaxDevices) return e != cudaSuccess ? set_cuda_error(e) : FASTLSH_EUNSUPPORTED;
    if (fastlsh_status so = smem_optin_once(reinterpret_cast<const void*>(keys_kernel)); so != FASTLSH_OK) return so;
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
