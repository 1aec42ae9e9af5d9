// e2lsh_tcgen05.cu — K4: dense E2LSH baseline on 5th-gen tensor cores.
//
// codes = floor((X . A^T + b) / w), E2LSH Eq. 1, with A[k][n] the dense
// coefficient matrix of the params (a_i itself for E2LSH params; the duplicates-merged sampled
// matrix for FastLSH params). fp32 accuracy from TF32 tensor cores by the 3xTF32 split
//     X.A ~= Xhi.Ahi + Xhi.Alo + Xlo.Ahi,   hi = fp32 with the low 13 mantissa bits cleared
// (precision 3; precision 1 = plain Xhi.Ahi, the ungated reference point), or at twice the MMA rate
// from fp16 tensor cores by the 3xFP16 split (precision 2, single-CTA kernel)
//     X.A ~= Xh.Ah + Xh.Al + Xl'.Ah',   Xh = fp16(x), Xl' = fp16((x - Xh) 2^11),
//                                        Ah = fp16(a), Al = fp16(a - Ah), Ah' = fp16(Ah 2^-11)
// (the 2^11 scaling keeps the low part of x out of fp16's subnormal range; all three products
// accumulate in one fp32 TMEM accumulator). Needs |x|, |a| < 65504: larger values overflow to inf
// and come back flagged like any non-finite projection.
//
// One CTA computes a 256-row x 256-hash output tile (non-persistent grid). fp32 operands make the
// GEMM bandwidth-hungry (A is re-read by every row tile), so rows per tile are 256: two UMMA
// M=128 halves accumulate into two 256-column TMEM accumulators (all 512 columns).
//   warp 0  : TMA producer — 2D tensor-map loads (64B swizzle, K-major) of the X tile
//             [256 rows x 16 floats] and the Ahi/Alo tiles [256 x 16] per K-block, 3 stages.
//   warps 2-9: split X in shared memory (in place: X -> Xhi, and Xlo into its own tile), then
//             after the main loop: tcgen05.ld the accumulators (warp%4 = TMEM lane quadrant) and
//             apply the fused +b, /w, floor epilogue (int32 codes or fp32 projections), stored
//             through a per-warp transpose buffer as coalesced 128-byte row segments.
//   warp 1  : TMEM allocation and the single-thread tcgen05.mma issue (kind::tf32, M=128,
//             N=256, K=8 per instruction; 2 halves x 2 k-steps x 3 products per K-block);
//             tcgen05.commit releases the smem stage and finally signals the epilogue.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.h"

namespace fastlsh {
namespace {

constexpr int BM = 256;         // rows per tile: two UMMA M=128 halves, two TMEM accumulators
constexpr int BN = 256;         // hashes per tile (UMMA N)
constexpr int BK = 16;          // floats per K-block (one 64-byte swizzle row)
constexpr int kMaxStagesE = 6;  // 3 stages of X|Xlo|Ahi|Alo (3xTF32) or 6 of X|Ahi (1xTF32): ~192 KB in flight
constexpr int kThreadsE = 320;  // 10 warps
constexpr uint32_t kXTileBytes = BM * BK * 4;   // 16 KB
constexpr uint32_t kATileBytes = BN * BK * 4;   // 16 KB
constexpr uint32_t kStageBytesE = 2 * kXTileBytes + 2 * kATileBytes;  // X, Xlo, Ahi, Alo
// 3xFP16 stages: the f32 X tile (converted in place into Xh | Xl', 8 KB each) and Ah | Al | Ah'
// (fp16 [256 x 16], 32-byte rows, 32-byte swizzle): 40 KB, 5 stages (C1: 5.01 / 4.70 / 4.51 ms at 3 / 4 / 5)
constexpr uint32_t kHTile = BN * BK * 2;                              // 8 KB
constexpr uint32_t kStageBytesH = kXTileBytes + 3 * kHTile;           // 40 KB
constexpr int kStagesH = 5;

struct E2Args {
    long long N;
    int n, k, kpad;
    const float* b;
    float w;
    int precision;
    int32_t* codes;
    float* proj;
    unsigned long long* flags;
    // FastLSH params on the dense path: canonical [k][m] samples and coefficients and the raw X rows,
    // for the exact re-evaluation of flagged elements (null for E2LSH params: the GEMM is the definition)
    const int* idx;
    const float* ca;
    int m;
    const float* X;
    // grid raster: 1 = hash tiles fastest (blockIdx.x), row tiles in blockIdx.y, so the CTAs resident
    // together share their X tiles through L2 (X is read from HBM once instead of kpad/256 times);
    // 0 = row tiles in blockIdx.x (more than 65535 row tiles)
    int hash_fast;
    int stages_h16;  // 3xFP16 ring depth (40 KB stages)
};

// A FastLSH hash sees only its sampled coordinates. The merged-coefficient GEMM
// multiplies every coordinate, so a non-finite coordinate no hash i samples still turns 0 * inf into
// NaN for hash i, and the fp32 rounding near |q| = 2^31 differs from a gather's. Elements the GEMM
// flags (non-finite or out-of-int32 quotient; non-finite projections) are therefore re-evaluated here
// as the gather itself — p = fma-chain over the m samples in the paper's order — before the flag is
// final. Rare by construction; the flagged lane alone, global loads.
__device__ __forceinline__ float gather_projection(const E2Args& a, long long row, int h) {
    const float* x = a.X + row * a.n;
    const int* id = a.idx + (long long)h * a.m;
    const float* co = a.ca + (long long)h * a.m;
    float p = __fmul_rn(x[id[0]], co[0]);
    for (int j = 1; j < a.m; ++j) p = __fmaf_rn(x[id[j]], co[j], p);
    return p;
}

// The flagged elements of one lane's 32-hash chunk (bit j: hash h0 + j of row `row`), after the
// chunk's fast pass wrote INT32_MIN / the raw projection into tb: re-evaluate (FastLSH params), count
// what stays flagged. Inlined in a cold branch after the unrolled loop (a real call costs the ABI's
// register saves and doubled C1's epilogue time).
__device__ __forceinline__ void fix_flagged(const E2Args& a, uint32_t* tb, uint32_t bits, int h0, long long row,
                                        bool w_pow2, float inv_w) {
    if (row >= a.N) return;  // rows past N are never stored
    while (bits) {
        const int j = __ffs(bits) - 1;
        bits &= bits - 1;
        const int h = h0 + j;
        if (a.proj) {  // only FastLSH params flag projections (non-finite): the gather decides
            tb[j] = __float_as_uint(gather_projection(a, row, h));
            continue;
        }
        float qv = 0.0f, f = 0.0f;
        bool ok = false;
        if (a.idx) {
            const float p = gather_projection(a, row, h);
            qv = w_pow2 ? __fmul_rn(__fadd_rn(p, a.b[h]), inv_w) : __fdiv_rn(__fadd_rn(p, a.b[h]), a.w);
            f = floorf(qv);
            ok = f > -2147483648.0f && f < 2147483648.0f;
        } else {
            qv = __uint_as_float(tb[j]);  // E2LSH params: the GEMM's quotient, kept by the fast pass
        }
        if (ok) {
            tb[j] = (uint32_t)(int)f;
        } else {
            atomicAdd(a.flags + (isfinite(qv) ? 1 : 0), 1ull);
            tb[j] = 0x80000000u;
        }
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "LAB_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LAB_WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
        : "memory");
}

// UMMA shared-memory descriptor, K-major, 64-byte swizzle: rows of 64 B, 8-row atoms of
// 512 B (SBO), LBO unused (1), version 1 (sm_100), layout type 4 = SWIZZLE_64B.
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;                 // LBO (16 B units)
    d |= (uint64_t)(512 >> 4) << 32;        // SBO
    d |= (uint64_t)1 << 46;                 // version
    d |= (uint64_t)4 << 61;                 // SWIZZLE_64B
    return d;
}

// K-major, 32-byte swizzle (fp16 rows of 16 elements): 8-row atoms of 256 B (SBO), layout type 6.
__device__ __forceinline__ uint64_t umma_desc_sw32(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;                 // LBO (16 B units)
    d |= (uint64_t)(256 >> 4) << 32;        // SBO
    d |= (uint64_t)1 << 46;                 // version
    d |= (uint64_t)6 << 61;                 // SWIZZLE_32B
    return d;
}

// Instruction descriptor: D f32, A/B f16, both K-major, N = 256, M = 128.
constexpr uint32_t kIdescF16 = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(kIdescF16), "r"(accumulate)
        : "memory");
}

// Instruction descriptor: D f32, A/B tf32, both K-major, N = 256, M = 128.
constexpr uint32_t kIdescTF32 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                ((uint32_t)(128 >> 4) << 24);

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(kIdescTF32), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(kThreadsE, 1)
e2lsh_tcgen05_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_ahi,
                     const __grid_constant__ CUtensorMap map_alo, const __grid_constant__ CUtensorMap map_ahs,
                     const E2Args a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-B alignment for the swizzle atoms
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // 1xTF32 stages carry only X and Ahi (32 KB), so twice as many fit: the same bytes in flight for
    // a third of the MMA work per stage (measured 4.19 ms on C1 with 3 stages: latency-bound)
    const bool h16 = a.precision == 2;
    const int kStagesE = h16 ? a.stages_h16 : a.precision == 3 ? 3 : 6;
    const uint32_t kStageBytes = h16 ? kStageBytesH : a.precision == 3 ? kStageBytesE : kXTileBytes + kATileBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStagesE * kStageBytes);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * kMaxStagesE + 1);
    constexpr int kConvThreads = kThreadsE - 64;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long m0 = (long long)(a.hash_fast ? blockIdx.y : blockIdx.x) * BM;
    const int h0 = (a.hash_fast ? blockIdx.x : blockIdx.y) * BN;
    const int KB = (a.n + BK - 1) / BK;

    const uint32_t sbase = smem_u32(smem);
    // stage layout: X | Ahi | Xlo | Alo (the last two only at 3xTF32)
    auto XT = [&](int s) { return sbase + s * kStageBytes; };
    auto AH = [&](int s) { return sbase + s * kStageBytes + kXTileBytes; };
    auto XL = [&](int s) { return sbase + s * kStageBytes + kXTileBytes + kATileBytes; };
    auto AL = [&](int s) { return sbase + s * kStageBytes + 2 * kXTileBytes + kATileBytes; };
    const uint32_t bar0 = smem_u32(bars);
    auto FULL = [&](int s) { return bar0 + 8u * s; };
    auto CONV = [&](int s) { return bar0 + 8u * (kMaxStagesE + s); };
    auto EMPTY = [&](int s) { return bar0 + 8u * (2 * kMaxStagesE + s); };
    const uint32_t ACC = bar0 + 8u * (3 * kMaxStagesE);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStagesE; ++s) {
            mbar_init(FULL(s), 1);
            mbar_init(CONV(s), kConvThreads);
            mbar_init(EMPTY(s), 1);
        }
        mbar_init(ACC, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(2 * BN)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            const uint32_t bytes = h16 ? kStageBytesH : kXTileBytes + (a.precision == 3 ? 2 : 1) * kATileBytes;
            for (int kb = 0; kb < KB; ++kb) {
                const int s = kb % kStagesE;
                if (kb >= kStagesE) mbar_wait(EMPTY(s), (uint32_t)(((kb - kStagesE) / kStagesE) & 1));
                mbar_arrive_tx(FULL(s), bytes);
                tma_load_2d(XT(s), &map_x, kb * BK, (int)m0, FULL(s));
                if (h16) {  // Ah | Al | Ah' behind the f32 X tile
                    tma_load_2d(XT(s) + kXTileBytes, &map_ahi, kb * BK, h0, FULL(s));
                    tma_load_2d(XT(s) + kXTileBytes + kHTile, &map_alo, kb * BK, h0, FULL(s));
                    tma_load_2d(XT(s) + kXTileBytes + 2 * kHTile, &map_ahs, kb * BK, h0, FULL(s));
                    continue;
                }
                tma_load_2d(AH(s), &map_ahi, kb * BK, h0, FULL(s));
                if (a.precision == 3) tma_load_2d(AL(s), &map_alo, kb * BK, h0, FULL(s));
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (one thread) ----------------
        if (lane == 0) {
            for (int kb = 0; kb < KB; ++kb) {
                const int s = kb % kStagesE;
                mbar_wait(CONV(s), (uint32_t)((kb / kStagesE) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (h16) {  // one K=16 MMA per product and row half: Xh.Ah + Xh.Al + Xl'.Ah'
                    const uint64_t dah = umma_desc_sw32(XT(s) + kXTileBytes);
                    const uint64_t dal = umma_desc_sw32(XT(s) + kXTileBytes + kHTile);
                    const uint64_t das = umma_desc_sw32(XT(s) + kXTileBytes + 2 * kHTile);
#pragma unroll
                    for (int mh = 0; mh < 2; ++mh) {
                        const uint32_t xo = mh * (kHTile / 2);  // rows 128*mh.. of Xh / Xl' (32 B each)
                        const uint32_t td = tmem + mh * BN;
                        const uint64_t dxh = umma_desc_sw32(XT(s) + xo);
                        umma_f16(td, dxh, dah, kb > 0 ? 1u : 0u);
                        umma_f16(td, dxh, dal, 1u);
                        umma_f16(td, umma_desc_sw32(XT(s) + kHTile + xo), das, 1u);
                    }
                    umma_commit(EMPTY(s));
                    continue;
                }
#pragma unroll
                for (int kk = 0; kk < BK / 8; ++kk) {
                    const uint32_t off = kk * 32;  // 8 tf32 = 32 bytes along K inside the swizzle row
                    const uint64_t dah = umma_desc_sw64(AH(s) + off);
                    const uint64_t dal = umma_desc_sw64(AL(s) + off);
                    const uint32_t acc0 = (kb > 0 || kk > 0) ? 1u : 0u;
#pragma unroll
                    for (int mh = 0; mh < 2; ++mh) {  // rows [128*mh, 128*mh+128) -> accumulator mh
                        const uint32_t xo = off + mh * (kXTileBytes / 2);
                        const uint64_t dxh = umma_desc_sw64(XT(s) + xo);
                        const uint32_t td = tmem + mh * BN;
                        umma_tf32(td, dxh, dah, acc0);
                        if (a.precision == 3) {
                            umma_tf32(td, dxh, dal, 1u);
                            umma_tf32(td, umma_desc_sw64(XL(s) + xo), dah, 1u);
                        }
                    }
                }
                umma_commit(EMPTY(s));  // stage s reusable once these MMAs complete
            }
            umma_commit(ACC);  // accumulator complete
        }
    } else {
        // ---------------- warps 2..9: split X in place, then the epilogue ----------------
        const int t = threadIdx.x - 64;  // 0..255
        for (int kb = 0; kb < KB; ++kb) {
            const int s = kb % kStagesE;
            mbar_wait(FULL(s), (uint32_t)((kb / kStagesE) & 1));
            if (h16) {
                // f32 tile [256 x 16] (64-byte rows, 64-byte swizzle: 16-byte chunk c of row r at
                // c ^ ((r >> 1) & 3)) -> Xh | Xl' fp16 [256 x 16] (32-byte rows, 32-byte swizzle: chunk
                // c at c ^ ((r >> 2) & 1)), in place: every converter thread reads its four float4s,
                // then all 256 meet at a named barrier before any writes
                unsigned char* st = smem + s * kStageBytes;
                float4 v[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) v[i] = reinterpret_cast<const float4*>(st)[t + kConvThreads * i];
                asm volatile("bar.sync 1, %0;" ::"r"(kConvThreads) : "memory");
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int u = t + kConvThreads * i;        // physical float4 slot of the f32 tile
                    const int r = u >> 2;
                    const int q = (u & 3) ^ ((r >> 1) & 3);    // logical float4 (columns 4q..4q+3)
                    const float x[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
                    __half2 hp[2], lp[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const __half h0 = __float2half_rn(x[2 * e]), h1 = __float2half_rn(x[2 * e + 1]);
                        hp[e] = __halves2half2(h0, h1);
                        lp[e] = __halves2half2(__float2half_rn((x[2 * e] - __half2float(h0)) * 2048.0f),
                                               __float2half_rn((x[2 * e + 1] - __half2float(h1)) * 2048.0f));
                    }
                    const uint32_t off = r * 32 + (((q >> 1) ^ ((r >> 2) & 1)) << 4) + ((q & 1) << 3);
                    *reinterpret_cast<uint2*>(st + off) =
                        make_uint2(*reinterpret_cast<uint32_t*>(&hp[0]), *reinterpret_cast<uint32_t*>(&hp[1]));
                    *reinterpret_cast<uint2*>(st + kHTile + off) =
                        make_uint2(*reinterpret_cast<uint32_t*>(&lp[0]), *reinterpret_cast<uint32_t*>(&lp[1]));
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            } else if (a.precision == 3) {
                float4* xt = reinterpret_cast<float4*>(smem + s * kStageBytes);
                float4* xl = reinterpret_cast<float4*>(smem + s * kStageBytes + kXTileBytes + kATileBytes);
#pragma unroll
                for (int i = 0; i < (int)(kXTileBytes / 16) / kConvThreads; ++i) {
                    float4 v = xt[t + kConvThreads * i];
                    float4 h, l;
                    h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u); l.x = v.x - h.x;
                    h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u); l.y = v.y - h.y;
                    h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u); l.z = v.z - h.z;
                    h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u); l.w = v.w - h.w;
                    xt[t + kConvThreads * i] = h;
                    xl[t + kConvThreads * i] = l;
                }
                // make the generic-proxy stores visible to the tensor core (async proxy)
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            }
            mbar_arrive(CONV(s));
        }
        // epilogue: TMEM lane quadrant = warp % 4, one output row per thread
        mbar_wait(ACC, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int quad = warp & 3;               // TMEM lane quadrant this warp may access
        const int half = (warp - 2) >> 2;        // accumulator (row half) of this warp
        const long long rbase = m0 + half * 128 + quad * 32;  // this warp's 32 rows
        const float w = a.w;
        const float inv_w = 1.0f / w;
        const bool w_pow2 = (__float_as_uint(w) & 0x007fffffu) == 0 && isfinite(inv_w) && inv_w != 0.0f;
        // 32x33 transpose buffer per warp (the operand stages are idle now): a lane computes one row,
        // then the warp stores row segments of 32 consecutive hashes (128 B, coalesced)
        uint32_t* tb = reinterpret_cast<uint32_t*>(smem) + (warp - 2) * 32 * 33;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(half * BN + c0), v);
            if (h0 + c0 >= a.k) break;
            uint32_t bad = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int h = h0 + c0 + j;
                const float p = __uint_as_float(v[j]);
                uint32_t out = v[j];
                if (h < a.k) {
                    if (!a.proj) {
                        const float num = __fadd_rn(p, a.b[h]);
                        const float qv = w_pow2 ? __fmul_rn(num, inv_w) : __fdiv_rn(num, w);
                        const float f = floorf(qv);
                        if (f > -2147483648.0f && f < 2147483648.0f) {
                            out = (uint32_t)(int)f;
                        } else {
                            bad |= 1u << j;
                            out = __float_as_uint(qv);  // fix_flagged decides
                        }
                    } else if (a.idx && !isfinite(p)) {
                        bad |= 1u << j;
                    }
                }
                tb[lane * 33 + j] = out;
            }
            if (bad) fix_flagged(a, tb + lane * 33, bad, h0 + c0, rbase + lane, w_pow2, inv_w);
            __syncwarp();
            const int h = h0 + c0 + lane;
#pragma unroll 4
            for (int r = 0; r < 32; ++r) {
                const long long row = rbase + r;
                if (row < a.N && h < a.k) {
                    const uint32_t val = tb[r * 33 + lane];
                    if (a.proj) a.proj[row * a.k + h] = __uint_as_float(val);
                    else a.codes[row * a.k + h] = (int32_t)val;
                }
            }
            __syncwarp();
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN) : "memory");
    }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (EncodeTiledFn) nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// 2D f32 tensor map over a row-major [rows][cols] matrix, box [box_rows][16 floats], 64B swizzle.
bool make_map(CUtensorMap* m, const float* base, long long rows, int cols, int box_rows) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
    cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ------------------------------------------------------------------------------------------
// CTA-pair form (cta_group::2). A cluster of two CTAs on one TPC computes a
// 256-row x 256-hash tile with M=256 UMMAs: each CTA stages its own 128 rows of X and its own half
// (128 hashes) of the coefficient tile, so per SM the operand bytes per MMA FLOP are those of the
// 256 x 256 single-CTA tile while each SM's TMEM holds only its 128 x 256 accumulator (256 columns).
//   warp 0    : TMA producer of this CTA's halves (signals its own FULL barrier)
//   warp 1    : TMEM allocation (cta_group::2) — and, in the leader CTA only, the MMA issue
//   warps 2-9 : split X into Xhi / Xlo in place, then arrive on the LEADER's CONV barrier (remote
//               mbarrier arrive through mapa); after the tile, the epilogue of this CTA's 128 rows
// The leader's commits are multicast to both CTAs' EMPTY / ACC barriers. Per output element the
// MMA sequence (K-blocks, k-steps, hi.hi / hi.lo / lo.hi) is the one of the single-CTA kernel.
// 3 stages of 32 KB (3xTF32: X|Bhi|Xlo|Blo of 8 KB each) or 6 of 16 KB (1xTF32: X|Bhi): ~97 KB of
// shared memory and 256 TMEM columns per CTA, so two pairs share each SM pair and one pair's prologue
// and epilogue overlap the other's MMAs (measured 6 / 12 stages at one CTA per SM: 8.2 ms on C1)
constexpr int kPairStages = 3;
constexpr int kPairStages1 = 6;
constexpr uint32_t kHalfTile = 128 * BK * 4;  // 8 KB: 128 rows (or hashes) x 16 floats
constexpr uint32_t kIdescTF32Pair = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                    ((uint32_t)(256 >> 4) << 24);

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t local_bar, uint32_t rank) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_bar), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void umma_tf32_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(kIdescTF32Pair), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(bar), "h"((uint16_t)3) : "memory");
}

__global__ void __launch_bounds__(kThreadsE, 1)
e2lsh_pair_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_ahi,
                  const __grid_constant__ CUtensorMap map_alo, const E2Args a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const bool x3 = a.precision == 3;
    const int NS = x3 ? kPairStages : kPairStages1;
    const uint32_t stage_bytes = x3 ? 4 * kHalfTile : 2 * kHalfTile;  // X | Bhi | Xlo | Blo
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)NS * stage_bytes);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * kPairStages1 + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    // the cluster pairs blockIdx.x 2j, 2j+1: j is the hash tile (hash_fast) or the row-tile pair
    const long long m0 = (long long)(a.hash_fast ? blockIdx.y : (blockIdx.x >> 1)) * 256 + rank * 128;  // this CTA's 128 rows
    const int h0 = (int)(a.hash_fast ? (blockIdx.x >> 1) : blockIdx.y) * BN;  // the pair's 256 hashes
    const int hb = h0 + (int)rank * 128;                                   // this CTA's 128 of them
    const int KB = (a.n + BK - 1) / BK;

    const uint32_t sbase = smem_u32(smem);
    auto XT = [&](int s) { return sbase + s * stage_bytes; };
    auto BH = [&](int s) { return sbase + s * stage_bytes + kHalfTile; };
    auto XL = [&](int s) { return sbase + s * stage_bytes + 2 * kHalfTile; };
    auto BL = [&](int s) { return sbase + s * stage_bytes + 3 * kHalfTile; };
    const uint32_t bar0 = smem_u32(bars);
    auto FULL = [&](int s) { return bar0 + 8u * s; };
    auto CONV = [&](int s) { return bar0 + 8u * (kPairStages1 + s); };   // used in the leader
    auto EMPTY = [&](int s) { return bar0 + 8u * (2 * kPairStages1 + s); };
    const uint32_t ACC = bar0 + 8u * (3 * kPairStages1);

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(FULL(s), 1);
            mbar_init(CONV(s), 2 * 8);  // one arrival per converter warp of both CTAs
            mbar_init(EMPTY(s), 1);
        }
        mbar_init(ACC, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(BN)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync_all();  // both CTAs' barriers initialised and TMEM allocated before any remote arrive / MMA
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            const uint32_t bytes = x3 ? 3 * kHalfTile : 2 * kHalfTile;  // Xlo is produced on chip
            for (int kb = 0; kb < KB; ++kb) {
                const int s = kb % NS;
                if (kb >= NS) mbar_wait(EMPTY(s), (uint32_t)(((kb - NS) / NS) & 1));
                mbar_arrive_tx(FULL(s), bytes);
                tma_load_2d(XT(s), &map_x, kb * BK, (int)m0, FULL(s));
                tma_load_2d(BH(s), &map_ahi, kb * BK, hb, FULL(s));
                if (x3) tma_load_2d(BL(s), &map_alo, kb * BK, hb, FULL(s));
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {
            for (int kb = 0; kb < KB; ++kb) {
                const int s = kb % NS;
                mbar_wait(CONV(s), (uint32_t)((kb / NS) & 1));  // both CTAs' stage s is converted
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int kk = 0; kk < BK / 8; ++kk) {
                    const uint32_t off = kk * 32;
                    const uint64_t dxh = umma_desc_sw64(XT(s) + off);
                    const uint64_t dbh = umma_desc_sw64(BH(s) + off);
                    const uint32_t acc0 = (kb > 0 || kk > 0) ? 1u : 0u;
                    umma_tf32_pair(tmem, dxh, dbh, acc0);
                    if (x3) {
                        umma_tf32_pair(tmem, dxh, umma_desc_sw64(BL(s) + off), 1u);
                        umma_tf32_pair(tmem, umma_desc_sw64(XL(s) + off), dbh, 1u);
                    }
                }
                umma_commit_pair(EMPTY(s));  // stage s of both CTAs reusable once these MMAs complete
            }
            umma_commit_pair(ACC);  // both CTAs' accumulators complete
        }
    } else {
        const int t = threadIdx.x - 64;  // 0..255
        for (int kb = 0; kb < KB; ++kb) {
            const int s = kb % NS;
            mbar_wait(FULL(s), (uint32_t)((kb / NS) & 1));
            if (x3) {
                float4* xt = reinterpret_cast<float4*>(smem + (size_t)s * stage_bytes);
                float4* xl = reinterpret_cast<float4*>(smem + (size_t)s * stage_bytes + 2 * kHalfTile);
#pragma unroll
                for (int i = 0; i < (int)(kHalfTile / 16) / 256; ++i) {
                    const float4 v = xt[t + 256 * i];
                    float4 h, l;
                    h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u); l.x = v.x - h.x;
                    h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u); l.y = v.y - h.y;
                    h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u); l.z = v.z - h.z;
                    h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u); l.w = v.w - h.w;
                    xt[t + 256 * i] = h;
                    xl[t + 256 * i] = l;
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores -> tensor core
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(CONV(s), 0);  // to the leader (also from the leader itself)
        }
        // epilogue: this CTA's 128 rows; TMEM lane quadrant = warp % 4, columns split by warp group
        mbar_wait(ACC, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int quad = warp & 3;
        const int chalf = (warp - 2) >> 2;  // columns [128 chalf, 128 chalf + 128)
        const long long rbase = m0 + quad * 32;
        const float w = a.w;
        const float inv_w = 1.0f / w;
        const bool w_pow2 = (__float_as_uint(w) & 0x007fffffu) == 0 && isfinite(inv_w) && inv_w != 0.0f;
        uint32_t* tb = reinterpret_cast<uint32_t*>(smem) + (warp - 2) * 32 * 33;  // stages are idle now
#pragma unroll 1
        for (int c0 = chalf * 128; c0 < chalf * 128 + 128; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)c0, v);
            if (h0 + c0 >= a.k) break;
            uint32_t bad = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int h = h0 + c0 + j;
                const float p = __uint_as_float(v[j]);
                uint32_t out = v[j];
                if (h < a.k) {
                    if (!a.proj) {
                        const float num = __fadd_rn(p, a.b[h]);
                        const float qv = w_pow2 ? __fmul_rn(num, inv_w) : __fdiv_rn(num, w);
                        const float f = floorf(qv);
                        if (f > -2147483648.0f && f < 2147483648.0f) {
                            out = (uint32_t)(int)f;
                        } else {
                            bad |= 1u << j;
                            out = __float_as_uint(qv);  // fix_flagged decides
                        }
                    } else if (a.idx && !isfinite(p)) {
                        bad |= 1u << j;
                    }
                }
                tb[lane * 33 + j] = out;
            }
            if (bad) fix_flagged(a, tb + lane * 33, bad, h0 + c0, rbase + lane, w_pow2, inv_w);
            __syncwarp();
            const int h = h0 + c0 + lane;
#pragma unroll 4
            for (int r = 0; r < 32; ++r) {
                const long long row = rbase + r;
                if (row < a.N && h < a.k) {
                    const uint32_t val = tb[r * 33 + lane];
                    if (a.proj) a.proj[row * a.k + h] = __uint_as_float(val);
                    else a.codes[row * a.k + h] = (int32_t)val;
                }
            }
            __syncwarp();
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync_all();  // both CTAs are done with TMEM (and the leader's MMAs with both CTAs' smem)
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN) : "memory");
    }
}

}  // namespace

// Dense hi/lo coefficient matrices on the device (once per params object and device).
static fastlsh_status ensure_dense(const fastlsh_params* p, DeviceCopy& d) {
    if (d.dense_hi) return FASTLSH_OK;
    const int kpad = (p->k + BN - 1) / BN * BN;
    std::vector<double> A((size_t)kpad * p->n, 0.0);
    for (int i = 0; i < p->k; ++i)
        for (int j = 0; j < p->m; ++j) A[(size_t)i * p->n + p->idx[(size_t)i * p->m + j]] += p->a[(size_t)i * p->m + j];
    std::vector<float> hi(A.size()), lo(A.size());
    for (size_t t = 0; t < A.size(); ++t) {
        const float f = (float)A[t];
        uint32_t u;
        std::memcpy(&u, &f, 4);
        u &= 0xFFFFE000u;
        float h;
        std::memcpy(&h, &u, 4);
        hi[t] = h;
        lo[t] = f - h;  // exact
    }
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&d.dense_hi), hi.size() * 4);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&d.dense_lo), lo.size() * 4);
    if (e == cudaSuccess) e = cudaMemcpy(d.dense_hi, hi.data(), hi.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d.dense_lo, lo.data(), lo.size() * 4, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(d.dense_hi); cudaFree(d.dense_lo);
        d.dense_hi = d.dense_lo = nullptr;
        return set_cuda_error(e);
    }
    d.dense_kpad = kpad;
    // FastLSH params: the canonical arrays for the exact re-evaluation of flagged elements
    if (!p->is_e2lsh && !d.j_idx) {
        int32_t* di = nullptr;
        float* da = nullptr;
        const size_t km = (size_t)p->k * p->m;
        e = cudaMalloc(reinterpret_cast<void**>(&di), km * 4);
        if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&da), km * 4);
        if (e == cudaSuccess) e = cudaMemcpy(di, p->idx.data(), km * 4, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(da, p->a.data(), km * 4, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(di); cudaFree(da);
            return set_cuda_error(e);
        }
        d.j_idx = di;
        d.j_a = da;
    }
    return FASTLSH_OK;
}

// 3xFP16 operands (precision 2): Ah | Al | Ah' as fp16 [3][kpad][n8] (n8 = n rounded up to 8: 16-byte
// row pitch for TMA; the padding columns are zero), from the same f32 coefficients as the tf32 split.
static fastlsh_status ensure_dense16(const fastlsh_params* p, DeviceCopy& d) {
    if (d.dense_h16) return FASTLSH_OK;
    const int kpad = (p->k + BN - 1) / BN * BN;
    const int n8 = (p->n + 7) / 8 * 8;
    std::vector<double> A((size_t)kpad * p->n, 0.0);
    for (int i = 0; i < p->k; ++i)
        for (int j = 0; j < p->m; ++j) A[(size_t)i * p->n + p->idx[(size_t)i * p->m + j]] += p->a[(size_t)i * p->m + j];
    const size_t plane = (size_t)kpad * n8;
    std::vector<__half> H(3 * plane, __float2half_rn(0.0f));
    for (int i = 0; i < kpad; ++i)
        for (int c = 0; c < p->n; ++c) {
            const float f = (float)A[(size_t)i * p->n + c];
            const __half h = __float2half_rn(f);
            const float hf = __half2float(h);
            H[(size_t)i * n8 + c] = h;
            H[plane + (size_t)i * n8 + c] = __float2half_rn(f - hf);
            H[2 * plane + (size_t)i * n8 + c] = __float2half_rn(hf * (1.0f / 2048.0f));
        }
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&d.dense_h16), H.size() * sizeof(__half));
    if (e == cudaSuccess) e = cudaMemcpy(d.dense_h16, H.data(), H.size() * sizeof(__half), cudaMemcpyHostToDevice);
    static_assert(sizeof(__half) == sizeof(uint16_t), "fp16 bits");
    if (e != cudaSuccess) {
        cudaFree(d.dense_h16);
        d.dense_h16 = nullptr;
        return set_cuda_error(e);
    }
    d.dense_n8 = n8;
    return FASTLSH_OK;
}

// 2D fp16 tensor map over [rows][n8], box [box_rows][16 halves] (32-byte rows), 32-byte swizzle.
static bool make_map_h16(CUtensorMap* m, const void* base, long long rows, int n8, int box_rows) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)n8, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)n8 * 2};
    cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

fastlsh_status launch_e2lsh(const fastlsh_params* p, DeviceCopy& d, const float* X, int64_t N, int32_t* codes,
                            float* proj, int precision, cudaStream_t stream) {
    if (p->n % 4 != 0 || (reinterpret_cast<uintptr_t>(X) & 15) != 0) return FASTLSH_EUNSUPPORTED;
    {
        std::lock_guard<std::mutex> g(const_cast<fastlsh_params*>(p)->dense_mu);
        fastlsh_status st = ensure_dense(p, d);
        if (st == FASTLSH_OK && precision == 2) st = ensure_dense16(p, d);
        if (st != FASTLSH_OK) return st;
    }
    CUtensorMap mx, mh, ml, ms;
    if (!make_map(&mx, X, N, p->n, BM)) return FASTLSH_EUNSUPPORTED;
    if (precision == 2) {
        const size_t plane = (size_t)d.dense_kpad * d.dense_n8;
        if (!make_map_h16(&mh, d.dense_h16, d.dense_kpad, d.dense_n8, BN) ||
            !make_map_h16(&ml, d.dense_h16 + plane, d.dense_kpad, d.dense_n8, BN) ||
            !make_map_h16(&ms, d.dense_h16 + 2 * plane, d.dense_kpad, d.dense_n8, BN))
            return FASTLSH_EUNSUPPORTED;
    } else if (!make_map(&mh, d.dense_hi, d.dense_kpad, p->n, BN) ||
               !make_map(&ml, d.dense_lo, d.dense_kpad, p->n, BN)) {
        return FASTLSH_EUNSUPPORTED;
    } else {
        ms = ml;  // unused
    }
    E2Args a;
    a.N = N;
    a.n = p->n;
    a.k = p->k;
    a.kpad = d.dense_kpad;
    a.b = d.b;
    a.w = p->w;
    a.precision = precision;
    a.codes = codes;
    a.proj = proj;
    a.flags = d.flags;
    a.idx = p->is_e2lsh ? nullptr : d.j_idx;
    a.ca = p->is_e2lsh ? nullptr : d.j_a;
    a.m = p->m;
    a.X = X;
    // The CTA pair wins at 3xTF32 (C1: 5.36 vs 5.49 ms; C3 chunk 8.2 vs 11.6 ms) and at 1xTF32 for short
    // K loops (C3: 7.35 vs 10.8 ms), but its converter relay costs more than it saves on long K loops
    // at 1xTF32 (C1: 4.54 vs 3.77 ms), where the single-CTA kernel stays.
    static const bool single = std::getenv("FASTLSH_K4_SINGLE") != nullptr;  // experiment knob, read once
    if (!single && precision != 2 && (precision == 3 || p->n <= 256)) {
        CUtensorMap px, ph, pl;
        if (!make_map(&px, X, N, p->n, 128) || !make_map(&ph, d.dense_hi, d.dense_kpad, p->n, 128) ||
            !make_map(&pl, d.dense_lo, d.dense_kpad, p->n, 128))
            return FASTLSH_EUNSUPPORTED;
        const size_t psmem = (size_t)kPairStages * 4 * kHalfTile + 1024 + 512;  // = 12 x 16 KB at 1xTF32
        static bool attr_done[kMaxDevices] = {};  // the attribute is per device
        int dev = 0;
        cudaError_t pe = cudaGetDevice(&dev);
        if (pe != cudaSuccess) return set_cuda_error(pe);
        if (!attr_done[dev]) {
            pe = cudaFuncSetAttribute(reinterpret_cast<const void*>(e2lsh_pair_kernel),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem);
            if (pe != cudaSuccess) return set_cuda_error(pe);
            attr_done[dev] = true;
        }
        cudaLaunchConfig_t cfg = {};
        const long long pairs = (N + 255) / 256;
        a.hash_fast = pairs <= 65535 ? 1 : 0;
        cfg.gridDim = a.hash_fast ? dim3((unsigned)(2 * (d.dense_kpad / BN)), (unsigned)pairs)
                                  : dim3((unsigned)(2 * pairs), (unsigned)(d.dense_kpad / BN));
        cfg.blockDim = dim3(kThreadsE);
        cfg.dynamicSmemBytes = psmem;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        pe = cudaLaunchKernelEx(&cfg, e2lsh_pair_kernel, px, ph, pl, a);
        return pe == cudaSuccess ? FASTLSH_OK : set_cuda_error(pe);
    }
    // 3 x 64 KB (3xTF32), 6 x 32 KB (1xTF32) or kStagesH x 40 KB (3xFP16)
    static const int stages_h16 = [] {  // experiment knob, read once
        const char* e = std::getenv("FASTLSH_K4_H16_STAGES");
        const int v = e ? std::atoi(e) : kStagesH;
        return v >= 2 && v <= kMaxStagesE && v * kStageBytesH + 1280 <= 227 * 1024 ? v : kStagesH;
    }();
    a.stages_h16 = stages_h16;
    const size_t smem = (precision == 2 ? (size_t)stages_h16 * kStageBytesH : 3 * kStageBytesE) + 1024 + 256;
    if (fastlsh_status so = smem_optin_once(reinterpret_cast<const void*>(e2lsh_tcgen05_kernel)); so != FASTLSH_OK)
        return so;
    cudaError_t e;
    const long long tiles = (N + BM - 1) / BM;
    a.hash_fast = tiles <= 65535 ? 1 : 0;
    dim3 grid = a.hash_fast ? dim3((unsigned)(d.dense_kpad / BN), (unsigned)tiles)
                            : dim3((unsigned)tiles, (unsigned)(d.dense_kpad / BN));
    e2lsh_tcgen05_kernel<<<grid, kThreadsE, smem, stream>>>(mx, mh, ml, ms, a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e);
    return FASTLSH_OK;
}

}  // namespace fastlsh
