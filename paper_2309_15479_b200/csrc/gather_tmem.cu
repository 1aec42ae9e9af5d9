// gather_tmem.cu — K1t: FastLSH hashing with TENSOR MEMORY as the gather source (sm_100a).
//
// For every row v and hash i: h_i(v) = floor((a_i . S_i(v) + b_i) / w)   (Eq. 5).
//
// Why TMEM (tools/microbench_tmem*.cu): the shared-memory gather of K1 is capped
// at one 128-B wavefront per SM per clock (G_s = 32 gathers/clk/SM). tcgen05.ld reads tensor
// memory through its own datapath: a warp-uniform column address returns one 32-bit word per
// lane — a conflict-free gather of 32 rows when lane = row — and .32x32b.x2 returns two adjacent
// columns, i.e. the same coordinate of two rows when rows are interleaved along columns.
// Measured on B200: 1.19x G_s for that loop with parameters broadcast from shared memory
// (2.8x G_s for the raw .x8 load), so the sampled projection is no longer bound by shared memory.
//
// Layout:
//  * One CTA per SM, 16 warps. TMEM: 128 lanes x 512 columns, two buffers of 256 columns.
//    Warp w accesses lanes 32*(w%4).. (its "quadrant" q = w%4). The four quadrants are independent
//    engines: each hashes its own stream of 64-row tiles; lane t of quadrant q holds rows t and
//    t+32 of the quadrant's tile, column 2*c + r for coordinate c of the current block.
//  * Coordinates are streamed in blocks of 128 (256 columns, double-buffered): TMA bulk copies
//    bring the block's 64 row segments into the quadrant's shared landing slot (row pitch 528 B,
//    conflict-free 128-bit reads), the 4 warps of the quadrant move it into TMEM (LDS.128 ->
//    tcgen05.st.32x32b.x8, interleaving the two rows), one block ahead of the gather.
//  * Hashes: a CTA serves a block of <= 4*NHW hashes; warp slot s = w/4 owns NHW consecutive
//    hashes and keeps their accumulators (2 rows each) in registers for the whole tile. The
//    (TMEM column, coefficient) records of its hashes' slots are grouped by (coordinate block,
//    hash) and broadcast from shared memory (LDS.128 = two slots).
//  * Per slot: tcgen05.ld.32x32b.x2 at the record's column + 2 FFMA (rows t, t+32).
//  * Epilogue at the last block of a tile: __fadd_rn(p, b), IEEE division by w (exact multiply
//    by 1/w for power-of-two w), floor, int32 store — the same arithmetic as K1.
// Summation order (fixed by the packing): coordinate blocks in order, slots in paper order within
// a block; one fp32 accumulator per (hash, row) over all m slots (m <= 128: gamma_m < 7.7e-6).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstring>
#include <vector>

#include "internal.h"

namespace fastlsh {

namespace {

constexpr int kTB = 128;                     // coordinates per TMEM block
constexpr int kTRows = 64;                   // rows per quadrant tile (32 lanes x 2)
constexpr int kNHW = 32;                     // max hashes per warp (register accumulators)
constexpr int kBox = 32;                     // coordinates per TMA box (128 B, 128-byte swizzle)
constexpr int kBoxBytes = kTRows * kBox * 4; // one box: 64 rows x 128 B
constexpr int kLandBytes = (kTB / kBox) * kBoxBytes;
constexpr size_t kSmemMax = 227 * 1024;
constexpr int kTMaxM = 128;

size_t tmem_smem_bytes(int recs_max, int nb, int kb_max) {
    size_t s = 4 * (size_t)kLandBytes;       // landing slots, one per quadrant
    s += (size_t)recs_max * 8;               // (column, coefficient) records
    s += 4 * (size_t)nb * 32;                // per (warp slot, block) hash slot counts (u8 x 32)
    s += 4 * (size_t)nb * 4;                 // per (warp slot, block) record offsets
    s += ((size_t)kb_max + 3) / 4 * 16;      // b of the block's hashes
    s += 4 * kTGroups * 4;                   // group starts of the 4 warp slots
    s += 8 * 8 + 16;                         // mbarriers + TMEM address slot
    return s;
}

}  // namespace

// Host packing for K1t (SURVEY.md §8(a) a1 "GPU packing"). Leaves tp.ok = false when the shape
// does not suit the TMEM kernel; the shared-memory kernel K1 then serves it.
void build_tmem_packing(const fastlsh_params& p, TPacking& tp) {
    tp = TPacking();
    const int n = p.n, m = p.m, k = p.k;
    if (n % 4 != 0 || m > kTMaxM) return;
    // coordinate blocks: an even count (block bk lives in TMEM buffer bk & 1, baked into its
    // records) of tb <= 128 coordinates, tb a multiple of the 32-coordinate TMA box
    int tb = kTB;
    if (n <= kTB) tb = std::max(kBox, (n / 2 + kBox - 1) / kBox * kBox);
    int nb = (n + tb - 1) / tb;
    nb += nb & 1;
    // hashes per warp: as many as the record region allows (records <= nh*4*(m+nb) with padding)
    int nhw = kNHW;
    while (nhw >= 4 && tmem_smem_bytes(4 * nhw * (m + nb), nb, 4 * nhw) > kSmemMax) nhw -= 4;
    if (nhw < 4) return;
    const int groups_total = (k + 3) / 4;
    if (groups_total < 4 * (nhw / 4)) nhw = 4 * std::max(1, (groups_total + 3) / 4);  // small k
    const int KB = 4 * nhw, GW = nhw / 4;  // hashes per CTA block, groups per warp slot
    const int HB = (k + KB - 1) / KB;
    if (HB > kTMaxHB) return;
    tp.nb = nb;
    tp.tb = tb;
    tp.nhw = nhw;
    tp.HB = HB;
    tp.hinfo.assign((size_t)HB * kTInfo, 0);
    tp.groups.assign((size_t)HB * 4 * kTGroups, -1);
    tp.counts.assign((size_t)HB * 4 * nb * 32, 0);
    tp.offs.assign((size_t)HB * 4 * nb, 0);
    // padded run length of hash h in coordinate block bk
    std::vector<int> cnt((size_t)k * nb, 0);
    for (int h = 0; h < k; ++h) {
        for (int t = 0; t < m; ++t) ++cnt[(size_t)h * nb + p.idx[(size_t)h * m + t] / tb];
        for (int bk = 0; bk < nb; ++bk) cnt[(size_t)h * nb + bk] += cnt[(size_t)h * nb + bk] & 1;
    }
    double bal_num = 0, bal_den = 0;
    for (int hb = 0; hb < HB; ++hb) {
        const int h0 = hb * KB, kb = std::min(KB, k - h0);
        const int G = (kb + 3) / 4;
        // cost of group g in block bk: its record pairs plus a per-hash loop overhead
        std::vector<int> cost((size_t)G * nb, 0);
        for (int g = 0; g < G; ++g)
            for (int u = 0; u < 4 && 4 * g + u < kb; ++u)
                for (int bk = 0; bk < nb; ++bk)
                    cost[(size_t)g * nb + bk] += cnt[(size_t)(h0 + 4 * g + u) * nb + bk] / 2 + 1;
        // assign groups to the 4 warp slots (<= GW each), minimising sum over blocks of the max load:
        // round robin, then pairwise swaps / moves while they improve
        std::vector<int> owner(G);
        for (int g = 0; g < G; ++g) owner[g] = g % 4;
        std::vector<int> load(4 * nb, 0), size(4, 0);
        for (int g = 0; g < G; ++g) {
            ++size[owner[g]];
            for (int bk = 0; bk < nb; ++bk) load[owner[g] * nb + bk] += cost[(size_t)g * nb + bk];
        }
        auto objective = [&]() {
            long long f = 0;
            for (int bk = 0; bk < nb; ++bk) {
                int mx = 0;
                for (int w = 0; w < 4; ++w) mx = std::max(mx, load[w * nb + bk]);
                f += mx;
            }
            return f;
        };
        long long best = objective();
        for (int pass = 0; pass < 50; ++pass) {
            bool improved = false;
            for (int g1 = 0; g1 < G; ++g1) {
                for (int g2 = g1 + 1; g2 < G; ++g2) {
                    const int w1 = owner[g1], w2 = owner[g2];
                    if (w1 == w2) continue;
                    for (int bk = 0; bk < nb; ++bk) {
                        const int d = cost[(size_t)g2 * nb + bk] - cost[(size_t)g1 * nb + bk];
                        load[w1 * nb + bk] += d;
                        load[w2 * nb + bk] -= d;
                    }
                    const long long f = objective();
                    if (f < best) {
                        best = f;
                        owner[g1] = w2;
                        owner[g2] = w1;
                        improved = true;
                    } else {
                        for (int bk = 0; bk < nb; ++bk) {
                            const int d = cost[(size_t)g2 * nb + bk] - cost[(size_t)g1 * nb + bk];
                            load[w1 * nb + bk] -= d;
                            load[w2 * nb + bk] += d;
                        }
                    }
                }
            }
            if (!improved) break;
        }
        {
            long long tot = 0;
            for (int v : load) tot += v;
            bal_num += (double)best;
            bal_den += (double)tot / 4.0;
        }
        int32_t* hi = &tp.hinfo[(size_t)hb * kTInfo];
        hi[0] = h0;
        hi[1] = kb;
        hi[2] = (int32_t)(tp.recs.size() / 2);
        std::vector<std::vector<int>> wg(4);
        for (int g = 0; g < G; ++g) wg[owner[g]].push_back(g);
        for (int s = 0; s < 4; ++s) {
            if ((int)wg[s].size() > GW) return;  // cannot happen: swaps keep the sizes of round robin
            hi[4 + s] = (int32_t)wg[s].size();
            for (size_t gi = 0; gi < wg[s].size(); ++gi)
                tp.groups[((size_t)hb * 4 + s) * kTGroups + gi] = h0 + 4 * wg[s][gi];
        }
        const size_t rec0 = tp.recs.size() / 2;
        for (int s = 0; s < 4; ++s) {
            for (int bk = 0; bk < nb; ++bk) {
                tp.offs[((size_t)hb * 4 + s) * nb + bk] = (uint32_t)(tp.recs.size() / 2 - rec0);
                for (size_t gi = 0; gi < wg[s].size(); ++gi) {
                    for (int u = 0; u < 4; ++u) {
                        const int h = h0 + 4 * wg[s][gi] + u;
                        if (h >= h0 + kb) break;
                        const int32_t* idx = &p.idx[(size_t)h * m];
                        const float* a = &p.a[(size_t)h * m];
                        int c = 0;
                        uint32_t last = 0;
                        for (int t = 0; t < m; ++t) {
                            if (idx[t] / tb != bk) continue;
                            last = (uint32_t)(2 * (idx[t] - bk * tb) + 256 * (bk & 1));
                            uint32_t cb;
                            std::memcpy(&cb, &a[t], 4);
                            tp.recs.push_back(last);
                            tp.recs.push_back(cb);
                            ++c;
                        }
                        if (c & 1) {  // pad to pairs (LDS.128 = two records): +0 * x at a used column
                            tp.recs.push_back(last);
                            tp.recs.push_back(0u);
                            ++c;
                        }
                        tp.counts[(((size_t)hb * 4 + s) * nb + bk) * 32 + 4 * gi + u] = (uint8_t)c;
                    }
                }
            }
        }
        hi[3] = (int32_t)(tp.recs.size() / 2 - rec0);
        tp.recs_max = std::max(tp.recs_max, hi[3]);
        tp.kb_max = std::max(tp.kb_max, kb);
    }
    tp.balance = bal_den > 0 ? bal_num / bal_den : 1.0;
    tp.smem = tmem_smem_bytes(tp.recs_max, nb, tp.kb_max);
    if (tp.smem > kSmemMax) return;
    tp.ok = true;
}

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct TArgs {
    CUtensorMap xmap;  // X [N][n] f32, box 32 coordinates x 64 rows, 128-byte swizzle
    const float* X;
    long long N;
    int n, nb, tb, k;
    const uint32_t* recs;
    const uint8_t* counts;
    const uint32_t* offs;
    const int32_t* hinfo;
    const int32_t* groups;
    const float* b;
    float w;
    int32_t* codes;
    float* proj;
    unsigned long long* flags;
    int recs_max, kb_max;
    int vec_store;
    int HB;
    int cta_first[kTMaxHB + 1];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t uni(uint32_t v) { return __shfl_sync(0xffffffffu, v, 0); }

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
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 32x32b.x2: this lane's TMEM lane, columns taddr and taddr+1 (rows t and t+32 of a coordinate)
__device__ __forceinline__ void tmem_ld2(uint32_t taddr, uint32_t& x0, uint32_t& x1) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(x0), "=r"(x1) : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st8(uint32_t taddr, float4 r0, float4 r1) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
                 "r"(__float_as_uint(r0.x)), "r"(__float_as_uint(r1.x)), "r"(__float_as_uint(r0.y)),
                 "r"(__float_as_uint(r1.y)), "r"(__float_as_uint(r0.z)), "r"(__float_as_uint(r1.z)),
                 "r"(__float_as_uint(r0.w)), "r"(__float_as_uint(r1.w))
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ int quantise(float p, float bh, float w, float inv_w, bool w_pow2,
                                        unsigned long long* flags, bool live) {
    const float num = __fadd_rn(p, bh);
    const float qv = w_pow2 ? __fmul_rn(num, inv_w) : __fdiv_rn(num, w);
    const float f = floorf(qv);
    int code = (int)f;
    if (!(f > -2147483648.0f && f < 2147483648.0f)) {
        code = INT_MIN;
        if (live) atomicAdd(flags + (isfinite(qv) ? 1 : 0), 1ull);
    }
    return code;
}

// Per-CTA state of one quadrant engine (shared-memory tables are this CTA's hash block).
struct Ctx {
    const unsigned char* landq;
    uint32_t landq_u32, recs_u32, counts_u32, bar_full, bar_empty;
    const uint32_t* soffs;
    const float* sb;
    const int32_t* sgroups;  // this warp slot's group starts
    int h0, hend, ng, s, lane, nb;
    long long e, E, G;
};

// Gather-FMA over this warp slot's hashes for coordinate block bk (TMEM buffer bk & 1). The TMEM
// address is the record itself: column with the buffer offset baked in, lane field 0 — for the
// .32x32b shape the hardware serves the warp's own lane quadrant whatever the lane field says
// (measured: tools/microbench_tmem_lane.cu; checked at kernel start). Each slot costs
// LDS.128/2 + R2UR + LDTM + 2 FFMA.
__device__ __forceinline__ void gather_block(const Ctx& c, float (&acc)[kNHW][2], int bk) {
    constexpr uint32_t IMM = 0;  // records carry column + buffer; the lane field may stay 0 (below)
    const int nh = 4 * c.ng;
    uint32_t rp = c.recs_u32 + 8u * uni(c.soffs[c.s * c.nb + bk]);
    const uint32_t cw = c.counts_u32 + (uint32_t)(c.s * c.nb + bk) * 32u;
    const uint4 c0 = lds128(cw), c1 = lds128(cw + 16);
    const uint32_t words[8] = {uni(c0.x), uni(c0.y), uni(c0.z), uni(c0.w),
                               uni(c1.x), uni(c1.y), uni(c1.z), uni(c1.w)};
#pragma unroll
    for (int j = 0; j < kNHW; ++j) {
        if (j < nh) {
            const uint32_t end = rp + ((words[j >> 2] >> (8 * (j & 3))) & 0xffu) * 8u;
            for (; rp + 32u <= end; rp += 32u) {
                const uint4 r0 = lds128(rp), r1 = lds128(rp + 16u);
                uint32_t v[8];
                tmem_ld2(r0.x + IMM, v[0], v[1]);
                tmem_ld2(r0.z + IMM, v[2], v[3]);
                tmem_ld2(r1.x + IMM, v[4], v[5]);
                tmem_ld2(r1.z + IMM, v[6], v[7]);
                tmem_wait_ld();
                acc[j][0] = fmaf(__uint_as_float(v[0]), __uint_as_float(r0.y), acc[j][0]);
                acc[j][1] = fmaf(__uint_as_float(v[1]), __uint_as_float(r0.y), acc[j][1]);
                acc[j][0] = fmaf(__uint_as_float(v[2]), __uint_as_float(r0.w), acc[j][0]);
                acc[j][1] = fmaf(__uint_as_float(v[3]), __uint_as_float(r0.w), acc[j][1]);
                acc[j][0] = fmaf(__uint_as_float(v[4]), __uint_as_float(r1.y), acc[j][0]);
                acc[j][1] = fmaf(__uint_as_float(v[5]), __uint_as_float(r1.y), acc[j][1]);
                acc[j][0] = fmaf(__uint_as_float(v[6]), __uint_as_float(r1.w), acc[j][0]);
                acc[j][1] = fmaf(__uint_as_float(v[7]), __uint_as_float(r1.w), acc[j][1]);
            }
            if (rp < end) {
                const uint4 r0 = lds128(rp);
                uint32_t v[4];
                tmem_ld2(r0.x + IMM, v[0], v[1]);
                tmem_ld2(r0.z + IMM, v[2], v[3]);
                tmem_wait_ld();
                acc[j][0] = fmaf(__uint_as_float(v[0]), __uint_as_float(r0.y), acc[j][0]);
                acc[j][1] = fmaf(__uint_as_float(v[1]), __uint_as_float(r0.y), acc[j][1]);
                acc[j][0] = fmaf(__uint_as_float(v[2]), __uint_as_float(r0.w), acc[j][0]);
                acc[j][1] = fmaf(__uint_as_float(v[3]), __uint_as_float(r0.w), acc[j][1]);
                rp += 16u;
            }
        }
    }
}

__device__ __forceinline__ void engine(const TArgs& a, const Ctx& c, int Q) {
    const int lane = c.lane, s = c.s, nb = c.nb;
    const bool leader = (s == 0);
    const uint32_t qcol = (uint32_t)(32 * Q) << 16;

    auto issue = [&](long long g) {  // leader lane 0: TMA boxes of block g (OOB rows/columns -> 0)
        if (lane != 0) return;
        const int row0 = (int)((c.e + (g / nb) * c.E) * kTRows);
        const int x0 = (int)(g % nb) * a.tb;
        int nbox = 0;
        for (int bx = 0; bx < a.tb / kBox; ++bx) nbox += (x0 + bx * kBox < a.n);
        mbar_arrive_tx(c.bar_full, (uint32_t)(nbox * kBoxBytes));
        for (int bx = 0; bx < a.tb / kBox; ++bx)
            if (x0 + bx * kBox < a.n)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3}], [%4];" ::"r"(c.landq_u32 + bx * kBoxBytes),
                    "l"(reinterpret_cast<uint64_t>(&a.xmap)), "r"(x0 + bx * kBox), "r"(row0), "r"(c.bar_full)
                    : "memory");
    };
    // this warp's box of block g (coordinates [32s, 32s+32)): landing -> TMEM buffer bk&1. Row r of
    // a box is 128 B whose 16-byte chunk j sits at chunk j ^ (r % 8) (128-byte swizzle), so the
    // lanes of a quarter-warp (rows t..t+7) read 8 different bank groups.
    auto stage = [&](long long g) {
        const int bk = (int)(g % nb);
        if (32 * s >= a.tb || bk * a.tb + 32 * s >= a.n) return;
        const uint32_t tcol = qcol + (uint32_t)(bk & 1) * 256u + 64u * s;
        const unsigned char* box = c.landq + s * kBoxBytes;
        const unsigned char* r0p = box + lane * 128;
        const unsigned char* r1p = box + (lane + 32) * 128;
        const int sw = lane & 7;  // (lane + 32) % 8 == lane % 8
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float4 v0 = *reinterpret_cast<const float4*>(r0p + 16 * (j ^ sw));
            const float4 v1 = *reinterpret_cast<const float4*>(r1p + 16 * (j ^ sw));
            tmem_st8(tcol + 8 * j, v0, v1);
        }
    };
    auto stage_and_refill = [&](long long g) {  // stage block g, then refill the landing with g+1
        mbar_wait(c.bar_full, (uint32_t)(g & 1));
        stage(g);
        __syncwarp();
        if (lane == 0) mbar_arrive(c.bar_empty);
        if (leader) {
            mbar_wait(c.bar_empty, (uint32_t)(g & 1));
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (g + 1 < c.G) issue(g + 1);
        }
    };
    auto sync_quadrant = [&]() {
        tmem_wait_st();
        tc_fence_before();
        asm volatile("bar.sync %0, 128;" ::"r"(1 + Q) : "memory");
        tc_fence_after();
    };

    const float w = a.w;
    const float inv_w = 1.0f / w;
    const bool w_pow2 = (__float_as_uint(w) & 0x007fffffu) == 0 && isfinite(inv_w) && inv_w != 0.0f;
    // rows past N in a tile were never loaded: their lanes read stale TMEM and their results are
    // discarded (no store, no flag)
    auto epilogue = [&](float (&acc)[kNHW][2], long long i) {
        const long long row0 = (c.e + i * c.E) * kTRows;
        const long long rA = row0 + lane, rB = row0 + lane + 32;
        const bool la = rA < a.N, lb = rB < a.N;
#pragma unroll
        for (int gi = 0; gi < kNHW / 4; ++gi) {
            if (gi < c.ng) {
                const int hs = c.sgroups[gi];
                const long long oA = rA * a.k + hs, oB = rB * a.k + hs;
                if (a.proj) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        if (hs + u < c.hend) {
                            if (la) a.proj[oA + u] = acc[4 * gi + u][0];
                            if (lb) a.proj[oB + u] = acc[4 * gi + u][1];
                        }
                    }
                } else if (a.vec_store && hs + 4 <= c.hend) {
                    const float b0 = c.sb[hs - c.h0], b1 = c.sb[hs - c.h0 + 1];
                    const float b2 = c.sb[hs - c.h0 + 2], b3 = c.sb[hs - c.h0 + 3];
                    int4 cA, cB;
                    cA.x = quantise(acc[4 * gi][0], b0, w, inv_w, w_pow2, a.flags, la);
                    cA.y = quantise(acc[4 * gi + 1][0], b1, w, inv_w, w_pow2, a.flags, la);
                    cA.z = quantise(acc[4 * gi + 2][0], b2, w, inv_w, w_pow2, a.flags, la);
                    cA.w = quantise(acc[4 * gi + 3][0], b3, w, inv_w, w_pow2, a.flags, la);
                    cB.x = quantise(acc[4 * gi][1], b0, w, inv_w, w_pow2, a.flags, lb);
                    cB.y = quantise(acc[4 * gi + 1][1], b1, w, inv_w, w_pow2, a.flags, lb);
                    cB.z = quantise(acc[4 * gi + 2][1], b2, w, inv_w, w_pow2, a.flags, lb);
                    cB.w = quantise(acc[4 * gi + 3][1], b3, w, inv_w, w_pow2, a.flags, lb);
                    if (la) *reinterpret_cast<int4*>(a.codes + oA) = cA;
                    if (lb) *reinterpret_cast<int4*>(a.codes + oB) = cB;
                } else {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        if (hs + u < c.hend) {
                            const float bh = c.sb[hs - c.h0 + u];
                            if (la) a.codes[oA + u] = quantise(acc[4 * gi + u][0], bh, w, inv_w, w_pow2, a.flags, la);
                            if (lb) a.codes[oB + u] = quantise(acc[4 * gi + u][1], bh, w, inv_w, w_pow2, a.flags, lb);
                        }
                    }
                }
            }
        }
    };

    float acc[kNHW][2];
    if (c.G > 0) {
        if (leader) issue(0);
        stage_and_refill(0);
        sync_quadrant();
    }
    for (long long g = 0; g < c.G; ++g) {
        if (g + 1 < c.G) stage_and_refill(g + 1);  // into the other TMEM buffer (nb is even; block g-1 is done)
        const int bk = (int)(g % nb);
        if (bk == 0) {
#pragma unroll
            for (int j = 0; j < kNHW; ++j) acc[j][0] = acc[j][1] = 0.f;
        }
        gather_block(c, acc, bk);
        if (bk == nb - 1) epilogue(acc, g / nb);
        sync_quadrant();
    }
}

__global__ void __launch_bounds__(512, 1) tmem_gather_kernel(const __grid_constant__ TArgs a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = warp & 3, s = warp >> 2;
    const int nb = a.nb;

    int hb = 0;
    while (hb + 1 < a.HB && (int)blockIdx.x >= a.cta_first[hb + 1]) ++hb;
    const int r = blockIdx.x - a.cta_first[hb];
    const int R = a.cta_first[hb + 1] - a.cta_first[hb];
    const int32_t* hi = a.hinfo + hb * kTInfo;
    const int h0 = hi[0], kb = hi[1], rec_base = hi[2], rec_count = hi[3];

    unsigned char* land = smem;
    uint32_t* srecs = reinterpret_cast<uint32_t*>(smem + 4 * kLandBytes);
    uint8_t* scounts = reinterpret_cast<uint8_t*>(srecs + 2 * (size_t)a.recs_max);
    uint32_t* soffs = reinterpret_cast<uint32_t*>(scounts + 4 * nb * 32);
    float* sb = reinterpret_cast<float*>(soffs + 4 * nb);
    int32_t* sgroups = reinterpret_cast<int32_t*>(sb + (a.kb_max + 3) / 4 * 4);
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(sgroups + 4 * kTGroups);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);

    {   // this block's tables
        const uint4* src = reinterpret_cast<const uint4*>(a.recs + 2 * (size_t)rec_base);
        uint4* dst = reinterpret_cast<uint4*>(srecs);
        for (int i = tid; i < rec_count / 2; i += 512) dst[i] = __ldg(src + i);
        const uint32_t* cs = reinterpret_cast<const uint32_t*>(a.counts + (size_t)hb * 4 * nb * 32);
        for (int i = tid; i < nb * 32; i += 512) reinterpret_cast<uint32_t*>(scounts)[i] = __ldg(cs + i);
        for (int i = tid; i < 4 * nb; i += 512) soffs[i] = __ldg(a.offs + (size_t)hb * 4 * nb + i);
        for (int i = tid; i < kb; i += 512) sb[i] = __ldg(a.b + h0 + i);
        for (int i = tid; i < 4 * kTGroups; i += 512) sgroups[i] = __ldg(a.groups + (size_t)hb * 4 * kTGroups + i);
    }
    const uint32_t bar0 = smem_u32(bars);
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) {
            mbar_init(bar0 + 8u * i, 1);
            mbar_init(bar0 + 8u * (4 + i), 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // all 512 columns are this CTA's, so the allocation starts at lane 0, column 0: the kernel folds
    // lane quadrant and buffer into immediate TMEM offsets
    if (*tmem_slot != 0u) __trap();
    if (smem_u32(smem) & 1023u) __trap();  // the 128-byte swizzle pattern assumes 1024-B aligned boxes

    Ctx c;
    c.landq = land + q * kLandBytes;
    c.landq_u32 = smem_u32(c.landq);
    c.recs_u32 = smem_u32(srecs);
    c.counts_u32 = smem_u32(scounts);
    c.bar_full = bar0 + 8u * q;
    c.bar_empty = bar0 + 8u * (4 + q);
    c.soffs = soffs;
    c.sb = sb;
    c.sgroups = sgroups + s * kTGroups;
    c.h0 = h0;
    c.hend = h0 + kb;
    c.ng = hi[4 + s];
    c.s = s;
    c.lane = lane;
    c.nb = nb;
    // this quadrant engine's tiles: e, e + E, ... (64 rows each)
    const long long tiles = (a.N + kTRows - 1) / kTRows;
    c.e = (long long)r * 4 + q;
    c.E = 4LL * R;
    const long long ntile = c.e < tiles ? (tiles - c.e + c.E - 1) / c.E : 0;
    c.G = ntile * nb;
    {   // self-check of the lane-field behaviour gather_block relies on: write this quadrant's
        // lane t at column 511 with its own lane field, read it back with lane field 0
        const uint32_t probe = 0x9e3779b9u ^ (uint32_t)((32 * q + lane) * 2654435761u);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(((uint32_t)(32 * q) << 16) + 511u),
                     "r"(probe)
                     : "memory");
        tmem_wait_st();
        uint32_t back;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(back) : "r"(511u));
        tmem_wait_ld();
        if (back != probe) __trap();
    }
    engine(a, c, q);

    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_slot), "r"(512)
                     : "memory");
    }
}

}  // namespace

fastlsh_status launch_gather_tmem(const fastlsh_params* p, const DeviceCopy& d, const float* X,
                                  int64_t N, int32_t* codes, float* proj, cudaStream_t stream) {
    const TPacking& tp = p->tpack;
    if (!tp.ok || !d.t_recs) return FASTLSH_EUNSUPPORTED;
    if (reinterpret_cast<uintptr_t>(X) & 15) return FASTLSH_EUNSUPPORTED;
    const bool vec_ok = (reinterpret_cast<uintptr_t>(codes) & 15) == 0;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (tp.HB > sms) return FASTLSH_EUNSUPPORTED;
    TArgs a;
    {
        static EncodeTiledFn enc = [] {
            void* fp = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess)
                return (EncodeTiledFn) nullptr;
            return reinterpret_cast<EncodeTiledFn>(fp);
        }();
        if (!enc || N > 0x7fffffffLL) return FASTLSH_EUNSUPPORTED;
        cuuint64_t dims[2] = {(cuuint64_t)p->n, (cuuint64_t)N};
        cuuint64_t strides[1] = {(cuuint64_t)p->n * 4};
        cuuint32_t box[2] = {(cuuint32_t)kBox, (cuuint32_t)kTRows};
        cuuint32_t estr[2] = {1, 1};
        if (enc(&a.xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return FASTLSH_EUNSUPPORTED;
    }
    a.X = X;
    a.N = N;
    a.n = p->n;
    a.nb = tp.nb;
    a.tb = tp.tb;
    a.k = p->k;
    a.recs = d.t_recs;
    a.counts = d.t_counts;
    a.offs = d.t_offs;
    a.hinfo = d.t_hinfo;
    a.groups = d.t_groups;
    a.b = d.b;
    a.w = p->w;
    a.codes = codes;
    a.proj = proj;
    a.flags = d.flags;
    a.recs_max = tp.recs_max;
    a.kb_max = tp.kb_max;
    a.vec_store = (vec_ok && p->k % 4 == 0) ? 1 : 0;
    a.HB = tp.HB;
    // CTAs per hash block in proportion to its hashes (one CTA per SM), capped by its tiles
    const long long tiles = (N + kTRows - 1) / kTRows;
    const long long cap = std::max(1LL, (tiles + 3) / 4);
    std::vector<long long> R(tp.HB, 1);
    int used = tp.HB;
    {
        std::vector<std::pair<double, int>> rem;
        for (int hb = 0; hb < tp.HB; ++hb) {
            const double share = (double)sms * tp.hinfo[(size_t)hb * kTInfo + 1] / p->k;
            R[hb] = std::max(1LL, std::min(cap, (long long)share));
            rem.push_back({share - (double)(long long)share, hb});
        }
        used = 0;
        for (long long v : R) used += (int)v;
        std::sort(rem.begin(), rem.end(), [](auto& x, auto& y) { return x.first > y.first; });
        for (size_t i = 0; used < sms && i < rem.size(); ++i)
            if (R[rem[i].second] < cap) { ++R[rem[i].second]; ++used; }
        while (used > sms) {  // more hash blocks than rounding allows: trim the largest
            int big = (int)(std::max_element(R.begin(), R.end()) - R.begin());
            if (R[big] <= 1) break;
            --R[big];
            --used;
        }
    }
    a.cta_first[0] = 0;
    for (int hb = 0; hb < tp.HB; ++hb) a.cta_first[hb + 1] = a.cta_first[hb] + (int)R[hb];
    const int grid = a.cta_first[tp.HB];
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(tmem_gather_kernel),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tp.smem);
    if (e != cudaSuccess) return set_cuda_error(e);
    tmem_gather_kernel<<<grid, 512, tp.smem, stream>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e);
    return FASTLSH_OK;
}

}  // namespace fastlsh
