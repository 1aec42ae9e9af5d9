// gather_tmem.cu — K1t: FastLSH hashing with TENSOR MEMORY as the gather source (sm_100a).
//
// For every row v and hash i: h_i(v) = floor((a_i . S_i(v) + b_i) / w)   (Eq. 5).
//
// Why TMEM (tools/microbench_tmem*.cu): the shared-memory gather of K1 is capped
// at one 128-B wavefront per SM per clock (G_s = 32 gathers/clk/SM). tcgen05.ld reads tensor
// memory through its own datapath: a warp-uniform column address returns one 32-bit word per
// lane — a conflict-free gather of 32 rows when lane = row — and .32x32b.x8 returns eight adjacent
// columns, i.e. the same coordinate of eight rows when rows are interleaved along columns.
// Measured on B200: the raw .x8 load gathers at 2.8x G_s, the .x4 loop with parameters broadcast
// from shared memory at 1.47x G_s.
// Status: parity-exact, opt-in (fastlsh_params_set_kernel(p, 2)). On C1 it is slower than K1
// (7.4 vs 5.2 ms): the per-slot parameter broadcast (LDS + R2UR + loop control) and the register
// budget for accumulators (which caps hashes per tile, so each staged element feeds few gathers)
// make it instruction-bound, not TMEM-bound. DESIGN.md "K1t" has the measurements.
//
// Layout:
//  * One CTA per SM, 16 warps; warp w works in TMEM lane quadrant q = w % 4 (the hardware rule for
//    tcgen05.ld/st.32x32b). A tile is 256 rows; lane t of EVERY quadrant holds rows t + 32 i
//    (i < 8) of the tile at columns 8*c + i (coordinate c of the current block).
//  * Coordinates stream in blocks of 64 (all 512 columns). TMA tensor copies (boxes of 32
//    coordinates x 256 rows, 128-byte swizzle, rows past N and columns past n read as 0) fill a
//    shared landing while the previous block is gathered; each quadrant's 4 warps then copy the
//    block into their own lanes (LDS.128 x 8 rows -> tcgen05.st.32x32b.x32) between two quadrant
//    barriers.
//  * Hashes: a CTA serves <= 128 hashes (16 warps x 2 groups of 4 consecutive hashes); every warp
//    keeps its 8 hashes' accumulators (8 rows each) in registers for the whole tile. The
//    (TMEM column, coefficient) records of its hashes' slots are grouped by (coordinate block,
//    hash) and broadcast from shared memory (LDS.64 per slot).
//  * Per slot: R2UR + tcgen05.ld.32x32b.x8 at the record's column + 8 FFMA (rows t+32i), in a
//    bra.uni loop per (hash, block) run, two slots per iteration.
//  * Epilogue after the last block of a tile: __fadd_rn(p, b), IEEE division by w (exact multiply
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

constexpr int kX = 8;                        // rows per lane (tcgen05.ld.32x32b.x8)
constexpr int kTRows = 32 * kX;              // rows per tile
constexpr int kTB = 512 / kX;                // coordinates per TMEM block (all 512 columns)
constexpr int kNHW = 4 * kTGroups;           // max hashes per warp (register accumulators)
constexpr int kBox = 32;                     // coordinates per TMA box (128 B, 128-byte swizzle)
constexpr int kBoxBytes = kTRows * kBox * 4; // one box: 256 rows x 128 B
constexpr int kLandBytes = (kTB / kBox) * kBoxBytes;
constexpr int kNL = 1;                       // landing slots
constexpr size_t kSmemMax = 227 * 1024;
constexpr int kTMaxM = 128;

size_t tmem_smem_bytes(int recs_max, int nb, int kb_max) {
    size_t s = kNL * (size_t)kLandBytes;        // landing slots
    s += (size_t)recs_max * 8 + 16;             // (column, coefficient) records + prefetch slack
    s += kTWarps * (size_t)nb * 16;             // per (warp, block) run lengths (u8 x 16)
    s += kTWarps * (size_t)nb * 4;              // per (warp, block) record offsets
    s += ((size_t)kb_max + 3) / 4 * 16;         // b of the block's hashes
    s += kTWarps * kTGroups * 4;                // group starts
    s += 8 * kNL + 4 * kNL + 16;                // mbarriers, consumption counters, TMEM address
    return s;
}

}  // namespace

// Host packing for K1t (SURVEY.md §8(a) a1 "GPU packing"). Leaves tp.ok = false when the shape
// does not suit the TMEM kernel; the shared-memory kernel K1 then serves it.
void build_tmem_packing(const fastlsh_params& p, TPacking& tp) {
    tp = TPacking();
    const int n = p.n, m = p.m, k = p.k;
    if (n % 4 != 0 || m > kTMaxM) return;
    const int nb = (n + kTB - 1) / kTB;
    // groups (of 4 hashes) per warp: as many as the record region allows
    int gw = kTGroups;
    while (gw >= 1 && tmem_smem_bytes(kTWarps * 4 * gw * m, nb, kTWarps * 4 * gw) > kSmemMax) --gw;
    if (gw < 1) return;
    const int groups_total = (k + 3) / 4;
    gw = std::min(gw, std::max(1, (groups_total + kTWarps - 1) / kTWarps));  // small k: fewer per warp
    const int KB = kTWarps * 4 * gw;
    const int HB = (k + KB - 1) / KB;
    if (HB > kTMaxHB) return;
    tp.nb = nb;
    tp.nhw = 4 * gw;
    tp.HB = HB;
    tp.hinfo.assign((size_t)HB * kTInfo, 0);
    tp.groups.assign((size_t)HB * kTWarps * kTGroups, -1);
    tp.counts.assign((size_t)HB * kTWarps * nb * 16, 0);
    tp.offs.assign((size_t)HB * kTWarps * nb, 0);
    // run length of hash h in coordinate block bk
    std::vector<int> cnt((size_t)k * nb, 0);
    for (int h = 0; h < k; ++h)
        for (int t = 0; t < m; ++t) ++cnt[(size_t)h * nb + p.idx[(size_t)h * m + t] / kTB];
    double crit = 0, mean = 0;
    for (int hb = 0; hb < HB; ++hb) {
        const int h0 = hb * KB, kb = std::min(KB, k - h0);
        const int G = (kb + 3) / 4;
        // cost of group g in block bk: its slots plus a per-run overhead (in slot units)
        std::vector<int> cost((size_t)G * nb, 0);
        for (int g = 0; g < G; ++g)
            for (int u = 0; u < 4 && 4 * g + u < kb; ++u)
                for (int bk = 0; bk < nb; ++bk) cost[(size_t)g * nb + bk] += cnt[(size_t)(h0 + 4 * g + u) * nb + bk] + 2;
        // groups -> warps (<= gw each): round robin over warps, then pairwise swaps that lower the
        // sum over blocks of the largest warp load (all warps meet once per block at the landing),
        // ties broken by the sum of squared loads
        std::vector<int> owner(G);
        for (int g = 0; g < G; ++g) owner[g] = g % kTWarps;
        std::vector<int> load((size_t)kTWarps * nb, 0);
        for (int g = 0; g < G; ++g)
            for (int bk = 0; bk < nb; ++bk) load[(size_t)owner[g] * nb + bk] += cost[(size_t)g * nb + bk];
        auto objective = [&](long long* total) {
            long long worst = 0, sum = 0;
            for (int bk = 0; bk < nb; ++bk) {
                int mx = 0, sm = 0;
                for (int w = 0; w < kTWarps; ++w) {
                    mx = std::max(mx, load[(size_t)w * nb + bk]);
                    sm += load[(size_t)w * nb + bk] * load[(size_t)w * nb + bk];
                }
                worst += mx;
                sum += sm;
            }
            *total = sum;
            return worst;
        };
        long long best_sum = 0, best = objective(&best_sum);
        for (int pass = 0; pass < 40; ++pass) {
            bool improved = false;
            for (int g1 = 0; g1 < G; ++g1) {
                for (int g2 = g1 + 1; g2 < G; ++g2) {
                    const int w1 = owner[g1], w2 = owner[g2];
                    if (w1 == w2) continue;
                    for (int bk = 0; bk < nb; ++bk) {
                        const int d = cost[(size_t)g2 * nb + bk] - cost[(size_t)g1 * nb + bk];
                        load[(size_t)w1 * nb + bk] += d;
                        load[(size_t)w2 * nb + bk] -= d;
                    }
                    long long sum = 0;
                    const long long f = objective(&sum);
                    if (f < best || (f == best && sum < best_sum)) {
                        best = f;
                        best_sum = sum;
                        owner[g1] = w2;
                        owner[g2] = w1;
                        improved = true;
                    } else {
                        for (int bk = 0; bk < nb; ++bk) {
                            const int d = cost[(size_t)g2 * nb + bk] - cost[(size_t)g1 * nb + bk];
                            load[(size_t)w1 * nb + bk] -= d;
                            load[(size_t)w2 * nb + bk] += d;
                        }
                    }
                }
            }
            if (!improved) break;
        }
        {
            long long tot = 0;
            for (int v : load) tot += v;
            crit += (double)best;
            mean += (double)tot / kTWarps;
        }
        int32_t* hi = &tp.hinfo[(size_t)hb * kTInfo];
        hi[0] = h0;
        hi[1] = kb;
        hi[2] = (int32_t)(tp.recs.size() / 2);
        std::vector<std::vector<int>> wg(kTWarps);
        for (int g = 0; g < G; ++g) wg[owner[g]].push_back(g);
        for (int w = 0; w < kTWarps; ++w) {
            if ((int)wg[w].size() > gw) return;  // cannot happen: swaps keep the round-robin sizes
            hi[4 + w] = (int32_t)wg[w].size();
            for (size_t gi = 0; gi < wg[w].size(); ++gi)
                tp.groups[((size_t)hb * kTWarps + w) * kTGroups + gi] = h0 + 4 * wg[w][gi];
        }
        const size_t rec0 = tp.recs.size() / 2;
        for (int w = 0; w < kTWarps; ++w) {
            for (int bk = 0; bk < nb; ++bk) {
                tp.offs[((size_t)hb * kTWarps + w) * nb + bk] = (uint32_t)(tp.recs.size() / 2 - rec0);
                for (size_t gi = 0; gi < wg[w].size(); ++gi) {
                    for (int u = 0; u < 4; ++u) {
                        const int h = h0 + 4 * wg[w][gi] + u;
                        if (h >= h0 + kb) break;
                        const int32_t* idx = &p.idx[(size_t)h * m];
                        const float* a = &p.a[(size_t)h * m];
                        int c = 0;
                        for (int t = 0; t < m; ++t) {
                            if (idx[t] / kTB != bk) continue;
                            uint32_t cb;
                            std::memcpy(&cb, &a[t], 4);
                            tp.recs.push_back((uint32_t)(kX * (idx[t] - bk * kTB)));
                            tp.recs.push_back(cb);
                            ++c;
                        }
                        tp.counts[(((size_t)hb * kTWarps + w) * nb + bk) * 16 + 4 * gi + u] = (uint8_t)c;
                    }
                }
            }
        }
        hi[3] = (int32_t)(tp.recs.size() / 2 - rec0);
        tp.recs_max = std::max(tp.recs_max, hi[3]);
        tp.kb_max = std::max(tp.kb_max, kb);
    }
    tp.balance = mean > 0 ? crit / mean : 1.0;
    tp.smem = tmem_smem_bytes(tp.recs_max, nb, tp.kb_max);
    if (tp.smem > kSmemMax) return;
    tp.ok = true;
}

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct TArgs {
    CUtensorMap xmap;  // X [N][n] f32, box 32 coordinates x 128 rows, 128-byte swizzle
    long long N;
    int n, nb, k;
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
__device__ __forceinline__ float4 lds128f(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t uni(uint32_t v) { return __shfl_sync(0xffffffffu, v, 0); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
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

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// 32 consecutive columns: coordinate-major, 8 rows each: (v0.x, v1.x, ..., v7.x, v0.y, ...)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float4 (&v)[8]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "f"(v[0].x), "f"(v[1].x), "f"(v[2].x), "f"(v[3].x), "f"(v[4].x), "f"(v[5].x), "f"(v[6].x), "f"(v[7].x),
        "f"(v[0].y), "f"(v[1].y), "f"(v[2].y), "f"(v[3].y), "f"(v[4].y), "f"(v[5].y), "f"(v[6].y), "f"(v[7].y),
        "f"(v[0].z), "f"(v[1].z), "f"(v[2].z), "f"(v[3].z), "f"(v[4].z), "f"(v[5].z), "f"(v[6].z), "f"(v[7].z),
        "f"(v[0].w), "f"(v[1].w), "f"(v[2].w), "f"(v[3].w), "f"(v[4].w), "f"(v[5].w), "f"(v[6].w), "f"(v[7].w)
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

// Per-warp state (shared-memory tables are this CTA's hash block).
struct Ctx {
    uint32_t land_u32, recs_u32, counts_u32, bar0;
    int* consumed;           // [kNL] warps that finished staging from each landing slot
    const uint32_t* soffs;   // this warp's [nb] record offsets
    const float* sb;
    const int32_t* sgroups;  // this warp's group starts
    int h0, hend, ng, wi, q, s, lane, nb;
    long long r, R, G;
};

// One hash's run of cnt records at shared address rp: acc_i += x[row t+32i][c] * a for each
// record (c as a TMEM column, a). Inline PTX so that the warp-uniform loop is a bra.uni loop,
// two records per iteration plus a one-record tail. The TMEM address is the record's
// column with lane field 0: for the .32x32b shapes the hardware serves the warp's own lane
// quadrant whatever the lane field says (measured: tools/microbench_tmem_lane.cu; checked at
// kernel start).
__device__ __forceinline__ void hash_run(float (&acc)[kX], uint32_t& rp, uint32_t cnt) {
    static_assert(kX == 8, "hash_run is written for 8 rows per lane");
    asm volatile(
        "{\n\t"
        ".reg .pred P;\n\t"
        ".reg .b32 e, e2, c0, c1;\n\t"
        ".reg .f32 f0, f1, u0, u1, u2, u3, u4, u5, u6, u7, w0, w1, w2, w3, w4, w5, w6, w7;\n\t"
        "mad.lo.u32 e, %9, 8, %8;\n\t"
        "sub.u32 e2, e, 8;\n\t"
        "setp.ge.u32 P, %8, e2;\n\t"
        "@P bra.uni HR_TAIL_%=;\n"
        "HR_LOOP_%=:\n\t"
        "ld.shared.v2.b32 {c0, f0}, [%8];\n\t"
        "ld.shared.v2.b32 {c1, f1}, [%8+8];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {u0, u1, u2, u3, u4, u5, u6, u7}, [c0];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {w0, w1, w2, w3, w4, w5, w6, w7}, [c1];\n\t"
        "add.u32 %8, %8, 16;\n\t"
        "setp.lt.u32 P, %8, e2;\n\t"
        "tcgen05.wait::ld.sync.aligned;\n\t"
        "fma.rn.f32 %0, u0, f0, %0;\n\t"
        "fma.rn.f32 %1, u1, f0, %1;\n\t"
        "fma.rn.f32 %2, u2, f0, %2;\n\t"
        "fma.rn.f32 %3, u3, f0, %3;\n\t"
        "fma.rn.f32 %4, u4, f0, %4;\n\t"
        "fma.rn.f32 %5, u5, f0, %5;\n\t"
        "fma.rn.f32 %6, u6, f0, %6;\n\t"
        "fma.rn.f32 %7, u7, f0, %7;\n\t"
        "fma.rn.f32 %0, w0, f1, %0;\n\t"
        "fma.rn.f32 %1, w1, f1, %1;\n\t"
        "fma.rn.f32 %2, w2, f1, %2;\n\t"
        "fma.rn.f32 %3, w3, f1, %3;\n\t"
        "fma.rn.f32 %4, w4, f1, %4;\n\t"
        "fma.rn.f32 %5, w5, f1, %5;\n\t"
        "fma.rn.f32 %6, w6, f1, %6;\n\t"
        "fma.rn.f32 %7, w7, f1, %7;\n\t"
        "@P bra.uni HR_LOOP_%=;\n"
        "HR_TAIL_%=:\n\t"
        "setp.ge.u32 P, %8, e;\n\t"
        "@P bra.uni HR_DONE_%=;\n\t"
        "ld.shared.v2.b32 {c0, f0}, [%8];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {u0, u1, u2, u3, u4, u5, u6, u7}, [c0];\n\t"
        "add.u32 %8, %8, 8;\n\t"
        "tcgen05.wait::ld.sync.aligned;\n\t"
        "fma.rn.f32 %0, u0, f0, %0;\n\t"
        "fma.rn.f32 %1, u1, f0, %1;\n\t"
        "fma.rn.f32 %2, u2, f0, %2;\n\t"
        "fma.rn.f32 %3, u3, f0, %3;\n\t"
        "fma.rn.f32 %4, u4, f0, %4;\n\t"
        "fma.rn.f32 %5, u5, f0, %5;\n\t"
        "fma.rn.f32 %6, u6, f0, %6;\n\t"
        "fma.rn.f32 %7, u7, f0, %7;\n"
        "HR_DONE_%=:\n\t"
        "}"
        : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3]), "+f"(acc[4]), "+f"(acc[5]), "+f"(acc[6]),
          "+f"(acc[7]), "+r"(rp)
        : "r"(cnt)
        : "memory");
}

// Gather-FMA over this warp's hashes for coordinate block bk.
__device__ __forceinline__ void gather_block(const Ctx& c, float (&acc)[kNHW][kX], int bk) {
    const int nh = 4 * c.ng;
    uint32_t rp = c.recs_u32 + 8u * uni(c.soffs[bk]);
    const uint4 cw = lds128(c.counts_u32 + (uint32_t)(c.wi * c.nb + bk) * 16u);
    const uint32_t words[4] = {uni(cw.x), uni(cw.y), uni(cw.z), uni(cw.w)};
#pragma unroll
    for (int j = 0; j < kNHW; ++j) {
        if (j < nh) {
            hash_run(acc[j], rp, (words[j >> 2] >> (8 * (j & 3))) & 0xffu);
        }
    }
}

__device__ __forceinline__ void engine(const TArgs& a, const Ctx& c) {
    const int lane = c.lane, nb = c.nb;
    const uint32_t qcol = (uint32_t)(32 * c.q) << 16;

    auto issue = [&](long long g) {  // one thread: TMA boxes of block g (OOB rows/columns -> 0)
        const int row0 = (int)((c.r + (g / nb) * c.R) * kTRows);
        const int x0 = (int)(g % nb) * kTB;
        int nbox = 0;
        for (int bx = 0; bx < kTB / kBox; ++bx) nbox += (x0 + bx * kBox < a.n);
        mbar_arrive_tx(c.bar0, (uint32_t)(nbox * kBoxBytes));
        for (int bx = 0; bx < kTB / kBox; ++bx)
            if (x0 + bx * kBox < a.n)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3}], [%4];" ::"r"(c.land_u32 + bx * kBoxBytes),
                    "l"(reinterpret_cast<uint64_t>(&a.xmap)), "r"(x0 + bx * kBox), "r"(row0), "r"(c.bar0)
                    : "memory");
    };
    // This warp's 16 coordinates [16s, 16s+16) of block g (half of TMA box s/2): landing -> this
    // quadrant's TMEM lanes. Row r of a box is 128 B whose 16-byte chunk j sits at chunk j ^ (r % 8)
    // (128-byte swizzle), so a quarter-warp (rows t..t+7) reads 8 different bank groups. The last
    // of the 16 warps to finish with the landing refills it with block g + 1.
    auto stage = [&](long long g) {
        mbar_wait(c.bar0, (uint32_t)(g & 1));
        const int bk = (int)(g % nb);
        if (bk * kTB + 16 * c.s < a.n) {
            const uint32_t box = c.land_u32 + (c.s >> 1) * kBoxBytes + lane * 128;
            const uint32_t tcol = qcol + (uint32_t)(kX * 16) * c.s;
            const int sw = lane & 7;  // (lane + 32 i) % 8 == lane % 8
#pragma unroll
            for (int cj = 0; cj < 4; ++cj) {
                const uint32_t off = 16u * (uint32_t)(((c.s & 1) * 4 + cj) ^ sw);
                float4 v[kX];
#pragma unroll
                for (int i = 0; i < kX; ++i) v[i] = lds128f(box + i * 32 * 128 + off);
                tmem_st32(tcol + 32u * cj, v);
            }
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            const int before = atomicAdd(c.consumed, 1);
            if (before % kTWarps == kTWarps - 1 && g + 1 < c.G) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(g + 1);
            }
        }
    };
    auto sync_quadrant = [&]() {
        tc_fence_before();
        asm volatile("bar.sync %0, 128;" ::"r"(1 + c.q) : "memory");
        tc_fence_after();
    };

    const float w = a.w;
    const float inv_w = 1.0f / w;
    const bool w_pow2 = (__float_as_uint(w) & 0x007fffffu) == 0 && isfinite(inv_w) && inv_w != 0.0f;
    // rows past N read zeros (TMA out-of-bounds fill); their results are discarded (no store, no flag)
    auto epilogue = [&](float (&acc)[kNHW][kX], long long i) {
        const long long row0 = (c.r + i * c.R) * kTRows;
#pragma unroll
        for (int gi = 0; gi < kNHW / 4; ++gi) {
            if (gi < c.ng) {
                const int hs = c.sgroups[gi];
                const bool full = hs + 4 <= c.hend;
                float bh[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) bh[u] = (hs + u < c.hend) ? c.sb[hs - c.h0 + u] : 0.f;
#pragma unroll
                for (int rr = 0; rr < kX; ++rr) {
                    const long long row = row0 + lane + 32 * rr;
                    const bool live = row < a.N;
                    const long long o = row * a.k + hs;
                    if (a.proj) {
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (live && hs + u < c.hend) a.proj[o + u] = acc[4 * gi + u][rr];
                        continue;
                    }
                    int cv[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        cv[u] = quantise(acc[4 * gi + u][rr], bh[u], w, inv_w, w_pow2, a.flags, live && hs + u < c.hend);
                    if (!live) continue;
                    if (a.vec_store && full) {
                        *reinterpret_cast<int4*>(a.codes + o) = make_int4(cv[0], cv[1], cv[2], cv[3]);
                    } else {
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (hs + u < c.hend) a.codes[o + u] = cv[u];
                    }
                }
            }
        }
    };

    // per block: stage (needs the quadrant done with the previous block) -> barrier -> gather ->
    // barrier. The landing refill for block g+1 overlaps the gather of block g.
    float acc[kNHW][kX];
    if (c.G > 0 && c.wi == 0 && lane == 0) issue(0);
    for (long long g = 0; g < c.G; ++g) {
        stage(g);
        tmem_wait_st();
        sync_quadrant();
        const int bk = (int)(g % nb);
        if (bk == 0) {
#pragma unroll
            for (int j = 0; j < kNHW; ++j)
#pragma unroll
                for (int i = 0; i < kX; ++i) acc[j][i] = 0.f;
        }
        gather_block(c, acc, bk);
        if (bk == nb - 1) epilogue(acc, g / nb);
        sync_quadrant();
    }
}

__global__ void __launch_bounds__(512, 1) tmem_gather_kernel(const __grid_constant__ TArgs a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nb = a.nb;

    int hb = 0;
    while (hb + 1 < a.HB && (int)blockIdx.x >= a.cta_first[hb + 1]) ++hb;
    const int r = blockIdx.x - a.cta_first[hb];
    const int R = a.cta_first[hb + 1] - a.cta_first[hb];
    const int32_t* hi = a.hinfo + hb * kTInfo;
    const int h0 = hi[0], kb = hi[1], rec_base = hi[2], rec_count = hi[3];

    unsigned char* land = smem;
    uint32_t* srecs = reinterpret_cast<uint32_t*>(smem + kNL * kLandBytes);
    uint8_t* scounts = reinterpret_cast<uint8_t*>(srecs + 2 * (size_t)a.recs_max + 4);  // + slack record, 16-B aligned
    uint32_t* soffs = reinterpret_cast<uint32_t*>(scounts + kTWarps * nb * 16);
    float* sb = reinterpret_cast<float*>(soffs + kTWarps * nb);
    int32_t* sgroups = reinterpret_cast<int32_t*>(sb + (a.kb_max + 3) / 4 * 4);
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(sgroups + kTWarps * kTGroups);
    int* consumed = reinterpret_cast<int*>(bars + kNL);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(consumed + kNL);

    {   // this hash block's tables
        const uint2* src = reinterpret_cast<const uint2*>(a.recs) + rec_base;
        uint2* dst = reinterpret_cast<uint2*>(srecs);
        for (int i = tid; i < rec_count; i += 512) dst[i] = __ldg(src + i);
        const uint32_t* cs = reinterpret_cast<const uint32_t*>(a.counts + (size_t)hb * kTWarps * nb * 16);
        for (int i = tid; i < kTWarps * nb * 4; i += 512) reinterpret_cast<uint32_t*>(scounts)[i] = __ldg(cs + i);
        for (int i = tid; i < kTWarps * nb; i += 512) soffs[i] = __ldg(a.offs + (size_t)hb * kTWarps * nb + i);
        for (int i = tid; i < kb; i += 512) sb[i] = __ldg(a.b + h0 + i);
        for (int i = tid; i < kTWarps * kTGroups; i += 512)
            sgroups[i] = __ldg(a.groups + (size_t)hb * kTWarps * kTGroups + i);
        if (tid < kNL) consumed[tid] = 0;
        if (tid == 0) reinterpret_cast<uint2*>(srecs)[rec_count] = make_uint2(0u, 0u);  // prefetch slack
    }
    const uint32_t bar0 = smem_u32(bars);
    if (tid == 0) {
        for (int i = 0; i < kNL; ++i) mbar_init(bar0 + 8u * i, 1);
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
    // all 512 columns are this CTA's, so the allocation starts at lane 0, column 0
    if (*tmem_slot != 0u) __trap();
    if (smem_u32(smem) & 1023u) __trap();  // the 128-byte swizzle pattern assumes 1024-B aligned boxes
    {   // self-check of the lane-field behaviour gather_block relies on: write this quadrant's
        // lane t at column 511 with its own lane field, read it back with lane field 0
        const int q = warp & 3;
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
    tc_fence_before();
    __syncthreads();  // the probe column is data from now on
    tc_fence_after();

    Ctx c;
    c.land_u32 = smem_u32(land);
    c.recs_u32 = smem_u32(srecs);
    c.counts_u32 = smem_u32(scounts);
    c.bar0 = bar0;
    c.consumed = consumed;
    c.soffs = soffs + warp * nb;
    c.sb = sb;
    c.sgroups = sgroups + warp * kTGroups;
    c.h0 = h0;
    c.hend = h0 + kb;
    c.ng = hi[4 + warp];
    c.wi = warp;
    c.q = warp & 3;
    c.s = warp >> 2;
    c.lane = lane;
    c.nb = nb;
    // this CTA's tiles: r, r + R, ... (128 rows each)
    const long long tiles = (a.N + kTRows - 1) / kTRows;
    c.r = r;
    c.R = R;
    const long long ntile = r < tiles ? (tiles - r + R - 1) / R : 0;
    c.G = ntile * nb;
    engine(a, c);

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
    a.N = N;
    a.n = p->n;
    a.nb = tp.nb;
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
    // CTAs per hash block in proportion to its hashes (one CTA per SM), capped by the tile count
    const long long tiles = (N + kTRows - 1) / kTRows;
    const long long cap = std::max(1LL, tiles);
    std::vector<long long> R(tp.HB, 1);
    {
        std::vector<std::pair<double, int>> rem;
        for (int hb = 0; hb < tp.HB; ++hb) {
            const double share = (double)sms * tp.hinfo[(size_t)hb * kTInfo + 1] / p->k;
            R[hb] = std::max(1LL, std::min(cap, (long long)share));
            rem.push_back({share - (double)(long long)share, hb});
        }
        int used = 0;
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
    if (fastlsh_status so = smem_optin_once(reinterpret_cast<const void*>(tmem_gather_kernel)); so != FASTLSH_OK)
        return so;
    cudaError_t e;
    tmem_gather_kernel<<<grid, 512, tp.smem, stream>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e);
    return FASTLSH_OK;
}

}  // namespace fastlsh
