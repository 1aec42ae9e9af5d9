// rpacker.cpp — bank scheduling for the row-major kernel K1r (SURVEY.md §8(a3)
// layout B "lane = hash, all lanes read the same row", bank-scheduled).
//
// Addition commutes, so the order of a hash's m products is free (Eq. 5 fixes the
// value, not the order). K1r stages rows row-major at a stride of S = 32*ceil(n/32) + 32 words, so
// coordinate c of any staged row sits in bank c mod 32, and a warp's LDS.32 at one slot position
// is a single wavefront when its 32 lanes read 32 distinct banks (or the same word). The packer:
//  1. splits k hashes into hash blocks (one CTA each) of <= 32/P * W hashes; block boundaries are
//     multiples of 4 so every block's codes of a row are a 16-byte aligned run (TMA bulk stores);
//  2. gives each warp hpw = 32/P hashes, hash slot j taking a hash congruent to j mod hpw (the
//     warp's code stores then hit distinct banks); starting from consecutive hashes, it swaps
//     same-slot hashes between warps to flatten every warp's per-bank load towards ceil(m/P)
//     (local search on F = sum over (warp, bank) of max(0, load - T)^2, T relaxed when stuck);
//  3. splits each hash's m slots into P parts (lanes j + hpw*q) and edge-colours the warp's
//     lanes x banks multigraph with Delta colours (König): a colour is a slot position;
//  4. where the stage class leaves room, coordinates [0, n1) are staged twice, the second copy
//     rotated by 16 banks; a warp's samples of those coordinates pick the copy that flattens its
//     bank loads (with one copy, the per-bank totals alone bound C3 at 80% useful slots);
//  5. fills free (lane, position) pairs with padding slots (coefficient 0, reading the zero word
//     of an unused bank in the staged row's 32-word zero tail), or, in the capped variant, folds
//     colours beyond the part size into existing positions (a few bank conflicts).
// A cost model (wavefronts per row / measured pipe rate) picks P, warps per CTA and the variant.
// Everything is deterministic, so every rank derives the identical packing and fp32 order.
#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <numeric>

#include "internal.h"

namespace fastlsh {
namespace {

// slot counts the kernel is instantiated for: even up to 64, multiples of 8 up to 128
int round_slots(int ms) {
    if (ms <= 64) return std::max(2, (ms + 1) & ~1);
    return (ms + 7) & ~7;
}

using Bank = std::array<int, 32>;

// Step 2: warps of a block. slot[w*hpw + j] = block-local hash or -1. Returns per-warp loads.
void balance_warps(const std::vector<Bank>& cnt, int kb, int hpw, int W, int T, std::vector<int>& slot,
                   std::vector<Bank>& load) {
    slot.assign((size_t)W * hpw, -1);
    load.assign(W, Bank{});
    for (int h = 0; h < kb; ++h) {
        slot[(size_t)(h / hpw) * hpw + h % hpw] = h;
        for (int b = 0; b < 32; ++b) load[h / hpw][b] += cnt[h][b];
    }
    if (W < 2) return;
    auto ex = [](int v, int Tt) { return v > Tt ? (long)(v - Tt) * (v - Tt) : 0L; };
    const Bank zero{};
    for (int Tt = T, guard = 0; guard < 256; ++Tt, ++guard) {
        bool any_excess = true;
        for (int sweep = 0; sweep < 64; ++sweep) {
            bool improved = false;
            any_excess = false;
            for (int w1 = 0; w1 < W; ++w1) {
                long e1 = 0;
                for (int b = 0; b < 32; ++b) e1 += ex(load[w1][b], Tt);
                if (e1 == 0) continue;
                any_excess = true;
                long best = 0;
                int bj = -1, bw = -1;
                for (int j = 0; j < hpw; ++j) {
                    const int h1 = slot[(size_t)w1 * hpw + j];
                    const Bank& c1 = h1 >= 0 ? cnt[h1] : zero;
                    for (int w2 = 0; w2 < W; ++w2) {
                        if (w2 == w1) continue;
                        const int h2 = slot[(size_t)w2 * hpw + j];
                        if (h1 < 0 && h2 < 0) continue;
                        const Bank& c2 = h2 >= 0 ? cnt[h2] : zero;
                        long d = 0;
                        for (int b = 0; b < 32; ++b) {
                            const int dl = c2[b] - c1[b];
                            if (dl == 0) continue;
                            d += ex(load[w1][b] + dl, Tt) - ex(load[w1][b], Tt) + ex(load[w2][b] - dl, Tt) -
                                 ex(load[w2][b], Tt);
                        }
                        if (d < best) { best = d; bj = j; bw = w2; }
                    }
                }
                if (bj < 0) continue;
                improved = true;
                const int h1 = slot[(size_t)w1 * hpw + bj], h2 = slot[(size_t)bw * hpw + bj];
                for (int b = 0; b < 32; ++b) {
                    const int dl = (h2 >= 0 ? cnt[h2][b] : 0) - (h1 >= 0 ? cnt[h1][b] : 0);
                    load[w1][b] += dl;
                    load[bw][b] -= dl;
                }
                std::swap(slot[(size_t)w1 * hpw + bj], slot[(size_t)bw * hpw + bj]);
            }
            if (!any_excess || !improved) break;
        }
        if (!any_excess) break;
    }
}

// One packing for P parts, at most Wmax warps per CTA, capped (fold beyond the part size) or not.
void try_rows(const fastlsh_params& p, int P, int Wmax, bool capped, RPacking& out, int dual_cls = -1) {
    const int n = p.n, m = p.m, k = p.k;
    RPacking pk;
    pk.parts = P;
    pk.cls = -1;
    pk.S0 = 32 * ((n + 31) / 32) + 32;  // copy 0: the row + a 32-word zero tail
    // short rows (n <= 512): a dual class, whose copy 1 holds all coordinates again at word
    // S0 + 16 + c, i.e. in bank (c + 16) mod 32: a sample may read either copy, so only the 16 pair
    // totals of a warp's bank loads matter (measured: a partial copy for longer rows cost more in
    // TMA issues than it saved). Longer rows: the smallest single-copy class.
    const bool no_copy1 = std::getenv("FASTLSH_NO_COPY1") != nullptr;  // experiment knob
    for (int c = 0; c < kRDualClasses && pk.cls < 0 && !no_copy1; ++c)
        if (n <= kRDualMaxN[c]) pk.cls = c;
    // dual_cls (4 or 6): a dual copy in a 2080-word class (4- or 8-row stages) for rows up to ~1000
    // words, tried beside the single-copy class by the cost model (C4: 2.15 -> 1.90 ms with 4-row
    // stages; C1 loses with them, 3.92 -> 4.42)
    if (pk.cls < 0 && dual_cls >= 0) {
        if (2 * pk.S0 - 16 > kRClasses[dual_cls].S) return;
        pk.cls = dual_cls;
    }
    if (pk.cls >= 0) {
        pk.n1 = n;
    } else {
        for (int c = 5; c >= kRDualClasses; --c)  // single-copy classes 3-5
            if (kRClasses[c].S >= pk.S0) pk.cls = c;
        if (pk.cls < 0) return;
        pk.n1 = 0;
    }
    pk.S = kRClasses[pk.cls].S;
    if (pk.n1 && pk.S0 + 16 + pk.n1 > pk.S) return;
    const int hpw = 32 / P;
    const int T = (m + P - 1) / P;
    if (T > kRMaxSlots) return;
    const int kb_cap = hpw * Wmax;
    // blocks: multiples of 4 hashes (the last takes the rest), balanced
    const int q4 = (k + 3) / 4;
    int HB = std::max(1, (k + kb_cap - 1) / kb_cap);
    while (4 * ((q4 + HB - 1) / HB) > kb_cap) ++HB;
    pk.hash_blocks = HB;
    pk.block_h0.resize(HB);
    pk.block_kb.resize(HB);
    for (int bl = 0, h0 = 0; bl < HB; ++bl) {
        const int quads = q4 / HB + (bl < q4 % HB ? 1 : 0);
        pk.block_h0[bl] = h0;
        pk.block_kb[bl] = std::min(4 * quads, k - h0);
        h0 += pk.block_kb[bl];
    }
    pk.kb_max = *std::max_element(pk.block_kb.begin(), pk.block_kb.end());
    const int W = (pk.kb_max + hpw - 1) / hpw;
    pk.warps = W;

    // per block: warp assignment, part split, colouring
    struct WarpPlan {
        std::vector<int> lane, bank, word;  // one entry per sample edge
        std::vector<float> coef;
        std::vector<int> col;
        int delta = 0;
    };
    std::vector<std::vector<WarpPlan>> plans(HB, std::vector<WarpPlan>(W));
    std::vector<std::vector<int>> slots_of(HB);
    int maxdelta = 0;
    for (int bl = 0; bl < HB; ++bl) {
        const int kb = pk.block_kb[bl], h0 = pk.block_h0[bl];
        // warp balance on bank loads; when every coordinate has two copies (n1 == n) a sample
        // can sit in bank b or b+16, so only the 16 pair totals matter (target 2T)
        const bool pairs = pk.n1 == n;
        std::vector<Bank> cnt(kb, Bank{});
        for (int h = 0; h < kb; ++h)
            for (int j = 0; j < m; ++j) cnt[h][p.idx[(size_t)(h0 + h) * m + j] & (pairs ? 15 : 31)]++;
        std::vector<Bank> load;
        balance_warps(cnt, kb, hpw, W, pairs ? 2 * T : T, slots_of[bl], load);
        for (int w = 0; w < W; ++w) {
            WarpPlan& wp = plans[bl][w];
            for (int j = 0; j < hpw; ++j) {
                const int h = slots_of[bl][(size_t)w * hpw + j];
                if (h < 0) continue;
                // parts: samples sorted by bank, dealt round-robin (part degrees floor/ceil m/P)
                std::vector<int> ord(m);
                std::iota(ord.begin(), ord.end(), 0);
                const int32_t* ix = &p.idx[(size_t)(h0 + h) * m];
                std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return (ix[x] & 31) < (ix[y] & 31); });
                for (int e = 0; e < m; ++e) {
                    const int jj = ord[e];
                    wp.lane.push_back(j + hpw * (e % P));
                    wp.bank.push_back(ix[jj] & 31);
                    wp.word.push_back(ix[jj]);
                    wp.coef.push_back(p.a[(size_t)(h0 + h) * m + jj]);
                }
            }
            // copies: samples of coordinates < n1 take the less loaded of banks c, c+16 (greedy in
            // order, then flips out of the fullest banks while they lower the maximum)
            Bank ld{};
            std::vector<int> flex;
            for (size_t e = 0; e < wp.word.size(); ++e) {
                if (wp.word[e] < pk.n1) flex.push_back((int)e);
                else ld[wp.bank[e]]++;
            }
            for (int e : flex) {
                const int b0 = wp.bank[e], b1 = (b0 + 16) & 31;
                if (ld[b1] < ld[b0]) {
                    wp.bank[e] = b1;
                    wp.word[e] += pk.S0 + 16;
                }
                ld[wp.bank[e]]++;
            }
            for (bool moved = !flex.empty(); moved;) {
                moved = false;
                for (int e : flex) {
                    const int b = wp.bank[e], b2 = (b + 16) & 31;
                    if (ld[b2] + 1 < ld[b]) {
                        ld[b]--;
                        ld[b2]++;
                        wp.bank[e] = b2;
                        wp.word[e] += wp.word[e] < pk.n1 ? pk.S0 + 16 : -(pk.S0 + 16);
                        moved = true;
                    }
                }
            }
            int d = T;
            for (int b = 0; b < 32; ++b) d = std::max(d, ld[b]);
            wp.delta = d;
            wp.col = color_bipartite(wp.lane, wp.bank, 32, 32, std::max(1, d));
            if (!wp.col.empty() && wp.col[0] < 0) return;  // cannot happen (König)
            maxdelta = std::max(maxdelta, d);
        }
    }
    int MS = round_slots(maxdelta);
    if (capped) MS = std::min(MS, round_slots(T));
    if (MS > kRMaxSlots) return;
    if (Wmax == 16 && MS > 64) return;  // 16 warps x 32 lanes need <= 128 registers per lane
    pk.slots = MS;

    const size_t lanes_total = (size_t)HB * W * 32;
    pk.offp.assign(lanes_total * (MS / 2), 0);
    pk.coef.assign(lanes_total * MS, 0.0f);
    pk.lane_hash.assign(lanes_total, (int16_t)-1);
    int64_t useful = 0, conflicts = 0;
    for (int bl = 0; bl < HB; ++bl) {
        for (int w = 0; w < W; ++w) {
            WarpPlan& wp = plans[bl][w];
            std::vector<int> tword((size_t)MS * 32, -1);
            std::vector<float> tcoef((size_t)MS * 32, 0.0f);
            std::vector<int> used((size_t)MS * 32, 0);  // lanes per (t, bank) reading distinct words
            std::vector<int> overflow;
            for (size_t e = 0; e < wp.lane.size(); ++e) {
                const int t = wp.col[e];
                if (t < MS) {
                    tword[(size_t)t * 32 + wp.lane[e]] = wp.word[e];
                    tcoef[(size_t)t * 32 + wp.lane[e]] = wp.coef[e];
                    used[(size_t)t * 32 + wp.bank[e]]++;
                } else {
                    overflow.push_back((int)e);
                }
            }
            for (int e : overflow) {  // fold: the free position of this lane with the least-used bank
                int bt = -1, bu = 1 << 30;
                for (int t = 0; t < MS; ++t) {
                    if (tword[(size_t)t * 32 + wp.lane[e]] >= 0) continue;
                    const int u = used[(size_t)t * 32 + wp.bank[e]];
                    if (u < bu) { bu = u; bt = t; }
                }
                if (bt < 0) return;  // lane degree > MS: cannot happen (MS >= T)
                tword[(size_t)bt * 32 + wp.lane[e]] = wp.word[e];
                tcoef[(size_t)bt * 32 + wp.lane[e]] = wp.coef[e];
                used[(size_t)bt * 32 + wp.bank[e]]++;
            }
            useful += (int64_t)wp.lane.size();
            for (int t = 0; t < MS; ++t) {
                // padding lanes read the zero word of a bank unused at t (least used if none)
                for (int l = 0; l < 32; ++l) {
                    if (tword[(size_t)t * 32 + l] >= 0) continue;
                    int bb = 0;
                    for (int b = 1; b < 32; ++b)
                        if (used[(size_t)t * 32 + b] < used[(size_t)t * 32 + bb]) bb = b;
                    used[(size_t)t * 32 + bb]++;
                    tword[(size_t)t * 32 + l] = pk.S0 - 32 + bb;
                    tcoef[(size_t)t * 32 + l] = 0.0f;
                }
                // extra wavefronts: distinct words sharing a bank (equal words are a broadcast)
                std::array<std::vector<int>, 32> words;
                for (int l = 0; l < 32; ++l) {
                    const int wd = tword[(size_t)t * 32 + l];
                    auto& v = words[wd & 31];
                    if (std::find(v.begin(), v.end(), wd) == v.end()) v.push_back(wd);
                }
                size_t mx = 1;
                for (auto& v : words) mx = std::max(mx, v.size());
                conflicts += (int64_t)mx - 1;
            }
            const size_t wl = (size_t)bl * W + w;
            for (int l = 0; l < 32; ++l) {
                for (int t = 0; t < MS; ++t) {
                    const uint32_t off = 4u * (uint32_t)tword[(size_t)t * 32 + l];
                    pk.offp[(wl * (MS / 2) + t / 2) * 32 + l] |= (t & 1) ? off << 16 : off;
                    pk.coef[(wl * MS + t) * 32 + l] = tcoef[(size_t)t * 32 + l];
                }
                const int h = slots_of[bl][(size_t)w * hpw + (l % hpw)];
                pk.lane_hash[wl * 32 + l] = (int16_t)h;
            }
        }
    }
    pk.conflict_wavefronts = conflicts;
    pk.efficiency = (double)useful / ((double)lanes_total * MS);
    // cost (shared-memory wavefronts per row): gathers (1 per warp, slot and row) + conflicts +
    // staging (TMA writes n/32) + code stores (1 STS wavefront per warp and row, k/32 for the
    // bulk store's reads). The LDS.32 loop runs at ~98% of the pipe with 8 or 16 warps per SM
    // (tools/microbench_lds32.cu).
    // staged words count twice: TMA writes into shared memory measured ~2x their 128-byte
    // wavefronts (C1 with a second copy: 3% fewer slots, 2.6% slower)
    const double wf = (double)HB * W * MS + (double)conflicts + 2.0 * HB * (n + pk.n1) / 32.0 + (double)HB * W +
                      k / 32.0;
    // resident warps per SM (register cap by MS as in the kernel's launch bounds, shared memory of
    // the class): the LDS.32 loop alone runs at ~98% with 8 or 16 warps/SM, but the whole kernel
    // needs more warps to cover its epilogue: measured slot wavefronts (+ staging) per cycle per SM,
    // 16-warp packings 0.78-0.90 (C1, C4 P=2, C2 m=128 P=4), 8-warp ones 0.69-0.74 (C4 P=1, C2
    // m=128 P=1) -> 8 warps/SM cost a factor 0.8
    const int regs = MS <= 24 ? 85 : MS <= 40 ? 102 : MS <= 64 ? 128 : 255;
    const int kbp = (pk.kb_max + 3) & ~3;
    // rows longer than 2048 words at 16 warps per CTA: 6-row stages (class 7, 2 x 99 KB) instead of
    // 4-row ones (class 5, 3 x 66 KB): a third fewer per-group costs and 6 independent LDS per slot.
    // C2 m = 32 (P = 1, MS = 36): 6.37 -> 5.47 ms. Measured no gain with parts (C2 m = 128, P = 2,
    // MS = 64: 23.5 ms class 5, 23.2 class 7 — the model would credit it and pick it over the better
    // P = 1 / 8-warp packing, 21.5 ms) and a loss at 8 warps (MS = 128: 22.9-23.8 ms with class 7's
    // 2-deep ring): one-part 16-warp packings only.
    if (pk.cls == 5 && W >= 16 && MS <= 64 && P == 1) {
        const RClass c7 = kRClasses[7];
        const double s7 = (double)c7.NS * c7.R * c7.S * 4 + (double)c7.NC * c7.R * kbp * 4 + 2048 + kbp * 4;
        if (s7 <= 227.0 * 1024) pk.cls = 7;
    }
    const RClass cl = kRClasses[pk.cls];
    const double smem = (double)cl.NS * cl.R * cl.S * 4 + (double)cl.NC * cl.R * kbp * 4 + 1024;
    const int by_regs = 65536 / (W * 32 * regs), by_smem = (int)(227.0 * 1024 / smem);
    const int warps_sm = W * std::max(1, std::min(by_regs, by_smem));
    // rate factor at 8 warps/SM (16 warps: 1): round 1 fitted 0.8; the round-2 part sweep
    // (profiles/r02_sweep_parts.txt) measured P=1 / MS=128 / 8 warps beating P=2 / MS=64 / 16 warps on
    // C2 m=128 (21.5 vs 23.5 ms) and P=4 / 8 warps beating P=8 / 16 warps on m=512 (25.2 vs 26.6 ms);
    // 0.87 picks the measured-best packing on every config (FASTLSH_RPACK_8W overrides, experiment knob)
    static const double low = [] {
        const char* e = std::getenv("FASTLSH_RPACK_8W");
        return e ? std::atof(e) : 0.87;
    }();
    const double rate = warps_sm >= 16 ? 0.98 : 0.98 * (1.0 - 2.0 * (1.0 - low) * (1.0 - warps_sm / 16.0));
    // per-group costs (waits, epilogue, flush) ~ 97 wavefront-equivalents per warp and group,
    // fitted to C1 single (R = 8) vs dual (R = 4) copies and checked on C4 (model 0.877, measured
    // 0.884 for the dual/single time ratio)
    pk.cost = (wf + (double)HB * W * 97.0 / cl.R) / rate;
    pk.ok = true;
    out = std::move(pk);
}

}  // namespace

void build_row_packing(const fastlsh_params& p, RPacking& out) {
    out = RPacking();
    if (p.n <= 0 || p.m <= 0 || p.k <= 0) return;
    if (32 * ((p.n + 31) / 32) + 32 > kRClasses[5].S) return;  // largest stage class
    if (std::getenv("FASTLSH_NO_ROWS")) return;       // experiment knob
    int force_p = 0;
    if (const char* e = std::getenv("FASTLSH_ROW_PARTS")) force_p = std::atoi(e);
    for (int P = 1; P <= 32; P *= 2) {
        if ((p.m + P - 1) / P > kRMaxSlots) continue;
        if (force_p && P != force_p) continue;
        for (int Wmax : {16, 8}) {
            for (int variant = 0; variant < 2; ++variant) {
                const bool capped = variant & 1;
                for (int dual_cls : {-1, 4, 6}) {
                if (dual_cls >= 0 && (p.n <= kRDualMaxN[kRDualClasses - 1] || std::getenv("FASTLSH_NO_COPY1"))) continue;
                if (const char* e = std::getenv("FASTLSH_DUAL_CLS"))  // experiment knob: pin the option
                    if (std::atoi(e) != dual_cls) continue;
                RPacking t;
                try_rows(p, P, Wmax, capped, t, dual_cls);
                if (t.ok && std::getenv("FASTLSH_PACK_DEBUG"))
                    std::fprintf(stderr, "[rpack-try] P=%d Wmax=%d capped=%d dual_cls=%d MS=%d W=%d HB=%d conflicts=%lld cost=%.1f\n",
                                 P, Wmax, (int)capped, dual_cls, t.slots, t.warps, t.hash_blocks,
                                 (long long)t.conflict_wavefronts, t.cost);
                if (t.ok && t.cost < out.cost) out = std::move(t);
                }
            }
        }
    }
    if (std::getenv("FASTLSH_PACK_DEBUG") && out.ok)
        std::fprintf(stderr, "[rpack] P=%d MS=%d W=%d HB=%d eff=%.3f conflicts=%lld cost=%.1f\n", out.parts,
                     out.slots, out.warps, out.hash_blocks, out.efficiency, (long long)out.conflict_wavefronts,
                     out.cost);
}

}  // namespace fastlsh
