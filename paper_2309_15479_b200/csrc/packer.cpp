// packer.cpp — offline bank scheduling of the sampled slots.
//
// Addition commutes, so the order in which a hash's m products are accumulated is free
// (Eq. 5 fixes the value, not the order). The packer uses that freedom so that the
// gather kernel's shared-memory loads are conflict-free:
//
//  1. Each hash's m slots (in paper order) are split into `parts` contiguous lane units.
//  2. The units of a CTA hash block are grouped 8 at a time into quarter-warps. One LDS.128
//     wavefront serves 8 lanes; two lanes conflict when their 16-B chunk positions differ but
//     fall in the same bank group (pos mod 8). Grouping balances the per-class load of each
//     quarter (greedy, then swap local search).
//  3. Each quarter's bipartite multigraph (lanes x 8 bank groups, one edge per slot) is edge
//     coloured with Delta colours by König's alternating-path method; a colour is a slot
//     position at which every lane and every bank group is used at most once.
//  4. Free (lane, position) pairs become padding slots: coefficient 0 reading a zero chunk of a
//     bank group unused at that position.
//  5. Lane positions inside a quarter are free for the schedule; they are chosen (König colouring
//     of quarters x (hash octet, part)) so that the epilogue's partial-sum reads are conflict-free.
//  Between 2 and 3, single slots move between the parts of a hash (the split into parts is free
//  too) to flatten each quarter's bank-group loads towards m/parts; each parts choice is then
//  costed with the padded slot count and with slots capped at the (even) part size, folding the
//  few remaining colours into conflicts.
//
// Everything is deterministic, so every rank derives the identical packing (and hence the
// identical fp32 summation order) from the same params.
#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "internal.h"

namespace fastlsh {
namespace {

struct Edge {
    int lane;   // lane within quarter
    int cls;    // bank group (pos mod 8)
    int pos;    // chunk position
    float coef;
    int color = -1;
};

struct Unit {
    int hash, part;
    std::vector<std::pair<int, float>> slots;  // (pos, coef)
    std::array<int, 8> cnt{};
    int deg = 0;
};

inline int chunk_pos(int c, int nq) { return (c & 3) * nq + (c >> 2); }

struct QuarterState {
    std::vector<int> members;  // unit ids
    std::array<int, 8> load{};
    int maxload() const { return *std::max_element(load.begin(), load.end()); }
    long sumsq() const {
        long s = 0;
        for (int v : load) s += (long)v * v;
        return s;
    }
};

// Group the units of one block into Q quarters of <= 8 lanes with balanced class loads.
std::vector<QuarterState> group_units(const std::vector<Unit>& units, int Q, int dmax) {
    std::vector<QuarterState> qs(Q);
    std::vector<int> order(units.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        int ma = *std::max_element(units[a].cnt.begin(), units[a].cnt.end());
        int mb = *std::max_element(units[b].cnt.begin(), units[b].cnt.end());
        return ma > mb;
    });
    // even fill: quarter capacity is ceil(U / Q) (<= 8) so empty lanes are spread out
    const int cap = std::min<int>(8, (int)((units.size() + Q - 1) / Q));
    for (int u : order) {
        int best = -1;
        long best_key0 = 0, best_key1 = 0;
        for (int q = 0; q < Q; ++q) {
            if ((int)qs[q].members.size() >= cap) continue;
            int ml = 0;
            long ss = 0;
            for (int c = 0; c < 8; ++c) {
                int v = qs[q].load[c] + units[u].cnt[c];
                ml = std::max(ml, v);
                ss += (long)v * v;
            }
            long k0 = ml, k1 = ss * 16 + (long)qs[q].members.size();
            if (best < 0 || k0 < best_key0 || (k0 == best_key0 && k1 < best_key1)) {
                best = q; best_key0 = k0; best_key1 = k1;
            }
        }
        qs[best].members.push_back(u);
        for (int c = 0; c < 8; ++c) qs[best].load[c] += units[u].cnt[c];
    }
    // local search on the excess over a target T: F = sum_q sum_c max(0, load - T)^2.
    // Start at T = dmax (perfect balance); if no swap/move lowers F any more, relax T by one.
    auto excess = [](const std::array<int, 8>& l, int T) {
        long e = 0;
        for (int v : l) if (v > T) e += (long)(v - T) * (v - T);
        return e;
    };
    int T = dmax;
    for (int guard = 0; guard < 64; ++guard, ++T) {
        bool any_excess = false;
        for (int sweep = 0; sweep < 24; ++sweep) {
            bool improved = false;
            any_excess = false;
            for (int q = 0; q < Q; ++q) {
                const long eq = excess(qs[q].load, T);
                if (eq == 0) continue;
                any_excess = true;
                long best = 0;
                int bi = -1, bq = -1, bj = -1;
                const auto& A = qs[q];
                for (int ii = 0; ii < (int)A.members.size(); ++ii) {
                    const Unit& u = units[A.members[ii]];
                    for (int q2 = 0; q2 < Q; ++q2) {
                        if (q2 == q) continue;
                        const auto& B = qs[q2];
                        const int n2 = (int)B.members.size();
                        const long e2 = excess(B.load, T);
                        for (int jj = -1; jj < n2; ++jj) {
                            if (jj < 0 && n2 >= 8) continue;
                            std::array<int, 8> a = A.load, b = B.load;
                            for (int c = 0; c < 8; ++c) { a[c] -= u.cnt[c]; b[c] += u.cnt[c]; }
                            if (jj >= 0) {
                                const Unit& v = units[B.members[jj]];
                                for (int c = 0; c < 8; ++c) { a[c] += v.cnt[c]; b[c] -= v.cnt[c]; }
                            }
                            const long d = excess(a, T) + excess(b, T) - eq - e2;
                            if (d < best) { best = d; bi = ii; bq = q2; bj = jj; }
                        }
                    }
                }
                if (bi < 0) continue;
                improved = true;
                auto& Am = qs[q];
                auto& Bm = qs[bq];
                const int u = Am.members[bi];
                for (int c = 0; c < 8; ++c) { Am.load[c] -= units[u].cnt[c]; Bm.load[c] += units[u].cnt[c]; }
                if (bj >= 0) {
                    const int v = Bm.members[bj];
                    for (int c = 0; c < 8; ++c) { Am.load[c] += units[v].cnt[c]; Bm.load[c] -= units[v].cnt[c]; }
                    Am.members[bi] = v;
                    Bm.members[bj] = u;
                } else {
                    Am.members.erase(Am.members.begin() + bi);
                    Bm.members.push_back(u);
                }
            }
            if (!any_excess || !improved) break;
        }
        if (!any_excess) break;
    }
    return qs;
}

// König edge colouring of a bipartite multigraph (lanes x 8 classes) with `ncol` colours,
// ncol >= max degree. Returns false if some edge could not be coloured (never for a valid ncol).
bool color_quarter(std::vector<Edge>& edges, int nlanes, int ncol) {
    std::vector<int> lane_col((size_t)nlanes * ncol, -1), cls_col((size_t)8 * ncol, -1);
    auto L = [&](int l, int t) -> int& { return lane_col[(size_t)l * ncol + t]; };
    auto C = [&](int c, int t) -> int& { return cls_col[(size_t)c * ncol + t]; };
    for (int e = 0; e < (int)edges.size(); ++e) {
        const int l = edges[e].lane, c = edges[e].cls;
        int alpha = -1, beta = -1;
        for (int t = 0; t < ncol && alpha < 0; ++t) if (L(l, t) < 0) alpha = t;
        for (int t = 0; t < ncol && beta < 0; ++t) if (C(c, t) < 0) beta = t;
        if (alpha < 0 || beta < 0) return false;
        if (C(c, alpha) >= 0) {
            // flip the alpha/beta alternating path that starts at class c
            std::vector<int> path;
            bool at_class = true;
            int v = c, col = alpha;
            for (;;) {
                int e2 = at_class ? C(v, col) : L(v, col);
                if (e2 < 0) break;
                path.push_back(e2);
                v = at_class ? edges[e2].lane : edges[e2].cls;
                at_class = !at_class;
                col = (col == alpha) ? beta : alpha;
            }
            for (int e2 : path) {
                L(edges[e2].lane, edges[e2].color) = -1;
                C(edges[e2].cls, edges[e2].color) = -1;
            }
            for (int e2 : path) {
                edges[e2].color = (edges[e2].color == alpha) ? beta : alpha;
                L(edges[e2].lane, edges[e2].color) = e2;
                C(edges[e2].cls, edges[e2].color) = e2;
            }
        }
        edges[e].color = alpha;
        L(l, alpha) = e;
        C(c, alpha) = e;
    }
    return true;
}

}  // namespace

// König edge colouring of a general bipartite multigraph (left x right nodes) with ncol >= max
// degree colours. Edge e joins left[e] and right[e]; returns the colour of every edge (-1 = failed).
std::vector<int> color_bipartite(const std::vector<int>& left, const std::vector<int>& right, int nleft,
                                 int nright, int ncol) {
    const int E = (int)left.size();
    std::vector<int> col(E, -1), lc((size_t)nleft * ncol, -1), rc((size_t)nright * ncol, -1);
    auto Lc = [&](int v, int t) -> int& { return lc[(size_t)v * ncol + t]; };
    auto Rc = [&](int v, int t) -> int& { return rc[(size_t)v * ncol + t]; };
    for (int e = 0; e < E; ++e) {
        const int l = left[e], r = right[e];
        int alpha = -1, beta = -1;
        for (int t = 0; t < ncol && alpha < 0; ++t) if (Lc(l, t) < 0) alpha = t;
        for (int t = 0; t < ncol && beta < 0; ++t) if (Rc(r, t) < 0) beta = t;
        if (alpha < 0 || beta < 0) return std::vector<int>(E, -1);
        if (Rc(r, alpha) >= 0) {  // flip the alpha/beta alternating path starting at r
            std::vector<int> path;
            bool at_right = true;
            int v = r, c = alpha;
            for (;;) {
                const int e2 = at_right ? Rc(v, c) : Lc(v, c);
                if (e2 < 0) break;
                path.push_back(e2);
                v = at_right ? left[e2] : right[e2];
                at_right = !at_right;
                c = (c == alpha) ? beta : alpha;
            }
            for (int e2 : path) { Lc(left[e2], col[e2]) = -1; Rc(right[e2], col[e2]) = -1; }
            for (int e2 : path) {
                col[e2] = (col[e2] == alpha) ? beta : alpha;
                Lc(left[e2], col[e2]) = e2;
                Rc(right[e2], col[e2]) = e2;
            }
        }
        col[e] = alpha;
        Lc(l, alpha) = e;
        Rc(r, alpha) = e;
    }
    return col;
}

namespace {

// Slot exchange between the parts of a hash (P >= 2): which of a hash's slots go to which part is
// free (addition commutes), so single slots are swapped between partner units in different
// quarters when that lowers F = sum over (quarter, bank group) of max(0, load - T)^2 with T = the
// part size (strict descent). Unit sizes do not change.
void exchange_slots(std::vector<Unit>& units, std::vector<QuarterState>& qs, int P, int T) {
    if (P < 2) return;
    std::vector<int> uq(units.size(), -1);
    for (int q = 0; q < (int)qs.size(); ++q)
        for (int u : qs[q].members) uq[u] = q;
    auto e2 = [T](int v) { return v > T ? (v - T) * (v - T) : 0; };
    for (int sweep = 0; sweep < 200; ++sweep) {
        bool improved = false;
        for (int q = 0; q < (int)qs.size(); ++q) {
            for (int g = 0; g < 8; ++g) {
                while (qs[q].load[g] > T) {
                    int best = 0, bu = -1, bu2 = -1, bg2 = -1;
                    for (int u : qs[q].members) {
                        if (units[u].cnt[g] == 0) continue;
                        const int base = u - units[u].part;  // units of a hash are consecutive
                        for (int pp = 0; pp < P; ++pp) {
                            const int u2 = base + pp;
                            const int q2 = uq[u2];
                            if (u2 == u || q2 < 0 || q2 == q) continue;
                            for (int g2 = 0; g2 < 8; ++g2) {
                                if (g2 == g || units[u2].cnt[g2] == 0) continue;
                                const auto& A = qs[q].load;
                                const auto& B = qs[q2].load;
                                const int d = e2(A[g] - 1) - e2(A[g]) + e2(A[g2] + 1) - e2(A[g2]) +
                                              e2(B[g] + 1) - e2(B[g]) + e2(B[g2] - 1) - e2(B[g2]);
                                if (d < best) { best = d; bu = u; bu2 = u2; bg2 = g2; }
                            }
                        }
                    }
                    if (bu < 0) break;
                    const int q2 = uq[bu2];
                    auto& sa = units[bu].slots;
                    auto& sb = units[bu2].slots;
                    int ia = -1, ib = -1;
                    for (int i = 0; i < (int)sa.size() && ia < 0; ++i) if ((sa[i].first & 7) == g) ia = i;
                    for (int i = 0; i < (int)sb.size() && ib < 0; ++i) if ((sb[i].first & 7) == bg2) ib = i;
                    std::swap(sa[ia], sb[ib]);
                    units[bu].cnt[g]--; units[bu].cnt[bg2]++;
                    units[bu2].cnt[bg2]--; units[bu2].cnt[g]++;
                    qs[q].load[g]--; qs[q].load[bg2]++;
                    qs[q2].load[bg2]--; qs[q2].load[g]++;
                    improved = true;
                }
            }
        }
        if (!improved) break;
    }
}

struct Trial {
    Packing pk;
    double cost = 1e300;
};

void try_parts(const fastlsh_params& p, int P, int lanes_cap, Trial& out, int ms_cap, bool direct = false) {
    direct = direct && P == 1;
    const int n = p.n, m = p.m, k = p.k;
    Packing pk;
    pk.parts = P;
    pk.nq = (n + 3) / 4;
    pk.stage_chunks = 4 * pk.nq + kPadChunks;
    const int dmax = (m + P - 1) / P;
    const int kb_cap = std::max(1, lanes_cap / P);
    // Hash blocks: k hashes split as evenly as possible into HB CTA blocks; with a table size T
    // (fastlsh_params_set_table_size) blocks hold whole tables of T consecutive hashes (the hashes
    // past the last whole table go to the last block), so keys can be built inside the kernel.
    const int T = (p.table_align > 1 && p.table_align <= kb_cap) ? p.table_align : 1;
    const int units = k / T, rem = k % T;
    int HB = (k + kb_cap - 1) / kb_cap;
    while (((units + HB - 1) / HB) * T + rem > kb_cap) ++HB;
    if (units > 0 && HB > units) HB = units;
    pk.hash_blocks = HB;
    pk.block_h0.resize(HB);
    pk.block_kb.resize(HB);
    int h0 = 0;
    for (int bl = 0; bl < HB; ++bl) {
        pk.block_kb[bl] = (units / HB + (bl < units % HB ? 1 : 0)) * T + (bl == HB - 1 ? rem : 0);
        pk.block_h0[bl] = h0;
        h0 += pk.block_kb[bl];
    }
    pk.kb_max = *std::max_element(pk.block_kb.begin(), pk.block_kb.end());
    pk.warps = (pk.kb_max * P + 31) / 32;
    const int Wn = pk.warps, Q = 4 * Wn;

    struct QuarterPlan {
        std::vector<int> members;
        std::vector<Edge> edges;
        int delta;
    };
    std::vector<std::vector<QuarterPlan>> plans(HB);
    std::vector<std::vector<Unit>> block_units(HB);
    int MS = 2;
    for (int bl = 0; bl < HB; ++bl) {
        auto& units = block_units[bl];
        for (int hh = 0; hh < pk.block_kb[bl]; ++hh) {
            const int h = pk.block_h0[bl] + hh;
            for (int q = 0; q < P; ++q) {
                Unit u;
                u.hash = hh;
                u.part = q;
                const int j0 = (int)((long)q * m / P), j1 = (int)((long)(q + 1) * m / P);
                for (int j = j0; j < j1; ++j) {
                    int pos = chunk_pos(p.idx[(size_t)h * m + j], pk.nq);
                    u.slots.push_back({pos, p.a[(size_t)h * m + j]});
                    u.cnt[pos & 7]++;
                }
                u.deg = j1 - j0;
                units.push_back(std::move(u));
            }
        }
        std::vector<QuarterState> qs;
        if (direct) {  // quarters of warp w take units (= hashes, P = 1) [32w, 32w+32) only
            qs.resize(Q);
            for (int w = 0; w < Wn; ++w) {
                const int u0 = 32 * w, u1 = std::min<int>((int)units.size(), u0 + 32);
                if (u0 >= u1) continue;
                std::vector<Unit> sub(units.begin() + u0, units.begin() + u1);
                auto sq = group_units(sub, 4, dmax);
                for (int qi = 0; qi < 4; ++qi) {
                    for (int& mbr : sq[qi].members) mbr += u0;
                    qs[4 * w + qi] = std::move(sq[qi]);
                }
            }
        } else {
            qs = group_units(units, Q, dmax);
            if (P <= 4) exchange_slots(units, qs, P, dmax);  // matters (and is cheap) for few parts
        }
        plans[bl].resize(Q);
        for (int q = 0; q < Q; ++q) {
            auto& qp = plans[bl][q];
            qp.members = qs[q].members;
            int d = 0;
            for (int li = 0; li < (int)qp.members.size(); ++li) {
                const Unit& u = units[qp.members[li]];
                d = std::max(d, u.deg);
                for (auto& s : u.slots) qp.edges.push_back(Edge{li, s.first & 7, s.first, s.second});
            }
            d = std::max(d, qs[q].maxload());
            qp.delta = d;
            if (!color_quarter(qp.edges, std::max<int>(1, qp.members.size()), std::max(1, d))) {
                qp.delta = -1;  // cannot happen for a valid Delta
            }
            MS = std::max(MS, d);
        }
    }
    if (std::getenv("FASTLSH_PACK_DEBUG")) {
        std::vector<int> hist(4 * kMaxSlots + 8, 0);
        for (int bl = 0; bl < HB; ++bl)
            for (auto& qp : plans[bl]) hist[std::min<int>(qp.delta, hist.size() - 1)]++;
        std::fprintf(stderr, "[pack] P=%d dmax=%d HB=%d W=%d delta histogram:", P, dmax, HB, Wn);
        for (size_t d = 0; d < hist.size(); ++d) if (hist[d]) std::fprintf(stderr, " %zu:%d", d, hist[d]);
        std::fprintf(stderr, "\n");
    }
    // fold colours beyond kMaxSlots into existing positions (creates bank conflicts)
    int64_t conflicts = 0;
    if (MS > kMaxSlots) MS = kMaxSlots;
    MS = (MS + 1) & ~1;  // the gather loop issues slots in pairs
    // ms_cap > 0: fold colours beyond the cap into existing positions (a few bank conflicts instead
    // of padding slots every lane pays); the cost model below compares both choices
    if (ms_cap < 0) ms_cap = (dmax + 1) & ~1;  // the even part size
    if (ms_cap > 0 && (ms_cap & ~1) >= dmax && (ms_cap & ~1) < MS) MS = ms_cap & ~1;
    if (const char* e = std::getenv("FASTLSH_MS_CAP")) {  // experiment knob: force a cap
        const int cap = std::atoi(e) & ~1;
        if (cap >= dmax && cap < MS) MS = cap;
    }
    pk.slots = MS;

    // Lane positions inside each quarter are free for the gather schedule (it is per lane). Choose
    // them so that the epilogue, which reads the partials of 8 consecutive hashes per quarter-warp
    // (one part at a time), hits 8 distinct bank groups: edge-colour the bipartite multigraph
    // quarters x (hash octet, part) with 8 colours (degrees <= 8, König) and use the colour as the
    // position. perm[bl][q][li] = position of member li (free lanes take the unused positions).
    std::vector<std::vector<std::array<int, 8>>> perm(HB, std::vector<std::array<int, 8>>(Q));
    for (int bl = 0; bl < HB; ++bl) {
        const auto& units = block_units[bl];
        std::vector<int> le, ri;
        const int octs = (pk.block_kb[bl] + 7) / 8;
        for (int q = 0; q < Q; ++q)
            for (int li : plans[bl][q].members) {
                le.push_back(q);
                ri.push_back((units[li].hash / 8) * P + units[li].part);
            }
        std::vector<int> col = color_bipartite(le, ri, Q, std::max(1, octs * P), 8);
        size_t e = 0;
        for (int q = 0; q < Q; ++q) {
            std::array<int, 8>& pm = perm[bl][q];
            bool used[8] = {false, false, false, false, false, false, false, false};
            const int nm = (int)plans[bl][q].members.size();
            bool ok = true;
            for (int li = 0; li < nm; ++li, ++e) {
                pm[li] = col[e];
                if (col[e] < 0 || used[col[e]]) ok = false;
                else used[col[e]] = true;
            }
            if (!ok) {  // cannot happen (König); keep the identity order
                for (int li = 0; li < 8; ++li) pm[li] = li;
                continue;
            }
            int nxt = 0;
            for (int li = nm; li < 8; ++li) {
                while (used[nxt]) ++nxt;
                pm[li] = nxt;
                used[nxt] = true;
            }
        }
    }

    const size_t lanes_total = (size_t)HB * Wn * 32;
    pk.offp.assign(lanes_total * MS, 0);
    pk.coef.assign(lanes_total * MS, 0.0f);
    pk.unit_lane.assign((size_t)HB * pk.kb_max * P, 0);
    int64_t useful = 0;
    for (int bl = 0; bl < HB; ++bl) {
        const auto& units = block_units[bl];
        for (int q = 0; q < Q; ++q) {
            auto& qp = plans[bl][q];
            const int w = q / 4, qi = q % 4;
            // slot table: pos[t][lane], coef[t][lane], -1 = free
            std::vector<int> tpos((size_t)MS * 8, -1);
            std::vector<float> tcoef((size_t)MS * 8, 0.0f);
            std::vector<int> used_cls((size_t)MS * 8, 0);  // #lanes per (t, class)
            std::vector<Edge*> overflow;
            for (auto& e : qp.edges) {
                if (e.color >= 0 && e.color < MS) {
                    tpos[(size_t)e.color * 8 + e.lane] = e.pos;
                    tcoef[(size_t)e.color * 8 + e.lane] = e.coef;
                    used_cls[(size_t)e.color * 8 + e.cls]++;
                } else {
                    overflow.push_back(&e);
                }
            }
            for (Edge* e : overflow) {
                int bt = -1, bu = 1 << 30;
                for (int t = 0; t < MS; ++t) {
                    if (tpos[(size_t)t * 8 + e->lane] >= 0) continue;
                    int u = used_cls[(size_t)t * 8 + e->cls];
                    if (u < bu) { bu = u; bt = t; }
                }
                tpos[(size_t)bt * 8 + e->lane] = e->pos;
                tcoef[(size_t)bt * 8 + e->lane] = e->coef;
                used_cls[(size_t)bt * 8 + e->cls]++;
            }
            for (int t = 0; t < MS; ++t) {
                int mx = 0;
                for (int c = 0; c < 8; ++c) mx = std::max(mx, used_cls[(size_t)t * 8 + c]);
                if (mx > 1) conflicts += mx - 1;
                // padding: every free lane reads the zero chunk of one unused bank group
                int freec = -1;
                for (int c = 0; c < 8 && freec < 0; ++c) if (used_cls[(size_t)t * 8 + c] == 0) freec = c;
                if (freec < 0) freec = 0;
                const int padpos = 4 * pk.nq + (((freec - 4 * pk.nq) % 8) + 8) % 8;
                for (int l = 0; l < 8; ++l) {
                    if (tpos[(size_t)t * 8 + l] < 0) { tpos[(size_t)t * 8 + l] = padpos; tcoef[(size_t)t * 8 + l] = 0.0f; }
                }
            }
            for (int l = 0; l < 8; ++l) {
                const int lane = qi * 8 + perm[bl][q][l];
                const size_t wl = ((size_t)bl * Wn + w);
                for (int t = 0; t < MS; ++t) {
                    const uint32_t off = (uint32_t)tpos[(size_t)t * 8 + l] * 16u;
                    pk.offp[(wl * MS + t) * 32 + lane] = off;
                    pk.coef[(wl * MS + t) * 32 + lane] = tcoef[(size_t)t * 8 + l];
                }
                if (l < (int)qp.members.size()) {
                    const Unit& u = units[qp.members[l]];
                    pk.unit_lane[((size_t)bl * pk.kb_max + u.hash) * P + u.part] = (uint16_t)(w * 32 + lane);
                    useful += u.deg;
                }
            }
        }
    }
    pk.conflict_wavefronts = conflicts;
    pk.efficiency = (double)useful / ((double)lanes_total * MS);
    // Cost model (shared-memory wavefronts per row / achievable pipe rate), from measurements on
    // B200 (tools/microbench_lds.cu): gather = one wavefront per LDS.128 per warp per slot per 4
    // rows -> HB*W*MS per row (+ scheduler conflicts); staging = landing read + transposed write of
    // the row per hash block -> HB*n/16; epilogue partial traffic ~ k*P/4. The pipe reaches ~98%
    // with 16 warps/SM (MS <= 32: <= 128 registers) but ~75% with 8 warps/SM (MS > 32).
    // The direct epilogue (P = 1) replaces the partial-sum traffic and item loop by one store per
    // lane and row.
    pk.direct = direct ? 1 : 0;
    const double epi = direct ? p.k / 16.0 : p.k * P / 4.0;
    const double wf = (double)HB * Wn * MS + (double)conflicts / 4.0 + (double)HB * p.n / 16.0 + epi;
    const double rate = MS <= 32 ? 0.98 : 0.75;
    out.cost = wf / rate;
    out.pk = std::move(pk);
}

}  // namespace

void build_packing(const fastlsh_params& p, Packing& out) {
    const int pmin = (p.m + kMaxSlots - 1) / kMaxSlots;
    int plo = pmin, phi = std::min(p.m, pmin + 2);
    // candidates: the fewest parts (<= 64 slots each), one or two more, and the split whose parts
    // of <= 28 slots usually schedule into MS <= 32 (16 warps per SM)
    const int p32 = std::min(p.m, (p.m + 27) / 28);
    std::vector<int> cands;
    for (int P = plo; P <= (pmin >= 16 ? plo : phi); ++P) cands.push_back(P);  // large m: fewer trials
    if (p32 > phi) cands.push_back(p32);
    int warps_force = 0;
    if (const char* e = std::getenv("FASTLSH_PARTS")) {  // experiment knob: force the split
        int v = std::atoi(e);
        if (v >= pmin && v <= p.m) cands.assign(1, v);
    }
    if (const char* e = std::getenv("FASTLSH_WARPS")) {  // experiment knob: warps per CTA
        int v = std::atoi(e);
        if (v >= 1 && v <= 16) warps_force = v;
    }
    const bool no_direct = std::getenv("FASTLSH_NO_DIRECT") != nullptr;  // experiment knob
    Trial best;
    for (int P : cands) {
        // beyond 256 lanes per hash the block holds a single hash; keep P <= 256
        if (P > 256) break;
        // 16 warps per CTA when the slots fit 128 registers per lane (MS <= 32), else 8
        for (int cap : {0, -1}) {  // padded slots, or slots capped at the part size with folding
            if (cap < 0 && P > 8) break;  // many parts: padding is already small
            for (int direct = 0; direct <= (P == 1 && !no_direct ? 1 : 0); ++direct) {
                Trial t;
                try_parts(p, P, (warps_force ? warps_force : 16) * 32, t, cap, direct);
                if (!warps_force && t.pk.slots > 32) {
                    t = Trial();
                    try_parts(p, P, 8 * 32, t, cap, direct);
                }
                if (t.cost < best.cost) best = std::move(t);
            }
        }
    }
    out = std::move(best.pk);
}

}  // namespace fastlsh
