// gather.cu — K1/K2: FastLSH sampled-projection hashing on sm_100a.
//
// For every row v and hash i: h_i(v) = floor((a_i . S_i(v) + b_i) / w)   (Eq. 5).
//
// Design: a persistent kernel, one CTA per (hash block, row stream).
//  * Each lane holds its hash part's slots in registers for the whole kernel: MS 32-bit smem
//    byte offsets and MS f32 coefficients, in the bank-scheduled order of packer.cpp.
//  * Rows are processed 4*RG at a time ("groups"). A stage is RG sub-stages of 4 rows, each
//    column-interleaved: the 16-byte chunk at pos(c) = (c%4)*nq + c/4 is (x0[c],..,x3[c]). One
//    LDS.128 per slot and sub-stage gathers the sampled coordinate of 4 rows; one FFMA per row
//    accumulates it. The packer guarantees the 8 lanes of each quarter-warp hit 8 distinct bank
//    groups at every slot, so each LDS.128 costs the ideal 4 wavefronts (32 gathers/wavefront).
//  * Staging: TMA bulk copies (cp.async.bulk ... complete_tx) bring each group's rows from HBM
//    into a row-major 2-slot landing ring with 128-bit transfers; the CTA's warps transpose
//    landing -> stage with conflict-free LDS.128 / STS.32. (Rows that are not 16-B aligned, or
//    too long for the landing ring, fall back to 4-byte cp.async into the transposed positions.)
//  * Pipeline without CTA barriers (mbarriers only, one iteration of slack): at iteration j every
//    thread transposes its share of group j+2, gathers group j, publishes its partials for j, and
//    finishes group j-1 (epilogue); thread 0 re-arms the landing slot freed by group j+2 with the
//    TMA copies of group j+4.
//  * Epilogue (fused): each thread takes a hash, sums its parts in fixed order for each row,
//    adds b (__fadd_rn), divides by w (__fdiv_rn; an exact multiply when w is a power of two),
//    floors toward -inf and writes int32 codes (coalesced over hashes).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <cstdlib>

#include "internal.h"

#include "gather_impl.cuh"

namespace fastlsh {
namespace k1 {

KernelFn select_kernel(int MS, int shape, bool fused) {
    if (MS < 2 || MS > 64 || (MS & 1)) return nullptr;
    switch ((MS - 2) / 16) {
        case 0: return kernel_for_ms_0(MS, shape, fused);
        case 1: return kernel_for_ms_1(MS, shape, fused);
        case 2: return kernel_for_ms_2(MS, shape, fused);
        default: return kernel_for_ms_3(MS, shape, fused);
    }
}

size_t smem_bytes(const Packing& pk, int shape, int tma, int landing_row, int keys_words) {
    const int rg = kShapes[shape].rg, ns = kShapes[shape].ns, nl = kShapes[shape].nl;
    return (size_t)ns * rg * pk.stage_chunks * 16 + (size_t)kPartSlots * rg * pk.warps * 32 * 16 +
           (tma ? (size_t)nl * 4 * rg * landing_row : 0) + (size_t)kBars * 8 +
           (size_t)(((pk.kb_max * pk.parts + 3) & ~3) * 2) + (size_t)((pk.kb_max + 1) & ~1) * 4 +
           (keys_words ? (size_t)2 * 4 * rg * pk.kb_max * 4 + (size_t)keys_words * 8 : 0);
}

int rows_per_group_override() {
    static const int v = [] {
        const char* e = std::getenv("FASTLSH_SHAPE");  // experiment knob: 1-based kShapes index
        return e ? std::atoi(e) : 0;
    }();
    return v;
}


}  // namespace k1

using namespace k1;

fastlsh_status launch_gather(const fastlsh_params* p, const DeviceCopy& d, const float* X,
                             int64_t N, int32_t* codes, float* proj, cudaStream_t stream,
                             const FusedKeys* fk) {
    const Packing& pk = p->pack;
    if (!d.offp) return FASTLSH_EUNSUPPORTED;  // packing skipped at upload (dense-path shape)
    const int landing_row = ((4 * p->n + 15) / 16) * 16;
    int tma = (p->n % 4 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
    const int fused = (fk && fk->keys) ? 1 : 0;  // codes may be null: keys only
    const int tables_max = fused ? pk.kb_max / fk->K + 1 : 0;
    const int keys_words = fused ? tables_max * (fk->K + 1) : 0;
    // Pipeline shape: among the shapes whose shared memory fits (with the TMA landing ring when
    // the rows allow TMA), the one with the most resident warps per SM up to 16 (measured: the
    // gather loop saturates the shared-memory pipe at 16 warps/SM, ~75% at 8), earlier (deeper,
    // larger) shapes on ties. Cached per device copy, TMA mode and fused-keys mode.
    constexpr size_t kSmemMax = 227 * 1024;
    const int threads = pk.warps * 32;
    int& cache = d.shape_cache[tma + 2 * fused];
    int enc = cache;  // shape + 16 * (uses TMA), -1 = not chosen yet
    if (enc < 0) {
        int best_score = -1;
        for (int pass = 0; pass < 2 && enc < 0; ++pass) {
            const int t = pass == 0 ? tma : 0;  // pass 1: no room for a landing ring -> cp.async
            if (pass == 1 && !tma) break;
            for (int s = 0; s < kNumShapes; ++s) {
                const size_t sm = smem_bytes(pk, s, t, landing_row, keys_words);
                if (sm > kSmemMax) continue;
                KernelFn f = select_kernel(pk.slots, s, fused);
                if (!f) return FASTLSH_EUNSUPPORTED;
                int occ = 0;
                cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(f),
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                if (e == cudaSuccess)
                    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, reinterpret_cast<const void*>(f), threads, sm);
                if (e != cudaSuccess) return set_cuda_error(e);
                const int score = occ * pk.warps < 16 ? occ * pk.warps : 16;
                if (occ > 0 && score > best_score) {
                    best_score = score;
                    enc = s + 16 * t;
                }
            }
        }
        if (enc < 0) return FASTLSH_EUNSUPPORTED;
        cache = enc;
    }
    int shape = enc % 16;
    tma = enc / 16;
    if (int o = rows_per_group_override()) {  // experiment knob: FASTLSH_SHAPE = 1..kNumShapes
        const int forced = (o >= 1 && o <= kNumShapes) ? o - 1 : 1;
        if (smem_bytes(pk, forced, tma, landing_row, keys_words) <= kSmemMax) shape = forced;
    }
    const int rg = kShapes[shape].rg;
    KernelFn fn = select_kernel(pk.slots, shape, fused);
    if (!fn) return FASTLSH_EUNSUPPORTED;
    GatherArgs a;
    a.X = X;
    a.N = N;
    a.n = p->n;
    a.nq = pk.nq;
    a.stage_chunks = pk.stage_chunks;
    a.offp = d.offp;
    a.coef = d.coef;
    a.unit_lane = d.unit_lane;
    a.b = d.b;
    a.block_h0 = d.block_h0;
    a.block_kb = d.block_kb;
    a.w = p->w;
    a.k = p->k;
    a.P = pk.parts;
    a.direct = (pk.direct && !fused) ? 1 : 0;
    a.W = pk.warps;
    a.HB = pk.hash_blocks;
    a.kb_max = pk.kb_max;
    a.groups = (N + 4 * rg - 1) / (4 * rg);
    a.codes = codes;
    a.proj = proj;
    a.flags = d.flags;
    a.tma = tma;
    a.landing_row = landing_row;
    a.kr = fused ? fk->r : nullptr;
    a.L = fused ? fk->L : 0;
    a.K = fused ? fk->K : 1;
    a.tables_max = tables_max;
    a.keys = fused ? fk->keys : nullptr;
    a.ldk = fused ? fk->ldk : 0;

    const size_t smem = smem_bytes(pk, shape, tma, landing_row, keys_words);
    if (fastlsh_status so = smem_optin_once(reinterpret_cast<const void*>(fn)); so != FASTLSH_OK) return so;
    cudaError_t e = cudaSuccess;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(fn), threads, smem);
    if (e != cudaSuccess) return set_cuda_error(e);
    if (per_sm < 1) return FASTLSH_EUNSUPPORTED;
    // persistent grid: as many row streams per hash block as fit resident at once
    const long long resident = (long long)sms * per_sm;
    long long gpr = resident / pk.hash_blocks;
    if (gpr > a.groups) gpr = a.groups;
    if (gpr < 1) gpr = 1;
    const long long grid = gpr * pk.hash_blocks;
    fn<<<(unsigned)grid, threads, smem, stream>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e);
    return FASTLSH_OK;
}

bool keys_fusable(const fastlsh_params* p, const fastlsh_keys* ks) {
    if (!p->packed || p->pack.slots <= 0 || p->table_align != ks->K || (int64_t)ks->L * ks->K > p->k) return false;
    const Packing& pk = p->pack;
    for (int bl = 0; bl < pk.hash_blocks; ++bl) {
        if (pk.block_h0[bl] % ks->K) return false;
        const int end = pk.block_h0[bl] + pk.block_kb[bl];
        if (end % ks->K && end < ks->L * ks->K) return false;  // a table split across blocks
    }
    return true;
}

}  // namespace fastlsh
