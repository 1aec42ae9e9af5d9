// gather_rows.cu — launcher of K1r, the row-major FastLSH hashing kernel (gather_rows.cuh;
// DESIGN.md "K1r", Eq. 5).
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstdlib>

#include "internal.h"

#include "gather_rows.cuh"

namespace fastlsh {
namespace k1r {

RowKernelFn select_row_kernel(int MS, int cls) {
    typedef RowKernelFn (*UnitFn)(int, int);
    static const UnitFn units[] = {row_kernel_ms_0, row_kernel_ms_1, row_kernel_ms_2,
                                   row_kernel_ms_3, row_kernel_ms_4, row_kernel_ms_5};
    for (UnitFn u : units)
        if (RowKernelFn f = u(MS, cls)) return f;
    return nullptr;
}

// stages + NC code buffers + barriers + key multipliers + counters + b
size_t row_smem_bytes(const RPacking& pk, int key_words = 0) {
    const RClass c = kRClasses[pk.cls];
    const int kbp = (pk.kb_max + 3) & ~3;
    return (size_t)c.NS * c.R * c.S * 4 + (size_t)c.NC * c.R * kbp * 4 + (size_t)((c.NS + 2 * c.NC + 1) & ~1) * 8 +
           (size_t)key_words * 16 + c.NS * 4 + (size_t)kbp * 4;  // key multipliers as uint4 limbs
}

}  // namespace k1r

using namespace k1r;

// A block [h0, h0 + kb) holds whole tables when h0 is a multiple of K and its end is too (or lies
// past the last table's codes, L*K <= k).
bool rows_keys_fusable(const RPacking& pk, int L, int K) {
    if (!pk.ok || K < 1) return false;
    for (int bl = 0; bl < pk.hash_blocks; ++bl) {
        if (pk.block_h0[bl] % K) return false;
        const int end = pk.block_h0[bl] + pk.block_kb[bl];
        if (end % K && end < L * K) return false;
    }
    return true;
}
int rows_key_tables_max(const RPacking& pk, int L, int K) {
    int t = 0;
    for (int bl = 0; bl < pk.hash_blocks; ++bl) {
        const int t0 = pk.block_h0[bl] / K, t1 = std::min(L, (pk.block_h0[bl] + pk.block_kb[bl]) / K);
        t = std::max(t, t1 - t0);
    }
    return t;
}

fastlsh_status launch_gather_rows(const fastlsh_params* p, const DeviceCopy& d, const float* X, int64_t N,
                                  int32_t* codes, float* proj, cudaStream_t stream, const FusedKeys* fk) {
    const RPacking& pk = p->rpack;
    if (!pk.ok || !d.r_offp) return FASTLSH_EUNSUPPORTED;
    // keys from the code tile need every table's codes in one block: blocks start on table
    // boundaries (K <= 1024: the limb sums of the flush are exact while K * 2^53 < 2^63)
    int key_words = 0;
    if (fk) {
        if (!rows_keys_fusable(pk, fk->L, fk->K) || (int64_t)fk->L * fk->K > p->k || fk->K > 1024)
            return FASTLSH_EUNSUPPORTED;
        key_words = rows_key_tables_max(pk, fk->L, fk->K) * (fk->K + 1);
    }
    // TMA bulk row copies need 16-byte aligned rows
    if ((p->n % 4) != 0 || (reinterpret_cast<uintptr_t>(X) & 15) != 0) return FASTLSH_EUNSUPPORTED;
    constexpr size_t kSmemMax = 227 * 1024;
    const int threads = pk.warps * 32;
    const size_t smem = row_smem_bytes(pk, key_words);
    if (smem > kSmemMax) return FASTLSH_EUNSUPPORTED;
    const int R = kRClasses[pk.cls].R;
    RowKernelFn fn = select_row_kernel(pk.slots, pk.cls);
    if (!fn) return FASTLSH_EUNSUPPORTED;
    RowArgs a;
    a.X = X;
    a.N = N;
    a.n = p->n;
    a.S = pk.S;
    a.S0 = pk.S0;
    a.n1 = pk.n1;
    a.offp = d.r_offp;
    a.coef = d.r_coef;
    a.lane_hash = d.r_lane_hash;
    a.b = d.b;
    a.block_h0 = d.r_block_h0;
    a.block_kb = d.r_block_kb;
    a.w = p->w;
    a.k = p->k;
    a.P = pk.parts;
    a.W = pk.warps;
    a.HB = pk.hash_blocks;
    a.kbp = (pk.kb_max + 3) & ~3;
    a.groups = (N + R - 1) / R;
    a.codes = codes;
    a.proj = proj;
    a.flags = d.flags;
    const void* out = proj ? static_cast<const void*>(proj) : static_cast<const void*>(codes);
    bool blocks_aligned = true;
    for (int bl = 0; bl < pk.hash_blocks; ++bl)
        if ((pk.block_h0[bl] % 4) || (pk.block_kb[bl] % 4)) blocks_aligned = false;
    a.vec = (p->k % 4 == 0) && blocks_aligned && ((reinterpret_cast<uintptr_t>(out) & 15) == 0) ? 1 : 0;
    if (std::getenv("FASTLSH_NO_VEC_STORE")) a.vec = 0;  // fallback-path test knob: read per call (the test toggles it)
    a.kr = fk ? fk->r : nullptr;
    a.L = fk ? fk->L : 0;
    a.K = fk ? fk->K : 1;
    a.kw = key_words;
    a.keys = fk ? fk->keys : nullptr;
    a.ldk = fk ? fk->ldk : 0;
    static const int debug = [] {  // experiment knob, read once
        const char* e = std::getenv("FASTLSH_K1R_DEBUG");
        return e ? std::atoi(e) : 0;
    }();
    a.debug = debug;

    // resident CTAs per device: queried once per (params, device, shared-memory size) — at C0's
    // 10^4 rows the attribute + occupancy queries per call cost as much as the kernel
    const int slot = fk ? 1 : 0;
    int resident = d.r_resident[slot];
    cudaError_t e;
    if (resident <= 0 || d.r_resident_smem[slot] != smem) {
        // the device maximum, never lowered: another params object sharing this kernel may launch
        // it with more shared memory than this one
        e = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kSmemMax);
        if (e != cudaSuccess) return set_cuda_error(e);
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(fn), threads, smem);
        if (e != cudaSuccess) return set_cuda_error(e);
        if (per_sm < 1) return FASTLSH_EUNSUPPORTED;
        resident = sms * per_sm;
        d.r_resident[slot] = resident;
        d.r_resident_smem[slot] = smem;
    }
    // persistent grid: as many row streams per hash block as fit resident at once
    long long gpr = (long long)resident / pk.hash_blocks;
    if (gpr > a.groups) gpr = a.groups;
    if (gpr < 1) gpr = 1;
    const long long grid = gpr * pk.hash_blocks;
    fn<<<(unsigned)grid, threads, smem, stream>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e);
    return FASTLSH_OK;
}

}  // namespace fastlsh
