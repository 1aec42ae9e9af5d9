// api.cu — the C ABI of include/fastlsh.h: validation, params/keys objects, per-device uploads,
// dispatch to the kernels, and the pipelined host-buffer entry point.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <new>
#include <string>

#include "internal.h"
#include "philox.h"

namespace fastlsh {

static thread_local std::string g_cuda_error;

fastlsh_status set_cuda_error(cudaError_t e) {
    g_cuda_error = std::string(cudaGetErrorName(e)) + ": " + cudaGetErrorString(e);
    return FASTLSH_ECUDA;
}

fastlsh_status smem_optin_once(const void* fn) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return set_cuda_error(e);
    static std::mutex mu;
    static std::vector<std::pair<const void*, int>> done;
    std::lock_guard<std::mutex> g(mu);
    for (const auto& d : done)
        if (d.first == fn && d.second == dev) return FASTLSH_OK;
    // the opt-in covers dynamic memory only: the kernel's static shared memory counts against 227 KB
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, fn);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - (int)fa.sharedSizeBytes);
    if (e != cudaSuccess) {
        cudaGetLastError();  // not sticky: keep it out of later launches' cudaGetLastError checks
        return set_cuda_error(e);
    }
    done.push_back({fn, dev});
    return FASTLSH_OK;
}

namespace {

#define FL_CUDA(call)                                  \
    do {                                               \
        cudaError_t _e = (call);                       \
        if (_e != cudaSuccess) return set_cuda_error(_e); \
    } while (0)

fastlsh_status current_device(int* dev) {
    FL_CUDA(cudaGetDevice(dev));
    if (*dev < 0 || *dev >= kMaxDevices) return FASTLSH_EUNSUPPORTED;
    return FASTLSH_OK;
}

fastlsh_status check_sm100(int dev) {
    int major = 0, minor = 0;
    FL_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    FL_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
    if (major != 10 || minor != 0) return FASTLSH_EUNSUPPORTED;
    return FASTLSH_OK;
}

bool valid_w(float w) { return std::isfinite(w) && w > 0.0f; }

template <typename T>
fastlsh_status upload_vec(T** dst, const std::vector<T>& src, cudaStream_t s) {
    if (src.empty()) { *dst = nullptr; return FASTLSH_OK; }
    FL_CUDA(cudaMalloc(reinterpret_cast<void**>(dst), src.size() * sizeof(T)));
    FL_CUDA(cudaMemcpyAsync(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    return FASTLSH_OK;
}

fastlsh_status new_params(int32_t n, int32_t m, int32_t k, float w, fastlsh_params** out) {
    if (!out) return FASTLSH_EINVAL;
    *out = nullptr;
    if (n <= 0 || m <= 0 || k <= 0 || !valid_w(w)) return FASTLSH_EINVAL;
    // beyond these, no specialised kernel packs the params and the generic K0 serves them
    if ((int64_t)k * m > ((int64_t)1 << 31)) return FASTLSH_EUNSUPPORTED;  // host arrays, int offsets
    fastlsh_params* p = new (std::nothrow) fastlsh_params();
    if (!p) return FASTLSH_ENOMEM;
    p->n = n; p->m = m; p->k = k; p->w = w;
    try {
        p->idx.resize((size_t)k * m);
        p->a.resize((size_t)k * m);
        p->b.resize(k);
    } catch (...) {
        delete p;
        return FASTLSH_ENOMEM;
    }
    *out = p;
    return FASTLSH_OK;
}

// params K1 / K1t / K1r can pack (shared-memory stages of 4 rows, <= kMaxSlots * 256 slots a hash)
bool packable(const fastlsh_params* p) { return p->n <= kMaxN && (int64_t)p->m <= (int64_t)kMaxSlots * 256; }

// full = false: params pinned to the dense path (kernel 5) skip the gather packings (seconds of host
// work for large k*m); pinning a gather kernel or exporting a packing asks for them (full).
fastlsh_status ensure_packed(fastlsh_params* p, bool full = false) {
    if (p->packed && !(full && p->pack_skipped)) return FASTLSH_OK;
    if (!packable(p)) {  // only the generic K0 (and K1j where it applies) will serve these params
        p->packed = true;
        return FASTLSH_OK;
    }
    if (!full && p->kernel == 5 && dense_shape(p)) {
        p->packed = p->pack_skipped = true;
        return FASTLSH_OK;
    }
    try {
        build_packing(*p, p->pack);
    } catch (...) {
        return FASTLSH_ENOMEM;
    }
    if (p->pack.slots <= 0) return FASTLSH_EUNSUPPORTED;
    try {
        if (!p->is_e2lsh) build_tmem_packing(*p, p->tpack);
        build_row_packing(*p, p->rpack);
    } catch (...) {
        return FASTLSH_ENOMEM;
    }
    p->packed = true;
    p->pack_skipped = false;
    return FASTLSH_OK;
}

fastlsh_status ready_params(const fastlsh_params* p, int* dev_out) {
    if (!p) return FASTLSH_EINVAL;
    int dev = 0;
    fastlsh_status st = current_device(&dev);
    if (st != FASTLSH_OK) return st;
    if (!p->dev[dev].ready) return FASTLSH_ESTATE;
    *dev_out = dev;
    return FASTLSH_OK;
}

void free_device_copy(DeviceCopy& d) {
    cudaFree(d.offp); cudaFree(d.coef); cudaFree(d.unit_lane); cudaFree(d.b);
    cudaFree(d.block_h0); cudaFree(d.block_kb); cudaFree(d.flags);
    cudaFree(d.dense_hi); cudaFree(d.dense_lo); cudaFree(d.dense_h16);
    cudaFree(d.t_recs); cudaFree(d.t_counts); cudaFree(d.t_offs); cudaFree(d.t_hinfo); cudaFree(d.t_groups);
    cudaFree(d.r_offp); cudaFree(d.r_coef); cudaFree(d.r_lane_hash); cudaFree(d.r_block_h0); cudaFree(d.r_block_kb);
    cudaFree(d.j_idx); cudaFree(d.j_a);
    for (int i = 0; i < 2; ++i) {
        cudaFree(d.ws_x[i]); cudaFree(d.ws_codes[i]); cudaFree(d.ws_keys[i]);
        if (d.ws_stream[i]) cudaStreamDestroy(d.ws_stream[i]);
    }
    for (int i = 0; i < 4; ++i) if (d.ws_event[i]) cudaEventDestroy(d.ws_event[i]);
    d = DeviceCopy();
}

}  // namespace

// K1t (TMEM gather) serves the call when pinned (kernel 2; an inapplicable call fails) or, in
// auto mode, when kAutoTmem is set and its packing exists and X is 16-B aligned.
constexpr bool kAutoTmem = false;  // K1t is still slower than K1 on the bench workload (C1)
bool tmem_selected(const fastlsh_params* p) {
    return p->kernel == 2 || (p->kernel == 0 && kAutoTmem && p->tpack.ok);
}
// K1r (row-major stages) serves the call when pinned (kernel 3) or, in auto mode, when its packing
// exists and its modelled cost is below K1's (K1's model omits its transposition stalls: the
// measured ratio is applied). Calls K1r cannot serve (n % 4 != 0, X not 16-B aligned) go to K1.
constexpr double kK1Derate = 1.25;
bool rows_selected(const fastlsh_params* p) {
    if (!p->rpack.ok) return false;
    if (p->kernel == 3) return true;
    if (p->n % 4) return false;  // rows are not 16-byte multiples: no bulk row copies
    return p->kernel == 0 && p->rpack.cost <= p->pack.cost * kK1Derate;
}
// Keys from K1r's code tile (every hash block builds the tables it holds) pay off when a block's key
// work (tables x K products per row, spread over the CTA) is small next to its gather work (W*MS
// LDS.32 wavefronts per row): measured C1 (500 vs 1024) 4.49 vs 4.59 ms for hash + keys, C3 (256
// vs 144) 10.9 vs 9.8 ms per 8M rows.
bool rows_keys_pay(const fastlsh_params* p, const fastlsh_keys* ks) {
    const RPacking& r = p->rpack;
    if (!rows_keys_fusable(r, ks->L, ks->K)) return false;
    return (double)rows_key_tables_max(r, ks->L, ks->K) * ks->K <= 0.75 * (double)r.warps * r.slots;
}
// K1j (params-specialised lane = row kernel, jit.cpp) serves the call when pinned (kernel 4) or, in
// auto mode, whenever it applies (n <= 128: the gathers become register operands, no shared-memory
// bound). Calls it cannot serve (alignment, compile failure) fall through unless pinned.
bool jit_selected(const fastlsh_params* p) {
    return p->kernel == 4 || (p->kernel == 0 && jit::applicable(*p));
}
// K4 on the duplicates-merged coefficient matrix: Eq. 5 as a dense 3xTF32
// tcgen05 GEMM, A[c][i] = sum_{j: idx_ij = c} a_ij. Opt-in only (kernel 5, fastlsh_params_set_kernel):
// north_star reserves the tensor cores for the dense E2LSH baseline — FastLSH's sampled projection is
// a gather — and SURVEY.md §8(f)3(iii) keeps this as analysis, so the automatic choice never takes it
// even where it is faster (C2 n = 4096: m = 512 K1r 25.2 vs dense 8.5 ms per 250k rows, m = 4096
// 17.4 vs 0.88 ms per 20k rows; bench.py reports it beside the gather kernel). The dense hi/lo
// matrices must stay small (kpad * n * 8 bytes <= 1 GiB).
bool dense_shape(const fastlsh_params* p) {
    if (p->n % 4) return false;
    const int64_t kpad = ((int64_t)p->k + 255) / 256 * 256;
    return kpad * p->n * 8 <= ((int64_t)1 << 30);
}
bool dense_selected(const fastlsh_params* p) { return p->kernel == 5; }
fastlsh_status launch_hash(const fastlsh_params* p, const DeviceCopy& d, const float* X, int64_t N,
                           int32_t* codes, float* proj, cudaStream_t stream) {
    if (dense_selected(p)) {
        // calls the GEMM cannot serve (X not 16-byte aligned) fall through to K1 (K0 when the gather
        // packings were skipped: dense pinned before the first info / upload)
        fastlsh_status st = launch_e2lsh(p, const_cast<DeviceCopy&>(d), X, N, codes, proj, 3, stream);
        if (st != FASTLSH_EUNSUPPORTED) return st;
    }
    if (jit_selected(p)) {
        fastlsh_status st = jit::launch(p, d, X, N, codes, proj, nullptr, nullptr, nullptr, 0, stream);
        if (st != FASTLSH_EUNSUPPORTED || p->kernel == 4) return st;
    }
    if (tmem_selected(p)) {
        fastlsh_status st = launch_gather_tmem(p, d, X, N, codes, proj, stream);
        if (st != FASTLSH_EUNSUPPORTED || p->kernel == 2) return st;
    }
    if (p->kernel == 3 || rows_selected(p)) {
        fastlsh_status st = launch_gather_rows(p, d, X, N, codes, proj, stream);
        if (st != FASTLSH_EUNSUPPORTED || p->kernel == 3) return st;
    }
    if (!packable(p) || !d.offp) return launch_generic(p, d, X, N, codes, proj, stream);
    return launch_gather(p, d, X, N, codes, proj, stream);
}

}  // namespace fastlsh

using namespace fastlsh;

extern "C" {

int32_t fastlsh_abi_version(void) { return 1; }

const char* fastlsh_status_string(fastlsh_status s) {
    switch (s) {
        case FASTLSH_OK: return "ok";
        case FASTLSH_EINVAL: return "invalid argument";
        case FASTLSH_ENOMEM: return "out of memory";
        case FASTLSH_ECUDA: return "CUDA error";
        case FASTLSH_EUNSUPPORTED: return "unsupported device or shape";
        case FASTLSH_ESTATE: return "params/keys not uploaded to the current device";
    }
    return "unknown status";
}

const char* fastlsh_last_cuda_error(void) { return g_cuda_error.c_str(); }

fastlsh_status fastlsh_params_create(int32_t n, int32_t m, int32_t k, float w, uint64_t seed,
                                     fastlsh_params** out) {
    fastlsh_status st = new_params(n, m, k, w, out);
    if (st != FASTLSH_OK) return st;
    fastlsh_params* p = *out;
    for (int32_t i = 0; i < k; ++i) {
        for (int32_t j = 0; j < m; ++j) {
            p->idx[(size_t)i * m + j] = draw_index(seed, (uint32_t)i, (uint32_t)j, (uint32_t)n);
            p->a[(size_t)i * m + j] = draw_gaussian(seed, (uint32_t)i, (uint32_t)j);
        }
        p->b[i] = draw_offset(seed, (uint32_t)i, w);
    }
    return FASTLSH_OK;
}

fastlsh_status fastlsh_params_create_from_arrays(int32_t n, int32_t m, int32_t k, float w,
                                                 const int32_t* idx, const float* a,
                                                 const float* b, fastlsh_params** out) {
    if (!idx || !a || !b) return FASTLSH_EINVAL;
    for (int64_t t = 0; t < (int64_t)k * m; ++t) {
        if (k > 0 && m > 0 && (idx[t] < 0 || idx[t] >= n)) return FASTLSH_EINVAL;
        if (!std::isfinite(a[t])) return FASTLSH_EINVAL;
    }
    for (int32_t i = 0; i < k; ++i) if (!std::isfinite(b[i])) return FASTLSH_EINVAL;
    fastlsh_status st = new_params(n, m, k, w, out);
    if (st != FASTLSH_OK) return st;
    fastlsh_params* p = *out;
    std::memcpy(p->idx.data(), idx, sizeof(int32_t) * (size_t)k * m);
    std::memcpy(p->a.data(), a, sizeof(float) * (size_t)k * m);
    std::memcpy(p->b.data(), b, sizeof(float) * (size_t)k);
    return FASTLSH_OK;
}

fastlsh_status e2lsh_params_create(int32_t n, int32_t k, float w, uint64_t seed,
                                   fastlsh_params** out) {
    fastlsh_status st = new_params(n, n, k, w, out);
    if (st != FASTLSH_OK) return st;
    fastlsh_params* p = *out;
    p->is_e2lsh = true;
    for (int32_t i = 0; i < k; ++i) {
        for (int32_t j = 0; j < n; ++j) {
            p->idx[(size_t)i * n + j] = j;
            p->a[(size_t)i * n + j] = draw_gaussian(seed, (uint32_t)i, (uint32_t)j);
        }
        p->b[i] = draw_offset(seed, (uint32_t)i, w);
    }
    return FASTLSH_OK;
}

void fastlsh_params_destroy(fastlsh_params* p) {
    if (!p) return;
    int cur = 0;
    cudaGetDevice(&cur);
    for (int d = 0; d < kMaxDevices; ++d) {
        DeviceCopy& dc = p->dev[d];
        bool any = dc.offp || dc.flags || dc.dense_hi || dc.ws_x[0];
        if (!any) continue;
        cudaSetDevice(d);
        free_device_copy(dc);
    }
    cudaSetDevice(cur);
    delete p;
}

fastlsh_status fastlsh_params_export(const fastlsh_params* p, int32_t* idx, float* a, float* b,
                                     float* w) {
    if (!p) return FASTLSH_EINVAL;
    if (idx) std::memcpy(idx, p->idx.data(), p->idx.size() * sizeof(int32_t));
    if (a) std::memcpy(a, p->a.data(), p->a.size() * sizeof(float));
    if (b) std::memcpy(b, p->b.data(), p->b.size() * sizeof(float));
    if (w) *w = p->w;
    return FASTLSH_OK;
}

fastlsh_status fastlsh_params_info(const fastlsh_params* cp, fastlsh_params_info_t* info) {
    if (!cp || !info) return FASTLSH_EINVAL;
    fastlsh_params* p = const_cast<fastlsh_params*>(cp);
    {
        std::lock_guard<std::mutex> g(p->mu);
        fastlsh_status st = ensure_packed(p);
        if (st != FASTLSH_OK) return st;
    }
    const Packing& pk = p->pack;
    info->n = p->n; info->m = p->m; info->k = p->k; info->w = p->w;
    info->is_e2lsh = p->is_e2lsh ? 1 : 0;
    info->parts = pk.parts;
    info->slots = pk.slots;
    info->units = p->k * pk.parts;
    info->warps_per_block = pk.warps;
    info->hash_blocks = pk.hash_blocks;
    info->rows_per_group = kRows;
    info->bank_efficiency = pk.efficiency;
    info->conflict_wavefronts = pk.conflict_wavefronts;
    info->kernel = dense_selected(p) ? 5 : jit_selected(p) ? 4 : !packable(p) ? 0 : tmem_selected(p) ? 2
                   : rows_selected(p) ? 3 : 1;
    info->tmem_hash_blocks = p->tpack.ok ? p->tpack.HB : 0;
    info->tmem_hashes_per_warp = p->tpack.ok ? p->tpack.nhw : 0;
    return FASTLSH_OK;
}

fastlsh_status fastlsh_params_packing(const fastlsh_params* cp, int32_t* sizes, uint32_t* offp,
                                      float* coef, uint16_t* unit_lane, int32_t* block_h0,
                                      int32_t* block_kb) {
    if (!cp) return FASTLSH_EINVAL;
    fastlsh_params* p = const_cast<fastlsh_params*>(cp);
    {
        std::lock_guard<std::mutex> g(p->mu);
        fastlsh_status st = ensure_packed(p, true);
        if (st != FASTLSH_OK) return st;
    }
    const Packing& pk = p->pack;
    if (sizes) {
        sizes[0] = pk.parts; sizes[1] = pk.slots; sizes[2] = pk.warps; sizes[3] = pk.hash_blocks;
        sizes[4] = pk.kb_max; sizes[5] = pk.nq; sizes[6] = pk.stage_chunks;
        sizes[7] = pk.hash_blocks * pk.warps * 32;
    }
    if (offp) std::memcpy(offp, pk.offp.data(), pk.offp.size() * sizeof(uint32_t));
    if (coef) std::memcpy(coef, pk.coef.data(), pk.coef.size() * sizeof(float));
    if (unit_lane) std::memcpy(unit_lane, pk.unit_lane.data(), pk.unit_lane.size() * sizeof(uint16_t));
    if (block_h0) for (size_t i = 0; i < pk.block_h0.size(); ++i) block_h0[i] = pk.block_h0[i];
    if (block_kb) for (size_t i = 0; i < pk.block_kb.size(); ++i) block_kb[i] = pk.block_kb[i];
    return FASTLSH_OK;
}

fastlsh_status fastlsh_params_row_packing(const fastlsh_params* cp, int32_t* sizes, uint32_t* offp, float* coef,
                                          int16_t* lane_hash, int32_t* block_h0, int32_t* block_kb) {
    if (!cp) return FASTLSH_EINVAL;
    fastlsh_params* p = const_cast<fastlsh_params*>(cp);
    {
        std::lock_guard<std::mutex> g(p->mu);
        fastlsh_status st = ensure_packed(p, true);
        if (st != FASTLSH_OK) return st;
    }
    const RPacking& pk = p->rpack;
    if (sizes) {
        sizes[0] = pk.ok ? 1 : 0; sizes[1] = pk.parts; sizes[2] = pk.slots; sizes[3] = pk.warps;
        sizes[4] = pk.hash_blocks; sizes[5] = pk.kb_max; sizes[6] = pk.S;
        sizes[7] = (int32_t)pk.conflict_wavefronts;
        sizes[8] = pk.S0; sizes[9] = pk.n1;
    }
    if (!pk.ok) return FASTLSH_OK;
    if (offp) std::memcpy(offp, pk.offp.data(), pk.offp.size() * sizeof(uint32_t));
    if (coef) std::memcpy(coef, pk.coef.data(), pk.coef.size() * sizeof(float));
    if (lane_hash) std::memcpy(lane_hash, pk.lane_hash.data(), pk.lane_hash.size() * sizeof(int16_t));
    if (block_h0) for (size_t i = 0; i < pk.block_h0.size(); ++i) block_h0[i] = pk.block_h0[i];
    if (block_kb) for (size_t i = 0; i < pk.block_kb.size(); ++i) block_kb[i] = pk.block_kb[i];
    return FASTLSH_OK;
}

fastlsh_status fastlsh_params_set_table_size(fastlsh_params* p, int32_t K) {
    if (!p || K < 1) return FASTLSH_EINVAL;
    std::lock_guard<std::mutex> g(p->mu);
    for (int d = 0; d < kMaxDevices; ++d)
        if (p->dev[d].ready) return FASTLSH_ESTATE;
    if (p->table_align != K) {
        p->table_align = K;
        p->packed = false;
        p->pack = Packing();
    }
    return FASTLSH_OK;
}

fastlsh_status fastlsh_params_upload(fastlsh_params* p, int32_t device, fastlsh_stream_t stream) {
    if (!p) return FASTLSH_EINVAL;
    int dev = 0;
    fastlsh_status st = current_device(&dev);
    if (st != FASTLSH_OK) return st;
    if (device != dev) return FASTLSH_EINVAL;
    st = check_sm100(dev);
    if (st != FASTLSH_OK) return st;
    std::lock_guard<std::mutex> g(p->mu);
    if (p->dev[dev].ready) return FASTLSH_OK;
    st = ensure_packed(p);
    if (st != FASTLSH_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    DeviceCopy& d = p->dev[dev];
    const Packing& pk = p->pack;
    std::vector<int32_t> h0(pk.block_h0.begin(), pk.block_h0.end());
    std::vector<int32_t> kb(pk.block_kb.begin(), pk.block_kb.end());
    if ((st = upload_vec(&d.offp, pk.offp, s)) != FASTLSH_OK ||
        (st = upload_vec(&d.coef, pk.coef, s)) != FASTLSH_OK ||
        (st = upload_vec(&d.unit_lane, pk.unit_lane, s)) != FASTLSH_OK ||
        (st = upload_vec(&d.b, p->b, s)) != FASTLSH_OK ||
        (st = upload_vec(&d.block_h0, h0, s)) != FASTLSH_OK ||
        (st = upload_vec(&d.block_kb, kb, s)) != FASTLSH_OK ||
        (p->tpack.ok && ((st = upload_vec(&d.t_recs, p->tpack.recs, s)) != FASTLSH_OK ||
                         (st = upload_vec(&d.t_counts, p->tpack.counts, s)) != FASTLSH_OK ||
                         (st = upload_vec(&d.t_offs, p->tpack.offs, s)) != FASTLSH_OK ||
                         (st = upload_vec(&d.t_hinfo, p->tpack.hinfo, s)) != FASTLSH_OK ||
                         (st = upload_vec(&d.t_groups, p->tpack.groups, s)) != FASTLSH_OK)) ||
        (p->rpack.ok && ((st = upload_vec(&d.r_offp, p->rpack.offp, s)) != FASTLSH_OK ||
                         (st = upload_vec(&d.r_coef, p->rpack.coef, s)) != FASTLSH_OK ||
                         (st = upload_vec(&d.r_lane_hash, p->rpack.lane_hash, s)) != FASTLSH_OK ||
                         (st = upload_vec(&d.r_block_h0, p->rpack.block_h0, s)) != FASTLSH_OK ||
                         (st = upload_vec(&d.r_block_kb, p->rpack.block_kb, s)) != FASTLSH_OK))) {
        free_device_copy(d);
        return st;
    }
    if ((jit::applicable(*p) || !packable(p) || p->pack_skipped) &&  // canonical arrays: K1j's slow path, K0
        ((st = upload_vec(&d.j_idx, p->idx, s)) != FASTLSH_OK || (st = upload_vec(&d.j_a, p->a, s)) != FASTLSH_OK)) {
        free_device_copy(d);
        return st;
    }
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&d.flags), 2 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemsetAsync(d.flags, 0, 2 * sizeof(unsigned long long), s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // host vectors may be reused right away
    if (e != cudaSuccess) {
        free_device_copy(d);
        return set_cuda_error(e);
    }
    d.ready = true;
    return FASTLSH_OK;
}


fastlsh_status fastlsh_params_set_kernel(fastlsh_params* p, int32_t kernel) {
    if (!p || kernel < 0 || kernel > 5) return FASTLSH_EINVAL;
    std::lock_guard<std::mutex> g(p->mu);
    if (kernel == 5) {  // pinned dense path: the gather packings are not needed (built on demand later)
        if (p->n % 4) return FASTLSH_EUNSUPPORTED;  // K4's K-major tensor maps
        p->kernel = 5;
        return ensure_packed(p, false);
    }
    // auto (0) and the gather kernels need the packings a pinned-dense params object skipped
    const bool gather = kernel <= 3;
    if (gather && p->pack_skipped) {
        // the gather packings were skipped (dense-path shape): build them now, unless a device copy
        // without them exists already
        for (int i = 0; i < kMaxDevices; ++i)
            if (p->dev[i].ready) return FASTLSH_ESTATE;
    }
    fastlsh_status st = ensure_packed(p, gather);
    if (st != FASTLSH_OK) return st;
    if (kernel == 2 && !p->tpack.ok) return FASTLSH_EUNSUPPORTED;
    if (kernel == 3 && !p->rpack.ok) return FASTLSH_EUNSUPPORTED;
    if (kernel == 4 && !jit::applicable(*p)) return FASTLSH_EUNSUPPORTED;
    p->kernel = kernel;
    return FASTLSH_OK;
}

static fastlsh_status hash_common(const fastlsh_params* p, const float* X, int64_t N,
                                  int32_t* codes, float* proj, fastlsh_stream_t stream) {
    if (!p || N < 0) return FASTLSH_EINVAL;
    if (N == 0) return FASTLSH_OK;
    if (!X || (!codes && !proj)) return FASTLSH_EINVAL;
    if ((reinterpret_cast<uintptr_t>(X) & 3) || (reinterpret_cast<uintptr_t>(codes) & 3) ||
        (reinterpret_cast<uintptr_t>(proj) & 3))
        return FASTLSH_EINVAL;
    int dev = 0;
    fastlsh_status st = ready_params(p, &dev);
    if (st != FASTLSH_OK) return st;
    return launch_hash(p, p->dev[dev], X, N, codes, proj, reinterpret_cast<cudaStream_t>(stream));
}

fastlsh_status fastlsh_hash(const fastlsh_params* p, const float* X, int64_t N, int32_t* codes,
                            fastlsh_stream_t stream) {
    if (!codes && N > 0) return FASTLSH_EINVAL;
    return hash_common(p, X, N, codes, nullptr, stream);
}

fastlsh_status fastlsh_project(const fastlsh_params* p, const float* X, int64_t N, float* proj,
                               fastlsh_stream_t stream) {
    if (!proj && N > 0) return FASTLSH_EINVAL;
    return hash_common(p, X, N, nullptr, proj, stream);
}

fastlsh_status e2lsh_hash(const fastlsh_params* p, const float* X, int64_t N, int32_t* codes,
                          int32_t precision, fastlsh_stream_t stream) {
    if (!p || N < 0 || (precision < 1 || precision > 3)) return FASTLSH_EINVAL;
    if (N == 0) return FASTLSH_OK;
    if (!X || !codes) return FASTLSH_EINVAL;
    int dev = 0;
    fastlsh_status st = ready_params(p, &dev);
    if (st != FASTLSH_OK) return st;
    fastlsh_params* mp = const_cast<fastlsh_params*>(p);
    return launch_e2lsh(mp, mp->dev[dev], X, N, codes, nullptr, precision,
                        reinterpret_cast<cudaStream_t>(stream));
}

fastlsh_status e2lsh_project(const fastlsh_params* p, const float* X, int64_t N, float* proj,
                             int32_t precision, fastlsh_stream_t stream) {
    if (!p || N < 0 || (precision < 1 || precision > 3)) return FASTLSH_EINVAL;
    if (N == 0) return FASTLSH_OK;
    if (!X || !proj) return FASTLSH_EINVAL;
    int dev = 0;
    fastlsh_status st = ready_params(p, &dev);
    if (st != FASTLSH_OK) return st;
    fastlsh_params* mp = const_cast<fastlsh_params*>(p);
    return launch_e2lsh(mp, mp->dev[dev], X, N, nullptr, proj, precision,
                        reinterpret_cast<cudaStream_t>(stream));
}

fastlsh_status fastlsh_keys_create(int32_t L, int32_t K, uint64_t seed, fastlsh_keys** out) {
    if (!out) return FASTLSH_EINVAL;
    *out = nullptr;
    if (L <= 0 || K <= 0 || (int64_t)L * (K + 1) > 8192) return FASTLSH_EINVAL;
    fastlsh_keys* ks = new (std::nothrow) fastlsh_keys();
    if (!ks) return FASTLSH_ENOMEM;
    ks->L = L; ks->K = K;
    ks->r.resize((size_t)L * (K + 1));
    for (int32_t l = 0; l < L; ++l)
        for (int32_t j = 0; j <= K; ++j)
            ks->r[(size_t)l * (K + 1) + j] = draw_key_multiplier(seed, (uint32_t)l, (uint32_t)j);
    *out = ks;
    return FASTLSH_OK;
}

fastlsh_status fastlsh_keys_create_from_arrays(int32_t L, int32_t K, const uint64_t* r,
                                               fastlsh_keys** out) {
    if (!out || !r) return FASTLSH_EINVAL;
    *out = nullptr;
    if (L <= 0 || K <= 0 || (int64_t)L * (K + 1) > 8192) return FASTLSH_EINVAL;
    for (int64_t t = 0; t < (int64_t)L * (K + 1); ++t) if (r[t] >= kP61) return FASTLSH_EINVAL;
    fastlsh_keys* ks = new (std::nothrow) fastlsh_keys();
    if (!ks) return FASTLSH_ENOMEM;
    ks->L = L; ks->K = K;
    ks->r.assign(r, r + (size_t)L * (K + 1));
    *out = ks;
    return FASTLSH_OK;
}

void fastlsh_keys_destroy(fastlsh_keys* ks) {
    if (!ks) return;
    int cur = 0;
    cudaGetDevice(&cur);
    for (int d = 0; d < kMaxDevices; ++d) {
        if (!ks->dev_r[d]) continue;
        cudaSetDevice(d);
        cudaFree(ks->dev_r[d]);
    }
    cudaSetDevice(cur);
    delete ks;
}

fastlsh_status fastlsh_keys_export(const fastlsh_keys* ks, uint64_t* r) {
    if (!ks || !r) return FASTLSH_EINVAL;
    std::memcpy(r, ks->r.data(), ks->r.size() * sizeof(uint64_t));
    return FASTLSH_OK;
}

static fastlsh_status keys_device(const fastlsh_keys* cks, int dev, const uint64_t** out) {
    fastlsh_keys* ks = const_cast<fastlsh_keys*>(cks);
    std::lock_guard<std::mutex> g(ks->mu);
    if (!ks->dev_r[dev]) {
        uint64_t* d = nullptr;
        FL_CUDA(cudaMalloc(reinterpret_cast<void**>(&d), ks->r.size() * sizeof(uint64_t)));
        cudaError_t e = cudaMemcpy(d, ks->r.data(), ks->r.size() * sizeof(uint64_t), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) { cudaFree(d); return set_cuda_error(e); }
        ks->dev_r[dev] = d;
    }
    *out = ks->dev_r[dev];
    return FASTLSH_OK;
}

fastlsh_status fastlsh_build_keys(const fastlsh_keys* ks, const int32_t* codes, int64_t N,
                                  int32_t k, uint64_t* keys_out, int64_t ldk,
                                  fastlsh_stream_t stream) {
    if (!ks || N < 0 || k <= 0) return FASTLSH_EINVAL;
    if ((int64_t)ks->L * ks->K > k) return FASTLSH_EINVAL;
    if (N == 0) return FASTLSH_OK;
    if (!codes || !keys_out || ldk < N) return FASTLSH_EINVAL;
    if ((reinterpret_cast<uintptr_t>(codes) & 3) || (reinterpret_cast<uintptr_t>(keys_out) & 7))
        return FASTLSH_EINVAL;
    int dev = 0;
    fastlsh_status st = current_device(&dev);
    if (st != FASTLSH_OK) return st;
    st = check_sm100(dev);
    if (st != FASTLSH_OK) return st;
    const uint64_t* dr = nullptr;
    st = keys_device(ks, dev, &dr);
    if (st != FASTLSH_OK) return st;
    return launch_build_keys(ks, dr, codes, N, k, keys_out, ldk, reinterpret_cast<cudaStream_t>(stream));
}

fastlsh_status fastlsh_tables_workspace(int32_t L, int64_t N, size_t* bytes) {
    if (L < 1 || N < 0 || N >= 0xffffffffLL || !bytes) return FASTLSH_EINVAL;
    *bytes = tables_workspace_bytes(L, N);
    return FASTLSH_OK;
}

fastlsh_status fastlsh_build_tables(const uint64_t* keys, int32_t L, int64_t N, int64_t ldk,
                                    uint64_t* sorted_keys, uint32_t* ids, uint32_t* bucket_start,
                                    int64_t* nbuckets, void* workspace, size_t workspace_bytes,
                                    fastlsh_stream_t stream) {
    if (L < 1 || N < 0 || N >= 0xffffffffLL || ldk < N) return FASTLSH_EINVAL;
    if (!bucket_start || !nbuckets || (reinterpret_cast<uintptr_t>(nbuckets) & 7) ||
        (reinterpret_cast<uintptr_t>(bucket_start) & 3))
        return FASTLSH_EINVAL;
    int dev = 0;
    fastlsh_status st = current_device(&dev);
    if (st != FASTLSH_OK) return st;
    st = check_sm100(dev);
    if (st != FASTLSH_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (N == 0) {  // empty tables: no buckets, bucket_start[l][0] = 0
        FL_CUDA(cudaMemsetAsync(nbuckets, 0, (size_t)L * sizeof(int64_t), s));
        FL_CUDA(cudaMemsetAsync(bucket_start, 0, (size_t)L * sizeof(uint32_t), s));
        return FASTLSH_OK;
    }
    if (!keys || !sorted_keys || !ids || !workspace || workspace_bytes < tables_workspace_bytes(L, N) ||
        (reinterpret_cast<uintptr_t>(keys) & 7) || (reinterpret_cast<uintptr_t>(sorted_keys) & 7) ||
        (reinterpret_cast<uintptr_t>(ids) & 3) || (reinterpret_cast<uintptr_t>(workspace) & 15))
        return FASTLSH_EINVAL;
    return launch_build_tables(keys, L, N, ldk, sorted_keys, ids, bucket_start,
                               reinterpret_cast<long long*>(nbuckets), workspace, s);
}

fastlsh_status fastlsh_query_workspace(int64_t N, int64_t nq, size_t* bytes) {
    if (N < 0 || nq < 0 || !bytes) return FASTLSH_EINVAL;
    *bytes = query_workspace_bytes(N, query_grid(nq));
    return FASTLSH_OK;
}

fastlsh_status fastlsh_query(const float* X, int64_t N, int32_t n, const uint64_t* sorted_keys,
                             const uint32_t* ids, int32_t L, const float* Q, const uint64_t* qkeys, int64_t nq,
                             int64_t ldq, int32_t topk, int32_t* out_ids, float* out_dist, int64_t* out_ncand,
                             void* workspace, size_t workspace_bytes, fastlsh_stream_t stream) {
    if (N < 0 || N >= 0xffffffffLL || n < 1 || L < 1 || L > 4096 || nq < 0 || ldq < nq || topk < 1 ||
        topk > 32)
        return FASTLSH_EINVAL;
    if (nq == 0) return FASTLSH_OK;
    if (!Q || !qkeys || !out_ids || !out_dist || !out_ncand || (N > 0 && (!X || !sorted_keys || !ids)) ||
        (reinterpret_cast<uintptr_t>(qkeys) & 7) || (reinterpret_cast<uintptr_t>(sorted_keys) & 7) ||
        (reinterpret_cast<uintptr_t>(out_ncand) & 7) || (reinterpret_cast<uintptr_t>(X) & 3) ||
        (reinterpret_cast<uintptr_t>(Q) & 3))
        return FASTLSH_EINVAL;
    if ((size_t)((n + 3) & ~3) * 4 + (size_t)L * 16 > 200 * 1024) return FASTLSH_EUNSUPPORTED;
    int dev = 0;
    fastlsh_status st = current_device(&dev);
    if (st != FASTLSH_OK) return st;
    st = check_sm100(dev);
    if (st != FASTLSH_OK) return st;
    if (!workspace || workspace_bytes < query_workspace_bytes(N, query_grid(nq))) return FASTLSH_EINVAL;
    return launch_query(X, N, n, sorted_keys, ids, L, Q, qkeys, nq, ldq, topk, out_ids, out_dist,
                        reinterpret_cast<long long*>(out_ncand), workspace, reinterpret_cast<cudaStream_t>(stream));
}

static fastlsh_status transform_checks(const float* X, int64_t N, int32_t n, const void* out) {
    if (N < 0 || n < 1) return FASTLSH_EINVAL;
    if (N > 0 && (!X || !out || (reinterpret_cast<uintptr_t>(X) & 3) || (reinterpret_cast<uintptr_t>(out) & 3)))
        return FASTLSH_EINVAL;
    int dev = 0;
    fastlsh_status st = current_device(&dev);
    if (st != FASTLSH_OK) return st;
    return check_sm100(dev);
}

fastlsh_status fastlsh_normalize_rows(const float* X, int64_t N, int32_t n, float* out, fastlsh_stream_t stream) {
    fastlsh_status st = transform_checks(X, N, n, out);
    if (st != FASTLSH_OK || N == 0) return st;
    return launch_normalize(X, N, n, out, reinterpret_cast<cudaStream_t>(stream));
}

fastlsh_status fastlsh_max_row_norm(const float* X, int64_t N, int32_t n, float* kappa, fastlsh_stream_t stream) {
    if (!kappa || (reinterpret_cast<uintptr_t>(kappa) & 3)) return FASTLSH_EINVAL;
    fastlsh_status st = transform_checks(X, N, n, kappa);
    if (st != FASTLSH_OK) return st;
    return launch_max_norm(X, N, n, kappa, reinterpret_cast<cudaStream_t>(stream));
}

fastlsh_status fastlsh_mips_transform(const float* X, int64_t N, int32_t n, const float* kappa, int32_t is_query,
                                      float* out, fastlsh_stream_t stream) {
    if (!is_query && (!kappa || (reinterpret_cast<uintptr_t>(kappa) & 3))) return FASTLSH_EINVAL;
    fastlsh_status st = transform_checks(X, N, n, out);
    if (st != FASTLSH_OK || N == 0) return st;
    return launch_mips(X, N, n, kappa, is_query ? 1 : 0, out, reinterpret_cast<cudaStream_t>(stream));
}

fastlsh_status fastlsh_hash_keys(const fastlsh_params* p, const fastlsh_keys* ks, const float* X,
                                 int64_t N, int32_t* codes, uint64_t* keys_out, int64_t ldk,
                                 fastlsh_stream_t stream) {
    if (!ks || !keys_out) return fastlsh_hash(p, X, N, codes, stream);
    if (!p || N < 0 || (int64_t)ks->L * ks->K > p->k) return FASTLSH_EINVAL;
    if (N == 0) return FASTLSH_OK;
    if (!X || ldk < N || (reinterpret_cast<uintptr_t>(X) & 3) || (reinterpret_cast<uintptr_t>(codes) & 3) ||
        (reinterpret_cast<uintptr_t>(keys_out) & 7))
        return FASTLSH_EINVAL;
    int dev = 0;
    fastlsh_status st = ready_params(p, &dev);
    if (st != FASTLSH_OK) return st;
    // dense path (kernel 5): codes from the GEMM, keys from them (keys only needs a gather kernel)
    if (codes && dense_selected(p)) {
        st = fastlsh_hash(p, X, N, codes, stream);
        if (st != FASTLSH_OK) return st;
        return fastlsh_build_keys(ks, codes, N, p->k, keys_out, ldk, stream);
    }
    // K1j: codes and keys in one launch, keys accumulated in registers; codes optional
    if (jit_selected(p)) {
        const uint64_t* dr = nullptr;
        st = keys_device(ks, dev, &dr);
        if (st != FASTLSH_OK) return st;
        st = jit::launch(p, p->dev[dev], X, N, codes, nullptr, ks, dr, keys_out, ldk, reinterpret_cast<cudaStream_t>(stream));
        if (st != FASTLSH_EUNSUPPORTED || p->kernel == 4) return st;
    }
    // K1r (hash blocks on table boundaries): keys built from the code tile in shared memory; codes not written
    // when codes == NULL. Falls through when K1r cannot serve the call.
    if (rows_selected(p) && (p->table_align <= 1 || p->table_align == ks->K) &&
        rows_keys_fusable(p->rpack, ks->L, ks->K) && (!codes || rows_keys_pay(p, ks))) {
        const uint64_t* dr = nullptr;
        st = keys_device(ks, dev, &dr);
        if (st != FASTLSH_OK) return st;
        FusedKeys fk{dr, ks->L, ks->K, keys_out, ldk};
        st = launch_gather_rows(p, p->dev[dev], X, N, codes, nullptr, reinterpret_cast<cudaStream_t>(stream), &fk);
        if (st != FASTLSH_EUNSUPPORTED) return st;
    }
    const bool fusable = keys_fusable(p, ks) && !tmem_selected(p);
    if (!codes && !fusable) return FASTLSH_EINVAL;  // keys only needs the fused kernel
    if (fusable) {  // keys built in K1's epilogue (codes not written when codes == NULL)
        const uint64_t* dr = nullptr;
        st = keys_device(ks, dev, &dr);
        if (st != FASTLSH_OK) return st;
        FusedKeys fk{dr, ks->L, ks->K, keys_out, ldk};
        return launch_gather(p, p->dev[dev], X, N, codes, nullptr, reinterpret_cast<cudaStream_t>(stream), &fk);
    }
    st = fastlsh_hash(p, X, N, codes, stream);
    if (st != FASTLSH_OK) return st;
    return fastlsh_build_keys(ks, codes, N, p->k, keys_out, ldk, stream);
}

fastlsh_status fastlsh_hash_keys_multicast(const fastlsh_params* p, const fastlsh_keys* ks, const float* X,
                                           int64_t N, int32_t* codes, uint64_t* keys_mc, int64_t ldk,
                                           fastlsh_stream_t stream) {
    if (!p || !ks || N < 0 || (int64_t)ks->L * ks->K > p->k) return FASTLSH_EINVAL;
    if (N == 0) return FASTLSH_OK;
    if (!X || !keys_mc || ldk < N || (reinterpret_cast<uintptr_t>(keys_mc) & 7)) return FASTLSH_EINVAL;
    int dev = 0;
    fastlsh_status st = ready_params(p, &dev);
    if (st != FASTLSH_OK) return st;
    if (!jit_selected(p)) return FASTLSH_EUNSUPPORTED;  // only K1j stores keys with multimem.st
    const uint64_t* dr = nullptr;
    st = keys_device(ks, dev, &dr);
    if (st != FASTLSH_OK) return st;
    return jit::launch(p, p->dev[dev], X, N, codes, nullptr, ks, dr, keys_mc, ldk,
                       reinterpret_cast<cudaStream_t>(stream), true);
}

fastlsh_status fastlsh_params_prepare(const fastlsh_params* p, const fastlsh_keys* ks, int32_t what) {
    if (!p || what < 0 || what > 7) return FASTLSH_EINVAL;
    if (!jit_selected(p)) return FASTLSH_OK;  // nothing to compile: K1r / K1 are built in
    fastlsh_status st = FASTLSH_OK;
    if ((what & 1) && (st = jit::prepare(p, 0, nullptr)) != FASTLSH_OK) return st;
    if ((what & 2) && (st = jit::prepare(p, 1, nullptr)) != FASTLSH_OK) return st;
    if ((what & 4) && ks && (st = jit::prepare(p, 0, ks)) != FASTLSH_OK && st != FASTLSH_EUNSUPPORTED) return st;
    return FASTLSH_OK;
}

fastlsh_status fastlsh_params_jit_check(const fastlsh_params* p, const fastlsh_keys* ks, int32_t what,
                                       double* compile_seconds, char* msg, int64_t msg_len) {
    if (!p || what < 0 || what > 31) return FASTLSH_EINVAL;
    std::string log;
    const fastlsh_status st = jit::compile_check(p, ks, what, compile_seconds, &log);
    if (msg && msg_len > 0) {
        const size_t n = log.size() < (size_t)msg_len - 1 ? log.size() : (size_t)msg_len - 1;
        std::memcpy(msg, log.data(), n);
        msg[n] = 0;
    }
    return st;
}

fastlsh_status fastlsh_params_jit_status(const fastlsh_params* p, double* compile_seconds, char* msg, int64_t msg_len) {
    if (!p) return FASTLSH_EINVAL;
    std::lock_guard<std::mutex> g(p->jit.mu);
    if (compile_seconds) *compile_seconds = p->jit.compile_seconds;
    if (msg && msg_len > 0) {
        const size_t n = p->jit.last_error.size() < (size_t)msg_len - 1 ? p->jit.last_error.size() : (size_t)msg_len - 1;
        std::memcpy(msg, p->jit.last_error.data(), n);
        msg[n] = 0;
    }
    return FASTLSH_OK;
}

fastlsh_status fastlsh_read_flags(const fastlsh_params* p, uint64_t* nonfinite,
                                  uint64_t* saturated, int32_t reset, fastlsh_stream_t stream) {
    int dev = 0;
    fastlsh_status st = ready_params(p, &dev);
    if (st != FASTLSH_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    unsigned long long h[2] = {0, 0};
    FL_CUDA(cudaMemcpyAsync(h, p->dev[dev].flags, sizeof(h), cudaMemcpyDeviceToHost, s));
    FL_CUDA(cudaStreamSynchronize(s));
    if (reset) {
        FL_CUDA(cudaMemsetAsync(p->dev[dev].flags, 0, sizeof(h), s));
        FL_CUDA(cudaStreamSynchronize(s));
    }
    if (nonfinite) *nonfinite = h[0];
    if (saturated) *saturated = h[1];
    return FASTLSH_OK;
}

// Host-buffer pipeline: chunk i is copied H2D on stream s[i%2], hashed (+keys) there, and its
// results copied D2H on the same stream; the two streams overlap copy with compute. The host
// buffers are used in place (pinned memory gives true async copies; pageable memory still works).
fastlsh_status fastlsh_hash_host(fastlsh_params* p, const fastlsh_keys* ks, const float* X_host,
                                 int64_t N, int32_t* codes_host, uint64_t* keys_host,
                                 int64_t chunk_rows) {
    if (!p || N < 0 || chunk_rows <= 0) return FASTLSH_EINVAL;
    if (N == 0) return FASTLSH_OK;
    if (!X_host || (!codes_host && !(ks && keys_host))) return FASTLSH_EINVAL;  // codes optional with keys
    if (ks && keys_host && (int64_t)ks->L * ks->K > p->k) return FASTLSH_EINVAL;
    int dev = 0;
    fastlsh_status st = ready_params(p, &dev);
    if (st != FASTLSH_OK) return st;
    DeviceCopy& d = p->dev[dev];
    const bool want_keys = ks && keys_host;
    const int L = want_keys ? ks->L : 0;
    std::lock_guard<std::mutex> g(p->mu);
    if (d.ws_rows < chunk_rows || d.ws_L < L) {
        for (int i = 0; i < 2; ++i) {
            cudaFree(d.ws_x[i]); cudaFree(d.ws_codes[i]); cudaFree(d.ws_keys[i]);
            d.ws_x[i] = nullptr; d.ws_codes[i] = nullptr; d.ws_keys[i] = nullptr;
        }
        for (int i = 0; i < 2; ++i) {
            FL_CUDA(cudaMalloc(reinterpret_cast<void**>(&d.ws_x[i]), (size_t)chunk_rows * p->n * sizeof(float)));
            FL_CUDA(cudaMalloc(reinterpret_cast<void**>(&d.ws_codes[i]), (size_t)chunk_rows * p->k * sizeof(int32_t)));
            if (L > 0) FL_CUDA(cudaMalloc(reinterpret_cast<void**>(&d.ws_keys[i]), (size_t)chunk_rows * L * sizeof(uint64_t)));
            if (!d.ws_stream[i]) FL_CUDA(cudaStreamCreateWithFlags(&d.ws_stream[i], cudaStreamNonBlocking));
        }
        d.ws_rows = chunk_rows;
        d.ws_L = L;
    }
    const uint64_t* dr = nullptr;
    if (want_keys) {
        st = keys_device(ks, dev, &dr);
        if (st != FASTLSH_OK) return st;
    }
    const bool dense = dense_selected(p);  // the GEMM makes the codes, K3 the keys
    const bool fuse = want_keys && !dense && keys_fusable(p, ks) && !tmem_selected(p);
    const int64_t nchunks = (N + chunk_rows - 1) / chunk_rows;
    for (int64_t c = 0; c < nchunks; ++c) {
        const int b = (int)(c & 1);
        cudaStream_t s = d.ws_stream[b];
        const int64_t r0 = c * chunk_rows;
        const int64_t rows = (N - r0 < chunk_rows) ? N - r0 : chunk_rows;
        FL_CUDA(cudaMemcpyAsync(d.ws_x[b], X_host + r0 * p->n, (size_t)rows * p->n * sizeof(float),
                                cudaMemcpyHostToDevice, s));
        bool fused_here = false;
        if (want_keys && jit_selected(p)) {  // codes not wanted on the host: they never leave the SM
            st = jit::launch(p, d, d.ws_x[b], rows, codes_host ? d.ws_codes[b] : nullptr, nullptr, ks, dr, d.ws_keys[b],
                             rows, s);
            fused_here = st == FASTLSH_OK;
            if (st != FASTLSH_OK && st != FASTLSH_EUNSUPPORTED) return st;
        }
        if (!fused_here && want_keys && !dense && rows_selected(p) &&
            (p->table_align <= 1 || p->table_align == ks->K) && rows_keys_pay(p, ks)) {
            FusedKeys fk{dr, ks->L, ks->K, d.ws_keys[b], rows};
            st = launch_gather_rows(p, d, d.ws_x[b], rows, codes_host ? d.ws_codes[b] : nullptr, nullptr, s, &fk);
            fused_here = st == FASTLSH_OK;
            if (st != FASTLSH_OK && st != FASTLSH_EUNSUPPORTED) return st;
        }
        if (fused_here) {
        } else if (fuse) {
            FusedKeys fk{dr, ks->L, ks->K, d.ws_keys[b], rows};
            st = launch_gather(p, d, d.ws_x[b], rows, d.ws_codes[b], nullptr, s, &fk);
            fused_here = true;
        } else {
            st = launch_hash(p, d, d.ws_x[b], rows, d.ws_codes[b], nullptr, s);
        }
        if (st != FASTLSH_OK) return st;
        if (codes_host)
            FL_CUDA(cudaMemcpyAsync(codes_host + r0 * p->k, d.ws_codes[b], (size_t)rows * p->k * sizeof(int32_t),
                                    cudaMemcpyDeviceToHost, s));
        if (want_keys) {
            if (!fused_here) st = launch_build_keys(ks, dr, d.ws_codes[b], rows, p->k, d.ws_keys[b], rows, s);
            if (st != FASTLSH_OK) return st;
            // keys of this chunk: [L][rows] on device -> columns r0.. of the [L][N] host matrix
            FL_CUDA(cudaMemcpy2DAsync(keys_host + r0, (size_t)N * sizeof(uint64_t), d.ws_keys[b],
                                      (size_t)rows * sizeof(uint64_t), (size_t)rows * sizeof(uint64_t), L,
                                      cudaMemcpyDeviceToHost, s));
        }
    }
    FL_CUDA(cudaStreamSynchronize(d.ws_stream[0]));
    FL_CUDA(cudaStreamSynchronize(d.ws_stream[1]));
    return FASTLSH_OK;
}

}  // extern "C"
