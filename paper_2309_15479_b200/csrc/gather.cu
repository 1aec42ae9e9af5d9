// gather.cu — K1/K2: FastLSH sampled-projection hashing on sm_100a.
//
// For every row v and hash i: h_i(v) = floor((a_i . S_i(v) + b_i) / w)   (Eq. 5).
//
// Design:
//  * One CTA owns a block of hashes; its lanes hold their hash part's slots in registers for the
//    whole kernel: MS 32-bit smem byte offsets and MS f32 coefficients, in the bank-scheduled
//    order produced by packer.cpp.
//  * Rows are processed 4 at a time. A stage holds 4 rows column-interleaved: the 16-byte chunk
//    at position pos(c) = (c%4)*nq + c/4 is (x0[c], x1[c], x2[c], x3[c]). One LDS.128 per slot
//    therefore gathers the sampled coordinate of 4 rows, and one FFMA per row accumulates it.
//    The packer guarantees the 8 lanes of each quarter-warp hit 8 distinct bank groups at every
//    slot position, so each LDS.128 costs the ideal 4 wavefronts (32 gathers per wavefront).
//  * Stages are double buffered: before gathering from stage j the CTA issues 4-byte cp.async
//    copies of group j+1 straight into their transposed positions of the other stage (no
//    registers held across the gather loop); they are waited for just before the stage barrier.
//  * Epilogue (fused): lanes deposit their 4 partial projections; after one CTA barrier each
//    thread takes a hash, sums its parts in fixed order for the 4 rows, adds b (__fadd_rn),
//    divides by w (__fdiv_rn), floors toward -inf and writes int32 codes (coalesced over hashes).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "internal.h"

namespace fastlsh {
namespace {

constexpr int kBatch = 4;  // float4 staging loads held in registers per thread

struct GatherArgs {
    const float* X;
    long long N;
    int n, nq, stage_chunks;
    const uint32_t* offp;
    const float* coef;
    const uint16_t* unit_lane;
    const float* b;
    const int* block_h0;
    const int* block_kb;
    float w;
    int k, P, W, HB, kb_max;
    long long groups;
    int32_t* codes;
    float* proj;
    unsigned long long* flags;
    int vec4;
};

__device__ __forceinline__ float4 lds128(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr));
    return v;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// Load float4 item `it` (row r = it % 4, quad q = it / 4) of the group starting at row `row0`.
__device__ __forceinline__ float4 load_item(const GatherArgs& a, long long row0, int it) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const int r = it & 3, q = it >> 2;
    const long long row = row0 + r;
    if (row < a.N) {
        const float* src = a.X + row * a.n;
        if (a.vec4) {
            v = __ldg(reinterpret_cast<const float4*>(src) + q);
        } else {
            const int c = 4 * q;
            v.x = (c + 0 < a.n) ? __ldg(src + c + 0) : 0.f;
            v.y = (c + 1 < a.n) ? __ldg(src + c + 1) : 0.f;
            v.z = (c + 2 < a.n) ? __ldg(src + c + 2) : 0.f;
            v.w = (c + 3 < a.n) ? __ldg(src + c + 3) : 0.f;
        }
    }
    return v;
}

// Column 4q+i of row r goes to chunk i*nq+q, component r.
__device__ __forceinline__ void store_item(float* stage, int nq, int it, const float4 v) {
    const int r = it & 3, q = it >> 2;
    float* d = stage + q * 4 + r;
    d[0 * 4 * nq] = v.x;
    d[1 * 4 * nq] = v.y;
    d[2 * 4 * nq] = v.z;
    d[3 * 4 * nq] = v.w;
}

// Items beyond the register batch (large n): synchronous load + store.
__device__ __forceinline__ void stage_rest(const GatherArgs& a, long long row0, float* stage, int from) {
    const int items = 4 * a.nq;
    for (int it = from; it < items; it += blockDim.x) store_item(stage, a.nq, it, load_item(a, row0, it));
}

// Asynchronous transposing stage fill: every float of the 4 rows is copied global -> shared by
// a 4-byte cp.async straight into its interleaved position (no registers held across the gather
// loop; rows past N and columns past n are zero-filled by the src-size operand).
__device__ __forceinline__ void cp_async4(uint32_t dst, const float* src, uint32_t src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void stage_async(const GatherArgs& a, long long row0, uint32_t stage_u32) {
    const int items = 4 * a.nq;
    const int nq4 = 16 * a.nq;  // bytes between the 4 column components of an item
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
        const int r = it & 3, q = it >> 2;
        const long long row = row0 + r;
        const bool live = row < a.N;
        const float* src = a.X + (live ? row : 0) * (long long)a.n + 4 * q;
        const uint32_t dst = stage_u32 + (uint32_t)(q * 16 + r * 4);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const bool ok = live && (4 * q + i < a.n);
            cp_async4(dst + i * nq4, ok ? src + i : a.X, ok ? 4u : 0u);
        }
    }
    cp_async_commit();
}

template <int MS>
__global__ void __launch_bounds__(256, (MS <= 32 ? 2 : 1)) gather_kernel(const GatherArgs a) {
    extern __shared__ __align__(128) float4 smem[];
    const int SC = a.stage_chunks;
    float4* part = smem + 2 * SC;  // [2][W*32]
    uint16_t* s_unit = reinterpret_cast<uint16_t*>(part + 2 * a.W * 32);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nthreads = blockDim.x;
    const int hb = blockIdx.x % a.HB;
    const long long gpr = gridDim.x / a.HB;
    const long long rs = blockIdx.x / a.HB;
    const int kb = a.block_kb[hb];
    const int h0 = a.block_h0[hb];
    const int P = a.P;
    float* s_b = reinterpret_cast<float*>(s_unit + ((a.kb_max * P + 1) & ~1));
    const int items = 4 * a.nq;

    // zero chunks (padding slots read these), hash metadata
    for (int i = tid; i < 2 * kPadChunks; i += nthreads)
        smem[(i / kPadChunks) * SC + 4 * a.nq + (i % kPadChunks)] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = tid; i < kb * P; i += nthreads)
        s_unit[i] = a.unit_lane[(size_t)hb * a.kb_max * P + i];
    for (int i = tid; i < kb; i += nthreads) s_b[i] = a.b[h0 + i];

    // this lane's slots: byte offsets into a stage and coefficients
    uint32_t op[MS];
    float cf[MS];
    {
        const size_t wl = (size_t)hb * a.W + warp;
        const uint32_t* po = a.offp + wl * MS * 32 + lane;
        const float* pc = a.coef + wl * MS * 32 + lane;
#pragma unroll
        for (int t = 0; t < MS; ++t) op[t] = __ldg(po + t * 32);
#pragma unroll
        for (int t = 0; t < MS; ++t) cf[t] = __ldg(pc + t * 32);
    }

    const uint32_t stage0_u32 = smem_u32(smem);
    const uint32_t stage_bytes = (uint32_t)SC * 16u;
    long long g = rs;
    if (g < a.groups) stage_async(a, g * 4, stage0_u32);
    cp_async_wait_all();
    __syncthreads();

    const float w = a.w;
    const float inv_w = 1.0f / w;
    const bool w_pow2 = (__float_as_uint(w) & 0x007fffffu) == 0 && isfinite(inv_w) && inv_w != 0.0f;
    int j = 0;
    for (; g < a.groups; g += gpr, ++j) {
        const long long gn = g + gpr;
        const bool has_next = gn < a.groups;
        // next group's rows stream into the other stage while this one is gathered
        if (has_next) stage_async(a, gn * 4, stage0_u32 + ((j + 1) & 1) * stage_bytes);

        // gather-FMA over the scheduled slots: 4 rows per LDS.128
        const uint32_t base = stage0_u32 + (j & 1) * stage_bytes;
        float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
#pragma unroll
        for (int t = 0; t < MS; t += 2) {
            const float4 v0 = lds128(base + op[t]);
            const float4 v1 = lds128(base + op[t + 1]);
            acc0 = fmaf(v0.x, cf[t], acc0);
            acc1 = fmaf(v0.y, cf[t], acc1);
            acc2 = fmaf(v0.z, cf[t], acc2);
            acc3 = fmaf(v0.w, cf[t], acc3);
            acc0 = fmaf(v1.x, cf[t + 1], acc0);
            acc1 = fmaf(v1.y, cf[t + 1], acc1);
            acc2 = fmaf(v1.z, cf[t + 1], acc2);
            acc3 = fmaf(v1.w, cf[t + 1], acc3);
        }
        part[(j & 1) * a.W * 32 + tid] = make_float4(acc0, acc1, acc2, acc3);
        cp_async_wait_all();
        __syncthreads();

        // epilogue: one hash per thread, its parts summed in fixed order for the 4 rows
        const float4* pb = part + (j & 1) * a.W * 32;
        const long long row0 = g * 4;
        const int nrows = (int)((a.N - row0) < 4 ? (a.N - row0) : 4);
        for (int h = tid; h < kb; h += nthreads) {
            float4 s = pb[s_unit[h * P]];
            for (int q = 1; q < P; ++q) {
                const float4 v = pb[s_unit[h * P + q]];
                s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
            }
            const float pr[4] = {s.x, s.y, s.z, s.w};
            const long long o0 = row0 * a.k + h0 + h;
            if (a.proj) {
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    if (r < nrows) a.proj[o0 + (long long)r * a.k] = pr[r];
            } else {
                const float bh = s_b[h];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    if (r >= nrows) break;
                    // w a power of two: x * (1/w) is exact, so it equals the IEEE quotient
                    const float num = __fadd_rn(pr[r], bh);
                    const float qv = w_pow2 ? __fmul_rn(num, inv_w) : __fdiv_rn(num, w);
                    const float f = floorf(qv);
                    int code = (int)f;
                    if (!(f > -2147483648.0f && f < 2147483648.0f)) {
                        code = INT_MIN;
                        atomicAdd(a.flags + (isfinite(qv) ? 1 : 0), 1ull);
                    }
                    a.codes[o0 + (long long)r * a.k] = code;
                }
            }
        }
    }
}

typedef void (*KernelFn)(GatherArgs);

template <int MS>
KernelFn kernel_for() { return gather_kernel<MS>; }

KernelFn select_kernel(int MS) {
    switch (MS) {
#define FASTLSH_CASE(X) case X: return kernel_for<X>();
        FASTLSH_CASE(2) FASTLSH_CASE(4) FASTLSH_CASE(6) FASTLSH_CASE(8) FASTLSH_CASE(10)
        FASTLSH_CASE(12) FASTLSH_CASE(14) FASTLSH_CASE(16) FASTLSH_CASE(18) FASTLSH_CASE(20)
        FASTLSH_CASE(22) FASTLSH_CASE(24) FASTLSH_CASE(26) FASTLSH_CASE(28) FASTLSH_CASE(30)
        FASTLSH_CASE(32) FASTLSH_CASE(34) FASTLSH_CASE(36) FASTLSH_CASE(38) FASTLSH_CASE(40)
        FASTLSH_CASE(42) FASTLSH_CASE(44) FASTLSH_CASE(46) FASTLSH_CASE(48) FASTLSH_CASE(50)
        FASTLSH_CASE(52) FASTLSH_CASE(54) FASTLSH_CASE(56) FASTLSH_CASE(58) FASTLSH_CASE(60)
        FASTLSH_CASE(62) FASTLSH_CASE(64)
#undef FASTLSH_CASE
        default: return nullptr;
    }
}

}  // namespace

fastlsh_status launch_gather(const fastlsh_params* p, const DeviceCopy& d, const float* X,
                             int64_t N, int32_t* codes, float* proj, cudaStream_t stream) {
    const Packing& pk = p->pack;
    KernelFn fn = select_kernel(pk.slots);
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
    a.W = pk.warps;
    a.HB = pk.hash_blocks;
    a.kb_max = pk.kb_max;
    a.groups = (N + 3) / 4;
    a.codes = codes;
    a.proj = proj;
    a.flags = d.flags;
    a.vec4 = (p->n % 4 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);

    const int threads = pk.warps * 32;
    const size_t smem = (size_t)2 * pk.stage_chunks * 16 + (size_t)2 * pk.warps * 32 * 16 +
                        (size_t)(((pk.kb_max * pk.parts + 1) & ~1) * 2) + (size_t)pk.kb_max * 4;
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_cuda_error(e);
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

}  // namespace fastlsh
