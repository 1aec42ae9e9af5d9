// jit.cpp — K1j: the params-specialised, lane = row hashing kernel, generated at params upload
// and compiled with NVRTC.
//
// For every row v and hash i: h_i(v) = floor((a_i . S_i(v) + b_i) / w)   (Eq. 5).
//
// Why: K1r/K1 read every sampled coordinate from shared memory (one 128-B wavefront per 32
// gathers), which bounds them at G_s = 9.3e12 gathers/s. For short rows (n <= 128: C0, C3) a whole
// row fits in a thread's registers, and once the params are fixed the sampled index set S_i is a
// compile-time constant: x[idx[i][j]] becomes a register operand and a[i][j], b[i] become
// instruction immediates. The gather then costs no shared-memory wavefront at all — one FFMA per
// sampled coordinate (O(m) per hash) — and the kernel is bound by instruction issue
// or by HBM (reading X, writing codes and keys), not by the shared-memory pipe.
//
// Kernel (one generated module per params object; one warp = 32 rows, lane = row):
//  * stage: TMA 2D tensor loads of the warp's 32-row tile of X as boxes of 32 rows x 32 floats
//    with the 128-byte swizzle (one box per 32 coordinates), complete_tx on a per-warp mbarrier;
//    lane t reads its row with LDS.128 at chunk (c ^ (t & 7)) — conflict-free quarter-warps. The
//    next tile's copy is issued as soon as the row is in registers (one stage per warp suffices:
//    a tile's compute is thousands of cycles).
//  * sample + project: per hash, p = x[i0]*a0 then fma(x[ij], aj, p) in the paper's slot order,
//    all straight-line code with immediate coefficients (fp32; parity bound as K1r's, m <= 128
//    terms: m * 2^-24 * ||a|| ||S(v)||).
//  * quantise: __fadd_rn(p, b), then * (1/w) (w a power of two: exact) or IEEE / w, F2I.FLOOR.
//    Out-of-range / non-finite quotients are detected by a per-lane flag; a warp with a flagged
//    row re-runs those rows in a generic slow path (canonical params from global memory, the same
//    operation sequence, so bit-identical values) which writes INT32_MIN and counts the flags.
//  * codes: every 32 hashes, a lane writes its 32 codes into a swizzled shared-memory box and one
//    lane issues a TMA tensor store (bulk_group, ring of NCB boxes); rows past N and hashes past k
//    are clipped by the tensor map.
//  * compound keys (R9), when a keys object is fused: the codes of table l
//    (hashes [lK, lK+K)) are accumulated as they are produced — three IMAD.WIDE.U32 with 21-bit
//    limbs of r[l][j+1] (kernel-parameter operands) — and key_l(v) = (r_{l,0} + S0 + S1*2^21 +
//    S2*2^42) mod 2^61-1 is stored as one coalesced 256-byte run per warp and table. Codes may
//    then stay on chip (keys only: X in, keys out).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

namespace fastlsh {
namespace jit {

// ------------------------------------------------------------------------------------------
// source generation
// ------------------------------------------------------------------------------------------

namespace {

void add_float(std::string& s, float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    char buf[48];
    std::snprintf(buf, sizeof buf, "__uint_as_float(0x%08xu)", u);
    s += buf;
}

void add_int(std::string& s, long long v) { s += std::to_string(v); }

bool pow2_w(float w) {
    uint32_t u;
    std::memcpy(&u, &w, 4);
    const float inv = 1.0f / w;
    return (u & 0x007fffffu) == 0 && std::isfinite(inv) && inv != 0.0f;
}

const char* kPrelude = R"FL(
typedef unsigned long long u64;
typedef unsigned int u32;
struct __align__(64) TMap { u64 v[16]; };
struct JArgs {
    long long N, tiles;
    int write_out;          // 0: keys only, the codes never leave the SM
    int* out;               // codes / projections [N][k] (slow path only; the fast path uses omap)
    u64* keys;              // [L][ldk]
    long long ldk, col0;
    u64* flags;             // [0] non-finite, [1] saturated
    const int* idx;         // canonical params [k][m], [k][m], [k] (slow path)
    const float* a;
    const float* b;
    const u64* kr;          // key multipliers [L][K+1] (slow path)
};
#define P61 ((1ull << 61) - 1ull)
__device__ __forceinline__ u64 mod61(u64 x) { x = (x & P61) + (x >> 61); return x >= P61 ? x - P61 : x; }
__device__ __forceinline__ u64 rotl61(u64 x, int j) { return ((x << j) & P61) | (x >> (61 - j)); }
__device__ __forceinline__ u32 su32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u32 bar, u32 c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(u32 bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(u32 bar, u32 ph) {
    asm volatile("{\n\t.reg .pred p;\nFLW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra FLW_%=;\n}"
                 ::"r"(bar), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma_load(u32 dst, const TMap* m, int x, int y, u32 bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(dst), "l"((u64)m), "r"(x), "r"(y), "r"(bar) : "memory");
}
__device__ __forceinline__ void tma_store(const TMap* m, u32 src, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];"
                 ::"l"((u64)m), "r"(src), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_ring() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(FL_NCB - 1) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// A compound key leaves either as a plain store into this GPU's [L][ldk] table or, with FL_MC, as a
// multimem store to the multicast address of a table replicated on every GPU of the NVLink domain
// (NVSwitch multicast: the key all-gather of SURVEY.md §8(a) a8 happens inside the hashing kernel).
__device__ __forceinline__ void key_store(u64* p, u64 key) {
#if FL_MC
    asm volatile("multimem.st.global.b64 [%0], %1;" ::"l"(p), "l"(key) : "memory");
#else
    *p = key;
#endif
}
// the fast path's form: one predicated store (rows past N skip it) instead of a branch per table
__device__ __forceinline__ void key_store_if(u32 live, u64* p, u64 key) {
#if FL_MC
    asm volatile("{\n\t.reg .pred kp;\n\tsetp.ne.b32 kp, %2, 0;\n\t@kp multimem.st.global.b64 [%0], %1;\n\t}"
                 ::"l"(p), "l"(key), "r"(live) : "memory");
#else
    asm volatile("{\n\t.reg .pred kp;\n\tsetp.ne.b32 kp, %2, 0;\n\t@kp st.global.b64 [%0], %1;\n\t}"
                 ::"l"(p), "l"(key), "r"(live) : "memory");
#endif
}

// Codes leave in groups of 32 hashes: a swizzled 32 x 32 box of the warp's ring, written 4 codes
// (one STS.128) at a time as they are produced, then one TMA tensor store per group.
__device__ __forceinline__ void group_begin(int lane) {
    if (lane == 0) bulk_wait_read_ring();  // the store that last read this ring box has read it
    __syncwarp();
}
__device__ __forceinline__ void put4(unsigned char* box_lane, u32 q, u32 sw, int c0, int c1, int c2, int c3) {
    *reinterpret_cast<int4*>(box_lane + ((q << 4) ^ sw)) = make_int4(c0, c1, c2, c3);
}
// Paired form (k % 32 == 0): the codes are viewed as a 3D tensor [N rows][k/32 groups][32 codes] and
// two consecutive groups leave in one box {32 codes, 2 groups, 32 rows} (8 KB, the whole ring), so each
// row gets 256 contiguous bytes per store instead of 128 (tools/microbench_wpattern.cu: 128-B
// segments at 1-KB stride reach 5.1-5.4 TB/s with 512 B/row of reads, 256-B segments 5.8).
// Box layout with the 128-B swizzle: flattened 128-B line f = 2 * row + group, chunk c at
// f * 128 + ((c ^ (f & 7)) << 4).
__device__ __forceinline__ void tma_store3(const TMap* m, u32 src, int x, int y, int z) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];"
                 ::"l"((u64)m), "r"(src), "r"(x), "r"(y), "r"(z) : "memory");
}
__device__ __forceinline__ void pair_begin(int lane) {
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // the previous pair is read
    __syncwarp();
}
__device__ __forceinline__ void pair_end(u32 cring_s, int lane, const TMap* om, int g0, long long t) {
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
        tma_store3(om, cring_s, 0, g0, (int)(32 * t));
        bulk_commit();
    }
}
__device__ __forceinline__ void group_end(u32 cring_s, int& cbi, int lane, const TMap* om, int g, long long t) {
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
        tma_store(om, cring_s + cbi * 4096, 32 * g, (int)(32 * t));
        bulk_commit();
    }
    cbi = cbi + 1 == FL_NCB ? 0 : cbi + 1;
}

// Generic path for a row with a flagged hash (non-finite or out-of-int32 quotient): the same
// operation sequence as the generated code (so bit-identical values), INT32_MIN + flag counts,
// codes rewritten in global memory, keys recomputed from the corrected codes.
__device__ __noinline__ void fix_row(const JArgs& a, float* scr, long long row, int lane) {
    int* sc = reinterpret_cast<int*>(scr + FL_N);
    for (int i = lane; i < FL_K; i += 32) {
        const int* id = a.idx + (long long)i * FL_M;
        const float* co = a.a + (long long)i * FL_M;
        float p = __fmul_rn(scr[id[0]], FL_COEF(co[0]));
        for (int j = 1; j < FL_M; ++j) p = __fmaf_rn(scr[id[j]], FL_COEF(co[j]), p);
        const float q = FL_Q(p, a.b[i]);
        int c = __float2int_rd(q);
        if (!(fabsf(q) < 2147483648.0f)) {
            c = (int)0x80000000;
            if (row < a.N) atomicAdd(a.flags + (isfinite(q) ? 1 : 0), 1ull);
        }
        sc[i] = c;
        if (a.write_out && row < a.N) a.out[row * FL_K + i] = c;
    }
    __syncwarp();
#if FL_L > 0
    for (int l = lane; l < FL_L; l += 32) {
        // the limb form of the generated code (exact for K <= 1024): S_q = sum limb_q(r) * u32(c).
        // (K1r's 128-bit lo/hi accumulation, written here first, gave wrong keys for K = 16 in this
        // NVRTC-compiled noinline function while exact for K <= 3 — not root-caused; the limb form is
        // the fast path's arithmetic and is verified by tests/test_gpu_jit.py flag tests.)
        const u64* rl = a.kr + l * (FL_KT + 1);
        u64 s0 = 0, s1 = 0, s2 = 0;
        for (int j = 0; j < FL_KT; ++j) {
            const u64 rv = rl[j + 1];
            const u64 u = (u32)sc[l * FL_KT + j];
            s0 += (rv & 0x1fffffull) * u;
            s1 += ((rv >> 21) & 0x1fffffull) * u;
            s2 += (rv >> 42) * u;
        }
        const u64 key = mod61(rl[0] + mod61(s0) + rotl61(mod61(s1), 21) + rotl61(mod61(s2), 42));
        if (row < a.N) key_store(a.keys + l * a.ldk + a.col0 + row, key);
    }
#endif
}
)FL";

// the per-tile prologue shared by both kernels: wait for the tile, load the lane's row into x[]
const char* kTileHead = R"FL(
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const u32 raw_s = su32(sm_raw);
    unsigned char* sm = sm_raw + (((raw_s + 1023u) & ~1023u) - raw_s);
    unsigned char* wb = sm + warp * FL_WB;
    unsigned char* cring = wb + FL_NBX * 4096;
    const u32 xs = su32(wb), cring_s = xs + FL_NBX * 4096;
    const u32 bar = su32(sm + FL_NW * FL_WB) + 8u * warp;
    if (lane == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    long long t = (long long)blockIdx.x * FL_NW + warp;
    const long long tstride = (long long)gridDim.x * FL_NW;
    if (lane == 0 && t < a.tiles) {
        mbar_expect(bar, FL_NBX * 4096);
#pragma unroll
        for (int bx = 0; bx < FL_NBX; ++bx) tma_load(xs + bx * 4096, &xmap, 32 * bx, (int)(32 * t), bar);
    }
    u32 ph = 0;
    int cbi = 0;  // ring box of the unpaired form
    (void)cbi;
    const u32 sw = (u32)(lane & 7) << 4;
    for (; t < a.tiles; t += tstride) {
        mbar_wait(bar, ph);
        ph ^= 1u;
        float x[FL_NX];
#pragma unroll
        for (int c = 0; c < FL_NX / 4; ++c) {
            const float4 v = *reinterpret_cast<const float4*>(wb + (c >> 3) * 4096 + lane * 128 + ((((u32)c & 7u) << 4) ^ sw));
            x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
        }
        __syncwarp();  // every lane's row is in registers: the stage may be refilled
        if (lane == 0 && t + tstride < a.tiles) {
            mbar_expect(bar, FL_NBX * 4096);
#pragma unroll
            for (int bx = 0; bx < FL_NBX; ++bx) tma_load(xs + bx * 4096, &xmap, 32 * bx, (int)(32 * (t + tstride)), bar);
        }
        const long long row = t * 32 + lane;
        (void)row;
)FL";

}  // namespace

// paired code stores (3D tensor map) need k % 32 == 0; FASTLSH_JIT_NOPAIR=1 keeps the 2D boxes
// (experiment knob, read once)
bool pair_stores(int k) {
    static const bool off = std::getenv("FASTLSH_JIT_NOPAIR") != nullptr;
    return k % 32 == 0 && !off;
}

std::string k1j_source(const Spec& s) {
    const int nbx = (s.n + 31) / 32;
    const int nx = (s.n + 3) / 4 * 4;
    const int wb = (nbx + s.ncb) * 4096;
    const int groups = (s.k + 31) / 32;
    const bool p2 = pow2_w(s.w);
    std::string src;
    src.reserve((size_t)s.k * s.m * 48 + 65536);
    auto def = [&](const char* name, long long v) {
        src += "#define ";
        src += name;
        src += " ";
        add_int(src, v);
        src += "\n";
    };
    src += "// K1j generated for n=" + std::to_string(s.n) + " m=" + std::to_string(s.m) + " k=" + std::to_string(s.k) +
           " (libfastlsh jit.cpp; DESIGN.md \"K1j\")\n";
    def("FL_N", s.n);
    def("FL_M", s.m);
    def("FL_K", s.k);
    def("FL_NX", nx);
    def("FL_NBX", nbx);
    def("FL_NW", s.warps);
    def("FL_NCB", s.ncb);
    def("FL_WB", wb);
    def("FL_L", s.L);
    def("FL_KT", s.K > 0 ? s.K : 1);
    def("FL_MC", s.mc ? 1 : 0);
    // Quantisation: q = (p + b) / w. For w a power of two, 1/w is folded into the
    // coefficients and b: every fp32 step then carries an exact power-of-two scale, so
    // fma-chain(a/w) + b/w == RN(p + b) / w bit for bit (outside subnormal / overflow ranges) and the
    // final multiply disappears. Otherwise IEEE division after the add, as in K1r.
    if (p2) {
        src += "#define FL_COEF(c) __fmul_rn((c), ";
        add_float(src, 1.0f / s.w);
        src += ")\n#define FL_Q(p, b) __fadd_rn((p), __fmul_rn((b), ";
        add_float(src, 1.0f / s.w);
        src += "))\n";
    } else {
        src += "#define FL_COEF(c) (c)\n#define FL_Q(p, b) __fdiv_rn(__fadd_rn((p), (b)), ";
        add_float(src, s.w);
        src += ")\n";
    }
    src += kPrelude;

    // One hash as one inline-PTX block: p in the paper's slot order with immediate coefficients,
    // then (codes) p + b, * 1/w or / w, floor. NVVM does not re-optimise asm: with plain C++
    // expressions the front end took ~14 s for the C3 shape, as asm ~2 s.
    auto hash_asm = [&](int i, const std::string& cj) {
        const int32_t* id = s.idx + (size_t)i * s.m;
        const float* co = s.a + (size_t)i * s.m;
        std::vector<int> ops;  // distinct coordinates -> asm operand numbers %1 ...
        std::vector<int> opnum(s.n, -1);
        for (int t = 0; t < s.m; ++t)
            if (opnum[id[t]] < 0) {
                opnum[id[t]] = (int)ops.size() + 1;
                ops.push_back(id[t]);
            }
        // codes: p and q live in a block-local register, only the code leaves; projections: p is %0
        const char* P = s.mode == 0 ? "q" : "%0";
        const float scale = (s.mode == 0 && p2) ? 1.0f / s.w : 1.0f;
        char buf[112];
        std::string h = s.mode == 0 ? "asm(\"{ .reg .f32 q; " : "{ float p; asm(\"";
        for (int t = 0; t < s.m; ++t) {
            const float c = co[t] * scale;  // exact: power-of-two scale
            uint32_t u;
            std::memcpy(&u, &c, 4);
            if (t == 0)
                std::snprintf(buf, sizeof buf, "mul.rn.f32 %s, %%%d, 0f%08X;", P, opnum[id[t]], u);
            else
                std::snprintf(buf, sizeof buf, " fma.rn.f32 %s, %%%d, 0f%08X, %s;", P, opnum[id[t]], u, P);
            h += buf;
        }
        if (s.mode == 0) {
            uint32_t ub, uw;
            if (p2) {
                const float bs = s.b[i] * scale;
                std::memcpy(&ub, &bs, 4);
                std::snprintf(buf, sizeof buf, " add.rn.f32 q, q, 0f%08X; cvt.rmi.s32.f32 %%0, q; }", ub);
            } else {
                std::memcpy(&ub, &s.b[i], 4);
                std::memcpy(&uw, &s.w, 4);
                std::snprintf(buf, sizeof buf, " add.rn.f32 q, q, 0f%08X; div.rn.f32 q, q, 0f%08X; cvt.rmi.s32.f32 %%0, q; }",
                              ub, uw);
            }
            h += buf;
            h += "\" : \"=r\"(" + cj + ") :";
        } else {
            h += "\" : \"=f\"(p) :";
        }
        for (size_t o = 0; o < ops.size(); ++o) {
            h += o ? ", " : " ";
            h += "\"f\"(x[" + std::to_string(ops[o]) + "])";
        }
        h += ");";
        if (s.mode == 1) h += " " + cj + " = __float_as_int(p); }";
        return h;
    };

    const bool keys = s.mode == 0 && s.L > 0;
    src += "\nextern \"C\" __global__ void __launch_bounds__(FL_NW * 32, 1)\n"
           "k1j(const __grid_constant__ TMap xmap, const __grid_constant__ TMap omap, const __grid_constant__ JArgs a) {\n";
    src += kTileHead;
    // Flags (codes mode): a per-row range check replaces a per-hash one. With a' = a (or a/w for a
    // power-of-two w) and S = sum_c |x_c| >= max_c |x_c|, every fp32 quotient obeys
    // |q_i| <= (1 + 1e-4) (A_i max|x| + |b'_i|) with A_i = sum_j |a'_ij|; a row whose fp32 S is below
    // T = (2^30 - max|b'|) / (1.01 max A_i) can therefore reach neither |q| >= 2^31 nor a non-finite
    // value, while NaN / Inf / huge inputs fail `S < T` and take the exact per-hash slow path.
    // (127 FADDs per row instead of k FSETPs.)
    if (s.mode == 0) {
        double amax = 0, bmax = 0;
        for (int i = 0; i < s.k; ++i) {
            double ai = 0;
            for (int j = 0; j < s.m; ++j) ai += std::fabs((double)s.a[(size_t)i * s.m + j]);
            amax = std::max(amax, ai / (p2 ? (double)s.w : 1.0));
            bmax = std::max(bmax, std::fabs((double)s.b[i]) / (p2 ? (double)s.w : 1.0));
        }
        // non-power-of-two w: q = (p + b) / w, so the bound is on |p + b| < 2^30 w
        const double lim = p2 ? 1073741824.0 : 1073741824.0 * (double)s.w;
        double T = amax > 0 ? (lim - bmax) / (1.01 * amax) : 3.0e38;
        if (!(T > 0)) T = 0;  // every row checked hash by hash
        float Tf = (float)T;
        if ((double)Tf > T) Tf = std::nextafter(Tf, 0.0f);
        // pairwise tree of |x_c| (coordinates past n are zero)
        std::vector<std::string> terms;
        for (int c = 0; c < s.n; ++c) terms.push_back("fabsf(x[" + std::to_string(c) + "])");
        while (terms.size() > 1) {
            std::vector<std::string> nx;
            for (size_t t = 0; t + 1 < terms.size(); t += 2) nx.push_back("(" + terms[t] + " + " + terms[t + 1] + ")");
            if (terms.size() & 1) nx.push_back(terms.back());
            terms.swap(nx);
        }
        src += "        const float sabs = " + terms[0] + ";\n        const bool bad = !(sabs < ";
        add_float(src, Tf);
        src += ");\n";
    }
    // codes stored (codes / projections) or kept on chip (keys only): a compile-time choice of the variant
    const bool store = s.mode == 1 || s.codes;
    const bool pair = pair_stores(s.k);  // 256-byte row segments per store (see pair_end)
    // quads of codes (4 per lane) computed before the wait for the pair box; FASTLSH_JIT_LATEWAIT
    // overrides (experiment knob). C3 chunk, codes + keys (tools/mb_jit.py): D = 0 2.70-2.72 ms, 1 2.63,
    // 2 2.59, 3 2.56, 4 2.58, 5 2.53, 6 2.51-2.52, 7 2.50, 8 (the whole group) 2.64 ms
    static const int late_depth = [] {
        const char* e = std::getenv("FASTLSH_JIT_LATEWAIT");
        return e ? std::atoi(e) : 7;
    }();
    if (keys) src += "        u64 s0, s1, s2;\n        const u32 live = row < a.N ? 1u : 0u;\n        u64* kp = a.keys + a.col0 + row;\n";
    char buf[160];
    for (int g = 0; g < groups; ++g) {
        if (!store)
            src += "        {\n";
        else if (!pair)
            src += "        {\n            group_begin(lane);\n"
                   "            unsigned char* box = cring + cbi * 4096 + lane * 128;\n";
        else
            src += std::string("        {\n") + ((g & 1) || late_depth > 0 ? "" : "            pair_begin(lane);\n") +
                   "            unsigned char* box = cring + lane * 256 + " + std::to_string((g & 1) * 128) + ";\n"
                   "            const u32 swp = (u32)((2 * lane + " + std::to_string(g & 1) + ") & 7) << 4;\n";
        // late wait (paired stores): the first D quads of a pair's first group are computed before the
        // wait for the pair box, their codes held in registers (e<q>_<r>), then stored
        const int nq = std::min(8, (s.k - 32 * g + 3) / 4);
        const int D = (store && pair && !(g & 1)) ? std::min(late_depth, nq) : 0;
        if (D) {
            src += "            int";
            for (int q = 0; q < D; ++q)
                for (int r = 0; r < 4; ++r) src += std::string(q || r ? ", " : " ") + "e" + std::to_string(q) + "_" + std::to_string(r);
            src += ";\n";
        }
        auto cname = [&](int q, int r) {
            return q < D ? "e" + std::to_string(q) + "_" + std::to_string(r) : "c" + std::to_string(r);
        };
        for (int q = 0; q < nq; ++q) {
            if (q >= D) src += "            { int c0, c1, c2, c3;\n";
            for (int j = 4 * q; j < 4 * q + 4; ++j) {
                const int i = 32 * g + j;
                src += "              " + hash_asm(i, cname(q, j & 3));
                if (keys && i < s.L * s.K) {
                    // key term (R9): the three 21-bit limbs of r[l][jj+1] (instruction
                    // immediates) times u32(code), exact 64-bit sums; S0 starts at r[l][0]
                    const int l = i / s.K, jj = i % s.K;
                    const uint64_t r = s.r[(size_t)l * (s.K + 1) + jj + 1];
                    if (jj == 0) {
                        std::snprintf(buf, sizeof buf, " s0 = 0x%llxull; s1 = 0; s2 = 0;",
                                      (unsigned long long)s.r[(size_t)l * (s.K + 1)]);
                        src += buf;
                    }
                    std::snprintf(buf, sizeof buf,
                                  " { const u64 u = (u32)%s; s0 += 0x%llxull * u; s1 += 0x%llxull * u; s2 += 0x%llxull * u; }",
                                  cname(q, j & 3).c_str(), (unsigned long long)(r & 0x1fffff), (unsigned long long)((r >> 21) & 0x1fffff),
                                  (unsigned long long)(r >> 42));
                    src += buf;
                    // key = (S0 + S1*2^21 + S2*2^42) mod 2^61-1 with S0 = r0 + ...: for K < 256, S1, S2 <
                    // K*2^53 < 2^61-1 are already reduced and S0 < 2^62, so one final reduction of a sum
                    // < 2^63 suffices
                    if (jj == s.K - 1) {
                        src += s.K < 256 ? "\n              { const u64 key = mod61(s0 + rotl61(s1, 21) + rotl61(s2, 42)); "
                                         : "\n              { const u64 key = mod61(mod61(s0) + rotl61(mod61(s1), 21) + "
                                           "rotl61(mod61(s2), 42)); ";
                        src += "key_store_if(live, kp + " + std::to_string(l) + "ll * a.ldk, key); }";
                    }
                }
                src += "\n";
            }
            if (q < D) {
                if (q == D - 1) {
                    src += "              pair_begin(lane);\n";  // the box is needed only now
                    for (int qq = 0; qq < D; ++qq)
                        src += "              put4(box, " + std::to_string(qq) + "u, swp, " + cname(qq, 0) + ", " + cname(qq, 1) +
                               ", " + cname(qq, 2) + ", " + cname(qq, 3) + ");\n";
                }
            } else {
                src += store ? "              put4(box, " + std::to_string(q) + (pair ? "u, swp" : "u, sw") + ", c0, c1, c2, c3); }\n"
                             : "              (void)c0; (void)c1; (void)c2; (void)c3; }\n";
            }
        }
        if (!store)
            src += "        }\n";
        else if (!pair)
            src += "            group_end(cring_s, cbi, lane, &omap, " + std::to_string(g) + ", t);\n        }\n";
        else if ((g & 1) || g == groups - 1)
            src += "            pair_end(cring_s, lane, &omap, " + std::to_string(g & ~1) + ", t);\n        }\n";
        else
            src += "        }\n";
    }
    if (s.mode == 0) {
        src += R"FL(
        if (__any_sync(0xffffffffu, bad)) {
            unsigned bm = __ballot_sync(0xffffffffu, bad);
            if (lane == 0) {
                bulk_wait_all();
                asm volatile("fence.proxy.async.global;" ::: "memory");
            }
            __syncwarp();
            float* scr = reinterpret_cast<float*>(cring);
            while (bm) {
                const int r = __ffs(bm) - 1;
                bm &= bm - 1;
#pragma unroll
                for (int c = 0; c < FL_N; ++c) {
                    const float v = __shfl_sync(0xffffffffu, x[c], r);
                    if (lane == 0) scr[c] = v;
                }
                __syncwarp();
                fix_row(a, scr, t * 32 + r, lane);
                __syncwarp();
            }
        }
)FL";
    }
    src += "    }\n    if (lane == 0) bulk_wait_all();\n}\n";
    return src;
}

// ------------------------------------------------------------------------------------------
// NVRTC (loaded at run time: without it K1j is simply unavailable and K1r serves the call)
// ------------------------------------------------------------------------------------------

namespace {

typedef int (*nvrtcCreateProgram_t)(void**, const char*, const char*, int, const char* const*, const char* const*);
typedef int (*nvrtcCompileProgram_t)(void*, int, const char* const*);
typedef int (*nvrtcGetSize_t)(void*, size_t*);
typedef int (*nvrtcGetBuf_t)(void*, char*);
typedef int (*nvrtcDestroyProgram_t)(void**);

struct Nvrtc {
    bool ok = false;
    nvrtcCreateProgram_t create = nullptr;
    nvrtcCompileProgram_t compile = nullptr;
    nvrtcGetSize_t log_size = nullptr, cubin_size = nullptr;
    nvrtcGetBuf_t log = nullptr, cubin = nullptr;
    nvrtcDestroyProgram_t destroy = nullptr;
};

const Nvrtc& nvrtc() {
    static Nvrtc lib = [] {
        Nvrtc r;
        const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12",
                               "/usr/local/cuda/lib64/libnvrtc.so"};
        void* h = nullptr;
        for (const char* nm : names)
            if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL)) != nullptr) break;
        if (!h) return r;
        r.create = (nvrtcCreateProgram_t)dlsym(h, "nvrtcCreateProgram");
        r.compile = (nvrtcCompileProgram_t)dlsym(h, "nvrtcCompileProgram");
        r.log_size = (nvrtcGetSize_t)dlsym(h, "nvrtcGetProgramLogSize");
        r.log = (nvrtcGetBuf_t)dlsym(h, "nvrtcGetProgramLog");
        r.cubin_size = (nvrtcGetSize_t)dlsym(h, "nvrtcGetCUBINSize");
        r.cubin = (nvrtcGetBuf_t)dlsym(h, "nvrtcGetCUBIN");
        r.destroy = (nvrtcDestroyProgram_t)dlsym(h, "nvrtcDestroyProgram");
        r.ok = r.create && r.compile && r.log_size && r.log && r.cubin_size && r.cubin && r.destroy;
        return r;
    }();
    return lib;
}

}  // namespace

bool nvrtc_available() { return nvrtc().ok; }

bool compile_cubin(const std::string& src, std::vector<char>& cubin, std::string& log, double* seconds) {
    const Nvrtc& nv = nvrtc();
    if (!nv.ok) {
        log = "libnvrtc not found";
        return false;
    }
    const auto t0 = std::chrono::steady_clock::now();
    void* prog = nullptr;
    if (nv.create(&prog, src.c_str(), "k1j.cu", 0, nullptr, nullptr) != 0) {
        log = "nvrtcCreateProgram failed";
        return false;
    }
    const char* opts[] = {"-arch=sm_100a", "--std=c++17", "-lineinfo", "--device-as-default-execution-space"};
    const int rc = nv.compile(prog, 4, opts);
    size_t ls = 0;
    nv.log_size(prog, &ls);
    log.assign(ls, '\0');
    if (ls) nv.log(prog, &log[0]);
    bool ok = rc == 0;
    if (ok) {
        size_t cs = 0;
        nv.cubin_size(prog, &cs);
        cubin.resize(cs);
        ok = cs > 0 && nv.cubin(prog, cubin.data()) == 0;
    }
    nv.destroy(&prog);
    if (seconds)
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return ok;
}


#ifndef FASTLSH_JIT_MAIN  // the standalone generator check below needs no CUDA runtime
// ------------------------------------------------------------------------------------------
// runtime: variants, module cache, tensor maps, launch
// ------------------------------------------------------------------------------------------

struct Module {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kern = nullptr;
    int warps = 0;
    size_t smem = 0;
    bool attr_set[kMaxDevices] = {};
    std::mutex mu;
};

namespace {

constexpr int kMaxN = 128;          // a row lives in registers: x[n] plus ~100 working registers
constexpr int kMaxCode = 16384;     // k*m straight-line FFMAs (16 B each: 256 KB of code)
constexpr int kNcb = 2;             // code boxes per warp (TMA store ring)
constexpr size_t kSmemBudget = 225 * 1024;

int warps_for(int n) {
    const int wb = ((n + 31) / 32 + kNcb) * 4096;
    int w = (int)(kSmemBudget / (size_t)(wb + 8));
    static const int cap = [] {  // experiment knob (FASTLSH_JIT_WARPS), read once
        const char* e = std::getenv("FASTLSH_JIT_WARPS");
        return e ? std::atoi(e) : 8;
    }();
    return w > cap ? cap : w;
}

size_t smem_bytes(int n, int warps) {
    return (size_t)warps * ((n + 31) / 32 + kNcb) * 4096 + 8 * (size_t)warps + 1024;
}

// process-wide cache: identical sources (same params arrays and variant) share one module
std::mutex g_cache_mu;
std::vector<std::pair<std::string, std::shared_ptr<Module>>>& cache() {
    static std::vector<std::pair<std::string, std::shared_ptr<Module>>> c;
    return c;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* q = nullptr;
        cudaDriverEntryPointQueryResult r;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r) != cudaSuccess ||
            r != cudaDriverEntryPointSuccess)
            return (EncodeTiledFn) nullptr;
        return reinterpret_cast<EncodeTiledFn>(q);
    }();
    return fn;
}

// codes / projections viewed as [rows][cols/32][32]: boxes {32, 2 groups, 32 rows}, 128-byte swizzle
bool make_map3(CUtensorMap* m, const void* base, long long rows, int cols, bool f32) {
    EncodeTiledFn enc = encode_fn();
    if (!enc || cols % 32) return false;
    cuuint64_t dims[3] = {32, (cuuint64_t)(cols / 32), (cuuint64_t)rows};
    cuuint64_t strides[2] = {128, (cuuint64_t)cols * 4};
    cuuint32_t box[3] = {32, 2, 32};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_INT32, 3, const_cast<void*>(base), dims,
               strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// [rows][cols] 4-byte elements, boxes of 32 rows x 32 elements (128 B), 128-byte swizzle
bool make_map(CUtensorMap* m, const void* base, long long rows, int cols, bool f32) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_INT32, 2, const_cast<void*>(base), dims,
               strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int sm_count(int dev) {
    static int cnt[kMaxDevices] = {};
    if (!cnt[dev]) {
        int c = 0;
        if (cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || c <= 0) c = 148;
        cnt[dev] = c;
    }
    return cnt[dev];
}

bool keys_fit(const fastlsh_params& p, const fastlsh_keys* ks) {
    return (int64_t)ks->L * ks->K <= p.k && ks->K <= 1024;  // K <= 1024: the 64-bit limb sums are exact
}

std::shared_ptr<Module> get_variant(const fastlsh_params* p, int mode, const fastlsh_keys* ks, bool mc, bool codes,
                                    fastlsh_status* st) {
    codes = codes || mode == 1 || !ks;  // only the keys variant can keep its codes on chip
    State& js = p->jit;
    std::lock_guard<std::mutex> g(js.mu);
    const int L = ks ? ks->L : 0, K = ks ? ks->K : 0;
    for (auto& v : js.variants)
        if (v.mode == mode && v.L == L && v.K == K && v.mc == mc && v.codes == codes && (!ks || v.r == ks->r))
            return v.mod;
    const int warps = warps_for(p->n);
    Spec s{p->n, p->m, p->k, p->w, p->idx.data(), p->a.data(), p->b.data(), L, K, ks ? ks->r.data() : nullptr,
           warps, kNcb, mode, mc ? 1 : 0, codes ? 1 : 0};
    std::string src = k1j_source(s);
    std::shared_ptr<Module> mod;
    {
        std::lock_guard<std::mutex> gc(g_cache_mu);
        for (auto& c : cache())
            if (c.first == src) mod = c.second;
    }
    if (!mod) {
        std::vector<char> cubin;
        std::string log;
        double sec = 0;
        if (!compile_cubin(src, cubin, log, &sec)) {
            js.last_error = "K1j compile failed: " + log.substr(0, 2000);
            *st = FASTLSH_EUNSUPPORTED;
            return nullptr;
        }
        js.compile_seconds += sec;
        mod = std::make_shared<Module>();
        cudaError_t e = cudaLibraryLoadData(&mod->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
        if (e == cudaSuccess) e = cudaLibraryGetKernel(&mod->kern, mod->lib, "k1j");
        if (e != cudaSuccess) {
            js.last_error = std::string("K1j module load failed: ") + cudaGetErrorString(e);
            *st = set_cuda_error(e);
            return nullptr;
        }
        mod->warps = warps;
        mod->smem = smem_bytes(p->n, warps);
        std::lock_guard<std::mutex> gc(g_cache_mu);
        cache().emplace_back(std::move(src), mod);
    }
    Variant v;
    v.mode = mode;
    v.L = L;
    v.K = K;
    v.mc = mc;
    v.codes = codes;
    if (ks) v.r = ks->r;
    v.mod = mod;
    js.variants.push_back(std::move(v));
    return mod;
}

}  // namespace

bool applicable(const fastlsh_params& p) {
    State& js = p.jit;
    std::lock_guard<std::mutex> g(js.mu);
    if (js.applicable < 0) {
        const char* off = std::getenv("FASTLSH_NO_JIT");
        const bool disabled = off && *off && std::strcmp(off, "0") != 0;
        js.applicable = !disabled && p.n <= kMaxN && p.n % 4 == 0 && p.k % 4 == 0 &&
                        (int64_t)p.k * p.m <= kMaxCode && (size_t)4 * (p.n + p.k) <= (size_t)kNcb * 4096 &&
                        warps_for(p.n) >= 1 && nvrtc_available();
    }
    return js.applicable == 1;
}

fastlsh_status prepare(const fastlsh_params* p, int mode, const fastlsh_keys* ks) {
    if (!applicable(*p)) return FASTLSH_EUNSUPPORTED;
    if (ks && (mode != 0 || !keys_fit(*p, ks))) return FASTLSH_EUNSUPPORTED;
    fastlsh_status st = FASTLSH_OK;
    return get_variant(p, mode, ks, false, true, &st) ? FASTLSH_OK : st;
}

fastlsh_status compile_check(const fastlsh_params* p, const fastlsh_keys* ks, int what, double* seconds,
                             std::string* log) {
    // generate and compile (no module load: works without a GPU) every variant selected by `what`:
    // bit 0 codes, 1 projections, 2 codes + keys, 3 keys only, 4 codes + keys with multicast stores
    if (!applicable(*p)) return FASTLSH_EUNSUPPORTED;
    double total = 0;
    for (int bit = 0; bit < 5; ++bit) {
        if (!(what & (1 << bit))) continue;
        const bool with_keys = bit >= 2;
        if (with_keys && (!ks || !keys_fit(*p, ks))) return FASTLSH_EINVAL;
        const fastlsh_keys* kk = with_keys ? ks : nullptr;
        const int warps = warps_for(p->n);
        Spec s{p->n, p->m, p->k, p->w, p->idx.data(), p->a.data(), p->b.data(), kk ? kk->L : 0, kk ? kk->K : 0,
               kk ? kk->r.data() : nullptr, warps, kNcb, bit == 1 ? 1 : 0, bit == 4 ? 1 : 0, bit == 3 ? 0 : 1};
        std::vector<char> cubin;
        std::string lg;
        double sec = 0;
        if (!compile_cubin(k1j_source(s), cubin, lg, &sec)) {
            if (log) *log = "variant " + std::to_string(bit) + ": " + lg.substr(0, 2000);
            return FASTLSH_EUNSUPPORTED;
        }
        total += sec;
    }
    if (seconds) *seconds = total;
    return FASTLSH_OK;
}

fastlsh_status launch(const fastlsh_params* p, const DeviceCopy& d, const float* X, int64_t N, int32_t* codes,
                      float* proj, const fastlsh_keys* ks, const uint64_t* dev_r, uint64_t* keys, int64_t ldk,
                      cudaStream_t stream, bool keys_mc) {
    if (!applicable(*p) || !d.j_idx) return FASTLSH_EUNSUPPORTED;
    if (keys_mc && !ks) return FASTLSH_EINVAL;
    void* out = proj ? static_cast<void*>(proj) : static_cast<void*>(codes);
    const int mode = proj ? 1 : 0;
    if (proj && ks) return FASTLSH_EUNSUPPORTED;
    if (!out && !ks) return FASTLSH_EINVAL;
    if (ks && (!keys_fit(*p, ks) || !keys || !dev_r)) return FASTLSH_EUNSUPPORTED;
    if ((reinterpret_cast<uintptr_t>(X) & 15) || (reinterpret_cast<uintptr_t>(out) & 15) ||
        N > (int64_t)0x7fffffff - 64)
        return FASTLSH_EUNSUPPORTED;
    fastlsh_status st = FASTLSH_OK;
    std::shared_ptr<Module> mod = get_variant(p, mode, ks, keys_mc, out != nullptr, &st);
    if (!mod) return st;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return set_cuda_error(e);
    {
        std::lock_guard<std::mutex> g(mod->mu);
        if (!mod->attr_set[dev]) {
            e = cudaKernelSetAttributeForDevice(mod->kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mod->smem, dev);
            if (e != cudaSuccess) return set_cuda_error(e);
            mod->attr_set[dev] = true;
        }
    }
    CUtensorMap xmap, omap;
    if (!make_map(&xmap, X, N, p->n, true)) return FASTLSH_EUNSUPPORTED;
    if (out) {
        const bool ok = pair_stores(p->k) ? make_map3(&omap, out, N, p->k, proj != nullptr)
                                       : make_map(&omap, out, N, p->k, proj != nullptr);
        if (!ok) return FASTLSH_EUNSUPPORTED;
    } else {
        omap = xmap;  // keys only: never used
    }
    struct JArgs {
        long long N, tiles;
        int write_out;
        int* out;
        uint64_t* keys;
        long long ldk, col0;
        unsigned long long* flags;
        const int* idx;
        const float* a;
        const float* b;
        const uint64_t* kr;
    } a;
    a.N = N;
    a.tiles = (N + 31) / 32;
    a.write_out = out ? 1 : 0;
    a.out = static_cast<int*>(out);
    a.keys = keys;
    a.ldk = ldk;
    a.col0 = 0;
    a.flags = d.flags;
    a.idx = d.j_idx;
    a.a = d.j_a;
    a.b = d.b;
    a.kr = dev_r;
    const long long ctas_needed = (a.tiles + mod->warps - 1) / mod->warps;
    const int grid = (int)(ctas_needed < sm_count(dev) ? ctas_needed : sm_count(dev));
    void* args[3] = {&xmap, &omap, &a};
    e = cudaLaunchKernel(reinterpret_cast<const void*>(mod->kern), dim3(grid), dim3(mod->warps * 32), args, mod->smem,
                         stream);
    if (e != cudaSuccess) return set_cuda_error(e);
    return FASTLSH_OK;
}

#endif  // FASTLSH_JIT_MAIN

}  // namespace jit
}  // namespace fastlsh

#ifdef FASTLSH_JIT_MAIN
// Standalone check of the generator + NVRTC (no GPU needed): prints the compile time and writes
// the source and cubin for inspection with cuobjdump.
#include "philox.h"
int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 128, m = argc > 2 ? atoi(argv[2]) : 16, k = argc > 3 ? atoi(argv[3]) : 256;
    const int L = argc > 4 ? atoi(argv[4]) : 16, K = argc > 5 ? atoi(argv[5]) : 16;
    const float w = 4.0f;
    std::vector<int32_t> idx((size_t)k * m);
    std::vector<float> a((size_t)k * m), b(k);
    for (int i = 0; i < k; ++i) {
        for (int j = 0; j < m; ++j) {
            idx[(size_t)i * m + j] = fastlsh::draw_index(1, i, j, n);
            a[(size_t)i * m + j] = fastlsh::draw_gaussian(1, i, j);
        }
        b[i] = fastlsh::draw_offset(1, i, w);
    }
    std::vector<uint64_t> r((size_t)L * (K + 1));
    for (int l = 0; l < L; ++l)
        for (int j = 0; j <= K; ++j) r[(size_t)l * (K + 1) + j] = fastlsh::draw_key_multiplier(1, l, j);
    fastlsh::jit::Spec s{n, m, k, w, idx.data(), a.data(), b.data(), L, K, r.data(), 8, 2, argc > 6 ? atoi(argv[6]) : 0,
                         argc > 7 ? atoi(argv[7]) : 0, argc > 8 ? atoi(argv[8]) : 1};
    const std::string src = fastlsh::jit::k1j_source(s);
    FILE* f = fopen("/tmp/k1j.cu", "w");
    fwrite(src.data(), 1, src.size(), f);
    fclose(f);
    std::vector<char> cubin;
    std::string log;
    double sec = 0;
    const bool ok = fastlsh::jit::compile_cubin(src, cubin, log, &sec);
    printf("source %zu bytes, compile %s in %.2f s, cubin %zu bytes\n%s\n", src.size(), ok ? "ok" : "FAILED", sec,
           cubin.size(), log.c_str());
    if (ok) {
        f = fopen("/tmp/k1j.cubin", "wb");
        fwrite(cubin.data(), 1, cubin.size(), f);
        fclose(f);
    }
    return ok ? 0 : 1;
}
#endif
