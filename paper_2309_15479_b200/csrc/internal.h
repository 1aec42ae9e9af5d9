// internal.h — host-side structures shared by the C ABI, the packer and the kernel launchers.
#pragma once
#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fastlsh.h"

namespace fastlsh {

constexpr int kMaxDevices = 16;
constexpr int kRows = 4;          // rows per stage: one LDS.128 gathers the same column of 4 rows
constexpr int kMaxSlots = 64;     // slot positions per lane held in registers
constexpr int kPadChunks = 8;     // zero chunks after the data: one per 16-B bank group
constexpr int kMaxN = 4400;       // 3 stages x (4*ceil(n/4)+8) x 16 B + partials <= 227 KB

// GPU packing of a params object.
//
// Shared-memory stage layout (one stage = kRows rows): the 16-byte chunk at position pos holds
// column c of all 4 rows, pos(c) = (c % 4) * nq + c / 4 with nq = ceil(n/4); chunks
// [4*nq, 4*nq + 8) are zero (targets of padding slots). A lane's slot is a byte offset 16*pos into
// the stage and a coefficient; one LDS.128 returns x[0..3][c].
//
// Lanes: each hash is split into `parts` lane units of <= ceil(m/parts) slots. Units of one CTA
// hash block are grouped into quarter-warps (8 lanes = one LDS.128 wavefront) whose slots are
// edge-coloured (König) so that at every slot position the 8 lanes touch distinct bank groups
// (pos mod 8).
struct Packing {
    int parts = 1;
    int slots = 0;            // MS: slot positions per lane (even)
    int warps = 0;            // W: warps per CTA
    int hash_blocks = 0;      // HB
    int kb_max = 0;           // max hashes per block
    int nq = 0;               // chunk columns per row-quarter
    int stage_chunks = 0;     // 4*nq + kPadChunks
    std::vector<int> block_h0, block_kb;       // hash range per block
    std::vector<uint32_t> offp;  // [HB][W][MS][32]: smem byte offset of slot t (16 * chunk position)
    std::vector<float> coef;     // [HB][W][MS][32]
    std::vector<uint16_t> unit_lane;  // [HB][kb_max][parts]: lane id (warp*32+lane) of each part
    double efficiency = 0;       // useful slots / (lanes * MS) over all warps
    double cost = 1e300;         // modelled shared-memory wavefronts per row / pipe rate
    int64_t conflict_wavefronts = 0;  // extra wavefronts per stage (all blocks) beyond 4 per LDS
    // direct epilogue (parts == 1): warp w of a block holds hashes [32w, 32w+32) of the block, so
    // each lane quantises its own sums and the warp's code stores are contiguous runs (no
    // partial-sum round trip through shared memory)
    int direct = 0;
};

// GPU packing for the TMEM kernel K1t (gather_tmem.cu). Hash block hb serves
// hashes [h0, h0+kb) as groups of 4 consecutive hashes spread over the CTA's 16 warps (<= 4 groups
// each; warp w works in TMEM lane quadrant w % 4), chosen so that every coordinate block costs the
// warps about the same. Records (TMEM column 8*(c - 64*block), coefficient bits) are grouped by
// (hb, warp, coordinate block, hash); counts[hb][warp][block][16]
// give the run lengths (hash j of a warp = group j/4, member j%4).
constexpr int kTMaxHB = 64;
constexpr int kTWarps = 16;
constexpr int kTGroups = 2;                  // max groups of 4 hashes per warp
constexpr int kTInfo = 4 + kTWarps;          // ints per hash block in TPacking::hinfo
struct TPacking {
    bool ok = false;
    int nb = 0, nhw = 0, HB = 0, recs_max = 0, kb_max = 0;  // nb coordinate blocks of 64
    size_t smem = 0;
    std::vector<int32_t> hinfo;    // [HB][20]: h0, kb, rec_base, rec_count, ngroups[16]
    std::vector<int32_t> groups;   // [HB][16][2]: first hash of each group of the warp
    std::vector<uint32_t> recs;    // [records][2]
    std::vector<uint8_t> counts;   // [HB][16][nb][16]
    std::vector<uint32_t> offs;    // [HB][16][nb] first record (relative to rec_base)
    double balance = 0;            // critical-path slots / mean slots per warp (>= 1)
};

// GPU packing for the row-major kernel K1r (gather_rows.cuh). Stages hold rows
// row-major at a stride of S words (a multiple of 32, fixed per class): copy 0 of the row at words
// [0, n), a 32-word zero tail at [S0-32, S0) (S0 = 32*ceil(n/32) + 32) read by padding slots, and,
// where the class leaves room, copy 1 of coordinates [0, n1) at word S0 + 16 + c (16 banks
// rotated). A coordinate's bank is thus the same in every staged row, and TMA bulk copies fill the
// stages directly. Hash block hb serves hashes [h0, h0+kb); a
// block's W warps hold hpw = 32/P hashes each, hash slot j of a warp in lanes j + hpw*q (q < P
// parts, summed by an xor butterfly), and the hash in slot j is congruent to j mod hpw so that the
// code stores of a warp hit distinct banks. At every slot position the 32 lanes of a warp read 32
// distinct banks (König colouring of lanes x banks), so one LDS.32 per slot and row is one
// wavefront. Slots are packed two per register (16-bit byte offsets within a row).
constexpr int kRMaxSlots = 128;
// Stage geometry per row-stride class (compile-time in the kernel, so the R rows of a stage are
// immediate offsets of one LDS address): S words per staged row, R rows per stage, NS stages, NC
// code buffers (a deep code ring lets fast warps run ahead of the flush of a slow warp's group).
struct RClass { int S, R, NS, NC, D; };  // D: code-ring flush lag (gather_rows.cuh)
// Classes 0-2 (n <= 128 / 256 / 512) stage a full second copy (n1 = n); classes 3-5 one copy.
constexpr RClass kRClasses[] = {{320, 8, 3, 5, 3}, {576, 8, 4, 6, 5}, {1088, 8, 3, 5, 4}, {1056, 8, 3, 6, 5},
                                {2080, 4, 4, 8, 7}, {4128, 4, 3, 3, 2},
                                {2080, 8, 2, 4, 3}, {4128, 6, 2, 2, 1}};
constexpr int kRDualClasses = 3;
constexpr int kRDualMaxN[kRDualClasses] = {128, 256, 512};
// class 6: 8-row dual stages for rows up to ~1000 words; class 7: 6-row stages of rows up to 4096
// words for 16-warp packings (rpacker.cpp)
constexpr int kNumRClasses = 8;
struct RPacking {
    bool ok = false;
    int parts = 1, slots = 0, warps = 0, hash_blocks = 0, kb_max = 0, S = 0, cls = 0;
    int S0 = 0, n1 = 0;  // copy 0 spans words [0, S0) (zero tail [S0-32, S0)); copy 1 = coords [0, n1) at S0+16
    std::vector<int> block_h0, block_kb;
    std::vector<uint32_t> offp;     // [HB][W][MS/2][32]: bits 0-15 slot 2t, bits 16-31 slot 2t+1
    std::vector<float> coef;        // [HB][W][MS][32]
    std::vector<int16_t> lane_hash; // [HB][W*32]: block-local hash of the lane's part, -1 = idle
    double efficiency = 0;          // useful slots / (lanes * MS)
    int64_t conflict_wavefronts = 0;  // extra wavefronts per row (all blocks) beyond 1 per LDS.32
    double cost = 1e300;            // modelled shared-memory wavefronts per row / pipe rate
};
// true when K1r can hash rows of this params object (packing exists) — X alignment is per call
void build_row_packing(const fastlsh_params& p, RPacking& out);

namespace jit {
struct Module;  // a compiled K1j variant (jit.cpp)
// K1j variants of one params object: (mode, keys multipliers) -> module; compiled on first use
struct Variant {
    int mode = 0, L = 0, K = 0;
    std::vector<uint64_t> r;  // key multipliers compiled into the module (empty: no keys)
    bool mc = false;          // keys stored to a multicast address
    bool codes = true;        // codes stored (false: keys only)
    std::shared_ptr<Module> mod;
};
struct State {
    std::mutex mu;
    int applicable = -1;  // -1 not decided yet
    std::vector<Variant> variants;
    std::string last_error;
    double compile_seconds = 0;  // total NVRTC time spent for this params object
};
}  // namespace jit

struct DeviceCopy {
    bool ready = false;
    int32_t* j_idx = nullptr;             // K1j slow path: canonical idx / a on the device
    float* j_a = nullptr;
    uint32_t* r_offp = nullptr;           // K1r packing (RPacking), when applicable
    float* r_coef = nullptr;
    int16_t* r_lane_hash = nullptr;
    mutable int r_resident[2] = {0, 0};          // K1r resident CTAs per device [plain, keys], cached
    mutable size_t r_resident_smem[2] = {0, 0};  // ... for this dynamic shared-memory size
    int32_t* r_block_h0 = nullptr;
    int32_t* r_block_kb = nullptr;
    uint32_t* offp = nullptr;
    float* coef = nullptr;
    uint16_t* unit_lane = nullptr;
    float* b = nullptr;
    int32_t* block_h0 = nullptr;
    int32_t* block_kb = nullptr;
    unsigned long long* flags = nullptr;  // [0] nonfinite, [1] saturated
    uint32_t* t_recs = nullptr;           // K1t packing (TPacking), when applicable
    uint8_t* t_counts = nullptr;
    uint32_t* t_offs = nullptr;
    int32_t* t_hinfo = nullptr;
    int32_t* t_groups = nullptr;
    float* dense_hi = nullptr;            // dense E2LSH operand A (tf32 hi) [kpad][n]
    float* dense_lo = nullptr;            // A - hi (tf32 lo)
    int dense_kpad = 0;
    uint16_t* dense_h16 = nullptr;        // 3xFP16 operands (fp16 bits) Ah | Al | Ah' (fp16 [3][kpad][dense_n8])
    int dense_n8 = 0;
    // host-pipeline workspace (fastlsh_hash_host)
    float* ws_x[2] = {nullptr, nullptr};
    int32_t* ws_codes[2] = {nullptr, nullptr};
    uint64_t* ws_keys[2] = {nullptr, nullptr};
    int64_t ws_rows = 0;
    int ws_L = 0;
    cudaStream_t ws_stream[2] = {nullptr, nullptr};
    cudaEvent_t ws_event[4] = {nullptr, nullptr, nullptr, nullptr};
    // gather pipeline shape chosen per TMA mode (index: rows 16-B aligned), -1 = not chosen yet
    mutable int shape_cache[4] = {-1, -1, -1, -1};  // [tma + 2 * fused keys]
};

}  // namespace fastlsh

struct fastlsh_params {
    int32_t n = 0, m = 0, k = 0;
    float w = 1.0f;
    bool is_e2lsh = false;
    std::vector<int32_t> idx;  // [k][m] canonical (paper) order
    std::vector<float> a;      // [k][m]
    std::vector<float> b;      // [k]
    fastlsh::Packing pack;
    fastlsh::TPacking tpack;
    fastlsh::RPacking rpack;
    bool packed = false;
    bool pack_skipped = false; // auto mode on a dense-path shape: K1 / K1t / K1r packings built on demand
    int32_t kernel = 0;        // fastlsh_params_set_kernel: 0 auto, 1 K1, 2 TMEM K1t, 3 row-major K1r, 4 K1j,
                               // 5 dense K4 on merged coefficients
    int32_t table_align = 1;   // hash blocks hold whole tables of this many hashes (fused keys)
    fastlsh::DeviceCopy dev[fastlsh::kMaxDevices];
    std::mutex mu;
    std::mutex dense_mu;       // guards DeviceCopy::dense_* (built on the first dense call; mu may be held)
    mutable fastlsh::jit::State jit;
};

struct fastlsh_keys {
    int32_t L = 0, K = 0;
    std::vector<uint64_t> r;  // [L][K+1]
    uint64_t* dev_r[fastlsh::kMaxDevices] = {};
    std::mutex mu;
};

namespace fastlsh {

// packer.cpp
void build_packing(const fastlsh_params& p, Packing& out);
// König edge colouring of a bipartite multigraph with ncol >= max degree colours; edge e joins
// left[e] and right[e]; returns each edge's colour (all -1 if ncol is too small)
std::vector<int> color_bipartite(const std::vector<int>& left, const std::vector<int>& right, int nleft,
                                 int nright, int ncol);

// gather.cu
struct FusedKeys {            // compound keys built in the hashing kernel's epilogue
    const uint64_t* r;        // device multipliers [L][K+1]
    int L, K;
    uint64_t* keys;           // device [L][ldk]
    int64_t ldk;
};
fastlsh_status launch_gather(const fastlsh_params* p, const DeviceCopy& d, const float* X,
                             int64_t N, int32_t* codes, float* proj, cudaStream_t stream,
                             const FusedKeys* fk = nullptr);
// true when every hash block of the packing holds whole tables of `keys`
bool keys_fusable(const fastlsh_params* p, const fastlsh_keys* keys);
// gather_tmem.cu
void build_tmem_packing(const fastlsh_params& p, TPacking& out);
fastlsh_status launch_gather_tmem(const fastlsh_params* p, const DeviceCopy& d, const float* X,
                                  int64_t N, int32_t* codes, float* proj, cudaStream_t stream);
// gather_rows.cu (fk: compound keys built in the flush of the code tile; needs one hash block)
struct FusedKeys;
// K1r keys from the code tile: every hash block holds whole tables; the most tables one block holds
bool rows_keys_fusable(const RPacking& pk, int L, int K);
int rows_key_tables_max(const RPacking& pk, int L, int K);
fastlsh_status launch_gather_rows(const fastlsh_params* p, const DeviceCopy& d, const float* X,
                                  int64_t N, int32_t* codes, float* proj, cudaStream_t stream,
                                  const FusedKeys* fk = nullptr);
// generic.cu: K0, the fallback for params no specialised kernel can pack (n > kMaxN, huge m)
fastlsh_status launch_generic(const fastlsh_params* p, const DeviceCopy& d, const float* X, int64_t N, int32_t* codes,
                              float* proj, cudaStream_t stream);
// the hashing dispatcher (api.cu): K1t when selected/applicable, else K1
fastlsh_status launch_hash(const fastlsh_params* p, const DeviceCopy& d, const float* X, int64_t N,
                           int32_t* codes, float* proj, cudaStream_t stream);
// keys.cu
fastlsh_status launch_build_keys(const fastlsh_keys* keys, const uint64_t* dev_r,
                                 const int32_t* codes, int64_t N, int32_t k, uint64_t* out,
                                 int64_t ldk, cudaStream_t stream);
// tables.cu
size_t tables_workspace_bytes(int L, long long N);
fastlsh_status launch_build_tables(const uint64_t* keys, int L, long long N, long long ldk, uint64_t* sorted_keys,
                                   uint32_t* ids, uint32_t* starts, long long* nbuckets, void* ws,
                                   cudaStream_t stream);
// query.cu
size_t query_workspace_bytes(long long N, int grid);
int query_grid(long long nq);
fastlsh_status launch_query(const float* X, long long N, int n, const uint64_t* sk, const uint32_t* ids, int L,
                            const float* Q, const uint64_t* qkeys, long long nq, long long ldq, int topk,
                            int32_t* out_ids, float* out_dist, long long* out_ncand, void* ws, cudaStream_t stream);
// transforms.cu
fastlsh_status launch_normalize(const float* X, long long N, int n, float* out, cudaStream_t s);
fastlsh_status launch_max_norm(const float* X, long long N, int n, float* kappa, cudaStream_t s);
fastlsh_status launch_mips(const float* X, long long N, int n, const float* kappa, int is_query, float* out,
                           cudaStream_t s);
// api.cu: params the dense path (K4 on merged coefficients) serves in automatic mode
bool dense_shape(const fastlsh_params* p);
// e2lsh_tcgen05.cu
fastlsh_status launch_e2lsh(const fastlsh_params* p, DeviceCopy& d, const float* X, int64_t N,
                            int32_t* codes, float* proj, int precision, cudaStream_t stream);

fastlsh_status set_cuda_error(cudaError_t e);
// cudaFuncAttributeMaxDynamicSharedMemorySize = 227 KB minus the kernel's static shared memory for
// kernel `fn` on the current device, once per (kernel, device) for the process (launchers call it
// before every launch; only the first call reaches the driver). Launches then pass their own
// dynamic size, which must fit that bound.
fastlsh_status smem_optin_once(const void* fn);

// jit.cpp — K1j, the params-specialised lane = row kernel
namespace jit {
struct Spec {
    int n, m, k;
    float w;
    const int32_t* idx;  // canonical [k][m]
    const float* a;      // [k][m]
    const float* b;      // [k]
    int L, K;            // fused compound keys (L = 0: none)
    const uint64_t* r;   // their multipliers [L][K+1] (compiled in as immediates)
    int warps, ncb;      // warps per CTA, code boxes per warp
    int mode;            // 0: codes (+ keys when L > 0), 1: projections
    int mc;              // keys stored with multimem.st to a multicast (NVLS) address
    int codes;           // mode 0: codes stored (1) or kept on chip, keys only (0)
};
std::string k1j_source(const Spec& s);
bool pair_stores(int k);
bool nvrtc_available();
bool compile_cubin(const std::string& src, std::vector<char>& cubin, std::string& log, double* seconds);
// K1j can serve this params object (shape limits, NVRTC present, not disabled by FASTLSH_NO_JIT)
bool applicable(const fastlsh_params& p);
// Hash (codes, or proj when proj != NULL) and optionally build compound keys in one launch.
// Returns FASTLSH_EUNSUPPORTED when K1j cannot serve this call (alignment, sizes, compile
// failure): the caller then uses K1r / K1.
fastlsh_status launch(const fastlsh_params* p, const DeviceCopy& d, const float* X, int64_t N, int32_t* codes,
                      float* proj, const fastlsh_keys* ks, const uint64_t* dev_r, uint64_t* keys, int64_t ldk,
                      cudaStream_t stream, bool keys_mc = false);
// compile (if needed) the variant a call with these arguments would use
fastlsh_status prepare(const fastlsh_params* p, int mode, const fastlsh_keys* ks);
// generate + compile the selected variants without loading them (no GPU needed)
fastlsh_status compile_check(const fastlsh_params* p, const fastlsh_keys* ks, int what, double* seconds,
                             std::string* log);
}  // namespace jit

}  // namespace fastlsh
