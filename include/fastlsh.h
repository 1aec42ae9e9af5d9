/*
 * fastlsh.h — C ABI of libfastlsh, a B200 (sm_100a) implementation of FastLSH hash evaluation
 * (Tan et al., "Fast Locality Sensitive Hashing with Theoretical Guarantee", arXiv 2309.15479).
 *
 * Method (§3.1, Eq. 5): for every row v of X[N x n] and hash i < k,
 *     h_i(v) = floor( (a_i . S_i(v) + b_i) / w )
 * where S_i(v) gathers m coordinates of v at a multiset of m indices drawn i.i.d. uniformly from
 * [0, n) with replacement, a_i ~ N(0,1)^m and b_i ~ U[0, w).
 * E2LSH (Eq. 1) is the special case m = n with the identity sample.
 *
 * Conventions for every call:
 *  - X, codes, proj and keys are DEVICE pointers owned by the caller, row-major, contiguous.
 *    X must be 4-byte aligned; 16-byte alignment and n % 4 == 0 select the 128-bit load path.
 *  - Calls are asynchronous and ordered on `stream` (a cudaStream_t; NULL = legacy default
 *    stream). No call synchronises except fastlsh_read_flags and the *_host entry points.
 *  - N == 0 is a no-op returning FASTLSH_OK.
 *  - Errors are returned, never aborted on. Data-dependent conditions inside a kernel (a
 *    non-finite projection, a quotient outside int32) write the sentinel INT32_MIN into that code
 *    and increment a per-params device counter, read back by fastlsh_read_flags.
 *  - Params and keys objects are immutable after creation/upload; concurrent calls on different
 *    streams with the same objects are safe.
 */
#ifndef FASTLSH_H
#define FASTLSH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* fastlsh_stream_t; /* == cudaStream_t */

typedef enum {
    FASTLSH_OK = 0,
    FASTLSH_EINVAL = -1,       /* bad argument: sizes, null/misaligned pointer, w <= 0 or NaN */
    FASTLSH_ENOMEM = -2,       /* host or device allocation failed */
    FASTLSH_ECUDA = -3,        /* a CUDA runtime call failed (see fastlsh_last_cuda_error) */
    FASTLSH_EUNSUPPORTED = -4, /* current device is not sm_100 (B200), or shape unsupported */
    FASTLSH_ESTATE = -5        /* params/keys not uploaded to the current device */
} fastlsh_status;

typedef struct fastlsh_params fastlsh_params; /* opaque: S_i, a_i, b_i, w + GPU packing */
typedef struct fastlsh_keys fastlsh_keys;     /* opaque: L, K, multipliers r[L][K+1]     */

/* Packing summary of a params object (filled by fastlsh_params_info). */
typedef struct {
    int32_t n, m, k;
    float w;
    int32_t is_e2lsh;          /* created by e2lsh_params_create (identity S, m == n)          */
    int32_t parts;             /* lanes per hash: each lane owns <= ceil(m/parts) slots         */
    int32_t slots;             /* slot positions per lane after bank scheduling (incl. padding) */
    int32_t units;             /* k * parts lane units                                          */
    int32_t warps_per_block;   /* warps in one CTA hash block                                    */
    int32_t hash_blocks;       /* CTAs per row group (disjoint hash ranges)                      */
    int32_t rows_per_group;    /* rows staged together per pipeline stage                        */
    double bank_efficiency;    /* useful gathers / (lanes * slots) over all warps                 */
    int64_t conflict_wavefronts; /* extra smem wavefronts per row left by the scheduler          */
    int32_t kernel;            /* hashing kernel for 16-B aligned X: 0 = generic K0 (n > 4400),
                                  1 = shared-memory gather K1,
                                  2 = tensor-memory gather K1t,
                                  3 = row-major gather K1r,
                                  4 = params-specialised lane = row kernel K1j,
                                  5 = dense 3xTF32 GEMM K4 on the merged coefficients */
    int32_t tmem_hash_blocks;  /* K1t: CTAs hash blocks (0 when K1t does not apply)              */
    int32_t tmem_hashes_per_warp; /* K1t: hashes (register accumulator pairs) per warp           */
} fastlsh_params_info_t;

/* ---- parameters: S_i, a_i, b_i, w --------------------- */

/* Draw params from `seed` with the library's counter-based Philox4x32-10 (R11):
 *   idx[i][j] = hi64(u64(philox(j,i,1)) * n),  a[i][j] = BoxMuller(philox(j,i,2)) as f32,
 *   b[i] = f32(w * u53(philox(0,i,3))) clamped to [0, w).
 * n, m, k >= 1; w finite and > 0; m > n is legal (sampling with replacement).
 * EINVAL otherwise; EUNSUPPORTED if k * m > 2^31. Params with n > 4400 (a 4-row stage of X no longer
 * fits in shared memory) or m > 16384 are served by the generic kernel K0 (global-memory gathers,
 * correctness path; fastlsh_params_info reports kernel 0). */
fastlsh_status fastlsh_params_create(int32_t n, int32_t m, int32_t k, float w, uint64_t seed,
                                     fastlsh_params** out);

/* Same, from caller-provided host arrays (copied): idx int32[k*m] (0 <= idx < n), a f32[k*m],
 * b f32[k] (any finite values). Used for parity with the oracle on shared seeded inputs. */
fastlsh_status fastlsh_params_create_from_arrays(int32_t n, int32_t m, int32_t k, float w,
                                                 const int32_t* idx, const float* a,
                                                 const float* b, fastlsh_params** out);

/* E2LSH params (Eq. 1): m = n, idx[i][j] = j; a and b drawn from the same
 * (seed, i, j) streams as fastlsh_params_create, so identity-FastLSH == E2LSH. */
fastlsh_status e2lsh_params_create(int32_t n, int32_t k, float w, uint64_t seed,
                                   fastlsh_params** out);

void fastlsh_params_destroy(fastlsh_params* p); /* frees host and all device copies; NULL ok */

/* Copy the canonical (paper-order) params out: idx int32[k*m], a f32[k*m], b f32[k], w.
 * Any output pointer may be NULL. */
fastlsh_status fastlsh_params_export(const fastlsh_params* p, int32_t* idx, float* a, float* b,
                                     float* w);

fastlsh_status fastlsh_params_info(const fastlsh_params* p, fastlsh_params_info_t* info);

/* Diagnostic: copy the GPU packing out (for host-side verification of the bank scheduler).
 * sizes[0..7] = {parts, slots, warps, hash_blocks, kb_max, nq, stage_chunks, n_lanes_total}.
 * Arrays (any may be NULL): offp u32[HB*W*slots*32] (smem byte offsets), coef f32[HB*W*slots*32],
 * unit_lane u16[HB*kb_max*parts], block_h0 int32[HB], block_kb int32[HB]. */
fastlsh_status fastlsh_params_packing(const fastlsh_params* p, int32_t* sizes, uint32_t* offp,
                                      float* coef, uint16_t* unit_lane, int32_t* block_h0,
                                      int32_t* block_kb);

/* Diagnostic: copy the K1r packing out (rpacker.cpp).
 * sizes[0..9] = {ok, parts P, slots MS, warps W, hash_blocks HB, kb_max, staged row stride S
 * (words), conflict wavefronts per row, S0, n1}: a staged row holds coordinates [0, n) at words
 * [0, n), zeros at [S0-32, S0), and coordinates [0, n1) again at words S0+16+c. When ok == 0
 * nothing else is written. Arrays (any may be
 * NULL): offp u32[HB*W*(MS/2)*32] (two 16-bit byte offsets into a staged row: bits 0-15 slot 2t,
 * bits 16-31 slot 2t+1), coef f32[HB*W*MS*32], lane_hash int16[HB*W*32] (block-local hash of the
 * lane's part, -1 idle; parts of hash slot j sit in lanes j + (32/P)q), block_h0/block_kb int32[HB]. */
fastlsh_status fastlsh_params_row_packing(const fastlsh_params* p, int32_t* sizes, uint32_t* offp,
                                          float* coef, int16_t* lane_hash, int32_t* block_h0,
                                          int32_t* block_kb);

/* Hint that keys of K consecutive codes will be built from these params: the GPU
 * packing then keeps whole tables inside each CTA hash block, which lets fastlsh_hash_keys build
 * the keys in the hashing kernel's epilogue (codes are still written). Must be called before the
 * first upload (ESTATE otherwise); K >= 1 (EINVAL otherwise). Results are identical either way. */
fastlsh_status fastlsh_params_set_table_size(fastlsh_params* p, int32_t K);

/* Pack the bank-scheduled GPU layout and copy it to the CURRENT device (cudaSetDevice first).
 * `device` must equal the current device. Idempotent per device. */
fastlsh_status fastlsh_params_upload(fastlsh_params* p, int32_t device, fastlsh_stream_t stream);

/* ---- hashing ----------------------------------------------------------- */

/* Choose the hashing kernel of these params (all compute Eq. 5, with the same
 * epilogue; only the summation order of the fp32 projection differs, within the same bound):
 *   0 = automatic (default), first applicable of: K1j (4); the row-major gather K1r when its packing exists and its cost model beats K1's,
 *       for calls with n % 4 == 0 and X 16-byte aligned; K0 for params nothing else packs; else K1;
 *   1 = always the shared-memory gather K1 (column-interleaved stages, LDS.128);
 *   2 = always K1t (calls on shapes or pointers it cannot serve return EUNSUPPORTED);
 *   3 = always K1r (row-major stages, LDS.32; likewise EUNSUPPORTED when it cannot serve);
 *   4 = always K1j, the params-specialised kernel: the library generates
 *       CUDA source in which S_i are register operands of a row held in registers (lane = row)
 *       and a_i, b_i, 1/w instruction immediates, compiles it with NVRTC for sm_100a on first
 *       use and caches the module (per process, keyed by the generated source). Applies when
 *       n <= 128, n % 4 == 0, k % 4 == 0, k*m <= 16384 and libnvrtc can be loaded; calls need X
 *       and codes/proj 16-byte aligned. In automatic mode K1j is preferred wherever it applies
 *       (set FASTLSH_NO_JIT=1 to disable it);
 *   5 = always the dense path: Eq. 5 as one tcgen05 3xTF32 GEMM against the
 *       coefficient matrix A[c][i] = sum of a_ij over the samples j of hash i with idx_ij = c
 *       (duplicates merged in double, rounded once to f32; built on the first call per device,
 *       kpad x n x 8 bytes), then the same epilogue (e2lsh_hash's kernel). Opt-in only (analysis):
 *       north_star reserves the tensor cores for the dense E2LSH baseline, so automatic mode never
 *       takes it, although for long densely-sampled rows (C2: n = 4096, m >= 512) it is faster than
 *       the gathers. Needs n % 4 == 0; calls with X not 16-byte aligned take the generic kernel K0.
 *       Pinning 5 before the first upload skips the gather packings; pinning 0-3 afterwards then
 *       returns ESTATE once a device copy exists (before it, the packings are built).
 * EINVAL for other values; EUNSUPPORTED for 2, 3, 4 or 5 when that kernel cannot serve the params. */
fastlsh_status fastlsh_params_set_kernel(fastlsh_params* p, int32_t kernel);

/* K1j only: compile ahead of time the variants a later call will use, so that the first
 * fastlsh_hash / fastlsh_project / fastlsh_hash_keys call does not pay the NVRTC compile
 * (seconds). what: bit 0 codes, bit 1 projections, bit 2 codes + keys of `keys` (its L and K;
 * the multipliers are kernel arguments, not compiled in). FASTLSH_OK and nothing done when the
 * params do not use K1j. EUNSUPPORTED when NVRTC fails (see fastlsh_params_jit_status). */
fastlsh_status fastlsh_params_prepare(const fastlsh_params* p, const fastlsh_keys* keys, int32_t what);

/* K1j diagnostic (no GPU needed): generate and compile, without loading, the variants selected by
 * `what` — bit 0 codes, 1 projections, 2 codes + keys, 3 keys only, 4 codes + keys with multicast key
 * stores (bits 2-4 need `keys`). EUNSUPPORTED when K1j does not apply or a compile fails (first
 * NVRTC log lines in msg), EINVAL for bad arguments. */
fastlsh_status fastlsh_params_jit_check(const fastlsh_params* p, const fastlsh_keys* keys, int32_t what,
                                       double* compile_seconds, char* msg, int64_t msg_len);

/* K1j diagnostics: total NVRTC compile time spent for these params and the last compile / load
 * error (empty when none); msg receives at most msg_len-1 bytes plus a NUL. */
fastlsh_status fastlsh_params_jit_status(const fastlsh_params* p, double* compile_seconds, char* msg,
                                         int64_t msg_len);

/* codes[r*k + i] = floor((a_i . S_i(X[r]) + b_i) / w) as int32, for r < N, i < k — Eq. 5.
 * fp32 accumulation (K1r: each lane sums <= 128 products in its bank-scheduled slot order, the
 * P <= 32 parts of a hash then by an xor butterfly; K1: chunks of <= 64 products; K1t: slots
 * grouped by 128-coordinate block, one accumulator over <= 128 products; K1j: the m products in the
 * paper's slot order, one accumulator), then
 * __fadd_rn(p, b), __fdiv_rn(., w), floor toward -inf. Non-finite or out-of-int32 quotients
 * write INT32_MIN and count in the params' flags. Requires fastlsh_params_upload. */
fastlsh_status fastlsh_hash(const fastlsh_params* p, const float* X, int64_t N, int32_t* codes,
                            fastlsh_stream_t stream);

/* proj[r*k + i] = a_i . S_i(X[r]) in fp32 (the projection before +b, /w, floor). */
fastlsh_status fastlsh_project(const fastlsh_params* p, const float* X, int64_t N, float* proj,
                               fastlsh_stream_t stream);

/* ---- dense E2LSH baseline on tcgen05 tensor cores ---------------------- */

/* codes = floor((X . A^T + b) / w) with A[k][n] the dense coefficient matrix of the params
 * (for E2LSH params, a_i itself; for FastLSH params, the duplicates-merged sampled matrix).
 * tcgen05 kind::tf32 MMAs with a 3xTF32 split (hi*hi + hi*lo + lo*hi), fp32 accumulation in TMEM,
 * fused +b, /w, floor epilogue. precision: 3 = 3xTF32 (parity-gated), 1 = plain TF32 (ungated),
 * 2 = 3xFP16: kind::f16 MMAs at twice the TF32 rate on Xh.Ah + Xh.Al + Xl'.Ah' with Xh = fp16(x),
 * Xl' = fp16((x - Xh) * 2^11), Ah = fp16(a), Al = fp16(a - Ah), Ah' = fp16(Ah * 2^-11) (parity-gated;
 * |x|, |a| must stay below 65504, fp16's range: an overflowing element comes back as INT32_MIN and
 * is counted as non-finite). Other precision values: EINVAL. Requires n % 4 == 0 and X 16-byte
 * aligned (else EUNSUPPORTED); the coefficient operands are built on the device on first use. */
fastlsh_status e2lsh_hash(const fastlsh_params* p, const float* X, int64_t N, int32_t* codes,
                          int32_t precision, fastlsh_stream_t stream);

/* proj = X . A^T in fp32 from the same GEMM (for projection parity). */
fastlsh_status e2lsh_project(const fastlsh_params* p, const float* X, int64_t N, float* proj,
                             int32_t precision, fastlsh_stream_t stream);

/* ---- compound bucket keys (§3.2) --------------------------- */

/* r[l][j] uniform in [0, 2^61-1) from Philox stream 4 (R9). L, K >= 1 and
 * L * (K + 1) <= 8192 (the multipliers live in shared memory), else EINVAL. */
fastlsh_status fastlsh_keys_create(int32_t L, int32_t K, uint64_t seed, fastlsh_keys** out);
fastlsh_status fastlsh_keys_create_from_arrays(int32_t L, int32_t K, const uint64_t* r,
                                               fastlsh_keys** out); /* r[L*(K+1)], each < 2^61-1 */
void fastlsh_keys_destroy(fastlsh_keys* keys);
fastlsh_status fastlsh_keys_export(const fastlsh_keys* keys, uint64_t* r);

/* keys[l*ldk + v] = (r[l][0] + sum_{j<K} r[l][j+1] * u32(codes[v*k + l*K + j])) mod (2^61-1)
 * for l < L, v < N; exact integer arithmetic. EINVAL if L*K > k or ldk < N. */
fastlsh_status fastlsh_build_keys(const fastlsh_keys* keys, const int32_t* codes, int64_t N,
                                  int32_t k, uint64_t* keys_out, int64_t ldk,
                                  fastlsh_stream_t stream);

/* Codes (as fastlsh_hash) and keys (as fastlsh_build_keys) for the same rows on `stream`; keys may
 * be NULL (codes only). When the params were packed with fastlsh_params_set_table_size(p, K) so that
 * every CTA hash block holds whole tables (K1j always; K1r when its hash blocks start on multiples
 * of K, e.g. C4's 4 blocks of 500 hashes with K = 10), the keys are built in the hashing kernel's epilogue
 * (codes never re-read); then `codes` may be NULL too — keys only, codes never written to HBM
 * (SURVEY.md §8(f)1). Otherwise codes == NULL is EINVAL. */
fastlsh_status fastlsh_hash_keys(const fastlsh_params* p, const fastlsh_keys* keys,
                                 const float* X, int64_t N, int32_t* codes, uint64_t* keys_out,
                                 int64_t ldk, fastlsh_stream_t stream);

/* ---- bucket tables (§3.2; reading R15) ------------ */

/* Table l is the multiset of pairs (key_l(v), v), v < N, built in canonical bulk form:
 *   sorted_keys[l*N + j]  keys of table l in ascending unsigned order (device u64 [L][N]),
 *   ids[l*N + j]          row id of entry j; equal keys (one bucket) in ascending id (u32 [L][N]),
 *   bucket_start[l*(N+1) + b]  first entry of bucket b for b < nbuckets[l], then N for the rest
 *                              of the row ([L][N+1] u32),
 *   nbuckets[l]           number of distinct keys of table l (device i64 [L]).
 * keys: device u64 [L][ldk] (e.g. fastlsh_build_keys output), ldk >= N. A stable radix sort per
 * table: for N <= 2^22 one global pass on the top 8 bits into 256 segments, each then sorted by one
 * CTA with 7 stable passes over bits 0-55 (in shared memory when it fits one 4096-entry tile);
 * larger N, 8 global LSD passes of 8 bits. Then bucket starts. `workspace` is a device
 * buffer of >= fastlsh_tables_workspace(L, N) bytes (16-byte aligned), owned by the caller.
 * EINVAL on bad sizes/pointers (N must be < 2^32 - 1); asynchronous on `stream`. */
fastlsh_status fastlsh_tables_workspace(int32_t L, int64_t N, size_t* bytes);
fastlsh_status fastlsh_build_tables(const uint64_t* keys, int32_t L, int64_t N, int64_t ldk,
                                    uint64_t* sorted_keys, uint32_t* ids, uint32_t* bucket_start,
                                    int64_t* nbuckets, void* workspace, size_t workspace_bytes,
                                    fastlsh_stream_t stream);

/* ---- query with exact re-ranking (§3.2; reading R16) ------ */

/* For every query q < nq (rows of Q f32 [nq][n], device): the candidates are the DISTINCT rows v of
 * the tables (fastlsh_build_tables output for the data X f32 [N][n]) whose key equals the query's
 * key qkeys[l*ldq + q] in at least one table l (qkeys from fastlsh_hash + fastlsh_build_keys with
 * the same params and keys objects); they are ranked by the exact squared l2 distance in fp32
 * (lane-strided sums, fixed warp reduction) and the first `topk` (1..32) by (distance, id) are
 * written to out_ids[q*topk + r] (int32) / out_dist (f32); fewer candidates pad with -1 / +inf.
 * out_ncand[q] (int64) = number of distinct candidates. workspace: >= fastlsh_query_workspace(N,
 * nq) bytes of device memory (visited bitmaps; zeroed by the call). EINVAL on bad arguments,
 * EUNSUPPORTED if n and L do not fit shared memory. Asynchronous on `stream`. */
fastlsh_status fastlsh_query_workspace(int64_t N, int64_t nq, size_t* bytes);
fastlsh_status fastlsh_query(const float* X, int64_t N, int32_t n, const uint64_t* sorted_keys,
                             const uint32_t* ids, int32_t L, const float* Q, const uint64_t* qkeys, int64_t nq,
                             int64_t ldq, int32_t topk, int32_t* out_ids, float* out_dist, int64_t* out_ncand,
                             void* workspace, size_t workspace_bytes, fastlsh_stream_t stream);

/* ---- extensions (§5, 830-834 App. B; reading R17) ------------- */

/* Angular similarity: out[r] = X[r] / ||X[r]||_2 (a zero row stays zero); out may equal X.
 * Device f32 [N][n], fp32 sums of squares, IEEE sqrt and division. */
fastlsh_status fastlsh_normalize_rows(const float* X, int64_t N, int32_t n, float* out, fastlsh_stream_t stream);
/* *kappa (device f32) = max_r ||X[r]||_2 (0 for N = 0). */
fastlsh_status fastlsh_max_row_norm(const float* X, int64_t N, int32_t n, float* kappa, fastlsh_stream_t stream);
/* MIPS transforms: data (is_query = 0) out[r] = (sqrt(max(kappa^2 - ||X[r]||^2, 0)), X[r]); queries
 * (is_query = 1) out[r] = (0, X[r]). out: device f32 [N][n+1] (kappa: device f32, data only);
 * hash the results with params of dimension n + 1. */
fastlsh_status fastlsh_mips_transform(const float* X, int64_t N, int32_t n, const float* kappa, int32_t is_query,
                                      float* out, fastlsh_stream_t stream);

/* ---- host-buffer entry point (end-to-end; SURVEY.md §3 "config 4 streaming") ----------------- */

/* Hash HOST rows: X_host f32[N*n] (pinned or pageable), codes_host int32[N*k], keys_host
 * uint64[L*N] table-major (may be NULL; `keys` may be NULL). codes_host may be NULL when keys are
 * requested: the codes then never cross PCIe (with K1j they never leave the SM). Rows are streamed in chunks of
 * `chunk_rows` through a double-buffered device workspace owned by the params object, with H2D
 * copies, hashing and D2H copies overlapped on two streams. Synchronous: returns when the host
 * outputs are complete. */
fastlsh_status fastlsh_hash_host(fastlsh_params* p, const fastlsh_keys* keys, const float* X_host,
                                 int64_t N, int32_t* codes_host, uint64_t* keys_host,
                                 int64_t chunk_rows);

/* Hash + keys with the key all-gather fused into the hashing kernel (a8): as
 * fastlsh_hash_keys, but `keys_mc` is the MULTICAST device address (NVSwitch / NVLS, e.g. torch
 * symmetric memory's multicast_ptr) of a [L][ldk] u64 table replicated on every GPU of the group,
 * already offset to this call's first column (global row offset of the rank's chunk). Every key is
 * written with multimem.st, so each GPU's copy of the table receives it; a group barrier after the
 * launches (on every rank) completes the all-gather. codes may be NULL (keys only). K1j only:
 * EUNSUPPORTED when the params are served by another kernel (use fastlsh_hash_keys + an NCCL
 * all-gather then). */
fastlsh_status fastlsh_hash_keys_multicast(const fastlsh_params* p, const fastlsh_keys* keys, const float* X,
                                           int64_t N, int32_t* codes, uint64_t* keys_mc, int64_t ldk,
                                           fastlsh_stream_t stream);

/* NVLS multicast table for the CURRENT device alone (mc.cpp): `bytes` of device memory mapped twice —
 * a unicast address (ordinary loads/stores, *unicast_ptr) and the address of an NVSwitch multicast
 * object bound to it (*multicast_ptr, for multimem.st, e.g. fastlsh_hash_keys_multicast). In a
 * multi-GPU job the multicast table comes from torch symmetric memory instead; this single-device
 * form lets the multimem path be exercised on one GPU. EUNSUPPORTED when the device or driver offers
 * no multicast (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, fabric). Release with fastlsh_multicast_free. */
fastlsh_status fastlsh_multicast_alloc(size_t bytes, void** unicast_ptr, void** multicast_ptr, void** handle);
void fastlsh_multicast_free(void* handle);

/* ---- flags / errors --------------------------------------------------------------------------- */

/* Read (and optionally reset) the per-device counters of sentinel codes written so far:
 * nonfinite (NaN/Inf projections), saturated (finite quotient outside int32). Synchronises
 * `stream`. */
fastlsh_status fastlsh_read_flags(const fastlsh_params* p, uint64_t* nonfinite,
                                  uint64_t* saturated, int32_t reset, fastlsh_stream_t stream);

/* Diagnostic (probe.cu): a plain streaming kernel that reads read_bytes and writes write_bytes per
 * row for `rows` rows (16-byte multiples; in / out 16-byte aligned device buffers of rows*read_bytes
 * and rows*write_bytes; out receives junk). Timing it gives the HBM ceiling of a hashing kernel's
 * own traffic mix, reported beside its roofline fraction (bench.py `roofline.mix_ceiling`). */
fastlsh_status fastlsh_bandwidth_probe(const void* in, void* out, int64_t rows, int32_t read_bytes,
                                       int32_t write_bytes, fastlsh_stream_t stream);

const char* fastlsh_status_string(fastlsh_status s);
const char* fastlsh_last_cuda_error(void); /* thread-local text of the last ECUDA */
int32_t fastlsh_abi_version(void);         /* 1 */

#ifdef __cplusplus
}
#endif
#endif /* FASTLSH_H */
