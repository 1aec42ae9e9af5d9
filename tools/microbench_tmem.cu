// Microbenchmark: can tensor memory serve as a gather source faster than shared memory?
// A lane = row layout in TMEM (thread t of a warp quadrant owns TMEM lane t) turns a warp-uniform
// column address into a conflict-free gather of 32 rows per tcgen05.ld.32x32b.x1; with rows
// interleaved along columns, .xX returns X rows' copies of one coordinate (32*X gathers).
// Also a hybrid: some warps gather from TMEM while the others run the K1 LDS.128 loop, to see
// whether the two read paths add.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbt tools/microbench_tmem.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int X>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&v)[X]);
template <>
__device__ __forceinline__ void tmem_ld<1>(uint32_t t, uint32_t (&v)[1]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v[0]) : "r"(t));
}
template <>
__device__ __forceinline__ void tmem_ld<2>(uint32_t t, uint32_t (&v)[2]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "r"(t));
}
template <>
__device__ __forceinline__ void tmem_ld<4>(uint32_t t, uint32_t (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(t));
}
template <>
__device__ __forceinline__ void tmem_ld<8>(uint32_t t, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                   "=r"(v[7])
                 : "r"(t));
}

__device__ __forceinline__ float4 lds128(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

// TW warps gather from TMEM (MS slots, X columns per load, B loads per wait), the rest from smem
template <int MS, int X, int B, int TW>
__global__ void __launch_bounds__(512, 1) mb(int iters, float* out, int chunks) {
    extern __shared__ float4 sm[];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < chunks * 2; i += blockDim.x) sm[i] = make_float4(1.f, 2.f, 3.f, 4.f);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&slot)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = slot + ((uint32_t)(32 * (warp & 3)) << 16);
    if (warp < 4) {  // initialise this quadrant's 512 columns
        for (int c = 0; c < 512; ++c) {
            const uint32_t v = __float_as_uint(1.0f + lane + c);
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tbase + c), "r"(v) : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    float s = 0.f;
    if (warp < TW) {
        uint32_t col[MS];
        float cf[MS];
#pragma unroll
        for (int t = 0; t < MS; ++t) {
            const uint32_t r = (uint32_t)(t * 2654435761u + warp * 40503u) >> 9;
            col[t] = (r % (512 / X)) * X;
            cf[t] = 1e-3f * (t + 1);
        }
        float acc[X];
#pragma unroll
        for (int x = 0; x < X; ++x) acc[x] = 0.f;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int t0 = 0; t0 < MS; t0 += B) {
                uint32_t v[B][X];
#pragma unroll
                for (int b = 0; b < B; ++b) tmem_ld<X>(tbase + col[t0 + b], v[b]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int b = 0; b < B; ++b)
#pragma unroll
                    for (int x = 0; x < X; ++x) acc[x] = fmaf(__uint_as_float(v[b][x]), cf[t0 + b], acc[x]);
            }
        }
#pragma unroll
        for (int x = 0; x < X; ++x) s += acc[x];
    } else {
        const int q8 = lane & 7;
        uint32_t op[32];
        float cf[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) {
            const uint32_t r = (uint32_t)(t * 2654435761u + threadIdx.x * 40503u) % (uint32_t)(chunks / 8);
            op[t] = (r * 8 + q8) * 16;
            cf[t] = 1e-3f * (t + 1);
        }
        const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
        const uint32_t sub = chunks * 16;
        float acc[2][4] = {};
        const int its = iters * MS * X / 64;  // comparable work per warp
        for (int it = 0; it < its; ++it) {
#pragma unroll
            for (int t = 0; t < 32; ++t) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const float4 v = lds128(base + u * sub + op[t]);
                    acc[u][0] = fmaf(v.x, cf[t], acc[u][0]);
                    acc[u][1] = fmaf(v.y, cf[t], acc[u][1]);
                    acc[u][2] = fmaf(v.z, cf[t], acc[u][2]);
                    acc[u][3] = fmaf(v.w, cf[t], acc[u][3]);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) s += acc[u][0] + acc[u][1] + acc[u][2] + acc[u][3];
    }
    if (s == 12345.f) out[0] = s;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512) : "memory");
    }
}

template <int MS, int X, int B, int TW>
void run(int warps) {
    const int chunks = 968;
    const int iters = 400;
    float* out;
    cudaMalloc(&out, 4);
    const size_t smem = (size_t)chunks * 2 * 16;
    cudaFuncSetAttribute(mb<MS, X, B, TW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = 148;
    mb<MS, X, B, TW><<<grid, warps * 32, smem>>>(4, out, chunks);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mb<MS, X, B, TW><<<grid, warps * 32, smem>>>(iters, out, chunks);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    const int tw = TW < warps ? TW : warps;
    const double g_t = (double)grid * tw * 32 * (double)iters * MS * X;
    const double g_s = (double)grid * (warps - tw) * 32 * (double)(iters * MS * X / 64) * 32 * 2 * 4;
    const double peak = 148.0 * 32 * 1.965e9;
    printf("MS=%d X=%d B=%d tmem_warps=%d/%d: %.3f ms  tmem %.3e + smem %.3e gathers/s = %.3f + %.3f of smem roofline %s\n",
           MS, X, B, tw, warps, ms, g_t / (ms / 1e3), g_s / (ms / 1e3), g_t / (ms / 1e3) / peak,
           g_s / (ms / 1e3) / peak, err ? cudaGetErrorString(err) : "");
    cudaFree(out);
}

int main() {
    run<64, 1, 8, 16>(16);
    run<64, 1, 16, 16>(16);
    run<64, 1, 16, 16>(8);
    run<64, 1, 16, 16>(4);
    run<64, 2, 8, 16>(16);
    run<64, 4, 8, 16>(16);
    run<64, 4, 4, 16>(8);
    run<64, 8, 4, 16>(16);
    run<64, 8, 8, 16>(8);
    run<64, 4, 8, 8>(16);   // 8 TMEM warps + 8 smem warps
    run<64, 4, 8, 4>(16);   // 4 TMEM warps + 12 smem warps
    run<64, 1, 16, 8>(16);
    run<64, 1, 16, 0>(16);  // smem only
    return 0;
}
