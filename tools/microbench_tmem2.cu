// Microbenchmark 2: the TMEM gather loop with realistic parameter delivery.
// Parameters (TMEM column, coefficient) per slot live in shared memory and are read with
// warp-uniform (broadcast) LDS.128 (2 slots per load); the column goes to a uniform register
// (R2UR) for tcgen05.ld.32x32b.xX; X FFMAs per slot; a partial (X floats per lane) is stored to
// shared memory every PART slots, like a hash part finishing. Prints gathers/s vs the smem roofline.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_tmem2 tools/microbench_tmem2.cu
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

__device__ __forceinline__ uint4 lds128u(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

// MODE 0: params via LDS.128 broadcast; MODE 1: params via __ldg (L1) broadcast
template <int X, int B, int PART, int MODE>
__global__ void __launch_bounds__(1024, 1) mb(int iters, float* out, const uint2* gparams, int S) {
    extern __shared__ __align__(16) uint2 prm[];  // [S] (col, coef bits)
    __shared__ uint32_t slot;
    __shared__ __align__(16) float partials[32][32 * 4];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < S; i += blockDim.x) prm[i] = gparams[i];
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
    if (warp < 4) {
        for (int c = 0; c < 512; ++c) {
            const uint32_t v = __float_as_uint(1.0f + lane + c);
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tbase + c), "r"(v) : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    const uint32_t p0 = (uint32_t)__cvta_generic_to_shared(prm);
    const int nw = blockDim.x >> 5;
    // each warp walks its own contiguous share of the slot list
    const int per = (S / nw) & ~(B - 1);
    const int first = warp * per;
    float acc[X];
#pragma unroll
    for (int x = 0; x < X; ++x) acc[x] = 0.f;
    float keep = 0.f;
    int cnt = 0;
    for (int it = 0; it < iters; ++it) {
        for (int t0 = first; t0 < first + per; t0 += B) {
            uint32_t col[B];
            float cf[B];
#pragma unroll
            for (int b = 0; b < B; b += 2) {
                uint4 q;
                if (MODE == 0) {
                    q = lds128u(p0 + (t0 + b) * 8);
                } else {
                    q = __ldg(reinterpret_cast<const uint4*>(gparams + t0 + b));
                }
                col[b] = q.x;
                cf[b] = __uint_as_float(q.y);
                col[b + 1] = q.z;
                cf[b + 1] = __uint_as_float(q.w);
            }
            uint32_t v[B][X];
#pragma unroll
            for (int b = 0; b < B; ++b) tmem_ld<X>(tbase + col[b], v[b]);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int b = 0; b < B; ++b) {
#pragma unroll
                for (int x = 0; x < X; ++x) acc[x] = fmaf(__uint_as_float(v[b][x]), cf[b], acc[x]);
            }
            cnt += B;
            if (cnt >= PART) {  // a hash part ends: publish the partial, restart
                cnt = 0;
#pragma unroll
                for (int x = 0; x < X; ++x) {
                    partials[warp][x * 32 + lane] = acc[x];
                    keep += acc[x];
                    acc[x] = 0.f;
                }
            }
        }
    }
#pragma unroll
    for (int x = 0; x < X; ++x) keep += acc[x];
    if (keep == 12345.f) out[0] = keep + partials[warp][lane];
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512) : "memory");
    }
}

template <int X, int B, int PART, int MODE>
void run(int warps, int S) {
    const int iters = 200;
    float* out;
    cudaMalloc(&out, 4);
    uint2* hp = new uint2[S];
    for (int i = 0; i < S; ++i) {
        const uint32_t r = (uint32_t)(i * 2654435761u) >> 9;
        hp[i].x = (r % (480 / X)) * X;
        float c = 1e-3f * (i % 97);
        hp[i].y = *reinterpret_cast<uint32_t*>(&c);
    }
    uint2* dp;
    cudaMalloc(&dp, S * 8);
    cudaMemcpy(dp, hp, S * 8, cudaMemcpyHostToDevice);
    const size_t smem = (size_t)S * 8;
    auto k = mb<X, B, PART, MODE>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = 148;
    k<<<grid, warps * 32, smem>>>(2, out, dp, S);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<grid, warps * 32, smem>>>(iters, out, dp, S);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    const int per = (S / warps) & ~(B - 1);
    const double g = (double)grid * warps * 32 * (double)iters * per * X;
    const double peak = 148.0 * 32 * 1.965e9;
    printf("X=%d B=%d PART=%d mode=%s warps=%d S=%d: %.3f ms  %.3e gathers/s = %.3f of smem roofline %s\n", X, B,
           PART, MODE ? "ldg" : "lds", warps, S, ms, g / (ms / 1e3), g / (ms / 1e3) / peak,
           err ? cudaGetErrorString(err) : "");
    cudaFree(out);
    cudaFree(dp);
    delete[] hp;
}

int main() {
    run<2, 8, 16, 0>(16, 16384);
    run<2, 16, 16, 0>(16, 16384);
    run<2, 8, 16, 0>(32, 16384);
    run<2, 8, 16, 0>(8, 16384);
    run<1, 8, 16, 0>(16, 16384);
    run<1, 16, 16, 0>(32, 16384);
    run<4, 8, 16, 0>(16, 16384);
    run<2, 8, 16, 1>(16, 16384);
    run<2, 8, 16, 1>(32, 16384);
    run<2, 8, 16, 1>(16, 65536);
    run<2, 8, 64, 0>(16, 16384);
    return 0;
}
