// Microbenchmark: achievable shared-memory gather rate of the K1 inner loop in isolation.
// Each lane holds MS conflict-free offsets (quarter-warp lanes read 8 distinct bank groups) and
// MS coefficients; per slot it issues RG LDS.128 and 4*RG FFMA, like gather_kernel. No staging,
// no epilogue. Prints gathers/s (4 rows x 32 lanes per LDS.128) vs 148*32*clock.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench_lds.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float4 lds128(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

template <int MS, int RG>
__global__ void __launch_bounds__(1024, 1) mb(int iters, float* out, int chunks) {
    extern __shared__ float4 sm[];
    for (int i = threadIdx.x; i < chunks * RG; i += blockDim.x) sm[i] = make_float4(1.f, 2.f, 3.f, 4.f);
    __syncthreads();
    const int lane = threadIdx.x & 31, q8 = lane & 7;
    uint32_t op[MS];
    float cf[MS];
#pragma unroll
    for (int t = 0; t < MS; ++t) {
        // chunk index = 8*(pseudo-random) + lane%8 -> 8 distinct bank groups per quarter
        const uint32_t r = (uint32_t)(t * 2654435761u + threadIdx.x * 40503u) % (uint32_t)(chunks / 8);
        op[t] = (r * 8 + q8) * 16;
        cf[t] = 1e-3f * (t + 1);
    }
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
    const uint32_t sub = chunks * 16;
    float acc[RG][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int t = 0; t < MS; ++t) {
#pragma unroll
            for (int u = 0; u < RG; ++u) {
                const float4 v = lds128(base + u * sub + op[t]);
                acc[u][0] = fmaf(v.x, cf[t], acc[u][0]);
                acc[u][1] = fmaf(v.y, cf[t], acc[u][1]);
                acc[u][2] = fmaf(v.z, cf[t], acc[u][2]);
                acc[u][3] = fmaf(v.w, cf[t], acc[u][3]);
            }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int u = 0; u < RG; ++u) s += acc[u][0] + acc[u][1] + acc[u][2] + acc[u][3];
    if (s == 12345.f) out[0] = s;
}

template <int MS, int RG>
void run(int warps, int ctas_per_sm) {
    const int chunks = 968;  // C1 sub-stage
    const int iters = 2000;
    float* out;
    cudaMalloc(&out, 4);
    size_t smem = (size_t)chunks * RG * 16;
    cudaFuncSetAttribute(mb<MS, RG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int grid = 148 * ctas_per_sm;
    mb<MS, RG><<<grid, warps * 32, smem>>>(10, out, chunks);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mb<MS, RG><<<grid, warps * 32, smem>>>(iters, out, chunks);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    double gathers = (double)grid * warps * 32 * (double)iters * MS * RG * 4;
    double peak = 148.0 * 32 * 1.965e9;
    printf("MS=%d RG=%d warps/CTA=%d CTAs/SM=%d: %.3f ms, %.3e gathers/s = %.3f of smem roofline %s\n", MS, RG, warps,
           ctas_per_sm, ms, gathers / (ms / 1e3), gathers / (ms / 1e3) / peak, err ? cudaGetErrorString(err) : "");
    cudaFree(out);
}

int main() {
    run<62, 1>(8, 1);
    run<62, 2>(8, 1);
    run<62, 2>(4, 2);
    run<32, 2>(16, 1);
    run<32, 1>(16, 1);
    run<32, 2>(8, 2);
    run<16, 2>(16, 2);
    run<62, 4>(8, 1);
    return 0;
}
