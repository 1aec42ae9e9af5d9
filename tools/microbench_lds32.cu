// Microbenchmark: gather rate of a lane = hash-part loop over ROW-MAJOR stages (no transposition).
// Each lane holds MS offsets whose banks are distinct across the warp at every slot position, and
// MS coefficients; per slot it issues R LDS.32 (one per row of the stage, rows STRIDE words apart)
// and R FFMA. Compared with microbench_lds.cu (LDS.128 over column-interleaved 4-row stages), this
// is the gather loop of a design whose stages TMA can fill directly.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_lds32 tools/microbench_lds32.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float lds32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

template <int MS, int R, int STRIDE, int NS>
__global__ void __launch_bounds__(768, 1) mb(int iters, float* out) {
    extern __shared__ float sm[];
    for (int i = threadIdx.x; i < NS * R * STRIDE; i += blockDim.x) sm[i] = 1e-3f * (i & 255);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    uint32_t op[MS];
    float cf[MS];
#pragma unroll
    for (int t = 0; t < MS; ++t) {
        const uint32_t blk = (uint32_t)(t * 2654435761u + threadIdx.x * 40503u) % (uint32_t)(STRIDE / 32);
        op[t] = (blk * 32 + ((lane + 7 * t) & 31)) * 4;  // bank (lane + 7t) mod 32: distinct per slot
        cf[t] = 1e-3f * (t + 1);
    }
    const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(sm);
    float acc[R] = {};
    for (int it = 0; it < iters; ++it) {
        const uint32_t base = s0 + (uint32_t)(it % NS) * (R * STRIDE * 4);
#pragma unroll
        for (int t = 0; t < MS; ++t) {
            const uint32_t a = base + op[t];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = fmaf(lds32(a + r * STRIDE * 4), cf[t], acc[r]);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) s += acc[r];
    if (s == 12345.f) out[0] = s;
}

template <int MS, int R, int STRIDE, int NS>
void run(int warps, int ctas_per_sm) {
    const int iters = 4000;
    float* out;
    cudaMalloc(&out, 4);
    size_t smem = (size_t)NS * R * STRIDE * 4;
    cudaFuncSetAttribute(mb<MS, R, STRIDE, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int grid = 148 * ctas_per_sm;
    mb<MS, R, STRIDE, NS><<<grid, warps * 32, smem>>>(10, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mb<MS, R, STRIDE, NS><<<grid, warps * 32, smem>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    double gathers = (double)grid * warps * 32 * (double)iters * MS * R;
    double peak = 148.0 * 32 * 1.965e9;
    printf("LDS.32 MS=%d R=%d stride=%d NS=%d warps/CTA=%d CTAs/SM=%d: %.3f ms, %.3e gathers/s = %.3f of G_s %s\n", MS,
           R, STRIDE, NS, warps, ctas_per_sm, ms, gathers / (ms / 1e3), gathers / (ms / 1e3) / peak,
           err ? cudaGetErrorString(err) : "");
    cudaFree(out);
}

int main() {
    run<32, 8, 1024, 4>(16, 1);
    run<32, 4, 1024, 4>(16, 1);
    run<32, 8, 1024, 4>(8, 1);
    run<32, 16, 1024, 2>(16, 1);
    run<30, 8, 1024, 4>(16, 1);
    run<20, 8, 128, 4>(16, 1);
    run<20, 16, 128, 4>(16, 1);
    run<20, 8, 128, 4>(24, 1);  // 768 threads
    run<32, 4, 4096, 2>(16, 1);
    run<48, 8, 1024, 4>(8, 1);
    return 0;
}
