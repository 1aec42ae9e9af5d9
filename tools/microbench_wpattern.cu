// Write-pattern check for K1j's code stores: a 32-row tile of 1 KB code rows written
// (a) row-contiguous (each warp instruction covers 512 contiguous bytes) or (b) as K1j's TMA boxes do:
// 8 groups of 128-B segments, one per row (rows 1 KB apart), group by group. Plus 512 B/row of reads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_wpat tools/microbench_wpattern.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void wr(const int4* __restrict__ in, int4* __restrict__ out, long long tiles, int boxed) {
    // boxed = 0: row-contiguous; otherwise segments of boxed * 128 B per row (1, 2, 4 groups)
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long t = warp; t < tiles; t += nw) {
        int4 acc = make_int4(lane, 1, 2, 3);
        const int4* src = in + t * 32 * 32;  // 32 rows x 512 B
        for (int i = lane; i < 32 * 32; i += 32) {
            const int4 v = __ldg(src + i);
            acc.x ^= v.x;
        }
        int4* dst = out + t * 32 * 64;  // 32 rows x 1 KB (64 int4)
        if (!boxed) {
            for (int i = lane; i < 32 * 64; i += 32) dst[i] = acc;
        } else {
            const int seg = 8 * boxed;                 // int4 per segment
            for (int g = 0; g < 64 / seg; ++g)         // segment g of every row
                for (int i = lane; i < 32 * seg; i += 32) {
                    const int r = i / seg, c = i % seg;
                    dst[r * 64 + g * seg + c] = acc;
                }
        }
    }
}

int main() {
    const long long tiles = 262144;  // 8.4M rows
    int4 *in, *out;
    cudaMalloc(&in, tiles * 32 * 512);
    cudaMalloc(&out, tiles * 32 * 1024);
    cudaMemset(in, 1, tiles * 32 * 512);
    for (int boxed : {0, 1, 2, 4}) {
        for (int it = 0; it < 2; ++it) wr<<<4 * 148, 512>>>(in, out, tiles, boxed);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        for (int it = 0; it < 10; ++it) wr<<<4 * 148, 512>>>(in, out, tiles, boxed);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 10;
        printf("segments %d B (0 = row-contiguous): %.3f ms, %.0f GB/s\n", boxed * 128, ms,
               tiles * 32.0 * 1536 / ms / 1e6);
    }
    return 0;
}
