// HBM bandwidth for the read/write mixes of the hashing kernels (no compute): rows of R bytes read,
// W bytes written per row (K1j on C3: R = 512 (X), W = 1024 (codes) + 128 (keys)). Plain 16-byte
// vector loads/stores, grid = 4 x 148 CTAs of 512 threads, grid-stride over rows.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_rw tools/microbench_rw.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void rw(const int4* __restrict__ in, int4* __restrict__ out, long long rows, int rq, int wq) {
    // rq / wq: 16-byte words read / written per row; each warp handles one row at a time
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long r = warp; r < rows; r += nw) {
        int4 acc = make_int4(0, 0, 0, 0);
        for (int i = lane; i < rq; i += 32) {
            const int4 v = __ldg(in + r * rq + i);
            acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
        }
        for (int i = lane; i < wq; i += 32) out[r * wq + i] = acc;
    }
}

int main(int argc, char** argv) {
    const long long rows = argc > 1 ? atoll(argv[1]) : 8388608;
    const int mixes[][2] = {{32, 72}, {32, 64}, {32, 32}, {32, 0}, {0, 64}, {32, 8}};
    for (auto& mx : mixes) {
        const int rq = mx[0], wq = mx[1];
        int4 *in = nullptr, *out = nullptr;
        cudaMalloc(&in, rows * (rq ? rq : 1) * 16);
        cudaMalloc(&out, rows * (wq ? wq : 1) * 16);
        cudaMemset(in, 1, rows * (rq ? rq : 1) * 16);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int it = 0; it < 2; ++it) rw<<<4 * 148, 512>>>(in, out, rows, rq, wq);
        cudaEventRecord(e0);
        const int iters = 10;
        for (int it = 0; it < iters; ++it) rw<<<4 * 148, 512>>>(in, out, rows, rq, wq);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= iters;
        const double bytes = (double)rows * (rq + wq) * 16;
        printf("read %4d B/row write %4d B/row: %.3f ms, %.0f GB/s\n", rq * 16, wq * 16, ms, bytes / ms / 1e6);
        cudaFree(in);
        cudaFree(out);
    }
    return 0;
}
