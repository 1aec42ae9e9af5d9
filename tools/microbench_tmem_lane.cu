// Does tcgen05.ld.32x32b honour or ignore the lane field of taddr? Each quadrant writes its own
// pattern; every warp then reads with lane field 0 and with its own quadrant base.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(uint32_t* out) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)), "r"(32) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t base = slot;
    const uint32_t own = base + ((uint32_t)(32 * (warp & 3)) << 16);
    uint32_t v = 1000u * (warp & 3) + lane;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(own), "r"(v) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t a, b;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(a) : "r"(own));
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(b) : "r"(base));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    out[threadIdx.x * 2] = a;
    out[threadIdx.x * 2 + 1] = b;
    out[512] = base;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(32) : "memory");
    }
}
int main() {
    uint32_t* d; cudaMalloc(&d, 4 * 520);
    cudaMemset(d, 0xff, 4 * 520);
    k<<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    uint32_t h[520]; cudaMemcpy(h, d, 4 * 520, cudaMemcpyDeviceToHost);
    printf("err=%s base=%u\n", cudaGetErrorString(e), h[512]);
    for (int w = 0; w < 4; ++w) printf("warp %d lane 5: own=%u lane0-field=%u\n", w, h[(w * 32 + 5) * 2], h[(w * 32 + 5) * 2 + 1]);
    return 0;
}
