"""Instruction-stream microbenchmark generator (design probe for a params-specialised kernel on long rows).

A lane = row kernel for n > 128 (C2) would run, per warp, a straight-line stream of LDS.128 (4 columns
of its row) and FFMAs with immediate coefficients into H register accumulators — one stream per hash
block, so 8 warps of a CTA run 8 DIFFERENT streams (k = 1000 / 125 hashes per warp). This generator
writes a kernel with exactly that instruction mix, in two flavours:
  spec   — warp w runs stream w (8 distinct streams per SM: instruction fetch is not shared)
  shared — every warp runs stream 0 (the fetch is shared, as in K1j)
and the main() times both; the ratio says whether L2 instruction fetch caps the design.

  python tools/gen_istream.py --fma 4000 --out /tmp/istream.cu   (m = 32 per-warp stream)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_istream /tmp/istream.cu
"""
import argparse
import random

ap = argparse.ArgumentParser()
ap.add_argument("--fma", type=int, default=4000, help="FFMAs per warp stream per tile")
ap.add_argument("--quads", type=int, default=1024, help="LDS.128 per warp stream per tile")
ap.add_argument("--hashes", type=int, default=125)
ap.add_argument("--streams", type=int, default=8)
ap.add_argument("--out", default="/tmp/istream.cu")
args = ap.parse_args()
H, Q = args.hashes, args.quads


def stream(seed):
    rnd = random.Random(seed)
    per_quad = [0] * Q
    for _ in range(args.fma):
        per_quad[rnd.randrange(Q)] += 1
    lines = []
    for q in range(Q):
        if q % 64 == 0:  # a new column chunk: the base comes from shared memory (as after an mbarrier wait)
            lines.append("  sb = ldbase(sb, z);")
        lines.append(f"  x = ld4(sb + {(q % 64) * 512});")
        for _ in range(per_quad[q]):
            h = rnd.randrange(H)
            comp = "xyzw"[rnd.randrange(4)]
            a = rnd.gauss(0, 1)
            lines.append(f"  acc[{h}] = fmaf(x.{comp}, {a:.8e}f, acc[{h}]);")
    return "\n".join(lines)


src = [r"""#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float4 ld4(unsigned a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ldbase(unsigned a, unsigned z) {
  unsigned v;  // sm[0] holds 0: the base is unchanged, but the compiler cannot know it
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(z) : "memory");
  return a + v;
}
"""]
for s in range(args.streams):
    src.append(f"__device__ __noinline__ void stream{s}(unsigned sb, unsigned z, float* out, int tiles) {{\n"
               f"  float acc[{H}];\n#pragma unroll\n  for (int i = 0; i < {H}; ++i) acc[i] = 0.f;\n"
               f"  for (int t = 0; t < tiles; ++t) {{\n  float4 x;\n{stream(s)}\n  }}\n"
               f"  float s = 0.f;\n#pragma unroll\n  for (int i = 0; i < {H}; ++i) s += acc[i];\n"
               f"  out[blockIdx.x * blockDim.x + threadIdx.x] = s;\n}}\n")
src.append(r"""
template <bool SPEC>
__global__ void __launch_bounds__(256, 1) kern(float* out, int tiles) {
  __shared__ __align__(16) float sm[64 * 128];
  for (int i = threadIdx.x; i < 64 * 128; i += blockDim.x) sm[i] = i ? 1e-3f * (i % 97) : 0.f;
  __syncthreads();
  unsigned z = (unsigned)__cvta_generic_to_shared(sm), sb = z + (threadIdx.x & 31) * 16;
  int w = SPEC ? threadIdx.x / 32 : 0;
  switch (w) {
""")
for s in range(args.streams):
    src.append(f"    case {s}: stream{s}(sb, z, out, tiles); break;\n")
src.append(r"""  }
}
int main() {
  float* out; cudaMalloc(&out, 148 * 256 * 4 * 8);
  int tiles = 16;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int spec = 0; spec < 2; ++spec) {
    for (int grid : {148, 296, 1184}) {
      auto go = [&] { if (spec) kern<true><<<grid, 256>>>(out, tiles); else kern<false><<<grid, 256>>>(out, tiles); };
      go(); cudaDeviceSynchronize();
      cudaEventRecord(e0);
      for (int i = 0; i < 5; ++i) go();
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
      double instr = (double)grid * 8 * tiles * (FMA + QUADS);  // warp instructions in the streams
      double ipc = instr / (ms * 1e-3) / 148 / 1.965e9;
      printf("%s grid=%d tiles=%d: %.3f ms, %.2f warp-instr/clk/SM (4 = issue peak), FFMA %.1f%% of peak\n",
             spec ? "spec  " : "shared", grid, tiles, ms, ipc, 100.0 * ipc * FMA / (FMA + QUADS) / 4);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
""")
text = "".join(src).replace("FMA + QUADS", f"{args.fma} + {Q}").replace("* FMA /", f"* {args.fma} /")
open(args.out, "w").write(text)
