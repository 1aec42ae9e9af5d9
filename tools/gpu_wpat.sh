# write-pattern microbench + K1j at 7 / 8 warps (segment size and occupancy for the C3 code stores)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_wpat tools/microbench_wpattern.cu && ./tools/mb_wpat > gpurun_out/r2i_wpat.txt 2>&1; cat gpurun_out/r2i_wpat.txt
for w in 8 7 6; do echo "warps $w"; FASTLSH_JIT_WARPS=$w timeout 300 python tools/mb_jit.py 2>&1 | head -8; done > gpurun_out/r2i_jit_warps.txt
cat gpurun_out/r2i_jit_warps.txt
