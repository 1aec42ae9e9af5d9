# session check: LDS.32 microbenchmark, GPU suite, default bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/mb.log 2>&1
timeout 120 ./tools/mb_lds32 >> gpurun_out/mb.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_lds tools/microbench_lds.cu && timeout 120 /tmp/mb_lds >> gpurun_out/mb.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cat gpurun_out/mb.log
