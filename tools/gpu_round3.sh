# round evidence (K1r + keys from its code tile): GPU suite, C1 bench, C3 bench, launch list, ncu full of K1r
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err; echo bench=$?
timeout 900 python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-dense --no-tables --e2e-steps 1 > gpurun_out/r1_bench_c3.json 2> gpurun_out/r1_bench_c3.err; echo bench_c3=$?
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r1_bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r1_ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:rows_kernel" -s 1 -c 1 -o gpurun_out/r1_rows_c1_keys python tools/prof_gather.py --config C1 --rows 262144 --iters 3 --fused-keys > gpurun_out/r1_ncu_full.log 2>&1; echo ncu2=$?
