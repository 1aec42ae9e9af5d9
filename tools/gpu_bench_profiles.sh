# bench line, launch list of the same command under ncu, ncu --set full of K1r on C1, per-config table
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err; echo bench=$?
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r1_bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r1_ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:rows_kernel" -s 1 -c 1 -o gpurun_out/r1_rows_c1 python tools/prof_gather.py --config C1 --rows 262144 --iters 3 > gpurun_out/r1_ncu_full.log 2>&1; echo ncu2=$?
timeout 1200 python tools/measure_configs.py --out gpurun_out/configs.jsonl > gpurun_out/configs.log 2>&1; echo configs=$?
