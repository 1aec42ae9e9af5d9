# round-2 closing evidence (r2h_ prefix): GPU suite with parity records, benches, per-config table,
# ncu launch list of the C3 bench, ncu --set full of the dense path (kernel 5) on C2 m = 512
mkdir -p gpurun_out
rm -f gpurun_out/r2h_parity.jsonl
FASTLSH_PARITY_LOG=gpurun_out/r2h_parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/r2h_gpu_tests.log 2>&1; echo tests=$?
tail -4 gpurun_out/r2h_gpu_tests.log
timeout 900 python bench.py > gpurun_out/r2h_bench_c3.json 2> gpurun_out/r2h_bench_c3.err; echo c3=$?
timeout 600 python bench.py --config C1 > gpurun_out/r2h_bench_c1.json 2> gpurun_out/r2h_bench_c1.err; echo c1=$?
timeout 900 python bench.py --config C4 --stream --batches 200 --steps 3 > gpurun_out/r2h_bench_c4s.json 2> gpurun_out/r2h_bench_c4s.err; echo c4s=$?
timeout 900 python bench.py --config C2 --sample-dims 512 --steps 5 > gpurun_out/r2h_bench_c2_m512.json 2> gpurun_out/r2h_bench_c2_m512.err; echo c2=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2h_bench_reference.json 2> gpurun_out/r2h_bench_reference.err; echo ref=$?
timeout 1500 python tools/measure_configs.py --out gpurun_out/r2h_configs.jsonl > gpurun_out/r2h_configs.log 2>&1; echo configs=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k1j|rows_kernel|keys_kernel|gather" -c 200 --csv \
  --log-file gpurun_out/r2h_launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-dense --e2e-steps 1 \
  > gpurun_out/r2h_ncu_bench.log 2>&1; echo ncu_list=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:e2lsh" -s 1 -c 1 -o gpurun_out/r2h_dense_c2_m512 -f \
  python tools/prof_dense.py > gpurun_out/r2h_ncu_dense.log 2>&1; echo ncu_dense=$?
