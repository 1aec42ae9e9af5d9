# round-2 final evidence: GPU suite (parity records), benches, ncu of the final K1j, launch list
mkdir -p gpurun_out
rm -f gpurun_out/r2g_parity.jsonl
FASTLSH_PARITY_LOG=gpurun_out/r2g_parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/r2g_gpu_tests.log 2>&1; echo tests=$?
tail -4 gpurun_out/r2g_gpu_tests.log
timeout 900 python bench.py > gpurun_out/r2g_bench_c3.json 2> gpurun_out/r2g_bench_c3.err; echo c3=$?
timeout 600 python bench.py --config C1 > gpurun_out/r2g_bench_c1.json 2> gpurun_out/r2g_bench_c1.err; echo c1=$?
timeout 900 python bench.py --config C4 --stream --batches 200 --steps 3 > gpurun_out/r2g_bench_c4s.json 2> gpurun_out/r2g_bench_c4s.err; echo c4s=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k1j|rows_kernel|keys_kernel|gather" -c 200 --csv \
  --log-file gpurun_out/r2g_launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-dense --e2e-steps 1 \
  > gpurun_out/r2g_ncu_bench.log 2>&1; echo ncu_list=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k1j" -s 1 -c 1 -o gpurun_out/r2g_k1j_c3_keys -f \
  python tools/prof_jit.py --mode keys > gpurun_out/r2g_ncu_k1j.log 2>&1; echo ncu_full=$?
