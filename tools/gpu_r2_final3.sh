# round-2 closing evidence after the K1j late wait and the K1r 6-row class (r2j_ prefix): GPU suite with
# parity records, benches (C3 default, C1, C2 m=32/128, C4 stream, reference arm), per-config table,
# ncu launch list of the C3 bench, ncu --set full of K1j (C3 chunk) and K1r (C2 m = 32)
mkdir -p gpurun_out
rm -f gpurun_out/r2j_parity.jsonl
FASTLSH_PARITY_LOG=gpurun_out/r2j_parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/r2j_gpu_tests.log 2>&1; echo tests=$?
tail -4 gpurun_out/r2j_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2j_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/r2j_bench_c3.json 2> gpurun_out/r2j_bench_c3.err; echo c3=$?
timeout 600 python bench.py --config C1 > gpurun_out/r2j_bench_c1.json 2> gpurun_out/r2j_bench_c1.err; echo c1=$?
for m in 32 128; do
timeout 900 python bench.py --config C2 --sample-dims $m --steps 5 > gpurun_out/r2j_bench_c2_m$m.json 2> gpurun_out/r2j_bench_c2_m$m.err; echo c2_m$m=$?
done
timeout 900 python bench.py --config C4 --stream --batches 200 --steps 3 > gpurun_out/r2j_bench_c4s.json 2> gpurun_out/r2j_bench_c4s.err; echo c4s=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2j_bench_reference.json 2> gpurun_out/r2j_bench_reference.err; echo ref=$?
timeout 1500 python tools/measure_configs.py --out gpurun_out/r2j_configs.jsonl > gpurun_out/r2j_configs.log 2>&1; echo configs=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k1j|rows_kernel|keys_kernel|gather" -c 200 --csv \
  --log-file gpurun_out/r2j_launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-dense --e2e-steps 1 \
  > gpurun_out/r2j_ncu_bench.log 2>&1; echo ncu_list=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k1j" -s 1 -c 1 -o gpurun_out/r2j_k1j_c3_keys -f \
  python tools/prof_jit.py --mode keys > gpurun_out/r2j_ncu_k1j.log 2>&1; echo ncu_k1j=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:rows_kernel" -s 1 -c 1 -o gpurun_out/r2j_rows_c2_m32 -f \
  python tools/prof_gather.py --config C2 --m 32 --rows 131072 --iters 2 --kernel rows > gpurun_out/r2j_ncu_c2.log 2>&1; echo ncu_c2=$?
