# round-2 closing evidence at HEAD (r2w_): GPU suite with parity records, smoke, C3 / C1 bench, C4 stream, reference arm,
# ncu launch list of the C3 bench, ncu --set full of the K4 3xFP16 comparator on C1, per-config table last
mkdir -p gpurun_out
rm -f gpurun_out/r2w_parity.jsonl
FASTLSH_PARITY_LOG=gpurun_out/r2w_parity.jsonl timeout 1800 python -m pytest tests -m gpu -q -rs > gpurun_out/r2w_gpu_tests.log 2>&1; echo tests=$?
tail -4 gpurun_out/r2w_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2w_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/r2w_smoke.log
timeout 900 python bench.py > gpurun_out/r2w_bench_c3.json 2> gpurun_out/r2w_bench_c3.err; echo c3=$?
timeout 600 python bench.py --config C1 > gpurun_out/r2w_bench_c1.json 2> gpurun_out/r2w_bench_c1.err; echo c1=$?
for f in r2w_bench_c3 r2w_bench_c1; do python - $f <<'PY'
import json, sys
d = json.loads(open("gpurun_out/%s.json" % sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "ms/step %.3f value %.4e frac %.4f launch %.4f clocks %s dense %s" % (d["ms_per_step"], d["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d["clocks"], {k: round(v["ms"], 3) for k, v in d["dense_e2lsh"].items() if isinstance(v, dict) and "ms" in v}))
PY
done
timeout 900 python bench.py --config C4 --stream > gpurun_out/r2w_bench_c4_stream.json 2> gpurun_out/r2w_bench_c4_stream.err; echo c4=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2w_bench_reference.json 2> gpurun_out/r2w_bench_reference.err; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k1j|rows_kernel|keys_kernel|gather" -c 200 --csv \
  --log-file gpurun_out/r2w_launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-dense --e2e-steps 1 \
  > gpurun_out/r2w_ncu_bench.log 2>&1; echo ncu_list=$?
timeout 120 python tools/prof_e2lsh.py --precision 2 > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:e2lsh_tcgen05" -s 1 -c 1 -o gpurun_out/r2w_k4_fp16_c1 -f python tools/prof_e2lsh.py --precision 2 > gpurun_out/r2w_ncu_k4.log 2>&1; echo ncu_k4=$?
timeout 1500 python tools/measure_configs.py --out gpurun_out/r2w_configs.jsonl > gpurun_out/r2w_configs.log 2>&1; echo configs=$?
