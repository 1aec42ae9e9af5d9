# final round-2 evidence (r2v_): GPU suite with parity records, smoke, C3 / C1 bench lines, C4 stream, per-config table,
# ncu --set full of the K4 3xFP16 comparator on C1
mkdir -p gpurun_out
rm -f gpurun_out/r2v_parity.jsonl
FASTLSH_PARITY_LOG=gpurun_out/r2v_parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/r2v_gpu_tests.log 2>&1; echo tests=$?
tail -4 gpurun_out/r2v_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2v_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/r2v_smoke.log
timeout 900 python bench.py > gpurun_out/r2v_bench_c3.json 2> gpurun_out/r2v_bench_c3.err; echo c3=$?
timeout 600 python bench.py --config C1 > gpurun_out/r2v_bench_c1.json 2> gpurun_out/r2v_bench_c1.err; echo c1=$?
for f in r2v_bench_c3 r2v_bench_c1; do python - $f <<'PY'
import json, sys
d = json.loads(open("gpurun_out/%s.json" % sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "ms/step %.3f value %.4e frac %.4f launch %.4f clocks %s dense %s" % (d["ms_per_step"], d["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d["clocks"], {k: round(v["ms"], 3) for k, v in d["dense_e2lsh"].items() if isinstance(v, dict) and "ms" in v}))
PY
done
timeout 1500 python tools/measure_configs.py --out gpurun_out/r2v_configs.jsonl > gpurun_out/r2v_configs.log 2>&1; echo configs=$?
timeout 120 python tools/prof_e2lsh.py --precision 2 > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:e2lsh_tcgen05" -s 1 -c 1 -o gpurun_out/r2v_k4_fp16_c1 -f python tools/prof_e2lsh.py --precision 2 > gpurun_out/r2v_ncu_k4.log 2>&1; echo ncu_k4=$?
