# re-entry after the K5 MSD commits (r2o_): full GPU suite with parity records, smoke, C3 (default) and C1 bench lines
mkdir -p gpurun_out
rm -f gpurun_out/r2o_parity.jsonl
FASTLSH_PARITY_LOG=gpurun_out/r2o_parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/r2o_gpu_tests.log 2>&1; echo tests=$?
tail -4 gpurun_out/r2o_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2o_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/r2o_smoke.log
timeout 900 python bench.py > gpurun_out/r2o_bench_c3.json 2> gpurun_out/r2o_bench_c3.err; echo c3=$?
timeout 600 python bench.py --config C1 > gpurun_out/r2o_bench_c1.json 2> gpurun_out/r2o_bench_c1.err; echo c1=$?
for f in r2o_bench_c3 r2o_bench_c1; do python - $f <<'PY'
import json, sys
d = json.loads(open("gpurun_out/%s.json" % sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "ms/step %.3f value %.4e frac %.4f launch %.4f clocks %s" % (d["ms_per_step"], d["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d["clocks"]))
PY
done
