# K1j late-wait default (D = 6): jit parity tests, depth A/B around 6, default bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_memsafety.py -q -x > gpurun_out/r2i_late_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/r2i_late_tests.log
run() { echo "$1: $(env $2 timeout 300 python tools/mb_jit.py 2>&1 | head -2 | tail -1 | cut -c1-120)"; }
for rep in 1 2; do
for d in 5 6 7; do run "late$d" "FASTLSH_JIT_LATEWAIT=$d"; done
done
timeout 900 python bench.py --no-dense > gpurun_out/r2i_bench_late.json 2> gpurun_out/r2i_bench_late.err; echo bench=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2i_bench_late.json").read().strip().splitlines()[-1])
print("ms/step %.3f value %.4e frac %.4f launch %.4f clocks %s" % (d["ms_per_step"], d["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d["clocks"]))
PY
