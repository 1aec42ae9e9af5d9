# dense fall-through fix + K1r limb keys: dense / rows-keys / keys tests, C1 bench (hash + keys from the code tile)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dense_path.py tests/test_gpu_parity.py -q -x -k "dense or keys or rows_kernel or host" > gpurun_out/r2l_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/r2l_tests.log
for i in 1 2; do
timeout 600 python bench.py --config C1 --no-dense --no-tables --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2l_bench_c1_$i.json 2> gpurun_out/r2l_bench_c1_$i.err; echo c1=$?
python - $i <<'PY'
import json, sys
d = json.loads(open("gpurun_out/r2l_bench_c1_%s.json" % sys.argv[1]).read().strip().splitlines()[-1])
print("C1 ms/step %.3f value %.4e frac %.4f launch %.4f clocks %s" % (d["ms_per_step"], d["value"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d["clocks"]))
PY
done
