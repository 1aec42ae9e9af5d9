# K1j late wait D = 7 + multi-row bandwidth probe: jit tests, two default bench runs, write-pattern microbench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_memsafety.py -q -x > gpurun_out/r2i_d7_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/r2i_d7_tests.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_wpat tools/microbench_wpattern.cu && ./tools/mb_wpat
for i in 1 2; do
timeout 900 python bench.py --no-dense > gpurun_out/r2i_bench_d7_$i.json 2> gpurun_out/r2i_bench_d7_$i.err; echo bench=$?
python - $i <<'PY'
import json, sys
d = json.loads(open("gpurun_out/r2i_bench_d7_%s.json" % sys.argv[1]).read().strip().splitlines()[-1])
r = d["roofline"]
print("ms/step %.3f value %.4e frac %.4f launch %.4f %s mix %.0f GB/s (%.3f) clocks %s" % (d["ms_per_step"], d["value"], r["frac"], r["launch_ms"], r["launch_ms_min_max"], r["mix_ceiling"]["gbs"], r["mix_ceiling"]["frac_of_ceiling"], d["clocks"]))
PY
done
