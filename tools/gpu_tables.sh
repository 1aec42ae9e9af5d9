# K5 MSD form: table / query tests (bit-exact vs the oracle), timing on random and C1 keys, sizes across the MSD threshold
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_memsafety.py -q -x -k "tables or query or guard or transforms or mips or chunked" > gpurun_out/r2n_tables_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/r2n_tables_tests.log
timeout 300 python tools/prof_tables.py 50 1000000
timeout 300 python tools/prof_tables.py 16 4194304
timeout 300 python tools/prof_tables.py 4 8000000
timeout 600 python bench.py --config C1 --no-dense --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2n_bench_c1.json 2> gpurun_out/r2n_bench_c1.err; echo c1=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2n_bench_c1.json").read().strip().splitlines()[-1])
print("tables", d["tables"]); print("queries", d["queries"])
PY
