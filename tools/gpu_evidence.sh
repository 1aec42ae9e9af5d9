# round evidence: GPU suite, smoke, default bench line, per-config table
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err; echo bench=$?
timeout 1200 python tools/measure_configs.py --out gpurun_out/configs.jsonl > gpurun_out/configs.log 2>&1; echo configs=$?
