mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
bash tools/gpu_round4.sh
timeout 900 python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-dense --no-tables --e2e-steps 1 > gpurun_out/r1_bench_c3.json 2> gpurun_out/r1_bench_c3.err; echo bench_c3=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1_ref.json 2> gpurun_out/r1_ref.err; echo ref=$?
