# re-entry check after the container was re-created: GPU suite, smoke, default (C3) bench
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/r2i_gpu_tests.log 2>&1; echo tests=$?
tail -4 gpurun_out/r2i_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2i_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/r2i_smoke.log
timeout 900 python bench.py > gpurun_out/r2i_bench_c3.json 2> gpurun_out/r2i_bench_c3.err; echo c3=$?
tail -c 3000 gpurun_out/r2i_bench_c3.json
