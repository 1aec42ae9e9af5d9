# after the dense path became opt-in (r2k_ prefix): GPU suite with parity records (C2 m = 512 / 4096 now
# through K1r), per-config table, C2 m = 512 / 4096 bench lines (K1r headline, kernel 5 as analysis)
mkdir -p gpurun_out
rm -f gpurun_out/r2k_parity.jsonl
FASTLSH_PARITY_LOG=gpurun_out/r2k_parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/r2k_gpu_tests.log 2>&1; echo tests=$?
tail -4 gpurun_out/r2k_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.log 2>&1; echo smoke=$?
timeout 1500 python tools/measure_configs.py --out gpurun_out/r2k_configs.jsonl > gpurun_out/r2k_configs.log 2>&1; echo configs=$?
timeout 900 python bench.py --config C2 --sample-dims 512 --steps 3 > gpurun_out/r2k_bench_c2_m512.json 2> gpurun_out/r2k_bench_c2_m512.err; echo c2_m512=$?
timeout 1200 python bench.py --config C2 --sample-dims 4096 --steps 3 > gpurun_out/r2k_bench_c2_m4096.json 2> gpurun_out/r2k_bench_c2_m4096.err; echo c2_m4096=$?
