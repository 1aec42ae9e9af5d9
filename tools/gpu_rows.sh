# K1r bring-up: parity tests of the row-major kernel, then K1 vs K1r timings per config
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "rows" > gpurun_out/rows_tests.log 2>&1; echo rows_tests=$? >> gpurun_out/rows_tests.log
tail -30 gpurun_out/rows_tests.log
for c in "C1 0 1000000" "C3 0 25000000" "C2 32 1000000" "C2 128 1000000" "C4 0 100000" "C0 0 10000"; do
  set -- $c
  for k in smem rows; do
    timeout 120 python tools/prof_gather.py --config $1 --m $2 --rows $3 --iters 2 --time --kernel $k 2>&1 | grep "ms/launch" | sed "s/; info=.*//;s/^/[$k] /"
  done
done > gpurun_out/rows_timing.log 2>&1
for pp in 1 2; do FASTLSH_ROW_PARTS=$pp timeout 120 python tools/prof_gather.py --config C1 --rows 1000000 --iters 2 --time --kernel rows 2>&1 | grep "ms/launch" | sed "s/; info=.*//;s/^/[rows P=$pp] /"; done >> gpurun_out/rows_timing.log 2>&1
cat gpurun_out/rows_timing.log
