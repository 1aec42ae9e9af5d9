# ncu --set full of K1r on C1 (262144 rows) and C3 (4M rows)
mkdir -p gpurun_out
timeout 120 python tools/prof_gather.py --config C1 --rows 262144 --iters 2 --kernel rows > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:rows_kernel" -s 1 -c 1 -o gpurun_out/rows_c1 python tools/prof_gather.py --config C1 --rows 262144 --iters 2 --kernel rows > gpurun_out/ncu_rows_c1.log 2>&1; echo c1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:rows_kernel" -s 1 -c 1 -o gpurun_out/rows_c3 python tools/prof_gather.py --config C3 --rows 4000000 --iters 2 --kernel rows > gpurun_out/ncu_rows_c3.log 2>&1; echo c3=$?
