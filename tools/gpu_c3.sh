for d in 0 1 2 3; do
  FASTLSH_K1R_DEBUG=$d timeout 120 python tools/prof_gather.py --config C3 --rows 25000000 --iters 2 --time --kernel rows 2>&1 | grep "ms/launch" | sed "s/; info=.*//;s/^/[debug=$d] /"
done > gpurun_out/c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:rows_kernel" -s 1 -c 1 -o gpurun_out/rows_c3 python tools/prof_gather.py --config C3 --rows 4000000 --iters 2 --kernel rows > gpurun_out/ncu_rows_c3.log 2>&1; echo c3=$?
cat gpurun_out/c3.log
