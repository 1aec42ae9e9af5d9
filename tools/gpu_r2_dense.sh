mkdir -p gpurun_out
timeout 600 python tools/dense_ref.py C1 > gpurun_out/r2_dense_ref.log 2>&1; cat gpurun_out/r2_dense_ref.log
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:e2lsh" -s 1 -c 1 -o gpurun_out/r2_k4_c1 -f \
  python tools/prof_gather.py --config C1 --rows 262144 --iters 1 --dense --dense-e2lsh > gpurun_out/r2_ncu_k4.log 2>&1; echo ncu_k4=$?
