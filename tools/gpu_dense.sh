# dense path for FastLSH params (kernel 5): tests + C2 m sweep timing
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dense_path.py tests/test_gpu_e2lsh.py -x -q > gpurun_out/dense_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/dense_tests.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "small_full_parity or full_size_sampled_parity and C2" > gpurun_out/dense_parity.log 2>&1; echo parity=$?
tail -3 gpurun_out/dense_parity.log
timeout 900 python tools/mb_dense.py > gpurun_out/dense_mb.log 2>&1; echo mb=$?
cat gpurun_out/dense_mb.log
