# K4 3xFP16 mode (precision 2): parity vs the oracle, then timing on C1 / C3 chunk / C2 (r2t_)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_e2lsh.py -q -x > gpurun_out/r2t_tests.log 2>&1; echo tests=$?; tail -15 gpurun_out/r2t_tests.log
timeout 600 python tools/mb_fp16.py 2>&1 | tail -5
