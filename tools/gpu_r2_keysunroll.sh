# K1r code-tile keys with the code loop unrolled by 4: timing (C1, C4) + key/code-tile parity (r2r_)
mkdir -p gpurun_out
timeout 300 python tools/mb_fused_keys.py 2>&1 | tail -4
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "code_tile or host_entry" > gpurun_out/r2r_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/r2r_tests.log
