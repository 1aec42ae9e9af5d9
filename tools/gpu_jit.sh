#!/bin/bash
# K1j: tests + microbenchmark (+ the whole GPU suite when FULL=1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jit.py -x -q > gpurun_out/jit_tests.log 2>&1
timeout 600 python tools/mb_jit.py > gpurun_out/jit_mb.log 2>&1
tail -3 gpurun_out/jit_tests.log; cat gpurun_out/jit_mb.log
if [ "$FULL" = 1 ]; then
  timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_suite.log 2>&1
  tail -5 gpurun_out/gpu_suite.log
fi
