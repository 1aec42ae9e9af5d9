# K1r gather loads as plain asm ordered by data dependencies (stage_base / acc_fence) instead of volatile + memory clobber (r2s_)
mkdir -p gpurun_out
timeout 300 python tools/mb_fused_keys.py 2>&1 | tail -3
timeout 300 python tools/mb_c2.py 2>&1 | tail -2 | cut -c1-120
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_memsafety.py -q -x > gpurun_out/r2s_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/r2s_tests.log
