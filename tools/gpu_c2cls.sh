# K1r C2 stage-geometry A/B (class 5 = n > 2016): parity on C2 shapes, then timing of m = 32 / 128
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "rows_kernel or small_full_parity or edge" > gpurun_out/r2i_c2cls_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/r2i_c2cls_tests.log
timeout 600 python tools/mb_c2.py
timeout 600 python tools/mb_c2.py
