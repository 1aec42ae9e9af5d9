# K1j shared X stage / two-box ring (FL_SHX) vs the one-box form: parity tests + timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jit.py -q -x > gpurun_out/r2i_shx_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/r2i_shx_tests.log
for v in 1 0 1 0; do
  if [ $v = 1 ]; then echo "shx"; timeout 300 python tools/mb_jit.py 2>&1 | head -2 | tail -1; else echo "noshx"; FASTLSH_JIT_NOSHX=1 timeout 300 python tools/mb_jit.py 2>&1 | head -2 | tail -1; fi
done
