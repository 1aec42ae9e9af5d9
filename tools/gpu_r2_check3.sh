mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_memsafety.py tests/test_gpu_nvls.py -q -rs > gpurun_out/r2_memsafety.log 2>&1; echo tests=$?
tail -15 gpurun_out/r2_memsafety.log
timeout 300 python tools/prof_gather.py --config C1 --rows 1000000 --iters 2 --kernel rows --time 2>&1 | tail -1
timeout 300 python tools/prof_gather.py --config C3 --rows 8388608 --iters 2 --kernel rows --time 2>&1 | tail -1
