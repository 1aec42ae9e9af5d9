mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -5 gpurun_out/gpu_tests.log
for c in "C1 0 1000000" "C3 0 25000000" "C2 32 1000000" "C4 0 100000"; do
  set -- $c
  timeout 120 python tools/prof_gather.py --config $1 --m $2 --rows $3 --iters 2 --time --kernel rows 2>&1 | grep "ms/launch" | sed "s/; info=.*//"
done
