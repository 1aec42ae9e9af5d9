# direct-epilogue A/B on the P = 1 configs, then the full GPU suite
for env in "" "FASTLSH_NO_DIRECT=1"; do
  for c in "C3 0 25000000" "C0 0 1000000" "C2 32 1000000" "C1 0 1000000"; do
    set -- $c
    env $env timeout 300 python tools/prof_gather.py --config $1 --m $2 --rows $3 --iters 2 --time 2>&1 | grep "ms/launch" | sed "s/; info=.*//;s/^/[$env] /"
  done
done > gpurun_out/direct.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log >> gpurun_out/direct.log
