# K1r ablation: full kernel vs no code output (1) vs no refills (2) vs both (3), C1 and C3
for d in 0 1 2 3; do
  for c in "C1 0 1000000" "C3 0 25000000" "C2 32 1000000"; do
    set -- $c
    FASTLSH_K1R_DEBUG=$d timeout 120 python tools/prof_gather.py --config $1 --m $2 --rows $3 --iters 2 --time --kernel rows 2>&1 | grep "ms/launch" | sed "s/; info=.*//;s/^/[debug=$d] /"
  done
done > gpurun_out/ablate.log 2>&1
cat gpurun_out/ablate.log
