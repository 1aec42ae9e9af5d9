for d in -1 4 6; do
  for c in "C1 0 1000000" "C4 0 100000"; do
    set -- $c
    FASTLSH_DUAL_CLS=$d timeout 120 python tools/prof_gather.py --config $1 --m $2 --rows $3 --iters 2 --time --kernel rows 2>&1 | grep "ms/launch" | sed "s/; info=.*//;s/^/[dual_cls=$d] /"
  done
done
