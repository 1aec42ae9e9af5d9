for c in "C4 0 100000" "C2 128 1000000" "C2 512 250000"; do
  set -- $c
  for pp in 0 1 2 4 8; do
    FASTLSH_ROW_PARTS=$pp timeout 120 python tools/prof_gather.py --config $1 --m $2 --rows $3 --iters 2 --time --kernel rows 2>&1 | grep "ms/launch" | sed "s/; info=.*//;s/^/[P=$pp] /"
  done
done
