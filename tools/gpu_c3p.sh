for pp in 0 2 4; do
  FASTLSH_ROW_PARTS=$pp timeout 120 python tools/prof_gather.py --config C3 --rows 25000000 --iters 2 --time --kernel rows 2>&1 | grep "ms/launch" | sed "s/; info=.*//;s/^/[P=$pp] /"
done
