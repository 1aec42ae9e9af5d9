for c in "C3 0 25000000" "C0 0 10000" "C1 0 1000000"; do
  set -- $c
  timeout 120 python tools/prof_gather.py --config $1 --m $2 --rows $3 --iters 2 --time 2>&1 | grep "ms/launch" | sed "s/; info=.*//"
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "rows or C3 or C0 or edge or keys" 2>&1 | tail -1
