for c in "C3 0 25000000" "C0 0 10000"; do
  set -- $c
  timeout 120 python tools/prof_gather.py --config $1 --m $2 --rows $3 --iters 2 --time --kernel rows 2>&1 | grep "ms/launch" | sed "s/; info=.*//"
done
timeout 300 python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-dense --no-tables --e2e-steps 1 > gpurun_out/c3.json 2>gpurun_out/c3.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/c3.json").read().strip().splitlines()[-1])
print("C3 bench ms/step %.3f" % d["ms_per_step"], "value %.3e" % d["value"], d["breakdown_ms"], d["keys_fused"], d["roofline"]["frac"])
PY
