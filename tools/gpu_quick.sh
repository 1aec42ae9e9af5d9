timeout 600 python -m pytest tests -m gpu -x -q -k "keys" 2>&1 | tail -1 > gpurun_out/qq.log
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-dense --no-tables --e2e-steps 1 > gpurun_out/q.json 2>gpurun_out/q.err
timeout 300 python bench.py --config C3 --steps 2 --no-cpu-baseline --no-dense --no-tables --e2e-steps 1 > gpurun_out/c3.json 2>gpurun_out/c3.err
python - <<'PY'
import json
for f in ("gpurun_out/q.json", "gpurun_out/c3.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, "ms/step %.3f" % d["ms_per_step"], "value %.3e" % d["value"], d["breakdown_ms"])
PY
cat gpurun_out/qq.log
