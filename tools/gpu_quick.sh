timeout 600 python -m pytest tests -m gpu -x -q -k "query" 2>&1 | tail -2 > gpurun_out/qq.log
timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-dense --e2e-steps 1 > gpurun_out/q.json 2>gpurun_out/q.err; echo bench=$?
tail -3 gpurun_out/q.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/q.json").read().strip().splitlines()[-1])
print("ms/step %.3f" % d["ms_per_step"], "value %.3e" % d["value"], d["tables"]["ms"], d["queries"])
PY
cat gpurun_out/qq.log
