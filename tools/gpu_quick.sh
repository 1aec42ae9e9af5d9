timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/q_pytest.log
cat gpurun_out/q_pytest.log
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-dense --e2e-steps 1 > gpurun_out/q.json 2>gpurun_out/q.err; echo bench=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/q.json").read().strip().splitlines()[-1])
print("ms/step %.3f" % d["ms_per_step"], "value %.3e" % d["value"], d["breakdown_ms"], "frac %.3f" % d["roofline"]["frac"], "e2e %.3e" % d["e2e"]["value"])
PY
