timeout 600 python -m pytest tests -m gpu -x -q -k "chunked or keys or host_entry or smoke" 2>&1 | tail -2
timeout 900 python bench.py --config C3 --steps 3 --e2e-steps 1 --no-dense --no-cpu-baseline > gpurun_out/c3.json 2>gpurun_out/c3.err; echo c3=$?
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-dense --e2e-steps 1 > gpurun_out/q.json 2>gpurun_out/q.err; echo bench=$?
python - <<'PY'
import json
for f in ("gpurun_out/c3.json", "gpurun_out/q.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, "ms/step %.3f" % d["ms_per_step"], "value %.3e" % d["value"], d["breakdown_ms"], "frac %.3f" % d["roofline"]["frac"], "e2e %.3e" % d["e2e"]["value"])
PY
