timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "rows or keys or host" 2>&1 | tail -3
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-dense --no-tables --e2e-steps 1 > gpurun_out/q.json 2>gpurun_out/q.err
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-dense --no-tables --e2e-steps 1 --separate-keys > gpurun_out/q2.json 2>gpurun_out/q2.err
python - <<'PY'
import json
for f in ("gpurun_out/q.json", "gpurun_out/q2.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, "ms/step %.3f" % d["ms_per_step"], "value %.3e" % d["value"], d["breakdown_ms"], d["keys_fused"], "e2e %.3e" % d["e2e"]["value"])
PY
