# quick GPU check: fused-keys + tmem parity tests, bench fused vs unfused (no cpu baseline / dense)
timeout 900 python -m pytest tests -m gpu -x -q -k "fused or tmem or host_entry or keys" 2>&1 | tail -5
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-dense --e2e-steps 1 > gpurun_out/q_fused.json 2>gpurun_out/q_fused.err; echo fused=$?
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-dense --e2e-steps 1 --unfused-keys > gpurun_out/q_unfused.json 2>gpurun_out/q_unfused.err; echo unfused=$?
python - <<'PY'
import json
for f in ("gpurun_out/q_fused.json", "gpurun_out/q_unfused.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, "ms/step %.3f" % d["ms_per_step"], "value %.3e" % d["value"], d["breakdown_ms"], "frac %.3f" % d["roofline"]["frac"])
    except Exception as e:
        print(f, "ERR", e, open(f.replace(".json", ".err")).read()[-800:])
PY
