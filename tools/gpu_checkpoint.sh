timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/ck_pytest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/ck_smoke.log 2>&1; echo smoke=$? >> gpurun_out/ck_smoke.log
timeout 900 python bench.py > gpurun_out/ck_bench.json 2> gpurun_out/ck_bench.err; echo bench=$?
cat gpurun_out/ck_pytest.log gpurun_out/ck_smoke.log
python - <<'PY'
import json
d = json.loads(open("gpurun_out/ck_bench.json").read().strip().splitlines()[-1])
print("ms/step %.3f" % d["ms_per_step"], "value %.3e" % d["value"], d["breakdown_ms"], "frac %.3f" % d["roofline"]["frac"], "e2e %.3e" % d["e2e"]["value"], "tables", d["tables"]["ms"], d["clocks"])
PY
