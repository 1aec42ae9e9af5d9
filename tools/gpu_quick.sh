timeout 600 python -m pytest tests -m gpu -x -q -k "fused or keys or host_entry" 2>&1 | tail -2 > gpurun_out/qq.log
timeout 900 python bench.py --config C3 --steps 3 --e2e-steps 1 --no-dense --no-cpu-baseline --fused-keys > gpurun_out/c3f.json 2>gpurun_out/c3f.err; echo c3f=$?
tail -2 gpurun_out/c3f.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/c3f.json").read().strip().splitlines()[-1])
print("C3 fused: ms/step %.3f" % d["ms_per_step"], "value %.3e" % d["value"], d["breakdown_ms"], "frac %.3f" % d["roofline"]["frac"], d["gpu_launches"])
PY
cat gpurun_out/qq.log
