timeout 1200 python tools/measure_configs.py --out gpurun_out/configs3.jsonl > gpurun_out/configs3.log 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/configs3.jsonl'):
    d=json.loads(l); k1=d.get('K1',{}); k1t=d.get('K1t',{}); d3=d.get('dense_tf32x3',{}); d1=d.get('dense_tf32x1',{})
    print(f"{d['config']} m={d['m']} N={d['rows']}: roof {d['t_roof_ms']:.3f} | K1 {k1.get('ms',float('nan')):.3f}ms frac {k1.get('roofline_frac',float('nan')):.3f} | K1t {k1t.get('ms',float('nan')):.3f} | x3 {d3.get('ms',float('nan')):.3f} x1 {d1.get('ms',float('nan')):.3f} | {d['packing']}")
PY
