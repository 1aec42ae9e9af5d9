# C2's m sweep through bench.py (auto kernel: K1r for m = 32 / 128, the dense path for 512 / 4096)
mkdir -p gpurun_out
for m in 32 128 512 4096; do
  timeout 900 python bench.py --config C2 --sample-dims $m --steps 5 --no-tables > gpurun_out/r2g_bench_c2_m$m.json 2> gpurun_out/r2g_bench_c2_m$m.err
  echo "m=$m rc=$?"; python - <<PY
import json
d=json.loads(open("gpurun_out/r2g_bench_c2_m$m.json").read().strip().splitlines()[-1])
r=d["roofline"]
print(d["value"], d["ms_per_step"], r["kernel"][:40], r["bound"], round(r["frac"],3), round(r.get("north_star_frac",0),3), d.get("parity",{}).get("out_of_band_mismatches"))
PY
done
