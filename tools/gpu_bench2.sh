# bench: C3 default (strong, 1 GPU), C1, C4 stream (short)
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err; echo c3=$?
timeout 600 python bench.py --config C1 --steps 10 > gpurun_out/b_c1.json 2> gpurun_out/b_c1.err; echo c1=$?
timeout 600 python bench.py --config C4 --stream --batches 50 --steps 3 > gpurun_out/b_c4s.json 2> gpurun_out/b_c4s.err; echo c4s=$?
tail -2 gpurun_out/b_c3.err gpurun_out/b_c1.err gpurun_out/b_c4s.err
python - <<'PY'
import json
for f in ("gpurun_out/b_c3.json", "gpurun_out/b_c1.json", "gpurun_out/b_c4s.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d["roofline"]
        print(f, "ms/step %.3f value %.3e" % (d["ms_per_step"], d["value"]), "frac %.3f %s" % (r["frac"], r["bound"]),
              "e2e %.3e" % d["e2e"]["value"], "parity", d.get("parity"), "overlap", d.get("overlap"))
    except Exception as e:
        print(f, "ERR", e)
PY
