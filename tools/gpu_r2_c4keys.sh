# K1r keys from the code tile with several hash blocks (C4: 4 blocks of 500 hashes, K = 10): parity, timing, C4 stream bench (r2p_)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_memsafety.py -q -x -k "code_tile or host_entry or fused or guard or race or chunked" > gpurun_out/r2p_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/r2p_tests.log
timeout 300 python tools/mb_fused_keys.py 2>&1 | tail -4
timeout 900 python bench.py --config C4 --stream > gpurun_out/r2p_bench_c4_stream.json 2> gpurun_out/r2p_bench_c4_stream.err; echo c4=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2p_bench_c4_stream.json").read().strip().splitlines()[-1])
r = d["roofline"]
print("C4 stream ms/step %.3f value %.4e frac %.4f launch %.4f e2e %.4e overlap %.3f identical %s launches %s clocks %s" % (
    d["ms_per_step"], d["value"], r["frac"], r["launch_ms"], d["e2e"]["value"], d["overlap"]["frac"],
    d["device_path_equals_hash_host"], d["gpu_launches"], d["clocks"]))
PY
