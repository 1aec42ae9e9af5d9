# Functional smoke test of bench.py's N > 1 orchestration on ONE GPU: 2 (and 3) ranks share cuda:0 and
# use gloo (host-staged collectives), so no rank's kernel waits on another's. Checks that every
# exchange mode runs to completion and prints its JSON line; the timings are not bench numbers.
mkdir -p gpurun_out
export FASTLSH_BENCH_BACKEND=gloo FASTLSH_BENCH_SHARE_GPU=1
run() {  # name nproc args...
  local name=$1 np=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $np --steps 2 --warmup 3 --no-cpu-baseline --no-dense \
    --no-tables --e2e-steps 1 "$@" > gpurun_out/mr_$name.json 2> gpurun_out/mr_$name.err
  echo "$name rc=$? $(tail -c 300 gpurun_out/mr_$name.json | tr -d '\n' | cut -c1-200)"
}
run c3_auto 2 --config C3 --rows 40000001 --chunk-rows 4194304
run c3_allgather 2 --config C3 --rows 40000000 --chunk-rows 4194304 --exchange allgather
run c3_a2a_serial 2 --config C3 --rows 40000000 --chunk-rows 4194304 --exchange alltoall --no-overlap
run c3_world3 3 --config C3 --rows 30000001 --chunk-rows 4194304
run c1 2 --config C1
run c4 2 --config C4
run c2_dense 2 --config C2 --sample-dims 512 --rows 200000
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29911 bench.py --gpus 2 --config C4 --stream --batches 20 --steps 2 --warmup 3 \
  > gpurun_out/mr_c4_stream.json 2> gpurun_out/mr_c4_stream.err
echo "c4_stream rc=$? $(tail -c 300 gpurun_out/mr_c4_stream.json | tr -d '\n' | cut -c1-200)"
for f in gpurun_out/mr_*.json; do python - "$f" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
av = d.get("allgather_variant") or {}
print(sys.argv[1], d.get("key_exchange"), d.get("exchange_check"), {k: av.get(k) for k in ("ms_per_step", "error")})
PY
done
