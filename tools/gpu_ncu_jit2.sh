# ncu --set full with source of K1j codes+keys and codes-only on a C3 chunk (stall reasons per SASS line)
mkdir -p gpurun_out
timeout 300 python tools/prof_jit.py --mode keys > /dev/null 2>&1 || echo "plain run failed"
for mode in keys codes; do
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k1j" -s 1 -c 1 -o gpurun_out/r2i_k1j_$mode -f python tools/prof_jit.py --mode $mode > gpurun_out/r2i_ncu_k1j_$mode.log 2>&1; echo $mode=$?
done
