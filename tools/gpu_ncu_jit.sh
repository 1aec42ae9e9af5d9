# ncu --set full of K1j on a C3 chunk (codes + keys, and keys only)
mkdir -p gpurun_out
timeout 300 python tools/prof_jit.py --mode keys > /dev/null 2>&1 || echo "plain run failed"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k1j" -s 1 -c 1 -o gpurun_out/k1j_c3_keys -f python tools/prof_jit.py --mode keys > gpurun_out/ncu_k1j.log 2>&1; echo keys=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k1j" -s 1 -c 1 -o gpurun_out/k1j_c3_keysonly -f python tools/prof_jit.py --mode keysonly >> gpurun_out/ncu_k1j.log 2>&1; echo keysonly=$?
