# ncu --set full of K1r with keys from its code tile (hash_keys): C1 (1 hash block, 262,144 rows) and C4 (4 blocks, 100,000 rows)
mkdir -p gpurun_out
timeout 120 python tools/prof_gather.py --config C1 --rows 262144 --iters 2 --fused-keys > /dev/null 2>&1; echo plain_c1=$?
timeout 120 python tools/prof_gather.py --config C4 --rows 100000 --iters 2 --fused-keys > /dev/null 2>&1; echo plain_c4=$?
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:rows_kernel" -s 1 -c 1 -o gpurun_out/r2q_rows_keys_c1 -f python tools/prof_gather.py --config C1 --rows 262144 --iters 2 --fused-keys > gpurun_out/r2q_ncu_c1.log 2>&1; echo c1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:rows_kernel" -s 1 -c 1 -o gpurun_out/r2q_rows_keys_c4 -f python tools/prof_gather.py --config C4 --rows 100000 --iters 2 --fused-keys > gpurun_out/r2q_ncu_c4.log 2>&1; echo c4=$?
