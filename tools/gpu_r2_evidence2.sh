# sanitizer pass, parity records, K1r C2 ncu captures
mkdir -p gpurun_out
bash tools/gpu_sanitize.sh > gpurun_out/r2_sanitize_summary.txt 2>&1
rm -f gpurun_out/r2_parity.jsonl
FASTLSH_PARITY_LOG=gpurun_out/r2_parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -k "parity or jit" > gpurun_out/r2_parity_tests.log 2>&1; echo parity_tests=$?
for m in 32 128; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:rows_kernel" -s 1 -c 1 -o gpurun_out/r2_rows_c2_m$m -f \
    python tools/prof_gather.py --config C2 --m $m --rows 131072 --iters 2 --kernel rows > gpurun_out/r2_ncu_c2_m$m.log 2>&1; echo ncu_c2_m$m=$?
done
cat gpurun_out/r2_sanitize_summary.txt
