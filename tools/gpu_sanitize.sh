# compute-sanitizer over every kernel family (tools/sanitize_run.py); logs to gpurun_out/r2_sanitize_*.log
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  for fam in K1j K1r K1 K1t K3 K4 K5 K7 probe; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_run.py --only $fam \
      > gpurun_out/r2_sanitize_${tool}_${fam}.log 2>&1
    echo "$tool $fam rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run ok' gpurun_out/r2_sanitize_${tool}_${fam}.log | tr '\n' ' ')"
  done
done
