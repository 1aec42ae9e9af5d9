for cfg in "C2 32 1000000" "C2 128 1000000" "C2 512 250000" "C4 0 100000" "C1 0 1000000"; do
  for pp in auto 1 2 4 8; do
    if [ $pp = auto ]; then unset FASTLSH_ROW_PARTS; else export FASTLSH_ROW_PARTS=$pp; fi
    timeout 120 python tools/sweep_parts.py $cfg 2>&1 | tail -1
  done
done
