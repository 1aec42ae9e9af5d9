# instruction-stream probe (tools/gen_istream.py): 8 distinct per-warp streams vs one shared stream
mkdir -p gpurun_out
for b in tools/mb_istream32 tools/mb_istream128; do
  [ -x $b ] && { echo "== $b"; timeout 300 $b; }
done > gpurun_out/istream.txt 2>&1
cat gpurun_out/istream.txt
