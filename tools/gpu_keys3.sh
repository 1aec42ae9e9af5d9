# K3 occupancy experiment: min blocks per SM 1 (default), 5, 6 — rebuild keys.cu only
for mb in 1 5 6; do
  touch paper_2309_15479_b200/csrc/keys.cu
  FASTLSH_NVCC_EXTRA="-DFASTLSH_KEYS_MINB=$mb" python -c "from paper_2309_15479_b200 import build as b; b.build()" > /dev/null 2>&1
  timeout 120 python tools/prof_gather.py --config C1 --rows 1000000 --iters 2 --keys > /dev/null 2>&1
  FASTLSH_NVCC_EXTRA="-DFASTLSH_KEYS_MINB=$mb" timeout 300 python tools/mb_fused_keys.py 2>&1 | sed "s/^/[minb=$mb] /"
done
