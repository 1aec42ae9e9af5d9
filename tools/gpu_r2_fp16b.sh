# K4 3xFP16: ring depth sweep (FASTLSH_K4_H16_STAGES = 3 / 4 / 5) on C1 / C3 chunk / C2 (r2u_)
for st in 3 4 5; do echo "stages=$st"; FASTLSH_K4_H16_STAGES=$st timeout 600 python tools/mb_fp16.py 2>&1 | tail -3; done
FASTLSH_K4_H16_STAGES=5 timeout 600 python -m pytest tests/test_gpu_e2lsh.py -q -x 2>&1 | tail -1
