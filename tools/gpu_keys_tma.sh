timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "keys or host" 2>&1 | tail -1
for env in "" "FASTLSH_KEYS_NO_TMA=1"; do env $env timeout 300 python tools/mb_fused_keys.py | sed "s/^/[$env] /"; done
