"""Time fastlsh_build_keys alone on the C1 / C3 / C4 shapes (random codes resident in HBM).
Usage: python tools/mb_keys.py [path/to/libfastlsh.so] — prints ms and achieved GB/s per shape."""
import sys

import torch

import paper_2309_15479_b200 as fl

if len(sys.argv) > 1:
    fl.load_library(sys.argv[1])
ONLY = __import__("os").environ.get("MB_KEYS_ONLY")
SHAPES = {"C1": (1_000_000, 500, 50, 10), "C3": (8_000_000, 256, 16, 16), "C4": (100_000, 2000, 200, 10)}
for name, (N, k, L, K) in SHAPES.items():
    if ONLY and name != ONLY:
        continue
    codes = torch.randint(-2**31, 2**31 - 1, (N, k), dtype=torch.int32, device="cuda")
    keys = fl.Keys.create(L, K, seed=7)
    out = torch.empty((L, N), dtype=torch.int64, device="cuda")
    for _ in range(3):
        fl.build_keys(keys, codes, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        fl.build_keys(keys, codes, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    gb = (4.0 * N * L * K + 8.0 * L * N) / 1e9
    print(f"{sys.argv[1] if len(sys.argv) > 1 else 'default'} {name}: {ms:.3f} ms  {gb / ms:.2f} TB/s")
