"""Time the bucket-table build on C1-sized keys (for ncu launch lists)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2309_15479_b200 as fl
L, N = int(sys.argv[1]) if len(sys.argv) > 1 else 50, int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
g = torch.Generator(device="cuda"); g.manual_seed(1)
keys = torch.randint(0, 2**61 - 1, (L, N), generator=g, device="cuda", dtype=torch.int64)
out = fl.build_tables(keys)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    fl.build_tables(keys, out=out)
e1.record(); torch.cuda.synchronize()
print(f"tables L={L} N={N}: {e0.elapsed_time(e1)/3:.3f} ms")
