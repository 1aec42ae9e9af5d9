"""C0 (10^4 rows, 7.7 MB of X + codes, L2-resident) timed warm (back-to-back
launches) and cold (a 512 MB write flushes the 126 MB L2 before every launch; only the hashing
launch is inside the events)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2309_15479_b200 as fl  # noqa: E402
from fastlsh_inputs import configs, data  # noqa: E402

c = configs.get("C0")
P = fl.Params.create(c.n, c.m, c.k, c.w, seed=c.seed)
X = data.generate(c.data, c.n, 0, c.N, seed=c.seed, device="cuda")
codes = torch.empty((c.N, c.k), dtype=torch.int32, device="cuda")
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for _ in range(5):
    fl.fastlsh_hash(P, X, out=codes)
torch.cuda.synchronize()
warm, cold = [], []
for _ in range(50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fl.fastlsh_hash(P, X, out=codes)
    e1.record()
    torch.cuda.synchronize()
    warm.append(e0.elapsed_time(e1))
    flush.fill_(1.0)
    e0.record()
    fl.fastlsh_hash(P, X, out=codes)
    e1.record()
    torch.cuda.synchronize()
    cold.append(e0.elapsed_time(e1))
warm.sort()
cold.sort()
print(f"C0 K1r: warm median {1e3 * warm[25]:.1f} us (min {1e3 * warm[0]:.1f}), "
      f"cold median {1e3 * cold[25]:.1f} us (min {1e3 * cold[0]:.1f}); kernel {P.info()['kernel']}")
