"""K1r: measured time per forced part count P (FASTLSH_ROW_PARTS) vs the packer's choice — run one P per
process (the packing is built once per params object): python tools/sweep_parts.py CONFIG M ROWS"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2309_15479_b200 as fl
from fastlsh_inputs import configs, data
name, m, rows = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
c = configs.get(name)
m = m or c.m
P = fl.Params.create(c.n, m, c.k, c.w, seed=1).set_kernel("rows")
rp = P.row_packing()
X = data.generate(c.data, c.n, 0, rows, seed=1, device="cuda")
out = torch.empty((rows, c.k), dtype=torch.int32, device="cuda")
fl.fastlsh_hash(P, X, out=out); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): fl.fastlsh_hash(P, X, out=out)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
frac = rows * c.k * m / (ms / 1e3) / (148 * 32 * 1.965e9)
print(f"{name} m={m} P_env={os.environ.get('FASTLSH_ROW_PARTS', 'auto')}: P={rp['parts']} MS={rp['slots']} W={rp['warps']} "
      f"HB={rp['hash_blocks']} conflicts={rp['conflicts']} S={rp['S']} -> {ms:.3f} ms, {frac:.3f} of G_s")
