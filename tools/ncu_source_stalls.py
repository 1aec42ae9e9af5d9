"""Per-opcode stall breakdown and main-loop share from an ncu report's source page."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
iSrc = hdr.index("Source")
tot = sum(int(r[iS]) for r in data)
print("stall samples", tot, "instructions", sum(int(r[iE]) for r in data))
byop, exe = Counter(), Counter()
for r in data:
    toks = r[iSrc].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    byop[op] += int(r[iS])
    exe[op] += int(r[iE])
for op, s in byop.most_common(14):
    print(f"  {op:10s} stall {100 * s / tot:5.1f}%  exec {exe[op]}")
idx = [i for i, r in enumerate(data) if "LDS.128" in r[iSrc]]
if idx:
    lo, hi = idx[0], idx[-1]
    loop = sum(int(r[iS]) for r in data[lo - 10:hi + 40])
    print(f"main gather loop (LDS.128 span {lo}-{hi}, {len(idx)} LDS.128): {100 * loop / tot:.1f}% of samples")

if len(sys.argv) > 2:
    top = int(sys.argv[2])
    iA = hdr.index("Address")
    ranked = sorted(range(len(data)), key=lambda i: -int(data[i][iS]))[:top]
    for i in sorted(ranked):
        r = data[i]
        print(f"  [{i:5d}] {int(r[iS]):6d} {100*int(r[iS])/tot:5.1f}%  exec={r[iE]:>10s}  {r[iSrc][:90]}")
