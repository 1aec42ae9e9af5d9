"""Markdown table of profiles/r01_configs.jsonl (tools/measure_configs.py output) for DESIGN.md."""
import json
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "profiles/r02_configs.jsonl"
print("| config | rows | t_roof | auto | auto frac | K1j | K1j frac | K1r | K1r frac | K1 | K1 frac | K1t | dense 3xTF32 | dense 3xFP16 | dense 1xTF32 | hash+keys (auto) | K1r packing |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for line in open(path):
    d = json.loads(line)
    def ms(k):
        v = d.get(k, {})
        return f"{v['ms']:.3g} ms" if "ms" in v else "—"
    def fr(k):
        v = d.get(k, {})
        return f"{v['roofline_frac']:.3f}" if "ms" in v else "—"
    name = f"{d['config']} m={d['m']}" if d["config"] == "C2" else d["config"]
    rp = d.get("row_packing") or {}
    pk = f"P={rp.get('parts')} MS={rp.get('slots')} W={rp.get('warps')} HB={rp.get('hash_blocks')}" if rp else "—"
    au = d.get("auto", {})
    auto = f"{au['kernel']} {au['ms']:.3g} ms" if "ms" in au else "—"
    print(f"| {name} | {d['rows']:.3g} | {d['t_roof_ms']:.3g} ms ({d['bound']}) | {auto} | {fr('auto')} | {ms('K1j')} | {fr('K1j')} | {ms('K1r')} | "
          f"{fr('K1r')} | {ms('K1')} | {fr('K1')} | {ms('K1t')} | {ms('dense_tf32x3')} | {ms('dense_fp16x3')} | {ms('dense_tf32x1')} | "
          f"{ms('hash_keys_auto')} | {pk} |")
