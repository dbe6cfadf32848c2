"""profiles/r02_configs.md from the gpurun_out/cfg_*.json lines of tools/gpu_configs.sh."""
import glob
import json
import os

import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import algo_bytes  # noqa: E402

lines = ["# bench.py per config and op (round 2; 20 steps back to back -- no L2 flush -- when the inputs exceed 2x the L2, "
         "else flushed; roofline frac of the dominant kernel vs the measured 6550 GB/s copy peak)", "",
         "| workload | op | BxLxHxd | dtype | path | Mtok/s | fwd us | bwd us | fwd+bwd GB/s | frac of copy peak | roofline frac (dominant) | timing |",
         "|---|---|---|---|---|---|---|---|---|---|---|---|"]
order = ["layer4k", "L8k", "L16k", "L32k", "L4k_b16", "bxh", "paper_d16", "layer4k_f32", "tiny"]
rows = []
for f in glob.glob("gpurun_out/cfg_*.json"):
    txt = open(f).read().strip()
    if not txt:
        continue
    d = json.loads(txt.splitlines()[-1])
    c = d["config"]
    rows.append((order.index(c["workload"]) if c["workload"] in order else 99, c["op"], c["path"], d))
for _, op, path, d in sorted(rows, key=lambda r: (r[0], r[2] != "auto", ["swr", "mix", "layer"].index(r[1]))):
    c = d["config"]
    by = algo_bytes(op, c["B_per_rank"], c["L"], c["H"], c["d_head"], d["dtype"])
    t = d["ms_per_step"] * 1e-3
    gbs = (by["fwd"] + by["bwd"]) / t / 1e9
    lines.append(f"| {c['workload']} | {op}{' (G=8)' if op == 'layer' else ''} | {c['B']}x{c['L']}x{c['H']}x{c['d_head']} | {d['dtype']} | "
                 f"{c['last_path']}{' (forced)' if path == 'ffma' else ''} | {d['value'] / 1e6:.1f} | {d['fwd_ms'] * 1e3:.1f} | "
                 f"{d['bwd_ms'] * 1e3:.1f} | {gbs:.0f} | {gbs / 6550.4:.2f} | {d['roofline']['frac']:.3f} | "
                 f"{'b2b' if 'back to back' in c['timing'] else 'flushed'} |")
open("profiles/r02_configs.md", "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
