"""profiles/r01_configs.md from the gpurun_out/cfg*.json lines of tools/gpu_configs.sh."""
import glob, json, os
lines = ["# bench.py per config (round 1, final kernels; 30 steps, L2 flushed between steps; roofline frac vs the 6650 GB/s fallback copy peak)", "",
         "| workload | op | BxLxHxd | dtype | path | Mtok/s | fwd us | bwd us | fwd+bwd GB/s | roofline frac (bwd) |",
         "|---|---|---|---|---|---|---|---|---|---|"]
def key(f):
    b = os.path.basename(f); return ("ffma" in b, "mix" in b, b)
for f in sorted(glob.glob("gpurun_out/cfg*.json"), key=key):
    d = json.loads(open(f).read().strip().splitlines()[-1]); c = d["config"]
    e = 4 if d["dtype"] in ("f32", "fp32", "float32") else 2
    D = c["d_head"]; n = c["B"] * c["L"] * c["H"]
    per = ((4 * D + 1) + (7 * D + 2)) if c["op"] == "mix" else ((2 * D + 1) + (3 * D + 2))
    t = (d["fwd_ms"] + d["bwd_ms"]) * 1e-3
    lines.append(f"| {c['workload']} | {c['op']} | {c['B']}x{c['L']}x{c['H']}x{D} | {d['dtype']} | {c['last_path']}"
                 f"{' (forced)' if c['path'] == 'ffma' else ''} | {d['value'] / 1e6:.1f} | {d['fwd_ms'] * 1e3:.1f} | "
                 f"{d['bwd_ms'] * 1e3:.1f} | {n * per * e / t / 1e9:.0f} | {d['roofline']['frac']:.3f} |")
lines += ["", "Run-to-run / box-to-box spread of the layer4k SWR line over this round's final runs: 259-271 Mtok/s (backward inside the step 75-80 us).",
          "The `(forced)` rows run the CUDA-core family on the graded bf16 shape (`--path ffma`): the tensor-core path is 1.5-1.6x (SWR) / 1.8-1.9x (mixer) faster there."]
open("profiles/r01_configs.md", "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
