"""Summarise ncu captures into profiles/ (run here, on the CPU box, after gpurun).

    python tools/ncu_summary.py <full.ncu-rep> <launches.csv> <tag>

Writes profiles/<tag>_kernels.md (per-kernel metrics of the --set full capture,
incl. DRAM bytes per launch), profiles/<tag>_launches.csv (the cold-cache launch
list) and updates profiles/traffic.json (DRAM bytes per launch, read by bench.py).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("launch__shared_mem_per_block_dynamic", "dynamic SMEM/CTA"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "SMEM bank conflicts"),
]
KEYS = {"swr_tc_kernel<0>": "swr_fwd", "swr_tc_kernel<1>": "swr_bwd",
        "swr_tc_kernel<2>": "mix_fwd", "swr_tc_kernel<3>": "mix_bwd",
        "swr_tc_kernel<4>": "layer_fwd", "swr_tc_kernel<5>": "layer_bwd", "swr_tc_kernel<8>": "layer_bwd"}


def to_bytes(val, unit):
    v = float(val)
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main(rep, launches, tag, config="layer4k_bf16", mode="L2 flushed before the kernel (ncu default)"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary ({tag})", "",
             f"Source: `{os.path.basename(rep)}` (one launch per kernel, `--clock-control none`, "
             f"config {config}; caches: {mode}).", ""]
    traffic_path = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        key = next((v for k, v in KEYS.items() if k in name), name)
        lines += [f"## {key}  (`{name}`)", "", "| metric | value |", "|---|---|"]
        for m, label in METRICS:
            if m in h:
                i = h.index(m)
                lines.append(f"| {label} (`{m}`) | {r[i]} {units[i]} |")
        rd = to_bytes(r[h.index("dram__bytes_read.sum")], units[h.index("dram__bytes_read.sum")])
        wr = to_bytes(r[h.index("dram__bytes_write.sum")], units[h.index("dram__bytes_write.sum")])
        lines += ["", f"DRAM traffic per launch: {rd + wr:.4g} B (read {rd:.4g} + write {wr:.4g}).", ""]
        if key in KEYS.values():
            op, dirn = key.split("_")
            traffic[f"{op}_{dirn}_{config}"] = {"bytes": rd + wr,
                                                "source": f"ncu --set full, profiles/{tag}_kernels.md ({mode})"}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_kernels.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=1)
    if launches == "-":
        print("wrote", f"profiles/{tag}_kernels.md", "profiles/traffic.json")
        return
    # launch list: keep only the CSV rows
    with open(launches) as f:
        body = [l for l in f if not l.startswith("==")]
    with open(os.path.join(ROOT, "profiles", f"{tag}_launches.csv"), "w") as f:
        f.writelines(body)
    print("wrote", f"profiles/{tag}_kernels.md", f"profiles/{tag}_launches.csv", "profiles/traffic.json")


if __name__ == "__main__":
    main(*sys.argv[1:])
