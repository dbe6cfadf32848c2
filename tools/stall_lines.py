"""Top source lines of one kernel by warp-stall samples, with their stall reasons.

    python tools/stall_lines.py <rep> <kernel substr> [top]"""
import csv, io, subprocess, sys
rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
raw2 = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                      capture_output=True, text=True).stdout
fn, f, hdr, seen, rows = None, None, None, set(), []
for r in csv.reader(io.StringIO(raw2)):
    if len(r) >= 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]; continue
    if len(r) >= 2 and r[0] == "Function Name":
        fn = r[1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if fn is None or kname not in fn or hdr is None or len(r) != len(hdr) or not r[0]:
        continue
    key = (f, r[0])
    if key in seen: continue
    seen.add(key)
    rows.append((f, int(r[0]), r[1].strip(), {h: float(r[i]) for i, h in enumerate(hdr)
                                              if (h.startswith("stall_") and "Not Issued" not in h) and r[i] not in ("", "-")},
                 float(r[hdr.index("Instructions Executed")] or 0)))
S = sum(sum(d.values()) for *_, d, _ in rows)
for f, ln, src, d, ie in sorted(rows, key=lambda x: -sum(x[3].values()))[:top]:
    s = sum(d.values())
    t = sorted(((v, k) for k, v in d.items()), reverse=True)[:3]
    print(f"{100*s/S:5.1f}% {f[:14]}:{ln:<4d} " + ",".join(f"{k[6:]} {100*v/max(s,1):.0f}" for v, k in t) + f" | {src[:70]}")
