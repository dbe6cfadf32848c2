"""Executed warp instructions of one kernel, split into SASS address regions at
the first instruction matching each marker (regions follow code order).

    python tools/sass_regions.py <rep> <kernel substr> name:regex|name:0xADDR [...]
(an address marker is relative to the kernel's first instruction)
"""
import csv, io, re, subprocess, sys
rep, kname = sys.argv[1], sys.argv[2]
marks = [(a.split(":", 1)[0], re.compile(a.split(":", 1)[1])) for a in sys.argv[3:]]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
fn, hdr, rows, done = None, None, [], set()
for r in csv.reader(io.StringIO(raw)):
    if len(r) >= 2 and r[0] in ("Function Name", "Kernel Name"):
        if fn is not None and kname in fn: done.add(fn)
        fn = r[1]; continue
    if r and r[0] == "Address":
        hdr = r; continue
    if fn is None or kname not in fn or fn in done or hdr is None or len(r) != len(hdr):
        continue
    try:
        rows.append((int(r[0], 16), r[1].strip(), float(r[hdr.index("Instructions Executed")]),
                     float(r[hdr.index("Warp Stall Sampling (All Samples)")]),
                     {h[6:]: float(r[i]) for i, h in enumerate(hdr)
                      if h.startswith("stall_") and "Not Issued" not in h and r[i] not in ("", "-")}))
    except ValueError:
        pass
rows.sort()
base = rows[0][0]
rows = [(ad - base, s, n, st, sr) for ad, s, n, st, sr in rows]
starts = []
for name, rx in marks:
    if rx.pattern.startswith("0x"):
        starts.append((name, int(rx.pattern, 16))); continue
    a = next((ad for ad, s, _, _, _ in rows if rx.search(s) and all(ad > x for _, x in starts)), None)
    if a is not None:
        starts.append((name, a))
bounds = [("prologue", rows[0][0])] + starts
tot = sum(r[2] for r in rows); tots = sum(r[3] for r in rows)
for i, (name, a) in enumerate(bounds):
    b = bounds[i + 1][1] if i + 1 < len(bounds) else 1 << 62
    sel = [r for r in rows if a <= r[0] < b]
    n = sum(r[2] for r in sel); s = sum(r[3] for r in sel)
    rs = {}
    for r in sel:
        for k, v in r[4].items(): rs[k] = rs.get(k, 0) + v
    rt = sum(rs.values()) or 1
    top = "  ".join(f"{k} {100*v/rt:.0f}%" for k, v in sorted(rs.items(), key=lambda kv: -kv[1])[:6])
    print(f"{name:10s} from {a:#x}: {n:12.0f} inst {100*n/tot:5.1f}%   stall samples {100*s/tots:5.1f}%   {top}")
