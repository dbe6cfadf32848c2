"""Stall-reason totals of one kernel, grouped by source-line range (role sections).

    python tools/stall_by_range.py <rep> <kernel substr> name:lo-hi [name:lo-hi ...]
SASS rows are attributed to the CUDA line they follow in the cuda,sass listing."""
import csv, io, subprocess, sys
rep, kname = sys.argv[1], sys.argv[2]
ranges = [(a.split(":")[0], *map(int, a.split(":")[1].split("-"))) for a in sys.argv[3:]]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fn, hdr, line, done = None, None, None, set()
tot = {}
for r in csv.reader(io.StringIO(raw)):
    if len(r) >= 2 and r[0] == "Function Name":
        if fn is not None and kname in fn: done.add(fn)
        fn = r[1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if fn is None or kname not in fn or fn in done or hdr is None or len(r) != len(hdr):
        continue
    if r[0]:
        line = int(r[0]); continue   # CUDA line row (aggregate); use the SASS rows below it
    if not r[2].startswith("0x"):
        continue
    name = next((n for n, lo, hi in ranges if lo <= line <= hi), "other")
    d = tot.setdefault(name, {})
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "(Not Issued)" not in h or h == "Instructions Executed":
            try: d[h] = d.get(h, 0) + float(r[i])
            except ValueError: pass
allst = sum(v for d in tot.values() for k, v in d.items() if k.startswith("stall_"))
for name, d in sorted(tot.items(), key=lambda kv: -sum(v for k, v in kv[1].items() if k.startswith("stall_"))):
    s = sum(v for k, v in d.items() if k.startswith("stall_"))
    top = sorted(((v, k) for k, v in d.items() if k.startswith("stall_")), reverse=True)[:6]
    print(f"{name:10s} inst {d.get('Instructions Executed',0):10.0f} samples {100*s/allst:5.1f}%  " +
          "  ".join(f"{k[6:]} {100*v/s:.0f}%" for v, k in top))
