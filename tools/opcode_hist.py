"""Executed-instruction histogram by SASS opcode of one kernel in an ncu report.

    python tools/opcode_hist.py <rep> <kernel substr> [top]
"""
import csv, io, subprocess, sys
rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
fn, hdr, acc, done = None, None, {}, set()
for r in csv.reader(io.StringIO(raw)):
    if len(r) >= 2 and r[0] in ("Function Name", "Kernel Name"):
        if fn is not None and kname in fn: done.add(fn)
        fn = r[1]; continue
    if r and r[0] == "Address":
        hdr = r; continue
    if fn is None or kname not in fn or fn in done or hdr is None or len(r) != len(hdr):
        continue
    src = r[hdr.index("Source")].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    try:
        acc[op] = acc.get(op, 0) + float(r[hdr.index("Instructions Executed")])
    except ValueError:
        pass
tot = sum(acc.values())
print(f"{kname}: {tot:.0f} warp instructions")
for op, n in sorted(acc.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{op:12s} {n:12.0f} {100*n/tot:5.1f}%")
