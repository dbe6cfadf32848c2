"""Executed instructions of one SASS opcode (prefix) per CUDA source line.

    python tools/op_by_line.py <rep> <kernel substr> <opcode prefix> [top]
"""
import csv, io, subprocess, sys
rep, kname, opp = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fn, hdr, line, done, acc, txt = None, None, None, set(), {}, {}
for r in csv.reader(io.StringIO(raw)):
    if len(r) >= 2 and r[0] in ("Function Name", "Kernel Name"):
        if fn is not None and kname in fn: done.add(fn)
        fn = r[1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if fn is None or kname not in fn or fn in done or hdr is None or len(r) != len(hdr):
        continue
    if r[0]:
        line = int(r[0]); txt[line] = r[1].strip(); continue
    s = r[3].strip() if len(r) > 3 else ""
    ops = s.split()
    if not ops: continue
    op = ops[1] if ops[0].startswith("@") else ops[0]
    if not op.startswith(opp): continue
    try:
        acc[line] = acc.get(line, 0) + float(r[hdr.index("Instructions Executed")])
    except ValueError:
        pass
tot = sum(acc.values())
print(f"{opp}: {tot:.0f}")
for ln, n in sorted(acc.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100*n/tot:5.1f}% L{ln}: {txt.get(ln, '')[:100]}")
