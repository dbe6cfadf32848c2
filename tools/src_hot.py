"""Per-source-line instruction and stall totals of one kernel in an ncu report.

    python tools/src_hot.py <rep.ncu-rep> <kernel substring, e.g. '(int)1>'> [top]
"""
import csv, io, subprocess, sys
rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
nth = int(sys.argv[4]) if len(sys.argv) > 4 else 0  # which launch of the kernel (0 = first)
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fn, hdr, acc, seen = None, None, {}, set()
count = {}
for r in csv.reader(io.StringIO(raw)):
    if len(r) >= 2 and r[0] == "Function Name":
        count[r[1]] = count.get(r[1], -1) + 1
        fn = r[1] if count[r[1]] == nth else None
        continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if fn is None or kname not in fn or hdr is None or len(r) < 8 or not r[0]:
        continue
    if (fn, r[0]) in seen:   # the report holds several launches: keep the first
        continue
    seen.add((fn, r[0]))
    ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    try:
        acc[int(r[0])] = (float(r[ie]), float(r[st]), r[1].strip())
    except ValueError:
        pass
ti = sum(v[0] for v in acc.values()); ts = sum(v[1] for v in acc.values())
print(f"{kname}: {ti:.0f} warp instructions, {ts:.0f} stall samples")
for ln, (i, s, src) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*i/ti:5.1f}% inst {100*s/ts:5.1f}% stall  L{ln}: {src[:95]}")
