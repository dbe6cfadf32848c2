"""Per-source-line shared-memory excess wavefronts (bank conflicts) of one kernel in an
ncu report:  python tools/src_conflicts.py <rep> <kernel substring> [top]"""
import csv, io, subprocess, sys
rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fn, hdr, acc, seen = None, None, {}, set()
for r in csv.reader(io.StringIO(raw)):
    if len(r) >= 2 and r[0] == "Function Name":
        fn = r[1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if fn is None or kname not in fn or hdr is None or len(r) < 8 or not r[0]:
        continue
    if (fn, r[0]) in seen:
        continue
    seen.add((fn, r[0]))
    try:
        ex = float(r[hdr.index("L1 Wavefronts Shared Excessive")])
        wf = float(r[hdr.index("L1 Wavefronts Shared")])
        acc[int(r[0])] = (ex, wf, r[1].strip())
    except (ValueError, IndexError):
        pass
tot = sum(v[0] for v in acc.values())
print(f"{kname}: {tot:.0f} excess shared wavefronts")
for ln, (ex, wf, src) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ex:10.0f} excess / {wf:10.0f}  L{ln}: {src[:100]}")
