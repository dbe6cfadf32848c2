"""Hottest basic blocks (by executed warp instructions) of a kernel in an ncu report."""
import csv, io, subprocess, sys
rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
ks, cur, hdr = [], None, None
for r in rows:
    if len(r) >= 2 and r[0] == "Kernel Name":
        cur = []; ks.append((r[1], cur)); continue
    if r and r[0] == "Address":
        hdr = r; continue
    if cur is not None and len(r) > 5 and r[0].startswith("0x"):
        cur.append(r)
ie = hdr.index("Instructions Executed")
st_i = hdr.index("Warp Stall Sampling (All Samples)")
for name, L in ks:
    if kname not in name:
        continue
    tot = sum(int(r[ie]) for r in L)
    stall = sum(int(r[st_i]) for r in L)
    print(name[:70], "executed", tot, "stall samples", stall)
    bbs, start = [], 0
    for i in range(1, len(L) + 1):
        if i == len(L) or L[i][ie] != L[start][ie]:
            n = int(L[start][ie])
            s = sum(int(r[st_i]) for r in L[start:i])
            bbs.append((n * (i - start), start, i - start, n, s)); start = i
    bbs.sort(reverse=True)
    for tb, st, sz, n, s in bbs[:top]:
        print(f"{tb:10d} ({100*tb/tot:4.1f}%) stall {s:5d} [{st:5d}+{sz:4d}] x{n:8d}  {L[st][1][:42]} .. {L[st+sz-1][1][:38]}")
    break
