"""Aggregate ncu source-page warp-stall samples per CUDA source line.
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None; hdr = None; res = []
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr and cur and len(r) == len(hdr) and r[2] == "-" and r[0]:
        try:
            s = int(r[4]); inst = int(r[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        res.append((s, inst, cur, int(r[0]), r[1].strip()[:95]))
tot = sum(x[0] for x in res)
res.sort(reverse=True)
print(f"total samples {tot}")
for s, inst, f, ln, src in res[:top]:
    print(f"{100*s/tot:5.1f}% inst={inst:>11d} {f}:{ln:<5d} {src}")
pf = defaultdict(int)
for s, _, f, _, _ in res: pf[f] += s
print({k: f"{100*v/tot:.1f}%" for k, v in pf.items()})
