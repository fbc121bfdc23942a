"""FP64 instructions (DFMA/DMUL/DADD, thread-level) executed per source line
of an ncu report (source page, cuda+sass view).
usage: python tools/ncu_fp64_lines.py report.ncu-rep units [top]"""
import csv, subprocess, sys
from collections import defaultdict
rep, units = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = hdr = None
src = None
agg = defaultdict(lambda: [0, 0, 0, ""])
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; ti = hdr.index("Thread Instructions Executed"); continue
    if not hdr or len(r) != len(hdr):
        continue
    if r[0]:
        src = (cur, int(r[0])); agg[src][3] = r[1].strip()[:80]; continue
    op = r[3].strip().split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    try:
        n = int(r[ti])
    except ValueError:
        continue
    k = 0 if o.startswith("DFMA") else 1 if o.startswith("DMUL") else 2 if o.startswith("DADD") else None
    if k is not None and src:
        agg[src][k] += n
tot = [sum(v[i] for v in agg.values()) for i in range(3)]
print(f"per unit: DFMA {tot[0]/units:.0f} DMUL {tot[1]/units:.0f} DADD {tot[2]/units:.0f} total {sum(tot)/units:.0f}")
rows = sorted(agg.items(), key=lambda kv: -(kv[1][0] + kv[1][1] + kv[1][2]))
for (f, ln), v in rows[:top]:
    s = sum(v[:3]) / units
    print(f"{s:7.1f}  fma {v[0]/units:6.1f} mul {v[1]/units:6.1f} add {v[2]/units:6.1f}  {f}:{ln} {v[3]}")
