"""Per-source-line executed instructions and stall samples of an ncu report.
usage: python tools/ncu_inst.py report.ncu-rep [top] [units]  (units: divisor for 'per unit' column)"""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
units = float(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = hdr = None
res = []
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr and cur and len(r) == len(hdr) and r[2] == "-" and r[0]:
        try:
            inst = int(r[hdr.index("Instructions Executed")] or 0); s = int(r[4])
        except ValueError:
            continue
        res.append((inst, s, cur, int(r[0]), r[1].strip()[:100]))
ti = sum(x[0] for x in res); ts = sum(x[1] for x in res)
print(f"total warp-inst {ti}" + (f"  per unit {32 * ti / units:.0f}" if units else ""))
res.sort(reverse=True)
for inst, s, f, ln, src in res[:top]:
    pu = f" {32 * inst / units:7.1f}/u" if units else ""
    print(f"{100 * inst / ti:5.1f}% inst {100 * s / max(ts, 1):5.1f}% stall{pu} {f}:{ln:<5d} {src}")
