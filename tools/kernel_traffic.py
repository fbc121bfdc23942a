"""profiles/kernel_traffic.json from an ncu --set full capture of one S2O4
step's kernels (3 face launches + 1 cell launch per stage, in launch order):
DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per stage for the
face pass and the cell kernel, plus each launch's FP64-pipe and issue share.

    python tools/kernel_traffic.py gpurun_out/step_full.ncu-rep [profiles/kernel_traffic.json]
"""
import csv
import json
import subprocess
import sys


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return float("nan")


def main():
    rep = sys.argv[1]
    out_path = sys.argv[2] if len(sys.argv) > 2 else "profiles/kernel_traffic.json"
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def get(v, name):
        i = h.index(name)
        return num(v[i]) * scale.get(units[i], 1)

    launches = []
    for v in rows[2:]:
        name = v[h.index("Kernel Name")]
        launches.append({
            "kernel": name,
            "ms": get(v, "gpu__time_duration.sum") / 1e6 if units[h.index("gpu__time_duration.sum")] == "nsecond"
            else num(v[h.index("gpu__time_duration.sum")]),
            "dram_read": get(v, "dram__bytes_read.sum"),
            "dram_write": get(v, "dram__bytes_write.sum"),
            "fp64_pipe_pct": num(v[h.index("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")]),
            "issue_pct": num(v[h.index("smsp__issue_active.avg.pct_of_peak_sustained_active")]),
            "regs": num(v[h.index("launch__registers_per_thread")]),
        })
    res = {"source": rep, "launches": launches, "face": {}, "cell": {}}
    stage = 0
    acc = {"face": [0.0, 0.0], "cell": [0.0, 0.0]}
    for L in launches:
        key = "face" if "face_kernel" in L["kernel"] else "cell" if "cell_kernel" in L["kernel"] else None
        if key is None:
            continue
        acc[key][stage] += L["dram_read"] + L["dram_write"]
        if key == "cell":
            stage = min(stage + 1, 1)
    for key in ("face", "cell"):
        res[key] = {"dram_bytes_stage1": acc[key][0], "dram_bytes_stage2": acc[key][1],
                    "dram_bytes_per_stage": 0.5 * (acc[key][0] + acc[key][1])}
    json.dump(res, open(out_path, "w"), indent=1)
    print(json.dumps({k: res[k] for k in ("face", "cell")}, indent=1))


if __name__ == "__main__":
    main()
