"""Summarise gpurun_out/ ncu artefacts into profiles/<tag>_*.{md,json}.

  python tools/profile_summary.py r01
reads gpurun_out/launches.csv (gpu__time_duration per launch), the
--set full reports gpurun_out/prof_face.ncu-rep / prof_cell.ncu-rep and
gpurun_out/bench.json; writes profiles/<tag>_ncu_summary.md,
profiles/<tag>_launches.csv (per-step DRAM traffic: tools/kernel_traffic.py ->
profiles/kernel_traffic.json, read by bench.py for roofline.traffic / hbm).
"""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return float("nan")


def to_bytes(v, unit):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return num(v) * f


def fp64_per_launch(rep):
    """Executed DFMA / DMUL / DADD thread instructions of the captured launch,
    summed over the source page's SASS rows."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    si, ti = h.index("Source"), h.index("Thread Instructions Executed")
    tot = {"dfma": 0.0, "dmul": 0.0, "dadd": 0.0}
    for r in rows[hi + 1:]:
        if len(r) != len(h):
            continue
        op = r[si].split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        for k in tot:
            if o.startswith(k.upper()):
                tot[k] += num(r[ti])
    return tot


FAMILIES = {"P2_visc": ("tgv", 2, 128), "P1_visc": ("tgv", 1, 128), "P3_visc": ("tgv", 3, 64),
            "P2_inv": ("adv3d", 2, 128), "P1_inv": ("adv3d", 1, 128), "P3_inv": ("adv3d", 3, 64)}


def exec_family(key):
    """Per-unit executed FP64 of one family from tools/exec_capture.sh's CSVs
    (face: one axis pass = cells * NFP points; cell: stage 1 and stage 2)."""
    case, deg, n = FAMILIES[key]
    ncells = n ** 3
    nfp = 9 if deg == 3 else 4
    out = {}
    for part, fname in (("face", f"exec_{key}_face.csv"), ("cell", f"exec_{key}_cell.csv")):
        path = os.path.join(OUT, fname)
        if not os.path.exists(path):
            return None
        rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
        per = defaultdict(dict)
        for r in rows:
            per[int(r[0])][r[12]] = num(r[14])
            per[int(r[0])]["kernel"] = r[4]
        face_rows = []
        for idx in sorted(per):
            m = per[idx]
            units = ncells * nfp if part == "face" else ncells
            e = {op: m.get(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum", 0.0) / units
                 for op in ("dfma", "dmul", "dadd")}
            e["fp64_flops"] = 2 * e["dfma"] + e["dmul"] + e["dadd"]
            e["kernel"] = m["kernel"][:60]
            if part == "face":
                face_rows.append(e)
            else:
                out["cell_stage" if ", 1>" in m["kernel"] else "cell_stage2"] = e
        if face_rows:
            # six launches = one step: stage 1 (x, y, z), stage 2 (Ft only); a
            # single launch (older captures) is stage 1
            def avg(rows):
                r = {k: sum(x[k] for x in rows) / len(rows) for k in ("dfma", "dmul", "dadd", "fp64_flops")}
                r["kernel"] = rows[0]["kernel"]
                return r
            out["face_point"] = avg(face_rows[:3])
            if len(face_rows) >= 6:
                out["face_point_stage2"] = avg(face_rows[3:6])
                out["face_point_mean"] = {k: 0.5 * (out["face_point"][k] + out["face_point_stage2"][k])
                                          for k in ("dfma", "dmul", "dadd", "fp64_flops")}
    if "cell_stage" in out and "cell_stage2" in out:
        out["cell_stage_mean"] = {k: 0.5 * (out["cell_stage"][k] + out["cell_stage2"][k])
                                  for k in ("dfma", "dmul", "dadd", "fp64_flops")}
    return out


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    md = [f"# ncu summary {tag}", ""]
    bench = None
    if os.path.exists(os.path.join(OUT, "bench.json")):
        txt = open(os.path.join(OUT, "bench.json")).read().strip().splitlines()
        bench = json.loads(txt[-1]) if txt else None
    if bench:
        md += [f"bench: value {bench['value']:.4g} {bench['unit']}, {bench['ms_per_step']:.2f} ms/step, "
               f"clocks {bench.get('clocks')}", ""]
    # launch list (cold-cache, serialised: shares only)
    lc = os.path.join(OUT, "launches.csv")
    if os.path.exists(lc):
        rows = list(csv.reader(open(lc)))
        hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        h = rows[hi]
        ki, vi = h.index("Kernel Name"), h.index("Metric Value")
        tot, cnt = defaultdict(float), defaultdict(int)
        for r in rows[hi + 1:]:
            if len(r) > vi:
                nm = r[ki].split("(")[0]
                tot[nm] += num(r[vi])
                cnt[nm] += 1
        # the DFMA-peak calibration and the initial projection run outside
        # the timed steps: listed, but not part of the step's shares
        outside = ("dfma_peak_kernel", "project_kernel")
        T = sum(v for k, v in tot.items() if not any(o in k for o in outside))
        md += ["## launch list (ncu gpu__time_duration, `bench.py --steps 2 --warmup 1`)", "",
               "share = fraction of the step kernels' time (calibration and setup kernels excluded)", "",
               "| kernel | launches | total ms | share of step |", "|---|---|---|---|"]
        for k in sorted(tot, key=lambda k: -tot[k]):
            sh = "outside the step" if any(o in k for o in outside) else f"{100 * tot[k] / T:.1f}%"
            md.append(f"| `{k}` | {cnt[k]} | {tot[k] / 1e6:.3f} | {sh} |")
        md.append("")
        shutil.copy(lc, os.path.join(PROF, f"{tag}_launches.csv"))
    traffic = {}
    for name in ("face", "cell"):
        rep = os.path.join(OUT, f"prof_{name}.ncu-rep")
        if not os.path.exists(rep):
            continue
        v, u = raw(rep)
        rd = to_bytes(v.get("dram__bytes_read.sum"), u.get("dram__bytes_read.sum"))
        wr = to_bytes(v.get("dram__bytes_write.sum"), u.get("dram__bytes_write.sum"))
        fp = sum(num(v.get(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed", 0))
                 for op in ("dfma", "dmul", "dadd"))
        dur_ms = num(v.get("gpu__time_duration.sum")) * (1e-3 if u.get("gpu__time_duration.sum") == "usecond" else 1.0)
        clk = num(v.get("sm__cycles_elapsed.avg.per_second")) * 1e9
        md += [f"## {name}: `{v.get('Kernel Name', '')[:110]}`", "",
               f"- duration {dur_ms:.3f} ms, SM clock {clk / 1e9:.3f} GHz, grid {v.get('launch__grid_size')} x "
               f"{v.get('launch__block_size')}, {v.get('launch__registers_per_thread')} regs/thread",
               f"- FP64 pipe active {num(v.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active')):.1f}% "
               f"(fp64 thread-inst/cycle over all SMs {fp:.0f} of {64 * 148})",
               f"- issue active {num(v.get('smsp__issue_active.avg.pct_of_peak_sustained_active')):.1f}%, warps active "
               f"{num(v.get('sm__warps_active.avg.pct_of_peak_sustained_active')):.1f}% of 64",
               f"- DRAM read {rd / 1e6:.1f} MB, write {wr / 1e6:.1f} MB per launch "
               f"({(rd + wr) / (dur_ms * 1e-3) / 1e9:.0f} GB/s)", ""]
        st = []
        for k, x in v.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                st.append((num(x), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        tot = sum(a for a, _ in st) or 1.0
        md.append("- stall samples: " + ", ".join(f"{n} {100 * a / tot:.0f}%" for a, n in sorted(st, reverse=True)[:8]))
        md.append("")
        traffic[name] = {"dram_bytes_per_launch": rd + wr, "read": rd, "write": wr, "duration_ms": dur_ms,
                         "kernel": v.get("Kernel Name", "")}
    # executed FP64 work per unit (bench.py's roofline basis): face launch = one
    # axis pass over ncells * NFP points; cell launch = one stage over ncells
    if bench and all(os.path.exists(os.path.join(OUT, f"prof_{n}.ncu-rep")) for n in ("face", "cell")):
        ncells = bench["config"]["cells"]
        nfp = {1: 4, 2: 4, 3: 9}[bench["config"]["degree"]]
        ex = {}
        for name, rep, units in (("face_point", "prof_face", ncells * nfp), ("cell_stage", "prof_cell", ncells),
                                 ("cell_stage2", "prof_cell2", ncells)):
            path = os.path.join(OUT, f"{rep}.ncu-rep")
            if not os.path.exists(path):
                continue
            t = fp64_per_launch(path)
            ex[name] = {k: v / units for k, v in t.items()}
            ex[name]["fp64_flops"] = 2 * ex[name]["dfma"] + ex[name]["dmul"] + ex[name]["dadd"]
            ex[name]["kernel"] = raw(path)[0].get("Kernel Name", "")[:60]
        if "cell_stage2" in ex:  # the two S2O4 stages differ (stage 2 computes only Lt)
            ex["cell_stage_mean"] = {k: 0.5 * (ex["cell_stage"][k] + ex["cell_stage2"][k])
                                     for k in ("dfma", "dmul", "dadd", "fp64_flops")}
        ex["source"] = f"ncu --set full source page, {tag}; units: face = cells*NFP points per launch, cell = cells"
        fam = {k: v for k, v in ((k, exec_family(k)) for k in FAMILIES) if v}
        if fam:
            ex["families"] = fam
            ex["families_source"] = ("tools/exec_capture.sh: ncu smsp__sass_thread_inst_executed_op_{dfma,dmul,dadd}"
                                     "_pred_on.sum of one face launch and both cell stages per family")
        json.dump(ex, open(os.path.join(PROF, "executed_fp64_per_unit.json"), "w"), indent=1)
        md += ["## executed FP64 per unit", "",
               f"- face point: {ex['face_point']['dfma']:.0f} DFMA + {ex['face_point']['dmul']:.0f} DMUL + "
               f"{ex['face_point']['dadd']:.0f} DADD = {ex['face_point']['fp64_flops']:.0f} flops "
               f"(reference op count 8,503)",
               f"- cell stage 1: {ex['cell_stage']['dfma']:.0f} DFMA + {ex['cell_stage']['dmul']:.0f} DMUL + "
               f"{ex['cell_stage']['dadd']:.0f} DADD = {ex['cell_stage']['fp64_flops']:.0f} flops"]
        if "cell_stage2" in ex:
            md += [f"- cell stage 2: {ex['cell_stage2']['dfma']:.0f} DFMA + {ex['cell_stage2']['dmul']:.0f} DMUL + "
                   f"{ex['cell_stage2']['dadd']:.0f} DADD = {ex['cell_stage2']['fp64_flops']:.0f} flops"]
        md += [""]
    open(os.path.join(PROF, f"{tag}_ncu_summary.md"), "w").write("\n".join(md) + "\n")
    if bench:
        json.dump(bench, open(os.path.join(PROF, f"{tag}_bench.json"), "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
