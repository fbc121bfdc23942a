"""Key metrics of an ncu --set full report (first kernel)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
def g(n):
    try: return v[h.index(n)]
    except ValueError: return "-"
keys = ["Kernel Name", "gpu__time_duration.sum", "launch__registers_per_thread", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_shared_st.sum",
        "smsp__inst_executed.sum", "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum", "sm__cycles_elapsed.avg.per_second"]
for k in keys: print(f"  {k:65s} {g(k)}")
fp = 0.0
for op in ("dfma", "dmul", "dadd"):
    n = f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed"
    try: fp += float(g(n))
    except ValueError: pass
print(f"  fp64 thread-inst per cycle (all SMs)                              {fp:.1f}")
st = []
for i, n in enumerate(h):
    if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
        try: st.append((float(v[i]), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError: pass
tot = sum(x for x, _ in st)
print("  stalls: " + ", ".join(f"{n} {100*x/tot:.0f}%" for x, n in sorted(st, reverse=True)[:8]))
