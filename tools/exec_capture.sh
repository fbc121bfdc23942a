#!/bin/bash
# Executed FP64 instruction counts (DFMA / DMUL / DADD, thread level) of the
# face pass and both cell stages for every bench-able (case, degree) family:
# the executed-FP64 roofline basis (tools/profile_summary.py ->
# profiles/executed_fp64_per_unit.json). Metric-only ncu runs (small CSVs).
set -u
mkdir -p gpurun_out
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,gpu__time_duration.sum
for spec in "tgv 2 128 P2_visc" "tgv 1 128 P1_visc" "tgv 3 64 P3_visc" "adv3d 2 128 P2_inv" "adv3d 1 128 P1_inv" "adv3d 3 64 P3_inv"; do
  set -- $spec
  CMD="python bench.py --case $1 --degree $2 --mesh $3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
  echo "== $4"
  $CMD > gpurun_out/plain_$4.log 2>&1 || { echo "plain run failed"; continue; }
  # one step's six face launches: stage 1 (F and Ft) x, y, z, then stage 2 (Ft only)
  timeout 600 ncu --metrics $M --clock-control none -k regex:face_kernel -s 6 -c 6 --csv --log-file gpurun_out/exec_$4_face.csv $CMD > /dev/null 2>&1; echo "face rc=$?"
  timeout 600 ncu --metrics $M --clock-control none -k regex:cell_kernel -s 2 -c 2 --csv --log-file gpurun_out/exec_$4_cell.csv $CMD > /dev/null 2>&1; echo "cell rc=$?"
done
