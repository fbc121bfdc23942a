#!/bin/bash
# One gpurun call that refreshes every measured artefact of the round:
# GPU tests, smoke, the bench line (+ the reference arm), executed-FP64 counts,
# the ncu launch list, --set full captures of the face and cell kernels and of
# one whole step, and the BASELINE config sweep.
#   gpurun --timeout 3600 -- 'bash tools/evidence_run.sh'
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
(lscpu; echo nproc=$(nproc); nvidia-smi -L) > gpurun_out/host.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
bash tools/exec_capture.sh > gpurun_out/exec_capture.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:face_kernel --launch-skip 3 --launch-count 1 -f \
  -o gpurun_out/prof_face python tools/probe.py 128 > gpurun_out/ncu_face.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:cell_kernel --launch-skip 2 --launch-count 1 -f \
  -o gpurun_out/prof_cell python tools/probe.py 128 > gpurun_out/ncu_cell.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:cell_kernel --launch-skip 3 --launch-count 1 -f \
  -o gpurun_out/prof_cell2 python tools/probe.py 128 > gpurun_out/ncu_cell2.log 2>&1
timeout 900 ncu --set full -k regex:"face_kernel|cell_kernel" --launch-skip 8 --launch-count 8 -f \
  -o gpurun_out/step_full python tools/probe.py 128 > gpurun_out/ncu_step.log 2>&1
bash tools/config_sweep.sh > gpurun_out/config_sweep.log 2>&1
