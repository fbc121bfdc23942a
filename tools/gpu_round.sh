#!/bin/bash
# One GPU verification round: tests, bench (both arms), ncu launch list + full captures.
set -u
mkdir -p gpurun_out
python paper_2202_13821_b200/build.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
make -s -C oracle oracle > /dev/null 2>&1
echo "== pytest -m gpu"; timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
echo "== bench"; timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
echo "== bench ref"; timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -c 1500 gpurun_out/bench_ref.json
if [ "${NCU:-1}" = "1" ]; then
  CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
  echo "== ncu launches"
  $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "rc=$?"
  echo "== ncu full face"
  $CMD > gpurun_out/plain2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:face_kernel -s 6 -c 1 -o gpurun_out/prof_face -f $CMD > gpurun_out/ncu_face.log 2>&1; echo "rc=$?"
  echo "== ncu full cell"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:cell_kernel -s 2 -c 1 -o gpurun_out/prof_cell -f $CMD > gpurun_out/ncu_cell.log 2>&1; echo "rc=$?"
  echo "== ncu full cell (stage 2)"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:cell_kernel -s 3 -c 1 -o gpurun_out/prof_cell2 -f $CMD > gpurun_out/ncu_cell2.log 2>&1; echo "rc=$?"
fi
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/host.txt
