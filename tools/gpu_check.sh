#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, compute-sanitizer on the multi-tile case.
#   gpurun --timeout 3000 -- 'bash tools/gpu_check.sh [pytest -k expr]'
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
K=${1:-}
(lscpu; echo nproc=$(nproc); nvidia-smi -L) > gpurun_out/host.txt 2>&1
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -rf -k "$K" > gpurun_out/pytest.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest.log 2>&1
fi
echo "pytest_rc=$?" >> gpurun_out/pytest.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench_rc=$?" >> gpurun_out/bench.log
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py > gpurun_out/$tool.log 2>&1
  echo "${tool}_rc=$?" >> gpurun_out/$tool.log
done
