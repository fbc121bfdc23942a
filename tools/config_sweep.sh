#!/bin/bash
# Secondary bench lines for BASELINE.json's other configs (device-resident value
# + roofline only; the headline line is bench.py's default TGV P2 128^3).
set -u
mkdir -p gpurun_out
python paper_2202_13821_b200/build.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
out=gpurun_out/config_sweep.jsonl
: > $out
for args in "--degree 2 --mesh 128" "--degree 2 --mesh 64" "--degree 1 --mesh 256" "--degree 2 --mesh 256" "--degree 3 --mesh 64" "--case adv3d --degree 2 --mesh 128"; do
  echo "== $args"
  timeout 600 python bench.py $args --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cs.json 2> gpurun_out/cs.err
  echo "rc=$?"; tail -3 gpurun_out/cs.err
  python - "$args" >> $out <<'PY'
import json, sys
l = json.loads(open("gpurun_out/cs.json").read().strip().splitlines()[-1])
r = l["roofline"]; ex = r.get("executed") or {}
print(json.dumps({"args": sys.argv[1], "workload": l["config"]["workload"], "value": l["value"],
                  "ms_per_step": l["ms_per_step"], "frac": r["frac"], "kernel": r["kernel"],
                  "face_pipe_frac": ex.get("face_pipe_frac"), "cell_pipe_frac": ex.get("cell_pipe_frac"),
                  "face_frac": ex.get("face_frac"), "cell_frac": ex.get("cell_frac"),
                  "clocks": l["clocks"], "gpu_launches": l["gpu_launches"]}))
PY
  tail -1 $out
done
