"""Per-rank step time of the z-slab data plane, measured on ONE GPU.

An 8-GPU run of TGV P2 128^3 gives each rank a 16-layer slab. Here a slab
solver of z_count layers is attached to NCCL with world = 1, so it is its own
z neighbour: every step runs exactly what a rank runs — the boundary-layer
pack, ncclSend/ncclRecv on the comm stream overlapped with the ghost-free
faces, the unpack and the two boundary z-face layers, the uint64 min
all-reduces of the dt bits and error keys, all inside the per-step CUDA graph
of the device loop — except that the halo bytes move through NCCL's local
path instead of NVLink and the all-reduces have one participant.

usage: python tools/nccl_ring_timing.py [n] [steps]   -> one JSON line (the last line
of stdout: NCCL prints its version banner first)
"""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2202_13821_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cfg = P.CaseConfig.named("tgv", n)
opt = P.RunOptions(degree=2)
cfl = P.default_cfl(2)


def timed(s):
    s.advance_records(1e9, cfl, max_steps=5)  # warm-up (graphs built)
    s.synchronize()
    t0 = time.perf_counter()
    done = s.advance_records(1e9, cfl, max_steps=steps)
    s.synchronize()
    assert done == steps
    return (time.perf_counter() - t0) / steps * 1e3


out = {"workload": f"tgv Re=1600 P2 {n}^3, device loop, {steps} steps, wall clock per step"}
full = P.setup_run(cfg, opt).solver
out["single_gpu_ms"] = t1 = timed(full)
full.close()
rows = {}
for world in (2, 4, 8):
    zc = n // world
    s = P.setup_run(cfg, opt, z_begin=0, z_count=zc).solver
    s.attach_nccl(P.Solver.nccl_unique_id(), 0, 1)
    ms = timed(s)
    s.close()
    rows[str(world)] = {"slab_layers": zc, "rank_step_ms": ms,
                        "efficiency_without_wire": t1 / (world * ms)}
out["ranks"] = rows
out["note"] = ("rank_step_ms: one rank's full step with the NCCL data plane (self-ring, world = 1); "
               "efficiency_without_wire = single_gpu_ms / (world * rank_step_ms). Not included: the "
               "NVLink transfer of 2 x 50 x n^2 doubles per stage (overlapped with the ghost-free "
               "faces) and the multi-participant all-reduce latency (2 per step).")
print(json.dumps(out))
