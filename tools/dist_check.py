"""Multi-process z-slab check (launched by torchrun; tests/test_gpu_dist.py).

Every rank owns a z-slab solver, wired with slabs.attach (the same code
bench.py uses); halos move over torch.distributed. With --backend gloo all
ranks may share one GPU (host-staged halos, no device-side waits between
ranks). Rank 0 gathers the slabs after K steps and compares them bitwise with
a single-solver run. Prints one JSON line on rank 0.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="tgv")
    ap.add_argument("--mesh", dest="n", type=int, default=12)
    ap.add_argument("--degree", type=int, default=2)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--backend", default="gloo")
    ap.add_argument("--device", type=int, default=-1, help="-1: LOCAL_RANK")
    a = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2202_13821_b200 as P
    from paper_2202_13821_b200 import slabs

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = a.device if a.device >= 0 else int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    if a.backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
    else:
        dist.init_process_group("gloo")
    cfg = P.CaseConfig.named(a.case, a.n)
    cfl = P.default_cfl(a.degree)
    zb, zc = slabs.slab_partition(a.n, world)[rank]
    r = P.setup_run(cfg, P.RunOptions(degree=a.degree, device=dev), z_begin=zb, z_count=zc)
    s = r.solver
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    s.set_stream(stream.cuda_stream)
    slabs.attach(s, rank, world, dev)
    dts = []
    for _ in range(a.steps):
        dt = s.compute_dt(cfl)
        dts.append(dt)
        s.step(dt)
    q = torch.from_numpy(s.get_state()[0])
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([q.numel()], dtype=torch.int64))
    if rank == 0:
        parts = [q] + [torch.empty(int(sz.item()), dtype=torch.float64) for sz in sizes[1:]]
        for src in range(1, world):
            dist.recv(parts[src], src)
        full = torch.cat(parts).numpy()
        ref = P.setup_run(cfg, P.RunOptions(degree=a.degree, device=dev))
        ref_dts = []
        for _ in range(a.steps):
            dt = ref.solver.compute_dt(cfl)
            ref_dts.append(dt)
            ref.solver.step(dt)
        qref = ref.solver.get_state()[0]
        print(json.dumps({"world": world, "bitwise": bool(np.array_equal(full, qref)), "dts": dts, "ref_dts": ref_dts,
                          "dts_equal": dts == ref_dts,
                          "max_abs_diff": float(np.max(np.abs(full - qref))) if full.shape == qref.shape else None}),
              flush=True)
    else:
        dist.send(q, 0)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
