"""Multi-process z-slab path end to end: torchrun with 2 and 3 ranks, halos
and dt min-allreduce over torch.distributed (gloo, host-staged, so every rank
can share the single GPU of a test box without device-side waits). The
gathered slabs must equal the single-solver run bit for bit."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,case,n", [(2, "tgv", 12), (3, "adv3d", 9)])
def test_torchrun_slabs_bitwise(hgks, world, case, n):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tools", "dist_check.py"), "--case", case, "--mesh", str(n), "--device", "0",
           "--backend", "gloo"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("{")][-1]
    res = json.loads(line)
    assert res["world"] == world
    assert res["dts_equal"]
    assert res["bitwise"], res


def test_bench_multirank_gloo(hgks):
    """bench.py's N>1 path (partition, attach, barriers, max-over-ranks timing,
    JSON) under torchrun with 2 ranks on one GPU via the gloo test mode."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "1", "--mesh", "32",
           "--dist-backend", "gloo", "--no-cpu-baseline"]
    env = dict(os.environ, HGKS_BENCH_DEVICE="0")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("{")][-1]
    res = json.loads(line)
    assert res["n_gpus"] == 2 and res["value"] > 0 and res["e2e"]["value"] > 0
    assert res["config"]["parallelism"] == "z-slab x2"
