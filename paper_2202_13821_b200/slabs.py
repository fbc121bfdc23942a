"""z-slab domain decomposition of the periodic box across ranks.

The reference has no distributed path (MPI is out of scope); its
only parallelism is contiguous index ranges per worker
(runtime.hpp:17-35). Here each rank owns a contiguous range of z layers
(contiguous in the x-fastest cell index, mesh.hpp:34); one layer of cell
coefficients moves to each z neighbour per stage, and each rank computes the
flux of its top boundary face redundantly from identical inputs, so results
are bitwise identical for any rank count. dt is a min-allreduce (order
independent, exact).

Two transports:

* NCCL (the product path on B200s): the library owns the data plane
  (hgks_attach_nccl). Rank 0's NCCL id is broadcast once over
  torch.distributed; after that the halo send/recv pair, the dt and
  error-key min-reductions all run inside libhgks_b200.so on device streams,
  captured in the per-step CUDA graph, with no Python on the step path.
* torch.distributed callbacks (gloo; the CPU tests and the one-GPU
  multi-rank test mode): the solver packs its boundary layers into
  contiguous device buffers (hgks_halo_pack), this module moves them, the
  solver unpacks (hgks_halo_unpack). The exchange is split
  (hgks_set_halo_exchange_split): it is enqueued right after the pack, the
  faces that need no ghost layer run while the layers are in flight, and the
  solver stream waits for the transfer only before the unpack and the two
  boundary z-face layers. dt bits, error keys and report values go through
  the host reduce hook (hgks_set_host_reduce), which every rank joins even
  when its own cells failed.
"""
from __future__ import annotations

from typing import List, Optional, Tuple


def slab_partition(nz: int, world: int) -> List[Tuple[int, int]]:
    """(z_begin, z_count) per rank: contiguous, the first nz % world ranks
    one layer larger (the reference's Partition::make rule, runtime.hpp:21-34)."""
    if world < 1:
        raise ValueError("slab_partition: world must be >= 1")
    if nz < world:
        raise ValueError(f"slab_partition: {nz} z layers cannot feed {world} ranks")
    base, rem = divmod(nz, world)
    out, z = [], 0
    for r in range(world):
        n = base + (1 if r < rem else 0)
        out.append((z, n))
        z += n
    return out


def ring_neighbors(rank: int, world: int) -> Tuple[int, int]:
    """(lower, upper) z neighbours on the periodic ring."""
    return (rank - 1) % world, (rank + 1) % world


def device_view(ptr: int, nbytes: int, device: int):
    """Zero-copy torch view of a device buffer owned by the C library."""
    import torch

    class _CAI:
        __cuda_array_interface__ = {"shape": (nbytes // 8,), "typestr": "<f8", "data": (ptr, False),
                                    "version": 3, "strides": None}

    return torch.as_tensor(_CAI(), device=f"cuda:{device}")


def torch_empty_like_cpu(t):
    import torch
    return torch.empty(t.shape, dtype=t.dtype)


def exchange_halos(send_lo, send_hi, recv_lo, recv_hi, rank: int, world: int, group=None):
    """send_lo -> lower neighbour's recv_hi, send_hi -> upper neighbour's recv_lo.

    Posting order is the same on every rank (down-going pair first), so for
    world == 2 — where lower == upper — point-to-point messages still match
    in order under NCCL (which ignores tags) and gloo (tags 0/1)."""
    import torch.distributed as dist

    if world == 1:
        recv_hi.copy_(send_lo)
        recv_lo.copy_(send_hi)
        return
    if send_lo.is_cuda and dist.get_backend(group) == "gloo":
        # host-staged exchange (gloo moves CPU tensors): the test mode that
        # runs several ranks' solvers on one GPU without device-side waits
        bufs = [t.cpu() for t in (send_lo, send_hi)] + [torch_empty_like_cpu(t) for t in (recv_lo, recv_hi)]
        exchange_halos(bufs[0], bufs[1], bufs[2], bufs[3], rank, world, group)
        recv_lo.copy_(bufs[2])
        recv_hi.copy_(bufs[3])
        return
    lower, upper = ring_neighbors(rank, world)
    ops = [
        dist.P2POp(dist.isend, send_lo, lower, group, 0),
        dist.P2POp(dist.irecv, recv_hi, upper, group, 0),
        dist.P2POp(dist.isend, send_hi, upper, group, 1),
        dist.P2POp(dist.irecv, recv_lo, lower, group, 1),
    ]
    for w in dist.batch_isend_irecv(ops):
        w.wait()


def start_halos(send_lo, send_hi, recv_lo, recv_hi, rank: int, world: int, group=None):
    """Enqueue the exchange (NCCL: behind the current stream, on its own
    stream) and return the pending work; finish_halos() makes the current
    stream wait for it. Same posting order as exchange_halos."""
    import torch.distributed as dist

    if world == 1 or (send_lo.is_cuda and dist.get_backend(group) == "gloo"):
        return None  # nothing to overlap: finish_halos does the whole exchange
    lower, upper = ring_neighbors(rank, world)
    ops = [
        dist.P2POp(dist.isend, send_lo, lower, group, 0),
        dist.P2POp(dist.irecv, recv_hi, upper, group, 0),
        dist.P2POp(dist.isend, send_hi, upper, group, 1),
        dist.P2POp(dist.irecv, recv_lo, lower, group, 1),
    ]
    return dist.batch_isend_irecv(ops)


def finish_halos(pending, send_lo, send_hi, recv_lo, recv_hi, rank: int, world: int, group=None):
    if pending is None:
        exchange_halos(send_lo, send_hi, recv_lo, recv_hi, rank, world, group)
        return
    for w in pending:
        w.wait()


def min_allreduce(value: float, device: Optional[str] = None, group=None) -> float:
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return float(t.item())


def sum_allreduce(values, device: Optional[str] = None, group=None):
    """Fixed-order sum over ranks: gather every rank's partials, add in rank
    order (deterministic, SURVEY §5 'per record')."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    acc = [0.0] * len(values)
    for o in out:
        for i, v in enumerate(o.tolist()):
            acc[i] += v
    return acc


def u64_min_allreduce(values, group=None):
    """In-place min over ranks of a uint64 array (error keys, dt bit patterns):
    the sign bit is flipped so the order survives the int64 all-reduce."""
    import numpy as np
    import torch
    import torch.distributed as dist

    flip = np.uint64(1 << 63)
    t = torch.from_numpy((values ^ flip).view(np.int64).copy())
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    values[:] = t.numpy().view(np.uint64) ^ flip


def host_reduce(op: int, values, group=None):
    """The solver's host reduce hook over torch.distributed (gloo)."""
    if op == 0:
        u64_min_allreduce(values, group=group)
    else:
        values[:] = sum_allreduce(values.tolist(), device="cpu", group=group)


def attach_nccl(solver, rank: int, world: int, group=None):
    """In-library NCCL data plane: rank 0 makes the NCCL id, torch.distributed
    broadcasts it once, every rank attaches (hgks_attach_nccl)."""
    import torch.distributed as dist

    obj = [solver.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    solver.attach_nccl(obj[0], rank, world)


def attach(solver, rank: int, world: int, device: int, group=None, transport: str = "auto"):
    """Wire a slab solver to its neighbours. transport "nccl" (default on an
    NCCL process group): the library's own data plane; "torch": halo exchange
    through torch.distributed callbacks on the solver's stream (which must be
    torch's current stream) and reductions through the host reduce hook."""
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    if transport == "auto":
        transport = "nccl" if backend == "nccl" else "torch"
    if transport == "nccl":
        attach_nccl(solver, rank, world, group)
        return None

    nbytes = solver.halo_bytes()
    ptrs = solver.halo_buffers()
    views = [device_view(p, nbytes, device) for p in ptrs]

    def same_stream():
        # the pack kernel runs on the solver's stream; torch's copies / NCCL ops
        # order against torch's current stream. When they are not the same
        # stream, order them explicitly (stream 0 is the legacy default
        # stream, never the solver's).
        ts = torch.cuda.current_stream(device)
        return ts, ts.cuda_stream != 0 and ts.cuda_stream == solver.stream()

    pending = {}

    def start(_s, which):
        ts, same = same_stream()
        if not same:
            solver.synchronize()
        pending[which] = start_halos(views[0], views[1], views[2], views[3], rank, world, group)

    def finish(_s, which):
        ts, same = same_stream()
        finish_halos(pending.pop(which, None), views[0], views[1], views[2], views[3], rank, world, group)
        if not same:
            ts.synchronize()

    # interior faces run while the layers are in flight
    solver.set_halo_exchange_split(start, finish)
    solver.set_host_reduce(lambda op, vals: host_reduce(op, vals, group=group))
    return views
