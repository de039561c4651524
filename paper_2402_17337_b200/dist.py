"""Multi-process plumbing for the slab-decomposed path.

One process per GPU.  torch.distributed is used only to broadcast the NCCL
unique id (the library builds its own NCCL communicator for the halo
exchanges and residual all-reduce) and to take the max of the per-rank timings.
The slab partition mirrors the library's (api.cu slab_rows): ny rows split into
near-equal contiguous ranges; every family uses the p-row range of its rank
and the last rank also owns v row ny.
"""
from __future__ import annotations


def slab_rows(ny: int, nranks: int, rank: int):
    """Global p-row range [j0, j1) of `rank` (same formula as the C library)."""
    if nranks < 1 or not 0 <= rank < nranks:
        raise ValueError("bad rank/nranks")
    base, rem = divmod(ny, nranks)
    j0 = rank * base + min(rank, rem)
    return j0, j0 + base + (1 if rank < rem else 0)


def slab_of(u, v, p, ny: int, nranks: int, rank: int):
    """This rank's rows of global u [ny][nx+1], v [ny+1][nx], p [ny][nx]."""
    j0, j1 = slab_rows(ny, nranks, rank)
    last = j1 == ny
    return u[j0:j1], v[j0:j1 + (1 if last else 0)], p[j0:j1]


def bootstrap_nccl_id(rank: int, id_fn=None, src: int = 0):
    """Rank `src` creates the 128-byte NCCL unique id (ibm_nccl_unique_id) and
    every rank receives it over the default torch.distributed group."""
    import torch.distributed as dist

    if id_fn is None:
        from .ibm import ibm_nccl_unique_id as id_fn
    obj = [id_fn() if rank == src else None]
    dist.broadcast_object_list(obj, src=src)
    nid = obj[0]
    if not isinstance(nid, (bytes, bytearray)) or len(nid) != 128:
        raise RuntimeError("bad NCCL unique id")
    return bytes(nid)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. elapsed ms) over the default group."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
