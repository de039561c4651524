"""World-size-2 tests of the multi-rank host logic on CPU (gloo): NCCL-id
bootstrap, slab partition / slab field slicing, max-over-ranks timing, and the
bench.py rank-0-only reporting.  The NCCL data path itself runs
only on GPUs; its decomposition is covered on one GPU by the loopback tests."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import ibm_inputs as I
from paper_2402_17337_b200.dist import slab_rows, slab_of


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2402_17337_b200.dist import bootstrap_nccl_id, max_over_ranks, slab_of

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fake = bytes(range(128))
        nid = bootstrap_nccl_id(rank, id_fn=lambda: fake)
        t = max_over_ranks(10.0 + rank)
        cfg = I.cfg1()
        u, v, p = I.initial_fields(cfg.nx, cfg.ny, cfg.perturb)
        us, vs, ps = slab_of(u, v, p, cfg.ny, world, rank)
        gathered = [None] * world
        dist.all_gather_object(gathered, (us, vs, ps))
        q.put((rank, nid == fake, t, [g[0].shape for g in gathered],
               np.array_equal(np.concatenate([g[0] for g in gathered]), u),
               np.array_equal(np.concatenate([g[1] for g in gathered]), v),
               np.array_equal(np.concatenate([g[2] for g in gathered]), p)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_bootstrap_and_slabs():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, id_ok, t, shapes, ok_u, ok_v, ok_p in res:
        assert id_ok                 # every rank received rank 0's id
        assert t == 11.0             # max over ranks
        assert ok_u and ok_v and ok_p  # slabs reassemble the global fields
        assert shapes == [(48, 129), (48, 129)]


@pytest.mark.parametrize("ny,P", [(96, 2), (97, 3), (8192, 8), (16384, 8), (130, 4)])
def test_slab_rows_partition(ny, P):
    rows = [slab_rows(ny, P, r) for r in range(P)]
    assert rows[0][0] == 0 and rows[-1][1] == ny
    for (a0, a1), (b0, b1) in zip(rows, rows[1:]):
        assert a1 == b0
    sizes = [b - a for a, b in rows]
    assert max(sizes) - min(sizes) <= 1


def test_slab_rows_match_library():
    """The Python partition equals the C library's (via the per-rank workspace size)."""
    import paper_2402_17337_b200.ibm as M
    M.lib()
    cfg = I.cfg1(ny=98)
    sizes = []
    for r in range(3):
        c = M.make_config(cfg.xn, cfg.yn, rank=r, nranks=3, nccl_id=bytes(128), **cfg.solver_kwargs())
        sizes.append(M.ibm_workspace_size(c))
    j = [slab_rows(98, 3, r) for r in range(3)]
    # ranks with more rows need more workspace; the last rank also owns v row ny
    assert (j[0][1] - j[0][0]) >= (j[2][1] - j[2][0])
    assert sizes[0] >= sizes[1]
