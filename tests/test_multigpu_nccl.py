"""Multi-GPU slab decomposition over NCCL (BJ configs[4]): one
process per GPU, grouped ncclSend/ncclRecv halos and ncclAllReduce(max) of the
SOR residual words.  Every reduction on the field path is a max, so the fields,
iteration counts and residuals must be bit-identical for any slab count, and
equal to the oracle.  Skipped unless the box has >= 2 GPUs (the driver's GPU
tier has one); the same decomposition runs on one GPU through the loopback
transport (tests/test_gpu_wavefront.py, tests/test_gpu_parity.py).

Cases: cfg1 (BJ configs[0]) at P = 2, 4, 8 (up to the device count) against the
oracle, with the fused pass's halo rows stored by the kernel into the neighbours'
CUDA-IPC-mapped buffers (IBM_PEER_HALO=1) and through NCCL send/recv
(IBM_PEER_HALO=0), and the 16384^2 mesh (BJ configs[4]) with capped SOR solves at P = 2,
4, 8 against P = 1 -- on the fields' checksums and a sampled row set."""
import os
import socket

import numpy as np
import pytest

import ibm_inputs as I

pytestmark = pytest.mark.gpu


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, q, peer="1"):
    import torch
    import torch.distributed as dist

    import paper_2402_17337_b200 as P
    from paper_2402_17337_b200.dist import bootstrap_nccl_id, slab_of

    os.environ["IBM_PEER_HALO"] = peer  # device-initiated halo (CUDA-IPC peer stores) or NCCL send/recv
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        nid = bootstrap_nccl_id(rank)
        cfg, steps, names = _case(case)
        u0, v0, p0 = I.initial_fields(cfg.nx, cfg.ny, cfg.perturb)
        g = P.Solver(cfg.xn, cfg.yn, device=rank, rank=rank, nranks=world, nccl_id=nid, **cfg.solver_kwargs())
        g.set_body(*cfg.body_args())
        g.set_fields(*slab_of(u0, v0, p0, cfg.ny, world, rank))
        st, stats = g.step(steps)
        out = {n: g.get(n) for n in names}
        out["peer_halo"] = g.query("peer_halo")
        rows = g.rows
        g.close()
        q.put((rank, st, stats, rows, out))
    finally:
        dist.destroy_process_group()


def _case(case):
    if case == "cfg1":
        return I.cfg1(), 10, ("u", "v", "p", "phi", "fu", "fv", "q")
    cfg = I.cfg5(maxit_p=60, maxit_uv=20)
    return cfg, 1, ("u", "v", "p")


def _run(world, case, peer="1"):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q, peer)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=1800) for _ in range(world)], key=lambda r: r[0])
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    stats = res[0][2]
    peers = {r[4].pop("peer_halo") for r in res}
    assert peers == {int(peer)}, peers  # every rank on the same halo path (IPC mapping agreed)
    for r in res[1:]:
        assert r[1] == res[0][1]
        assert np.array_equal(r[2], stats)  # same iteration counts, residuals, forces on every rank
    fields = {n: np.concatenate([r[4][n] for r in res]) for n in res[0][4]}
    return res[0][1], stats, fields


@pytest.mark.parametrize("peer", ["1", "0"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_nccl_slabs_cfg1_equal_oracle(oracle_mod, world, peer):
    if _ngpu() < world:
        pytest.skip("needs %d GPUs" % world)
    cfg, steps, names = _case("cfg1")
    st, stats, fields = _run(world, "cfg1", peer)
    u0, v0, p0 = I.initial_fields(cfg.nx, cfg.ny, cfg.perturb)
    o = oracle_mod.Oracle(cfg.xn, cfg.yn, **cfg.solver_kwargs())
    o.set_body(*cfg.body_args())
    o.set_fields(u0, v0, p0)
    so, sto = o.step(steps)
    assert st == so
    assert np.array_equal(stats[:, 1:5], sto[:, 1:5])
    for n in names:
        assert np.array_equal(fields[n], o.get(n)), n


@pytest.mark.parametrize("world", [2, 4, 8])
def test_nccl_slabs_16384_equal_one_gpu(world):
    if _ngpu() < world:
        pytest.skip("needs %d GPUs" % world)
    import paper_2402_17337_b200 as P
    cfg, steps, names = _case("16384")
    st, stats, fields = _run(world, "16384")
    g = P.Solver(cfg.xn, cfg.yn, device=0, **cfg.solver_kwargs())
    g.set_body(*cfg.body_args())
    g.set_fields(*I.initial_fields(cfg.nx, cfg.ny, cfg.perturb))
    s1, st1 = g.step(steps)
    assert s1 == st
    assert np.array_equal(st1[:, 1:5], stats[:, 1:5])
    for n in names:
        assert np.array_equal(g.get(n), fields[n]), n
    g.close()
