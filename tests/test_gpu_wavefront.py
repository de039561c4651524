"""GPU parity of the temporally blocked Poisson pass (k_sor_wf):
sor_fuse = m fuses m red-black iterations per HBM pass.  It must give the
oracle's fields bit for bit and the same iteration counts, including solves that
stop inside a fused pass (replayed from the pass's input buffer), segment
boundaries every few rows (IBM_WF_ROWS), ragged strips, stretched rows and the
body (predicated chunks).  sor_batch > 0 keeps small grids off the persistent
cooperative solve so that the fused pass is the one under test."""
import numpy as np
import pytest

import ibm_inputs as I
from test_gpu_parity import assert_parity, mods, run_pair  # noqa: F401

pytestmark = pytest.mark.gpu

FUSE = [2, 3, 4]


@pytest.fixture
def wf_rows(monkeypatch):
    def set_rows(n):
        if n:
            monkeypatch.setenv("IBM_WF_ROWS", str(n))
        else:
            monkeypatch.delenv("IBM_WF_ROWS", raising=False)
    return set_rows


@pytest.mark.parametrize("m", FUSE)
@pytest.mark.parametrize("rows", [0, 6, 14])
def test_cfg1_fused(mods, wf_rows, m, rows):
    """BJ configs[0] (foil, 128 x 96, perturbed start), 4 steps, every segment length."""
    wf_rows(rows)
    cfg = I.cfg1(steps=4, maxit_p=900)
    o, g, ro, rg = run_pair(mods, cfg, cfg.steps, sor_batch=5, sor_fuse=m)
    assert_parity(o, g, ro, rg)
    g.close()


@pytest.mark.parametrize("m", FUSE)
@pytest.mark.parametrize("nx,ny", [(130, 98), (257, 131), (64, 36), (61, 40)])
def test_ragged_fused(mods, wf_rows, m, nx, ny):
    wf_rows(10)
    cfg = I.cfg1(nx=nx, ny=ny, steps=2, maxit_p=500)
    o, g, ro, rg = run_pair(mods, cfg, cfg.steps, sor_batch=7, sor_fuse=m)
    assert_parity(o, g, ro, rg)


@pytest.mark.parametrize("m", FUSE)
def test_stretched_fused(mods, wf_rows, m):
    """Non-uniform rows: chunks fall back to the predicated path."""
    wf_rows(0)
    xn = I.stretched_axis(-3.0, 6.0, -0.8, 1.2, 1.0 / 40, 1.06)
    yn = I.stretched_axis(-2.5, 2.5, -0.45, 0.45, 1.0 / 40, 1.06)
    cfg = I.Config("stretched", xn, yn, Re=500.0, dt=1e-3, body=I.Body(), steps=3, maxit_p=800, perturb=0.01)
    o, g, ro, rg = run_pair(mods, cfg, cfg.steps, sor_batch=9, sor_fuse=m)
    assert_parity(o, g, ro, rg)


@pytest.mark.parametrize("m", FUSE)
def test_cylinder_fused(mods, wf_rows, m):
    wf_rows(8)
    cfg = I.cfg2(nx=96, ny=72, steps=3, maxit_p=400)
    o, g, ro, rg = run_pair(mods, cfg, cfg.steps, sor_batch=4, sor_fuse=m)
    assert_parity(o, g, ro, rg)


@pytest.mark.parametrize("m", FUSE)
def test_check_every_fused(mods, wf_rows, m):
    wf_rows(0)
    cfg = I.cfg1(steps=3, check_every=3, maxit_p=2000)
    o, g, ro, rg = run_pair(mods, cfg, cfg.steps, sor_batch=16, sor_fuse=m)
    assert_parity(o, g, ro, rg)


@pytest.mark.parametrize("m", FUSE)
def test_converged_fused(mods, wf_rows, m):
    """Solves that converge (status 0) at arbitrary iterations."""
    wf_rows(0)
    cfg = I.cfg1(nx=64, ny=48, steps=4, omega_p=1.8, tol_p=1e-8, maxit_p=20000)
    o, g, ro, rg = run_pair(mods, cfg, cfg.steps, sor_batch=32, sor_fuse=m)
    assert ro[0] == 0
    assert_parity(o, g, ro, rg)


@pytest.mark.parametrize("m", FUSE)
@pytest.mark.parametrize("iters", [1, 2, 5, 7, 12])
def test_poisson_iterate_fused_vs_unfused(mods, wf_rows, m, iters):
    """Fixed iteration counts (tolerance off): a fused solve and a one-iteration-
    per-pass solve leave identical phi and residual, whatever iters mod m is."""
    O, P = mods
    wf_rows(12)
    cfg = I.cfg1(steps=1, maxit_p=300)
    out = []
    for fuse in (1, m):
        g = P.Solver(cfg.xn, cfg.yn, sor_batch=3, sor_fuse=fuse, **cfg.solver_kwargs())
        g.set_body(*cfg.body_args())
        g.set_fields(*I.initial_fields(cfg.nx, cfg.ny, cfg.perturb))
        g.step(1)
        rho = g.poisson_iterate(iters)
        out.append((g.get("phi"), rho))
        g.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1] or (np.isnan(out[0][1]) and np.isnan(out[1][1]))


@pytest.mark.parametrize("m", FUSE)
@pytest.mark.parametrize("P", [2, 3])
def test_loopback_slabs_fused(mods, wf_rows, m, P):
    """Slab decomposition with the fused pass: 2m halo rows exchanged per pass, the
    m residuals reduced after it -- bit-identical to the oracle."""
    wf_rows(10)
    cfg = I.cfg1(steps=3, maxit_p=700)
    o, g, ro, rg = run_pair(mods, cfg, cfg.steps, nranks=P, loopback=True, sor_batch=5, sor_fuse=m)
    assert_parity(o, g, ro, rg)


@pytest.mark.parametrize("peer", ["1", "0"])
@pytest.mark.parametrize("m", [2, 3, 4])
@pytest.mark.parametrize("P,nx,ny", [(2, 128, 96), (3, 130, 98), (4, 257, 131)])
def test_loopback_peer_halo(mods, wf_rows, monkeypatch, peer, m, P, nx, ny):
    """Device-initiated halo: with IBM_PEER_HALO on, each slab's
    fused pass stores its 2m boundary rows straight into the neighbours' ghost rows
    (no exchange between passes); off, the rows go through the overlapped exchange.
    Both bit-identical to the oracle, over ragged slabs and short segments."""
    monkeypatch.setenv("IBM_PEER_HALO", peer)
    wf_rows(10)
    cfg = I.cfg1(nx=nx, ny=ny, steps=3, maxit_p=700)
    o, g, ro, rg = run_pair(mods, cfg, cfg.steps, nranks=P, loopback=True, sor_batch=5, sor_fuse=m)
    assert g.query("peer_halo") == int(peer)
    assert_parity(o, g, ro, rg)


@pytest.mark.parametrize("fuse", [1, 3])
@pytest.mark.parametrize("P,ny", [(2, 50), (2, 53), (3, 98)])
def test_loopback_odd_slab_rows(mods, wf_rows, fuse, P, ny):
    """Slabs whose first global row is odd (colour template TP = 1): the one-
    iteration pass loads its row coefficients by a 1-D TMA box, which must start
    16-B aligned (an odd fp64 start raised "illegal instruction" before the fix)."""
    wf_rows(0)
    cfg = I.cfg1(nx=64, ny=ny, steps=2, maxit_p=500)
    o, g, ro, rg = run_pair(mods, cfg, cfg.steps, nranks=P, loopback=True, sor_batch=5, sor_fuse=fuse)
    assert_parity(o, g, ro, rg)


@pytest.mark.parametrize("m", [3])
def test_loopback_cylinder_fused(mods, wf_rows, m):
    """Body crossing a slab boundary (cylinder centred on the domain's mid row)."""
    wf_rows(0)
    cfg = I.cfg2(nx=96, ny=72, steps=3, maxit_p=400)
    o, g, ro, rg = run_pair(mods, cfg, cfg.steps, nranks=2, loopback=True, sor_fuse=m)
    assert_parity(o, g, ro, rg)


@pytest.mark.parametrize("nr", [1, 2])
@pytest.mark.parametrize("m", FUSE)
@pytest.mark.parametrize("K", [37, 38, 39])
def test_provisional_stop_not_confirmed(mods, wf_rows, m, K, nr):
    """The fused pass decides on a lower bound of rho (its high 32 bits).  With
    tol set to that bound at iteration K (taken from the oracle: rho_K with its
    low word cleared, < rho_K), the pass holding K stops provisionally, the exact
    replay finds rho_K > tol and the solve carries on -- to the oracle's own stop.
    nr = 2: the same through the decomposed path (bounds reduced across slabs,
    k_sor_check, replay with halo exchanges)."""
    import struct
    O, P = mods
    wf_rows(0)
    probe = I.cfg1(nx=64, ny=48, steps=1, maxit_p=K)
    o = O.Oracle(probe.xn, probe.yn, **probe.solver_kwargs())
    o.set_body(*probe.body_args())
    o.set_fields(*I.initial_fields(probe.nx, probe.ny, probe.perturb))
    _, st = o.step(1)
    assert st[0, 2] == K
    bits = struct.unpack("<Q", struct.pack("<d", st[0, 4]))[0]
    assert bits & 0xFFFFFFFF, "rho_K has an empty low word: pick another K"
    tol = struct.unpack("<d", struct.pack("<Q", bits & ~0xFFFFFFFF))[0]
    cfg = I.cfg1(nx=64, ny=48, steps=1, tol_p=tol, maxit_p=5000)
    kw = dict(nranks=2, loopback=True) if nr > 1 else {}
    o2, g, ro, rg = run_pair(mods, cfg, cfg.steps, sor_batch=4, sor_fuse=m, **kw)
    assert ro[1][0, 2] > K  # the oracle goes past K
    assert_parity(o2, g, ro, rg)
    g.close()


@pytest.mark.parametrize("m", FUSE)
def test_nan_in_fused_poisson_is_divergence(mods, wf_rows, m):
    """A NaN that first appears in the Poisson solve (warm-start phi) is caught by
    the fused pass's approximate residual (high word 0x7fffffff), confirmed by the
    exact replay, and reported as divergence -- as by the one-iteration pass."""
    O, P = mods
    wf_rows(0)
    cfg = I.cfg1(nx=64, ny=48, steps=1, maxit_p=200)
    u0, v0, p0 = I.initial_fields(cfg.nx, cfg.ny, cfg.perturb)
    phi0 = np.zeros((cfg.ny, cfg.nx))
    phi0[20, 30] = np.nan
    for fuse in (1, m):
        g = P.Solver(cfg.xn, cfg.yn, sor_batch=4, sor_fuse=fuse, **cfg.solver_kwargs())
        g.set_body(*cfg.body_args())
        g.set_fields(u0, v0, p0, phi=phi0)
        st, _ = g.step(1)
        assert st == 3, (fuse, st)
        g.close()
