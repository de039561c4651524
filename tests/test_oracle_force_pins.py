"""Pins for the oracle's forcing targets (all four directions) and force
coefficients (row a8), and a cross-check of the SOR rounding contract.

Each test checks the oracle against something other than itself: a closed form
of continuum mechanics evaluated on the discrete body (Archimedes' force of a
uniform pressure gradient, the viscous force of a parabolic shear flow), an
exact cancellation the force formula must show for a body started from rest,
the discrete momentum balance built from separately pinned operators, brute
force (bisection intercepts + numpy.polyfit lines), and the plain IEEE form of
the SOR update.

Citations: P:NN = PAPER.md line, S:NN = SPEC.md line; R-numbers = DESIGN.md §2.
These run without a GPU.
"""
import math

import numpy as np
import pytest

import ibm_inputs as I


def _inside(X, Y, a, b, x0, yb):
    dxn, dyn = (X - x0) / a, (Y - yb) / b
    return (dxn * dxn + dyn * dyn) <= 1.0


def _tags_brute(xs, ys, a, b, x0, yb):
    """Independent classification: 0 Fluid, 1 Solid, 2 Forcing."""
    X, Y = np.meshgrid(xs, ys)
    ins = _inside(X, Y, a, b, x0, yb)
    nj, ni = ins.shape
    tag = np.zeros((nj, ni), dtype=np.uint8)
    for j, i in zip(*np.nonzero(ins)):
        nb = [(i + 1, j), (i - 1, j), (i, j + 1), (i, j - 1)]
        fluid = any(0 <= p < ni and 0 <= q < nj and not ins[q, p] for p, q in nb)
        tag[j, i] = 2 if fluid else 1
    return tag


def _metrics(cfg):
    xn, yn = cfg.xn, cfg.yn
    xc, yc = 0.5 * (xn[1:] + xn[:-1]), 0.5 * (yn[1:] + yn[:-1])
    dx, dy = np.diff(xn), np.diff(yn)
    hxc = np.concatenate([[0.0], np.diff(xc)])
    hyc = np.concatenate([[0.0], np.diff(yc)])
    return xc, yc, dx, dy, hxc, hyc


def _body_volumes(cfg, yb):
    """Discrete body volumes of the u and v families: sum of the control volumes
    (hxc dy, dx hyc; R20) of the Solid and Forcing interior nodes."""
    b = cfg.body
    xc, yc, dx, dy, hxc, hyc = _metrics(cfg)
    tu = _tags_brute(cfg.xn, yc, b.a, b.b, b.x0, yb)
    tv = _tags_brute(xc, cfg.yn, b.a, b.b, b.x0, yb)
    nx, ny = cfg.nx, cfg.ny
    dVu = dy[:, None] * np.append(hxc, 0.0)[None, :]   # u nodes i = 0..nx (boundary ones masked)
    dVv = np.append(hyc, 0.0)[:, None] * dx[None, :]   # v nodes j = 0..ny
    mu = tu != 0
    mu[:, 0] = mu[:, nx] = False
    mv = tv != 0
    mv[0, :] = mv[ny, :] = False
    return (dVu * mu).sum(), (dVv * mv).sum(), mu, mv, dVu, dVv


def _oracle(oracle_mod, cfg):
    o = oracle_mod.Oracle(cfg.xn, cfg.yn, **cfg.solver_kwargs())
    o.set_body(*cfg.body_args())
    return o


# ------------------------------------------------------------------ forces (a8)
@pytest.mark.parametrize("body", ["foil", "cylinder"])
def test_force_uniform_pressure_gradient_is_archimedes(oracle_mod, body):
    """A fluid at rest with a uniform pressure gradient G pushes an immersed body
    with F = -G V (Archimedes: -closed-surface integral of p n = -volume integral
    of grad p).  Stationary body, u = v = 0, p = Gx x + Gy y: the oracle's c_d, c_l
    must equal 2 (-Gx V_u, -Gy V_v) on the discrete body volumes to round-off, and
    V must approximate pi a b.  Pins the sign (+x downstream, +y up), the
    factor 2 and that f is summed over every node where the momentum
    equation is replaced (R19b) -- a Forcing-only sum misses the Solid volume."""
    cfg = I.cfg1(steps=1)
    if body == "cylinder":
        cfg.body = I.Body(a=0.4, b=0.4, hbar=0.0, k=1.0)
    cfg.body.hbar = 0.0
    o = _oracle(oracle_mod, cfg)
    xc, yc, *_ = _metrics(cfg)
    Gx, Gy = 0.3, -0.7
    nx, ny = cfg.nx, cfg.ny
    p = Gx * xc[None, :] + Gy * yc[:, None]
    o.set_fields(np.zeros((ny, nx + 1)), np.zeros((ny + 1, nx)), p)
    st, stats = o.step(1)
    assert st in (0, 1)
    Vu, Vv, *_ = _body_volumes(cfg, cfg.body.y0)
    cd, cl = stats[0, 5], stats[0, 6]
    assert abs(cd - 2.0 * (-Gx * Vu)) <= 1e-10 * abs(2 * Gx * Vu), (cd, -2 * Gx * Vu)
    assert abs(cl - 2.0 * (-Gy * Vv)) <= 1e-10 * abs(2 * Gy * Vv), (cl, -2 * Gy * Vv)
    assert cl > 0  # pressure falling upward pushes the body up
    area = math.pi * cfg.body.a * cfg.body.b
    tol = 0.1 if body == "foil" else 0.02  # the foil is ~4 cells thick
    assert abs(Vu - area) < tol * area and abs(Vv - area) < tol * area


def test_force_parabolic_shear_is_viscous_closed_form(oracle_mod):
    """u = y^2, v = 0, p = 0 around a stationary body: convection vanishes, grad^2 u
    = 2, so the viscous force on the body is F_x = nu * volume integral of grad^2 u
    = 2 V / Re (divergence theorem on the shear stress), F_y = 0.  Pins the viscous
    part of u_hat in f (R19) and the momentum term's cancellation of the targets."""
    cfg = I.cfg1(steps=1)
    cfg.body.hbar = 0.0
    o = _oracle(oracle_mod, cfg)
    xc, yc, *_ = _metrics(cfg)
    nx, ny = cfg.nx, cfg.ny
    u = np.repeat((yc ** 2)[:, None], nx + 1, axis=1)
    o.set_fields(u, np.zeros((ny + 1, nx)), np.zeros((ny, nx)))
    st, stats = o.step(1)
    assert st in (0, 1)
    Vu, Vv, *_ = _body_volumes(cfg, cfg.body.y0)
    ref = 2.0 * (2.0 * Vu / cfg.Re)
    assert abs(stats[0, 5] - ref) <= 1e-8 * ref, (stats[0, 5], ref)
    assert abs(stats[0, 6]) <= 1e-8 * ref


def test_force_body_started_from_rest_cancels(oracle_mod):
    """Fluid at rest (u = v = p = 0), plunging body at its first step:
    u_hat = u^n = 0 at every body node, so the momentum forcing (-sum f dV) and the
    body-momentum change (dM/dt) are the same sum with opposite signs and the force
    vanishes to round-off, although each term is O(k h V / dt).  Pins the relative
    sign and weight of the two terms of S:355 and that both run over the same
    nodes (Solid and Forcing, R19b/R20)."""
    cfg = I.cfg1(steps=1)
    o = _oracle(oracle_mod, cfg)
    nx, ny = cfg.nx, cfg.ny
    o.set_fields(np.zeros((ny, nx + 1)), np.zeros((ny + 1, nx)), np.zeros((ny, nx)))
    st, stats = o.step(1)
    assert st in (0, 1)
    b = cfg.body
    _, ydot = oracle_mod.plunge(cfg.dt, b.hbar, b.k)
    _, Vv, *_ = _body_volumes(cfg, b.y0 + oracle_mod.plunge(cfg.dt, b.hbar, b.k)[0])
    scale = 2.0 * abs(ydot) * Vv / cfg.dt  # size of either term in c_l units (~50)
    assert scale > 10.0
    assert abs(stats[0, 5]) <= 1e-12 * scale and abs(stats[0, 6]) <= 1e-12 * scale, stats[0, 5:7]


def test_force_discrete_momentum_budget(oracle_mod):
    """the force equals the direct momentum balance of the body region.
    With unchanged tags (h = 0) and f = (u* - u_hat)/dt at every body node,
    F = sum_body (u_hat - u^n)/dt dV = sum_body (-C - G p + (1/Re) L u) dV at the
    first step (Euler, R8).  Built here from the separately pinned convection and
    Laplacian operators and a numpy pressure difference, on a perturbed state;
    agreement within 1e-10 relative."""
    cfg = I.cfg1(steps=1)
    cfg.body.hbar = 0.0
    o = _oracle(oracle_mod, cfg)
    u, v, p = I.initial_fields(cfg.nx, cfg.ny, 0.05)
    p = 0.2 * I.random_field(p.shape, seed=5)
    o.set_fields(u, v, p)
    xc, yc, dx, dy, hxc, hyc = _metrics(cfg)
    cu, cv = o.convection(u, v)
    Lu, Lv = o.laplacian(0, u), o.laplacian(1, v)
    nx, ny = cfg.nx, cfg.ny
    Gu = np.zeros_like(u)
    Gu[:, 1:nx] = (p[:, 1:] - p[:, :-1]) / hxc[None, 1:]
    Gv = np.zeros_like(v)
    Gv[1:ny, :] = (p[1:, :] - p[:-1, :]) / hyc[1:, None]
    _, _, mu, mv, dVu, dVv = _body_volumes(cfg, cfg.body.y0)
    Fx = ((-cu - Gu + Lu / cfg.Re) * dVu)[mu].sum()
    Fy = ((-cv - Gv + Lv / cfg.Re) * dVv)[mv].sum()
    st, stats = o.step(1)
    assert st in (0, 1)
    for got, ref in ((stats[0, 5], 2 * Fx), (stats[0, 6], 2 * Fy)):
        assert abs(got - ref) <= 1e-10 * max(abs(ref), 1e-3), (got, ref)


# ------------------------------------------------------------------ forcing targets (a3)
def _bisect_intercept(g, lo, hi, iters=200):
    """root of g on [lo, hi] with g(lo) <= 0 < g(hi) (inside -> outside)."""
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        if g(mid) <= 0:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def _target_brute(xs, ys, tag, field, i, j, body, yb, uB):
    """R14/R14b by brute force: per direction E, W, N, S with an in-range Fluid
    neighbour, the intercept by bisection, the line through (B, uB) and the
    neighbour (through N2 when d_N < d_F and N2 is Fluid) by numpy.polyfit,
    evaluated at the forcing node; the mean over the directions."""
    a, b, x0 = body.a, body.b, body.x0
    f = lambda x, y: ((x - x0) / a) ** 2 + ((y - yb) / b) ** 2 - 1.0
    nj, ni = tag.shape
    vals = []
    for di, dj in ((1, 0), (-1, 0), (0, 1), (0, -1)):
        i1, j1 = i + di, j + dj
        if not (0 <= i1 < ni and 0 <= j1 < nj) or tag[j1, i1] != 0:
            continue
        if di:
            xB = _bisect_intercept(lambda s: f(s, ys[j]), xs[i], xs[i1]) if di > 0 else \
                -_bisect_intercept(lambda s: f(-s, ys[j]), -xs[i], -xs[i1])
            dF, dN = abs(xB - xs[i]), abs(xs[i1] - xB)
        else:
            yB = _bisect_intercept(lambda s: f(xs[i], s), ys[j], ys[j1]) if dj > 0 else \
                -_bisect_intercept(lambda s: f(xs[i], -s), -ys[j], -ys[j1])
            dF, dN = abs(yB - ys[j]), abs(ys[j1] - yB)
        uN = field[j1, i1]
        if dN < dF:
            i2, j2 = i1 + di, j1 + dj
            if 0 <= i2 < ni and 0 <= j2 < nj and tag[j2, i2] == 0:
                dN = dN + (abs(xs[i2] - xs[i1]) if di else abs(ys[j2] - ys[j1]))
                uN = field[j2, i2]
        vals.append(np.polyval(np.polyfit([0.0, dN], [uB, uN], 1), -dF))
    return float(np.mean(vals))


@pytest.mark.parametrize("shape", [(0.5, 0.3), (0.45, 0.45), (0.3, 0.5)])
def test_forcing_target_linear_exact_horizontal(oracle_mod, shape):
    """R14 / R14b, horizontal branch (E/W): for forcing nodes whose only Fluid
    neighbour lies east or west, a field linear along the row that takes the body
    velocity at the row's intercept is reproduced exactly -- through N and, when
    d_N < d_F, through N2.  A wrong x-distance (d_F or d_N) or node breaks it."""
    cfg = I.cfg1()
    cfg.body = I.Body(a=shape[0], b=shape[1])
    o = _oracle(oracle_mod, cfg)
    t = 0.07
    o.classify_at(t)
    b = cfg.body
    ybar, ydot = oracle_mod.plunge(t, b.hbar, b.k)
    yb = b.y0 + ybar
    xc, yc, *_ = _metrics(cfg)
    seen = {True: 0, False: 0}
    for fam, name, xs, ys, uB in ((0, "tu", cfg.xn, yc, 0.0), (1, "tv", xc, cfg.yn, ydot)):
        tag = o.get(name)
        nj, ni = tag.shape
        X, Y = np.meshgrid(xs, ys)
        for j, i in zip(*np.nonzero(tag == 2)):
            nbs = [(di, dj) for di, dj in ((1, 0), (-1, 0), (0, 1), (0, -1))
                   if 0 <= i + di < ni and 0 <= j + dj < nj and tag[j + dj, i + di] == 0]
            if len(nbs) != 1 or nbs[0][0] == 0:
                continue
            di = nbs[0][0]
            eta = (ys[j] - yb) / b.b
            xB = b.x0 + di * b.a * math.sqrt(1.0 - eta * eta)
            dF, dN = abs(xB - xs[i]), abs(xs[i + di] - xB)
            field = uB + 0.7 * (X - xB)
            got = o.forcing_target(fam, field, int(i), int(j))
            assert abs(got - (uB + 0.7 * (xs[i] - xB))) < 1e-12
            seen[bool(dN < dF)] += 1
    assert seen[True] >= 2 and seen[False] >= 2, seen


@pytest.mark.parametrize("shape,t", [((0.5, 0.06), 0.07), ((0.5, 0.3), 0.21), ((0.35, 0.35), 0.0)])
def test_forcing_target_brute_force_all_nodes(oracle_mod, shape, t):
    """Every forcing node of both families, any number of Fluid neighbours: the
    oracle's target equals the brute-force one (bisection intercepts, polyfit
    lines, N2 switch, mean over directions) on a random field, within 1e-10."""
    cfg = I.cfg1()
    cfg.body = I.Body(a=shape[0], b=shape[1])
    o = _oracle(oracle_mod, cfg)
    o.classify_at(t)
    b = cfg.body
    ybar, ydot = oracle_mod.plunge(t, b.hbar, b.k)
    yb = b.y0 + ybar
    xc, yc, *_ = _metrics(cfg)
    multi = 0
    for fam, name, xs, ys, uB in ((0, "tu", cfg.xn, yc, 0.0), (1, "tv", xc, cfg.yn, ydot)):
        tag = o.get(name)
        field = I.random_field(tag.shape, seed=31 + fam)
        for j, i in zip(*np.nonzero(tag == 2)):
            ref = _target_brute(xs, ys, tag, field, int(i), int(j), b, yb, uB)
            got = o.forcing_target(fam, field, int(i), int(j))
            assert abs(got - ref) < 1e-10 * (1.0 + abs(ref)), (fam, i, j, got, ref)
            nb = sum(1 for di, dj in ((1, 0), (-1, 0), (0, 1), (0, -1))
                     if 0 <= i + di < tag.shape[1] and 0 <= j + dj < tag.shape[0] and tag[j + dj, i + di] == 0)
            multi += nb > 1
    assert multi > 4


# ------------------------------------------------------------------ SOR rounding contract (R13)
def test_sor_contract_vs_plain_ieee(oracle_mod):
    """R13 is a rounding choice, not a different method: the FMA-chain/reciprocal
    contract and the plain IEEE form of SURVEY §8(c) (s, gs = (b+s)/aP,
    x = (1-w)x + w gs) give identical SOR iteration counts on cfg1 over 10 steps
    and fields within 1e-12 relative L2."""
    cfg = I.cfg1()
    u0, v0, p0 = I.initial_fields(cfg.nx, cfg.ny, cfg.perturb)
    out = []
    try:
        for plain in (False, True):
            oracle_mod.set_sor_form(plain)
            o = _oracle(oracle_mod, cfg)
            o.set_fields(u0, v0, p0)
            st, stats = o.step(cfg.steps)
            out.append((stats, {k: o.get(k) for k in ("u", "v", "p")}))
    finally:
        oracle_mod.set_sor_form(False)
    (s0, f0), (s1, f1) = out
    assert np.array_equal(s0[:, 1:3], s1[:, 1:3])
    for k in ("u", "v", "p"):
        rel = np.linalg.norm(f0[k] - f1[k]) / np.linalg.norm(f0[k])
        assert rel < 1e-12, (k, rel)
    assert not np.array_equal(f0["p"], f1["p"])  # the two forms really differ in rounding


# ------------------------------------------------------------------ oracle_omp
@pytest.mark.parametrize("case", ["cfg1", "stretched-cylinder"])
def test_oracle_omp_bitwise_equal_seq(oracle_mod, case):
    """The OpenMP build of the oracle (rows of one colour / disjoint writes split
    over threads, sums kept serial) is bitwise identical to the one-thread build:
    fields, iteration counts, residuals and forces."""
    if case == "cfg1":
        cfg = I.cfg1(steps=6)
    else:
        xn = I.stretched_axis(-3.0, 6.0, -0.8, 1.2, 1.0 / 40, 1.06)
        yn = I.stretched_axis(-2.5, 2.5, -0.6, 0.6, 1.0 / 40, 1.06)
        cfg = I.Config("stretched-cyl", xn, yn, Re=100.0, dt=2e-3, body=I.Body(a=0.4, b=0.4, hbar=0.1, k=3.0),
                       steps=4, maxit_p=400, perturb=0.01)
    u0, v0, p0 = I.initial_fields(cfg.nx, cfg.ny, cfg.perturb)
    res = []
    for omp in (False, True):
        o = oracle_mod.Oracle(cfg.xn, cfg.yn, omp=omp, **cfg.solver_kwargs())
        o.set_body(*cfg.body_args())
        o.set_fields(u0, v0, p0)
        st, stats = o.step(cfg.steps)
        res.append((st, stats, {k: o.get(k) for k in ("u", "v", "p", "phi", "fu", "fv", "q")}))
    (s0, t0, f0), (s1, t1, f1) = res
    assert s0 == s1
    assert np.array_equal(t0, t1)
    for k in f0:
        assert np.array_equal(f0[k], f1[k]), k


@pytest.mark.parametrize("threads", ["2", "4"])
def test_oracle_omp_bitwise_equals_seq(oracle_mod, monkeypatch, threads):
    """oracle_omp (the same C source with -fopenmp, the all-core CPU baseline of
    bench.py and the SOL1 analogue of the performance report) must give the
    one-thread oracle's fields and statistics bit for bit: its loops split rows of
    one colour / one kernel, and the only sums on the step path (forces) stay
    serial.  BJ configs[0] with the body, 4 steps (converged and capped solves)."""
    monkeypatch.setenv("OMP_NUM_THREADS", threads)
    cfg = I.cfg1(steps=4, maxit_p=600)
    u0, v0, p0 = I.initial_fields(cfg.nx, cfg.ny, cfg.perturb)
    out = []
    for omp in (False, True):
        o = oracle_mod.Oracle(cfg.xn, cfg.yn, omp=omp, **cfg.solver_kwargs())
        o.set_body(*cfg.body_args())
        o.set_fields(u0, v0, p0)
        st, stats = o.step(cfg.steps)
        out.append((st, stats, {n: o.get(n) for n in ("u", "v", "p", "phi", "fu", "fv", "q")}))
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1])
    for n in out[0][2]:
        assert np.array_equal(out[0][2][n], out[1][2][n]), n
