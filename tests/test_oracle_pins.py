"""Pins for the CPU oracle: each function checked against something other than
itself -- closed forms, brute force, library routines, invariants.

Citations: P:NN = PAPER.md line, S:NN = SPEC.md line.  These run without a GPU.
"""
import json
import math
import os

import numpy as np
import pytest

import ibm_inputs as I

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- kinematics
def test_plunge_closed_form(oracle_mod):
    """Eqs. (1)-(2): y(0)=0, ydot(0)=k h; y(pi/2k)=h, ydot(pi/2k)=0."""
    k, h = 2 * math.pi, 0.16
    y, yd = oracle_mod.plunge(0.0, h, k)
    assert y == 0.0 and yd == k * h
    y, yd = oracle_mod.plunge(math.pi / (2 * k), h, k)
    assert abs(y - h) < 1e-15 and abs(yd) < 1e-15
    # P:150 "k h = 1.0 with k = 2 pi and h = 0.16" (paper rounds 1.00531)
    assert abs(k * h - 1.0) < 6e-3


def test_plunge_fd_and_period(oracle_mod):
    """central FD of y matches ydot (rel < 1e-6 at dt = 1e-4); period 2 pi / k."""
    k, h, dt = 2 * math.pi, 0.16, 1e-4
    for t in np.linspace(0.01, 1.7, 23):
        yp, _ = oracle_mod.plunge(t + dt, h, k)
        ym, _ = oracle_mod.plunge(t - dt, h, k)
        _, yd = oracle_mod.plunge(t, h, k)
        fd = (yp - ym) / (2 * dt)
        assert abs(fd - yd) <= 1e-6 * max(abs(yd), 1e-3 * k * h)
        y1, _ = oracle_mod.plunge(t, h, k)
        y2, _ = oracle_mod.plunge(t + 2 * math.pi / k, h, k)
        assert abs(y1 - y2) < 1e-12


# ---------------------------------------------------------------- geometry
def test_inside_examples(oracle_mod):
    """S:172-174 worked example: a=0.5, b=0.06, (0.3, 0.04): 0.36 + 0.4444 <= 1."""
    assert oracle_mod.inside(0.3, 0.04, 0.5, 0.06, 0.0, 0.0)
    assert oracle_mod.inside(0.0, 0.0, 0.5, 0.06, 0.0, 0.0)
    assert not oracle_mod.inside(10.0, 10.0, 0.5, 0.06, 0.0, 0.0)
    assert oracle_mod.inside(0.5, 0.0, 0.5, 0.06, 0.0, 0.0)  # boundary inclusive
    assert not oracle_mod.inside(0.3, 0.05, 0.5, 0.06, 0.0, 0.0)  # 0.36 + 0.694 > 1


def test_intercept_vs_bisection(oracle_mod):
    """closed-form intercept vs bisection within 1e-10; ellipse residual < 1e-12."""
    rng = np.random.default_rng(7)
    a, b, xb, yb = 0.5, 0.06, 0.1, -0.03
    f = lambda x, y: ((x - xb) / a) ** 2 + ((y - yb) / b) ** 2 - 1.0
    n = 0
    while n < 200:
        axis = int(rng.integers(0, 2))
        d = int(rng.choice([-1, 1]))
        xF = xb + a * rng.uniform(-0.95, 0.95)
        yF = yb + b * rng.uniform(-0.95, 0.95)
        if f(xF, yF) > 0:
            continue
        if axis == 0:
            xN, yN = xF + d * 2.5 * a, yF
        else:
            xN, yN = xF, yF + d * 2.5 * b
        B = oracle_mod.intercept(axis, d, xF, yF, a, b, xb, yb)
        lo, hi = (xF, xN) if axis == 0 else (yF, yN)
        g = (lambda s: f(s, yF)) if axis == 0 else (lambda s: f(xF, s))
        for _ in range(200):
            mid = 0.5 * (lo + hi)
            if g(mid) <= 0:
                lo = mid
            else:
                hi = mid
        assert abs(B - 0.5 * (lo + hi)) < 1e-10
        assert abs(g(B)) < 1e-12
        n += 1
    # through the centre: x = +-a
    assert oracle_mod.intercept(0, 1, 0.0, 0.0, 0.5, 0.06, 0.0, 0.0) == 0.5
    assert oracle_mod.intercept(0, -1, 0.0, 0.0, 0.5, 0.06, 0.0, 0.0) == -0.5


def test_target_dir_is_linear_extrapolation(oracle_mod):
    """R14 / S:254: the target is the line through (B, uB), (N, uN) evaluated at F,
    which lies at distance dF on the other side of B; pinned against numpy.polyfit."""
    rng = np.random.default_rng(11)
    for _ in range(200):
        uB, uN = rng.uniform(-2, 2, 2)
        dF, dN = rng.uniform(0.01, 1.0, 2)
        ref = np.polyval(np.polyfit([0.0, dN], [uB, uN], 1), -dF)
        assert abs(oracle_mod.target_dir(uB, uN, dF, dN) - ref) < 1e-10 * (1 + abs(ref))
    # zero distance -> body velocity exactly; uN == uB -> uB
    assert oracle_mod.target_dir(0.3, 5.0, 0.0, 0.2) == 0.3
    assert oracle_mod.target_dir(0.3, 0.3, 0.7, 0.2) == 0.3


def _classify_brute(xn, yn, body, t):
    """Independent full-scan classification with numpy."""
    a, b, x0, y0, hbar, k = body
    yb = y0 + hbar * math.sin(k * t)
    xc, yc = 0.5 * (xn[1:] + xn[:-1]), 0.5 * (yn[1:] + yn[:-1])
    out = {}
    for name, (xs, ys) in {"tu": (xn, yc), "tv": (xc, yn), "tp": (xc, yc)}.items():
        X, Y = np.meshgrid(xs, ys)
        dxn, dyn = (X - x0) / a, (Y - yb) / b
        ins = (dxn * dxn + dyn * dyn) <= 1.0
        tag = np.zeros(ins.shape, dtype=np.uint8)
        nj, ni = ins.shape
        for j in range(nj):
            for i in range(ni):
                if not ins[j, i]:
                    continue
                nb = [(i + 1, j), (i - 1, j), (i, j + 1), (i, j - 1)]
                fluid = any(0 <= p < ni and 0 <= q < nj and not ins[q, p] for p, q in nb)
                tag[j, i] = 2 if fluid else 1
        out[name] = tag
    return out


@pytest.mark.parametrize("t", [0.0, 0.013, 0.25, 0.6])
def test_classification_brute_force(oracle_mod, t):
    """tag counts (and every tag) equal a brute-force re-classification."""
    cfg = I.cfg1()
    o = oracle_mod.Oracle(cfg.xn, cfg.yn, **cfg.solver_kwargs())
    o.set_body(*cfg.body_args())
    o.classify_at(t)
    ref = _classify_brute(cfg.xn, cfg.yn, cfg.body_args(), t)
    for name in ("tu", "tv", "tp"):
        got = o.get(name)
        assert np.array_equal(got, ref[name]), name
        assert (got == 2).sum() > 0 and (got == 1).sum() > 0


def test_classification_area(oracle_mod):
    """(#Solid+Forcing p cells) x cell area ~ pi a b within 5%."""
    cfg = I.cfg1()
    o = oracle_mod.Oracle(cfg.xn, cfg.yn, **cfg.solver_kwargs())
    o.set_body(*cfg.body_args())
    h = cfg.xn[1] - cfg.xn[0]
    area = (o.get("tp") != 0).sum() * h * h
    b = cfg.body
    assert abs(area - math.pi * b.a * b.b) / (math.pi * b.a * b.b) < 0.05


def test_forcing_target_uniform_body_velocity(oracle_mod):
    """when the fluid neighbours carry the body velocity, every target is the
    body velocity (u_B = 0 for u, ydot for v)."""
    cfg = I.cfg1()
    o = oracle_mod.Oracle(cfg.xn, cfg.yn, **cfg.solver_kwargs())
    o.set_body(*cfg.body_args())
    t = 0.07
    o.classify_at(t)
    _, yd = oracle_mod.plunge(t, cfg.body.hbar, cfg.body.k)
    tu, tv = o.get("tu"), o.get("tv")
    u0 = np.zeros(o.shape("u"))
    v0 = np.full(o.shape("v"), yd)
    for (j, i) in zip(*np.nonzero(tu == 2)):
        assert o.forcing_target(0, u0, int(i), int(j)) == 0.0
    for (j, i) in zip(*np.nonzero(tv == 2)):
        assert abs(o.forcing_target(1, v0, int(i), int(j)) - yd) < 1e-14


# ---------------------------------------------------------------- operators
def _unit_grid(n, Lx=2.0, Ly=1.0):
    return I.uniform_axis(0.0, Lx, 2 * n), I.uniform_axis(0.0, Ly, n)


def test_convection_uniform_flow_zero(oracle_mod):
    """uniform flow u=1, v=0 gives C = 0 exactly."""
    cfg = I.cfg1()
    o = oracle_mod.Oracle(cfg.xn, cfg.yn, **cfg.solver_kwargs())
    o.clear_body()
    u, v, _ = I.initial_fields(cfg.nx, cfg.ny)
    cu, cv = o.convection(u, v)
    assert np.all(cu == 0.0) and np.all(cv == 0.0)


def test_convection_second_order(oracle_mod):
    """smooth field vs analytic div(uu); max error falls ~4x per halving.
    v vanishes on the walls and the inlet and has zero x-slope at the outlet,
    matching the wall / inlet / outlet closures of R10."""
    Lx, Ly = 2.0, 1.0
    errs = []
    for n in (16, 32, 64):
        xn, yn = _unit_grid(n, Lx, Ly)
        o = oracle_mod.Oracle(xn, yn, Re=100.0, dt=1e-3)
        o.clear_body()
        xc, yc = 0.5 * (xn[1:] + xn[:-1]), 0.5 * (yn[1:] + yn[:-1])
        al, be = math.pi / (2 * Lx), math.pi / Ly
        U = lambda x, y: 1.0 + 0.5 * np.cos(1.3 * x) * np.cos(0.7 * y + 0.2)
        Ux = lambda x, y: -0.65 * np.sin(1.3 * x) * np.cos(0.7 * y + 0.2)
        Uy = lambda x, y: -0.35 * np.cos(1.3 * x) * np.sin(0.7 * y + 0.2)
        Vf = lambda x, y: 0.4 * np.sin(al * x) * np.sin(be * y)
        Vx = lambda x, y: 0.4 * al * np.cos(al * x) * np.sin(be * y)
        Vy = lambda x, y: 0.4 * be * np.sin(al * x) * np.cos(be * y)
        Xu, Yu = np.meshgrid(xn, yc)
        Xv, Yv = np.meshgrid(xc, yn)
        cu, cv = o.convection(U(Xu, Yu), Vf(Xv, Yv))
        # d(uu)/dx + d(uv)/dy ; d(uv)/dx + d(vv)/dy
        cu_ex = 2 * U(Xu, Yu) * Ux(Xu, Yu) + Uy(Xu, Yu) * Vf(Xu, Yu) + U(Xu, Yu) * Vy(Xu, Yu)
        cv_ex = Ux(Xv, Yv) * Vf(Xv, Yv) + U(Xv, Yv) * Vx(Xv, Yv) + 2 * Vf(Xv, Yv) * Vy(Xv, Yv)
        eu = np.abs(cu - cu_ex)[:, 1:-1].max()
        ev = np.abs(cv - cv_ex)[1:-1, :].max()
        errs.append((eu, ev))
    for k in range(2):
        for c in range(2):
            r = errs[k][c] / errs[k + 1][c]
            assert 3.2 <= r <= 4.8, (k, c, errs)


def test_laplacian_second_order(oracle_mod):
    """Viscous / pressure Laplacians on the MAC grid (R10): fields that satisfy
    each family's boundary closure -- slip walls, Dirichlet v=0 at the inlet face,
    phi = 0 at the outlet face -- converge at second order in the max norm."""
    Lx, Ly = 2.0, 1.0
    al, be = math.pi / (2 * Lx), math.pi / Ly
    errs = {0: [], 1: [], 2: []}
    for n in (16, 32, 64):
        xn, yn = _unit_grid(n, Lx, Ly)
        o = oracle_mod.Oracle(xn, yn, Re=100.0, dt=1e-3)
        xc, yc = 0.5 * (xn[1:] + xn[:-1]), 0.5 * (yn[1:] + yn[:-1])
        # u: cos(be y) (slip walls), any x-profile; outlet column excluded (zero-gradient closure)
        X, Y = np.meshgrid(xn, yc)
        f = np.exp(0.3 * X) * np.cos(be * Y)
        lap = (0.09 - be * be) * f
        L = o.laplacian(0, f)
        errs[0].append(np.abs(L - lap)[:, 1:-2].max())
        # v: sin(1.1 x) sin(be y) (odd about the inlet face -> Dirichlet v=0 there)
        X, Y = np.meshgrid(xc, yn)
        f = np.sin(1.1 * X) * np.sin(be * Y)
        lap = -(1.21 + be * be) * f
        L = o.laplacian(1, f)
        errs[1].append(np.abs(L - lap)[1:-1, :-1].max())
        # p: cos(al x) cos(be y): Neumann W/S/N, phi=0 on the outlet face (all cells)
        X, Y = np.meshgrid(xc, yc)
        f = np.cos(al * X) * np.cos(be * Y)
        lap = -(al * al + be * be) * f
        L = o.laplacian(2, f)
        errs[2].append(np.abs(L - lap).max())
    for fam, e in errs.items():
        for k in range(2):
            assert 3.2 <= e[k] / e[k + 1] <= 4.8, (fam, e)


# ---------------------------------------------------------------- SOR
def _dirichlet16(n=16):
    aP = np.full((n, n), 4.0)
    aE = np.ones((n, n)); aW = np.ones((n, n)); aN = np.ones((n, n)); aS = np.ones((n, n))
    T = 2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    A = np.kron(np.eye(n), T) + np.kron(T, np.eye(n))   # row-major (j, i), x fastest
    return aP, aE, aW, aN, aS, A


def test_sor_dense_direct(oracle_mod):
    """S:286 / S:563: 16x16 Dirichlet Poisson by red-black SOR vs numpy dense solve,
    max difference < 1e-8 at tol = 1e-10; omega = 1.5 needs fewer sweeps than 1.0."""
    n = 16
    aP, aE, aW, aN, aS, A = _dirichlet16(n)
    b = I.random_field((n, n), seed=3)
    upd = np.ones((n, n), dtype=np.uint8)
    x_ref = np.linalg.solve(A, b.ravel()).reshape(n, n)
    x15, it15, rho15, st = oracle_mod.sor_generic(aP, aE, aW, aN, aS, b, upd, np.zeros((n, n)), 1.5, 1e-10, 100000)
    assert st == 0 and rho15 <= 1e-10
    assert np.abs(x15 - x_ref).max() < 1e-8
    x10, it10, _, _ = oracle_mod.sor_generic(aP, aE, aW, aN, aS, b, upd, np.zeros((n, n)), 1.0, 1e-10, 100000)
    assert np.abs(x10 - x_ref).max() < 1e-8
    assert it15 < it10


def test_sor_exact_initial_guess(oracle_mod):
    """rhs = A x0 with initial guess x0 converges in one sweep pair."""
    n = 16
    aP, aE, aW, aN, aS, A = _dirichlet16(n)
    x0 = I.random_field((n, n), seed=5)
    b = (A @ x0.ravel()).reshape(n, n)
    upd = np.ones((n, n), dtype=np.uint8)
    x, it, rho, st = oracle_mod.sor_generic(aP, aE, aW, aN, aS, b, upd, x0, 1.5, 1e-12, 100)
    assert it == 1 and rho <= 1e-12 and st == 0


def test_sor_nan_is_divergence(oracle_mod):
    n = 8
    aP, aE, aW, aN, aS, A = _dirichlet16(n)
    b = np.zeros((n, n)); b[3, 4] = np.nan
    upd = np.ones((n, n), dtype=np.uint8)
    x, it, rho, st = oracle_mod.sor_generic(aP, aE, aW, aN, aS, b, upd, np.zeros((n, n)), 1.5, 1e-8, 50)
    assert st == 3 and it == 1 and math.isnan(rho)


def test_sor_maxit_reported(oracle_mod):
    n = 16
    aP, aE, aW, aN, aS, A = _dirichlet16(n)
    b = I.random_field((n, n), seed=9)
    upd = np.ones((n, n), dtype=np.uint8)
    x, it, rho, st = oracle_mod.sor_generic(aP, aE, aW, aN, aS, b, upd, np.zeros((n, n)), 1.5, 1e-14, 7)
    assert it == 7 and st == 1 and rho > 1e-14


def test_poisson_manufactured(oracle_mod):
    """S:294 / BJ: manufactured phi = cos(pi x/(2Lx)) cos(pi y/Ly) (Neumann W/S/N,
    phi = 0 on the outlet face); discrete error falls 3.2-4.8x per halving."""
    Lx, Ly = 2.0, 1.0
    al, be = math.pi / (2 * Lx), math.pi / Ly
    errs = []
    for n in (8, 16, 32):
        xn, yn = _unit_grid(n, Lx, Ly)
        o = oracle_mod.Oracle(xn, yn, Re=100.0, dt=1e-3, omega_p=1.8, tol_p=1e-13, maxit_p=200000)
        o.clear_body()
        xc, yc = 0.5 * (xn[1:] + xn[:-1]), 0.5 * (yn[1:] + yn[:-1])
        X, Y = np.meshgrid(xc, yc)
        ex = np.cos(al * X) * np.cos(be * Y)
        rhs = -(al * al + be * be) * ex
        phi, it, rho, st = o.poisson(rhs)
        assert st == 0, (it, rho)
        errs.append(np.abs(phi - ex).max())
    for k in range(2):
        assert 3.2 <= errs[k] / errs[k + 1] <= 4.8, errs


# ---------------------------------------------------------------- full step invariants
def test_uniform_flow_fixed_point(oracle_mod):
    """no body, uniform flow is a fixed point of the full step."""
    cfg = I.cfg1()
    o = oracle_mod.Oracle(cfg.xn, cfg.yn, **cfg.solver_kwargs())
    o.clear_body()
    u, v, p = I.initial_fields(cfg.nx, cfg.ny)
    o.set_fields(u, v, p)
    st, stats = o.step(3)
    assert st == 0
    assert np.abs(o.get("u") - 1.0).max() <= 1e-12
    assert np.abs(o.get("v")).max() <= 1e-12
    assert np.abs(o.get("p")).max() <= 1e-12
    assert np.all(stats[:, 2] == 1)  # Poisson: b = 0 -> converged at the first sweep pair


def test_uniform_flow_fixed_point_stretched(oracle_mod):
    """Same invariant on a geometrically stretched grid (S:45-53 axis)."""
    xn = I.stretched_axis(-3.0, 6.0, -1.0, 2.0, 0.1, 1.08)
    yn = I.stretched_axis(-3.0, 3.0, -0.6, 0.6, 0.1, 1.08)
    o = oracle_mod.Oracle(xn, yn, Re=500.0, dt=2e-3)
    o.clear_body()
    nx, ny = len(xn) - 1, len(yn) - 1
    u, v, p = I.initial_fields(nx, ny)
    o.set_fields(u, v, p)
    st, _ = o.step(2)
    assert st == 0
    assert np.abs(o.get("u") - 1.0).max() <= 1e-12 and np.abs(o.get("v")).max() <= 1e-12


def _divergence(o, u, v):
    xn, yn = o.xn, o.yn
    dx, dy = np.diff(xn), np.diff(yn)
    return (u[:, 1:] - u[:, :-1]) / dx[None, :] + (v[1:, :] - v[:-1, :]) / dy[:, None]


def test_projection_divergence_bound(oracle_mod):
    """S:303 / S:318: after correction max |div u - q| <= 10 tol_p / dt on active
    cells; with a tight tolerance it is at round-off level (BJ 'discrete
    divergence-free velocity to round-off after projection')."""
    for tol, bound in ((1e-6, None), (1e-13, 1e-8)):
        cfg = I.cfg1(steps=2, tol_p=tol, maxit_p=400000)
        o = oracle_mod.Oracle(cfg.xn, cfg.yn, **cfg.solver_kwargs())
        o.set_body(*cfg.body_args())
        o.set_fields(*I.initial_fields(cfg.nx, cfg.ny, cfg.perturb))
        st, stats = o.step(2)
        assert st == 0, stats
        d = _divergence(o, o.get("u"), o.get("v")) - o.get("q")
        act = o.get("act").astype(bool)
        err = np.abs(d[act]).max()
        assert err <= 10 * tol / cfg.dt
        if bound is not None:
            assert err <= bound, err


def test_mirror_symmetry(oracle_mod):
    """zero-amplitude plunge, symmetric foil and grid -> v antisymmetric and
    u symmetric about the foil centreline (tight tolerances, since colour parity
    is not mirror-symmetric for even ny)."""
    cfg = I.cfg1(perturb=0.0, tol_p=1e-12, tol_uv=1e-14, maxit_p=400000)
    cfg.body.hbar = 0.0
    o = oracle_mod.Oracle(cfg.xn, cfg.yn, **cfg.solver_kwargs())
    o.set_body(*cfg.body_args())
    o.set_fields(*I.initial_fields(cfg.nx, cfg.ny))
    st, _ = o.step(3)
    assert st == 0
    u, v = o.get("u"), o.get("v")
    assert np.abs(v + v[::-1, :]).max() < 1e-8
    assert np.abs(u - u[::-1, :]).max() < 1e-8
    tp = o.get("tp")
    assert np.array_equal(tp, tp[::-1, :])


def test_forces_zero_flow_stationary_body(oracle_mod):
    """zero flow and a stationary body give c_l = c_d = 0."""
    cfg = I.cfg1()
    cfg.body.hbar = 0.0
    o = oracle_mod.Oracle(cfg.xn, cfg.yn, **cfg.solver_kwargs())
    o.set_body(*cfg.body_args())
    nx, ny = cfg.nx, cfg.ny
    o.set_fields(np.zeros((ny, nx + 1)), np.zeros((ny + 1, nx)), np.zeros((ny, nx)))
    st, stats = o.step(2)
    assert st == 0
    assert np.all(stats[:, 5] == 0.0) and np.all(stats[:, 6] == 0.0)


def test_forces_pressure_constant_invariance(oracle_mod):
    """adding a uniform constant to p leaves c_l, c_d unchanged."""
    res = []
    for c0 in (0.0, 0.75):
        cfg = I.cfg1(steps=1)
        o = oracle_mod.Oracle(cfg.xn, cfg.yn, **cfg.solver_kwargs())
        o.set_body(*cfg.body_args())
        u, v, p = I.initial_fields(cfg.nx, cfg.ny, cfg.perturb)
        p = 0.01 * I.random_field(p.shape, seed=17) + c0
        o.set_fields(u, v, p)
        st, stats = o.step(1)
        res.append(stats[0, 5:7])
    assert np.allclose(res[0], res[1], rtol=1e-6, atol=1e-9)


def test_helmholtz_solution_satisfies_system(oracle_mod):
    """The predictor u* solves (I - beta L) u* = rhs at Fluid nodes, using
    L pinned independently above; residual bounded by diag x tol_uv."""
    cfg = I.cfg1(steps=1, tol_uv=1e-12)
    o = oracle_mod.Oracle(cfg.xn, cfg.yn, **cfg.solver_kwargs())
    o.set_body(*cfg.body_args())
    o.set_fields(*I.initial_fields(cfg.nx, cfg.ny, cfg.perturb))
    st, stats = o.step(1)
    assert st in (0, 1) and stats[0, 1] < cfg.maxit_uv  # Poisson may stop at maxit_p
    beta = cfg.dt * 0.5 / cfg.Re
    us, rhs = o.get("us"), o.get("rhs_u")
    us_pre = us.copy()
    us_pre[:, -1] = 0.0  # outlet fill happened after the solve; the nx-1 row has cE = 0
    r = us - beta * o.laplacian(0, us_pre) - rhs
    fluid = (o.get("tu") == 0)
    fluid[:, 0] = False
    fluid[:, -1] = False
    assert np.abs(r[fluid]).max() < 1e-10


def test_paper_constants_golden():
    """tests/golden/paper_constants.json holds numbers the paper prints (cited);
    the input generators use exactly those."""
    with open(os.path.join(GOLDEN, "paper_constants.json")) as f:
        g = json.load(f)
    assert tuple(g["domain"]["value"]) == I.PAPER_DOMAIN
    assert g["thickness_ratio"]["value"] == I.THICKNESS_RATIO
    assert g["Re"]["value"] == I.PAPER_RE
    assert g["hbar"]["value"] == I.PAPER_HBAR
    assert g["dt"]["value"] == I.PAPER_DT
    assert abs(g["k"]["value"] - I.PAPER_K) < 1e-15
    b = I.Body()
    assert b.b / b.a == I.THICKNESS_RATIO


def test_forcing_target_linear_exact_including_second_node(oracle_mod):
    """R14 / R14b: for forcing nodes with a single fluid neighbour (vertical), a
    field linear along the column that takes the body velocity at the boundary
    intercept is reproduced exactly -- both when the target extrapolates through
    the neighbour N and when it switches to N2 (d_N < d_F).  A wrong distance or
    node in either branch breaks the exactness."""
    cfg = I.cfg1()
    o = oracle_mod.Oracle(cfg.xn, cfg.yn, **cfg.solver_kwargs())
    o.set_body(*cfg.body_args())
    t = 0.07
    o.classify_at(t)
    b = cfg.body
    ybar, ydot = oracle_mod.plunge(t, b.hbar, b.k)
    yb = b.y0 + ybar
    xc, yc = 0.5 * (cfg.xn[1:] + cfg.xn[:-1]), 0.5 * (cfg.yn[1:] + cfg.yn[:-1])
    seen = {True: 0, False: 0}
    for fam, name, xs, ys, uB in ((0, "tu", cfg.xn, yc, 0.0), (1, "tv", xc, cfg.yn, ydot)):
        tag = o.get(name)
        nj, ni = tag.shape
        X, Y = np.meshgrid(xs, ys)
        for j, i in zip(*np.nonzero(tag == 2)):
            nbs = [(di, dj) for di, dj in ((1, 0), (-1, 0), (0, 1), (0, -1))
                   if 0 <= i + di < ni and 0 <= j + dj < nj and tag[j + dj, i + di] == 0]
            if len(nbs) != 1 or nbs[0][1] == 0:
                continue
            dj = nbs[0][1]
            z = (xs[i] - b.x0) / b.a
            yB = yb + dj * b.b * math.sqrt(1.0 - z * z)
            dF, dN = abs(yB - ys[j]), abs(ys[j + dj] - yB)
            field = uB + 0.7 * (Y - yB)
            got = o.forcing_target(fam, field, int(i), int(j))
            assert abs(got - (uB + 0.7 * (ys[j] - yB))) < 1e-12
            seen[bool(dN < dF)] += 1
    assert seen[True] > 5 and seen[False] > 5


def test_long_run_bounded(oracle_mod):
    """R9b / R14b: with the open-face pressure gradient and the N2 switch the
    cfg1 foil stays bounded over 60 steps with converged Poisson solves (the
    SPEC-literal readings diverge within ~40 steps)."""
    cfg = I.cfg1(perturb=0.0, steps=60, omega_p=1.9, maxit_p=100000)
    o = oracle_mod.Oracle(cfg.xn, cfg.yn, **cfg.solver_kwargs())
    o.set_body(*cfg.body_args())
    o.set_fields(*I.initial_fields(cfg.nx, cfg.ny))
    st, stats = o.step(cfg.steps)
    assert st == 0
    assert np.abs(o.get("u")).max() < 3.0 and np.abs(o.get("v")).max() < 3.0
    assert np.all(np.isfinite(stats[:, 5:7]))


def test_temporal_order_second(oracle_mod):
    """P:54 (R7): AB2 convection + CN diffusion + incremental projection are second
    order in time.  Self-convergence on a fixed 48x32 grid from a discretely
    divergence-free start (streamfunction on cell corners, vanishing at the inlet
    and walls): successive differences at T fall 4x per dt halving (3.2-4.8).
    This also pins the outlet reading R10b -- the SPEC-literal zero-gradient
    fill makes these differences stagnate."""
    nx, ny, L, H = 48, 32, 3.0, 2.0
    xn, yn = I.uniform_axis(0.0, L, nx), I.uniform_axis(-1.0, 1.0, ny)
    Xc, Yc = np.meshgrid(xn, yn)
    psi = Yc + 0.05 * np.sin(math.pi * Xc / L) ** 2 * np.sin(math.pi * (Yc + 1) / H) ** 2
    u0 = (psi[1:, :] - psi[:-1, :]) / np.diff(yn)[:, None]
    v0 = -(psi[:, 1:] - psi[:, :-1]) / np.diff(xn)[None, :]
    u0[:, 0], v0[0, :], v0[-1, :] = 1.0, 0.0, 0.0
    T, res = 0.02, []
    for dt in (0.01, 0.005, 0.0025, 0.00125):
        o = oracle_mod.Oracle(xn, yn, Re=50.0, dt=dt, omega_p=1.8, tol_p=1e-13, maxit_p=200000, omega_uv=1.2,
                              tol_uv=1e-14, maxit_uv=10000)
        o.clear_body()
        o.set_fields(u0, v0, np.zeros((ny, nx)))
        st, _ = o.step(int(round(T / dt)))
        assert st == 0
        res.append((o.get("u"), o.get("v")))
    for k in (0, 1):
        e = [np.abs(res[i][k] - res[i + 1][k]).max() for i in range(3)]
        for i in range(2):
            assert 3.2 <= e[i] / e[i + 1] <= 4.8, (k, e)


def test_production_mesh_presets():
    """cfg3 mesh levels (reading R28): nx*ny within 1 % of 6/12/18 lakh,
    axes span the paper domain exactly, uniform patch at h_min with a
    whole number of cells, geometric ratio 1.05 outside except the
    clamped last cell, M1 at h_min ~ 0.004."""
    x0, x1, y0, y1 = I.PAPER_DOMAIN
    for level, cells in I.MESH_LEVEL_CELLS.items():
        c = I.cfg3(level=level)
        assert abs(c.nx * c.ny - cells) <= 0.01 * cells
        h = c.extra["h_min"]
        for ax, lo, hi, ulo, uhi in ((c.xn, x0, x1, -1.0, 2.0), (c.yn, y0, y1, -0.75, 0.75)):
            assert ax[0] == lo and ax[-1] == hi
            d = np.diff(ax)
            assert np.all(d > 0)
            core = (ax[:-1] >= ulo - 1e-12) & (ax[1:] <= uhi + 1e-12)
            assert np.allclose(d[core], h, rtol=1e-9, atol=0)
            iu = np.nonzero(core)[0]
            right = d[iu[-1] + 1:-1]          # stretched cells, clamped last one excluded
            left = d[1:iu[0]][::-1]
            for side in (right, left):
                r = side[1:] / side[:-1]
                assert np.allclose(r, 1.05, rtol=1e-9)
                assert abs(side[0] / h - 1.05) < 1e-9
    assert abs(I.cfg3(level=1).extra["h_min"] - 0.004) < 0.0005
