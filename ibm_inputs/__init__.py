"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no stencil, no SOR, no forcing):
only grid-node coordinates, body parameters, solver settings and seeded initial
fields -- the inputs both sides receive.  It imports neither ``oracle`` nor the
product package.

Recipes follow SURVEY.md §8(d) / DESIGN.md §5:
  cfg1  plunging foil Re=500, 128x96 uniform on [-1.5,2.5]x[-1.5,1.5], h=1/32
  cfg2  stationary cylinder Re=100, 512x384 uniform on [-8,24]x[-12,12], h=1/16
  cfg3  paper domain [-7.5,24]x[-12.5,12.5], uniform patch + geometric stretch
  cfg4  N x N uniform on the paper domain, N in 256..8192 (input-scaling sweep)
  cfg5  16384 x 16384 uniform on the paper domain (slab-decomposed)
Physics constants: t/c = 0.12; Re = 500, k = 2 pi, h = 0.16;
dt = 1e-4 on the production grid.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, asdict

import numpy as np

SEED = 240217337
PAPER_DOMAIN = (-7.5, 24.0, -12.5, 12.5)
THICKNESS_RATIO = 0.12
PAPER_RE, PAPER_K, PAPER_HBAR = 500.0, 2.0 * math.pi, 0.16
PAPER_DT = 1e-4


def uniform_axis(lo: float, hi: float, n: int) -> np.ndarray:
    """n cells, n+1 node coordinates."""
    return np.linspace(lo, hi, n + 1)


def stretched_axis(domain_lo, domain_hi, uniform_lo, uniform_hi, h_min, ratio=1.05):
    """Uniform patch of spacing h_min on [uniform_lo, uniform_hi], geometric
    progression (factor `ratio`) toward both domain ends, last cell clamped so
    the end node equals the domain bound exactly."""
    if not (domain_lo < uniform_lo < uniform_hi < domain_hi) or h_min <= 0 or ratio < 1:
        raise ValueError("stretched_axis: invalid bounds")
    n_uni = int(round((uniform_hi - uniform_lo) / h_min))
    core = uniform_lo + h_min * np.arange(n_uni + 1)
    core[-1] = uniform_hi

    def side(length):
        widths, w, tot = [], h_min, 0.0
        while tot < length - 1e-12:
            w = w * ratio
            if tot + w >= length or tot + w + w * ratio > length + 0.5 * w * ratio:
                widths.append(length - tot)
                break
            widths.append(w)
            tot += w
        return np.array(widths)

    right = side(domain_hi - uniform_hi)
    left = side(uniform_lo - domain_lo)
    xr = uniform_hi + np.cumsum(right)
    xr[-1] = domain_hi
    xl = uniform_lo - np.cumsum(left)
    xl[-1] = domain_lo
    return np.concatenate([xl[::-1], core, xr])


@dataclass
class Body:
    a: float = 0.5                      # chord/2
    b: float = 0.5 * THICKNESS_RATIO    # thickness/2  (t/c = 0.12)
    x0: float = 0.0
    y0: float = 0.0
    hbar: float = PAPER_HBAR
    k: float = PAPER_K


@dataclass
class Config:
    name: str
    xn: np.ndarray
    yn: np.ndarray
    Re: float
    dt: float
    body: Body | None
    steps: int
    omega_p: float = 1.5
    tol_p: float = 1e-6
    maxit_p: int = 10000
    omega_uv: float = 1.2
    tol_uv: float = 1e-8
    maxit_uv: int = 1000
    check_every: int = 1
    perturb: float = 0.0
    seed: int = SEED
    extra: dict = field(default_factory=dict)

    @property
    def nx(self):
        return len(self.xn) - 1

    @property
    def ny(self):
        return len(self.yn) - 1

    def solver_kwargs(self):
        return dict(Re=self.Re, dt=self.dt, omega_p=self.omega_p, tol_p=self.tol_p,
                    maxit_p=self.maxit_p, omega_uv=self.omega_uv, tol_uv=self.tol_uv,
                    maxit_uv=self.maxit_uv, check_every=self.check_every)

    def body_args(self):
        b = self.body
        return None if b is None else (b.a, b.b, b.x0, b.y0, b.hbar, b.k)

    def describe(self):
        d = {k: v for k, v in asdict(self).items() if k not in ("xn", "yn", "extra")}
        d.update(nx=self.nx, ny=self.ny)
        return d


def cfg1(perturb=0.01, nx=128, ny=96, steps=10, **kw) -> Config:
    """BJ configs[0]: plunging foil, Re=500, 128x96, 10 steps; h = 1/32."""
    h = 1.0 / 32.0 * (128 / nx)
    xn = uniform_axis(-1.5, -1.5 + h * nx, nx)
    yn = uniform_axis(-0.5 * h * ny, 0.5 * h * ny, ny)
    return Config("cfg1-foil-%dx%d" % (nx, ny), xn, yn, Re=PAPER_RE, dt=2e-3, body=Body(),
                  steps=steps, perturb=perturb, **kw)


def cfg2(nx=512, ny=384, steps=2000, **kw) -> Config:
    """BJ configs[1]: stationary circular cylinder Re=100, 512x384, h=1/16.
    omega_p = 1.9: with the S:327 default 1.5 the Poisson solve cannot reach
    tol 1e-8 within 10^4 iterations on this grid and the under-converged
    projection diverges by t ~ 1.4 (measured)."""
    xn = uniform_axis(-8.0, 24.0, nx)
    yn = uniform_axis(-12.0, 12.0, ny)
    body = Body(a=0.5, b=0.5, hbar=0.0, k=1.0)
    kw.setdefault("tol_p", 1e-8)
    kw.setdefault("omega_p", 1.9)
    return Config("cfg2-cylinder-%dx%d" % (nx, ny), xn, yn, Re=100.0, dt=0.02, body=body,
                  steps=steps, perturb=0.0, **kw)


# Production mesh levels of the paper's input-scaling study (Table 2
# P:175-186): M1/M2/M3 = 6/12/18 lakh cells.  The paper gives the domain
# and Delta x = Delta y = 0.004 but not the uniform patch or stretch ratio
# (S:80-81 open question): reading R28 -- uniform patch x in [-1, 2] (chord plus
# near wake), y in [-0.75, 0.75] (plunge envelope +-(h + b) plus a 0.5c margin),
# geometric ratio 1.05 outside, h_min chosen per level so that nx*ny hits
# the level's cell count within 1 %.  M1 comes out at h_min ~ 0.004.
MESH_LEVEL_CELLS = {1: 600_000, 2: 1_200_000, 3: 1_800_000}
PAPER_UNIFORM_PATCH = (-1.0, 2.0, -0.75, 0.75)


def production_axes(cells: int, ratio: float = 1.05):
    """(xn, yn, h_min) of the stretched paper-domain grid with nx*ny within 1 %
    of `cells`.  h_min = 3/n with n even, so both uniform patches (3 and 1.5
    chords) hold a whole number of cells; the count is monotone in n."""
    x0, x1, y0, y1 = PAPER_DOMAIN
    ux0, ux1, uy0, uy1 = PAPER_UNIFORM_PATCH
    best = None
    for n in range(100, 4000, 2):
        h = (ux1 - ux0) / n
        xn = stretched_axis(x0, x1, ux0, ux1, h, ratio)
        yn = stretched_axis(y0, y1, uy0, uy1, h, ratio)
        cnt = (len(xn) - 1) * (len(yn) - 1)
        if best is None or abs(cnt - cells) < abs(best[3] - cells):
            best = (xn, yn, h, cnt)
        if cnt > cells:
            break
    if abs(best[3] - cells) > 0.01 * cells:
        raise ValueError("production_axes: no grid within 1 %% of %d cells" % cells)
    return best[0], best[1], best[2]


def cfg3(level=1, steps=1000, **kw) -> Config:
    """BJ configs[2]: plunging foil, Re = 500, k = 2 pi, h = 0.16 on the
    paper's stretched production mesh M1/M2/M3 (reading R28), dt = 1e-4
    (P:59), impulsive start; timing over the first 1000 steps (Table 2)."""
    xn, yn, h = production_axes(MESH_LEVEL_CELLS[level])
    c = Config("cfg3-foil-M%d-%dx%d" % (level, len(xn) - 1, len(yn) - 1), xn, yn, Re=PAPER_RE,
               dt=kw.pop("dt", PAPER_DT), body=Body(), steps=steps, **kw)
    c.extra["h_min"] = h
    c.extra["level"] = level
    return c


def cfg4(n=8192, steps=3, **kw) -> Config:
    """BJ configs[3]: N x N uniform grid on the paper domain, foil as the
    paper's validation case, impulsive start, tol_p = 1e-6."""
    x0, x1, y0, y1 = PAPER_DOMAIN
    xn = uniform_axis(x0, x1, n)
    yn = uniform_axis(y0, y1, n)
    h = min(31.5 / n, 25.0 / n)
    dt = kw.pop("dt", min(PAPER_DT * max(1.0, h / 0.004), 2e-3))
    return Config("cfg4-foil-%dx%d" % (n, n), xn, yn, Re=PAPER_RE, dt=dt, body=Body(),
                  steps=steps, **kw)


def cfg5(n=16384, steps=5, **kw) -> Config:
    """BJ configs[4]: 16384^2 on the paper domain, maxit_p capped at 500."""
    kw.setdefault("maxit_p", 500)
    c = cfg4(n=n, steps=steps, **kw)
    c.name = "cfg5-foil-%dx%d" % (n, n)
    return c


def initial_fields(nx: int, ny: int, perturb: float = 0.0, seed: int = SEED):
    """Impulsive start u = 1, v = 0, p = 0 (R11) plus an optional seeded
    perturbation u += perturb*xi, v = perturb*eta, xi, eta ~ U(-1, 1).
    Inlet column u[:, 0] = 1 and wall rows v[0, :] = v[ny, :] = 0 are kept."""
    u = np.ones((ny, nx + 1))
    v = np.zeros((ny + 1, nx))
    p = np.zeros((ny, nx))
    if perturb:
        rng = np.random.default_rng(seed)
        u += perturb * rng.uniform(-1.0, 1.0, size=u.shape)
        v += perturb * rng.uniform(-1.0, 1.0, size=v.shape)
        u[:, 0] = 1.0
        v[0, :] = 0.0
        v[ny, :] = 0.0
    return u, v, p


def random_field(shape, seed=SEED, lo=-1.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, size=shape)
