"""ctypes wrapper for the CPU fp64 oracle (oracle/ibm_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg.  The product package
(paper_2402_17337_b200) never imports this module, and this module never
imports the product package.  Arrays are numpy, global row-major:
u [ny][nx+1], v [ny+1][nx], p/phi/q [ny][nx].
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "ibm_oracle.c")
LIB = os.path.join(HERE, "libibm_oracle.so")          # oracle_seq: one thread (the checker)
LIB_OMP = os.path.join(HERE, "libibm_oracle_omp.so")  # oracle_omp: same source, -fopenmp (host baseline)

# plain C, no FMA contraction, no fast-math (DESIGN.md §3 R13)
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def _build_one(path, extra):
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(SRC):
        tmp = path + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", *CFLAGS, *extra, "-o", tmp, SRC, "-lm"])
        os.replace(tmp, path)
    return path


def build(force: bool = False) -> str:
    """Builds both oracle libraries (seq and OpenMP); returns the seq one."""
    if force:
        for p in (LIB, LIB_OMP):
            if os.path.exists(p):
                os.remove(p)
    _build_one(LIB_OMP, ["-fopenmp"])
    return _build_one(LIB, [])


_libs = {}


def lib(omp: bool = False):
    """ctypes handle of oracle_seq (default) or oracle_omp (threads: OMP_NUM_THREADS)."""
    if omp not in _libs:
        build()
        L = C.CDLL(LIB_OMP if omp else LIB)
        dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
        bp = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
        d, i, vp = C.c_double, C.c_int, C.c_void_p
        L.orc_plunge.argtypes = [d, d, d, dp]
        L.orc_inside.argtypes = [d, d, d, d, d, d]
        L.orc_inside.restype = i
        L.orc_intercept.argtypes = [i, i, d, d, d, d, d, d]
        L.orc_intercept.restype = d
        L.orc_target_dir.argtypes = [d, d, d, d]
        L.orc_target_dir.restype = d
        L.orc_create.argtypes = [i, i, dp, dp, d, d, d, d, i, d, d, i, i]
        L.orc_create.restype = vp
        L.orc_destroy.argtypes = [vp]
        L.orc_set_body.argtypes = [vp, d, d, d, d, d, d]
        L.orc_set_body.restype = i
        L.orc_clear_body.argtypes = [vp]
        L.orc_clear_body.restype = i
        L.orc_set_fields.argtypes = [vp, vp, vp, vp]
        L.orc_set_fields.restype = i
        L.orc_step.argtypes = [vp, i, dp]
        L.orc_step.restype = i
        L.orc_get.argtypes = [vp, i, dp]
        L.orc_get.restype = i
        L.orc_get_tags.argtypes = [vp, i, bp]
        L.orc_get_tags.restype = i
        L.orc_forces.argtypes = [vp, dp]
        L.orc_timers.argtypes = [vp, dp]
        L.orc_classify_at.argtypes = [vp, d]
        L.orc_convection.argtypes = [vp, dp, dp, dp, dp]
        L.orc_laplacian.argtypes = [vp, i, dp, dp]
        L.orc_poisson.argtypes = [vp, dp, dp, C.POINTER(d), C.POINTER(i)]
        L.orc_poisson.restype = i
        L.orc_forcing_target.argtypes = [vp, i, dp, i, i]
        L.orc_forcing_target.restype = d
        L.orc_sor_generic.argtypes = [i, i, dp, dp, dp, dp, dp, dp, bp, dp, d, d, i, i,
                                      C.POINTER(d), C.POINTER(i)]
        L.orc_sor_generic.restype = i
        L.orc_set_sor_form.argtypes = [i]
        _libs[omp] = L
    return _libs[omp]


FIELDS = {"u": 0, "v": 1, "p": 2, "phi": 3, "fu": 4, "fv": 5, "q": 6, "cu_prev": 7,
          "cv_prev": 8, "us": 9, "vs": 10, "bp": 11, "rhs_u": 12, "rhs_v": 13}
TAGS = {"tu": 0, "tv": 1, "tp": 2, "act": 3, "open_u": 4, "open_v": 5}
STATUS = {0: "OK", 1: "WARN_NOCONV", 2: "ERR_CONFIG", 3: "ERR_DIVERGED"}


def plunge(t, hbar, k):
    out = np.zeros(2)
    lib().orc_plunge(t, hbar, k, out)
    return out[0], out[1]


def inside(x, y, a, b, xb, yb):
    return bool(lib().orc_inside(x, y, a, b, xb, yb))


def intercept(axis, direction, xF, yF, a, b, xb, yb):
    return lib().orc_intercept(axis, direction, xF, yF, a, b, xb, yb)


def target_dir(uB, uN, dF, dN):
    return lib().orc_target_dir(uB, uN, dF, dN)


def set_sor_form(plain: bool) -> None:
    """Selects the SOR node-update form for the whole process: False = the
    arithmetic contract R13 (default), True = the plain IEEE form (pin only)."""
    lib().orc_set_sor_form(1 if plain else 0)


def sor_generic(aP, aE, aW, aN, aS, b, upd, x0, omega, tol, maxit, check_every=1):
    nj, ni = aP.shape
    x = np.ascontiguousarray(x0, dtype=np.float64).copy()
    rho, st = C.c_double(0.0), C.c_int(0)
    f = lambda a: np.ascontiguousarray(a, dtype=np.float64)
    it = lib().orc_sor_generic(ni, nj, f(aP), f(aE), f(aW), f(aN), f(aS), f(b),
                               np.ascontiguousarray(upd, dtype=np.uint8), x, omega, tol, maxit,
                               check_every, C.byref(rho), C.byref(st))
    return x, it, rho.value, st.value


class Oracle:
    """One oracle solver instance (mirrors the C-ABI calls of include/ibm.h)."""

    def __init__(self, xn, yn, Re, dt, omega_p=1.5, tol_p=1e-6, maxit_p=10000,
                 omega_uv=1.2, tol_uv=1e-8, maxit_uv=1000, check_every=1, omp=False):
        self.xn = np.ascontiguousarray(xn, dtype=np.float64)
        self.yn = np.ascontiguousarray(yn, dtype=np.float64)
        self.nx, self.ny = len(self.xn) - 1, len(self.yn) - 1
        self._L = lib(omp)
        self._c = self._L.orc_create(self.nx, self.ny, self.xn, self.yn, Re, dt, omega_p, tol_p,
                                   maxit_p, omega_uv, tol_uv, maxit_uv, check_every)
        if not self._c:
            raise ValueError("oracle: invalid configuration")

    def __del__(self):
        c = getattr(self, "_c", None)
        if c:
            self._L.orc_destroy(c)
            self._c = None

    def shape(self, name):
        nx, ny = self.nx, self.ny
        fam = {"u": "u", "fu": "u", "cu_prev": "u", "us": "u", "rhs_u": "u", "tu": "u", "open_u": "u",
               "v": "v", "fv": "v", "cv_prev": "v", "vs": "v", "rhs_v": "v", "tv": "v", "open_v": "v"}
        f = fam.get(name, "p")
        return {"u": (ny, nx + 1), "v": (ny + 1, nx), "p": (ny, nx)}[f]

    def set_body(self, a, b, x0, y0, hbar, k):
        st = self._L.orc_set_body(self._c, a, b, x0, y0, hbar, k)
        if st:
            raise ValueError("oracle: invalid body")

    def clear_body(self):
        self._L.orc_clear_body(self._c)

    def set_fields(self, u=None, v=None, p=None):
        keep = []

        def ptr(a, name):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=np.float64)
            assert a.shape == self.shape(name), (name, a.shape)
            keep.append(a)
            return a.ctypes.data

        self._L.orc_set_fields(self._c, ptr(u, "u"), ptr(v, "v"), ptr(p, "p"))

    def step(self, nsteps=1):
        """Returns (status, stats[nsteps, 8]) with columns
        t, it_uv, it_p, rho_uv, rho_p, cd, cl, status."""
        stats = np.zeros((max(nsteps, 1), 8))
        st = self._L.orc_step(self._c, nsteps, stats)
        return st, stats[:nsteps]

    def get(self, name):
        if name in TAGS:
            out = np.zeros(self.shape(name), dtype=np.uint8)
            self._L.orc_get_tags(self._c, TAGS[name], out)
            return out
        out = np.zeros(self.shape(name))
        self._L.orc_get(self._c, FIELDS[name], out)
        return out

    def timers(self):
        """Region wall times (s) since the last call: flagging, predictor+forcing, U-V SOR,
        Poisson rhs, P SOR, correction, forces (Table 1 layout)."""
        out = np.zeros(7)
        self._L.orc_timers(self._c, out)
        return out

    def forces(self):
        out = np.zeros(3)
        self._L.orc_forces(self._c, out)
        return tuple(out)

    def classify_at(self, t):
        self._L.orc_classify_at(self._c, t)

    def convection(self, u, v):
        cu = np.zeros(self.shape("u"))
        cv = np.zeros(self.shape("v"))
        self._L.orc_convection(self._c, np.ascontiguousarray(u, dtype=np.float64),
                             np.ascontiguousarray(v, dtype=np.float64), cu, cv)
        return cu, cv

    def laplacian(self, fam, x):
        name = {0: "u", 1: "v", 2: "p"}[fam]
        out = np.zeros(self.shape(name))
        self._L.orc_laplacian(self._c, fam, np.ascontiguousarray(x, dtype=np.float64), out)
        return out

    def poisson(self, rhs, phi0=None):
        phi = np.zeros(self.shape("p")) if phi0 is None else np.ascontiguousarray(phi0, dtype=np.float64).copy()
        rho, st = C.c_double(0.0), C.c_int(0)
        it = self._L.orc_poisson(self._c, np.ascontiguousarray(rhs, dtype=np.float64), phi,
                               C.byref(rho), C.byref(st))
        return phi, it, rho.value, st.value

    def forcing_target(self, fam, x, i, j):
        return self._L.orc_forcing_target(self._c, fam, np.ascontiguousarray(x, dtype=np.float64), i, j)
