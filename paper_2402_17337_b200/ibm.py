"""Thin ctypes binding of include/ibm.h (argument marshalling only).

Every step of the hot path runs in the CUDA kernels of libibm_b200.so; this
module only converts Python / numpy / torch arguments to the C ABI.  PyTorch
provides the device workspace, the current CUDA stream and (multi-GPU) the
process group used to broadcast the NCCL unique id.  There is no CPU fallback:
a missing library or CUDA device raises.

Function names mirror the C ABI (ibm_init, ibm_set_body, ibm_step,
ibm_get_fields, ibm_forces, ...); `Solver` bundles them for convenience.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# (IBM_LIB_VARIANT=name loads libibm_b200_<name>.so: kernel tuning experiments only,
# built by scripts/build_variants.py)
LIB_PATH = os.path.join(HERE, "libibm_b200%s.so" % (("_" + os.environ["IBM_LIB_VARIANT"])
                                                    if os.environ.get("IBM_LIB_VARIANT") else ""))

IBM_OK, IBM_WARN_NOCONV, IBM_ERR_CONFIG, IBM_ERR_DIVERGED = 0, 1, 2, 3
IBM_ERR_ARG, IBM_ERR_CUDA, IBM_ERR_NCCL, IBM_ERR_STATE = 4, 5, 6, 7
STATUS_NAMES = {0: "OK", 1: "WARN_NOCONV", 2: "ERR_CONFIG", 3: "ERR_DIVERGED", 4: "ERR_ARG",
                5: "ERR_CUDA", 6: "ERR_NCCL", 7: "ERR_STATE"}
IBM_HOST, IBM_DEVICE = 0, 1
FIELD_BITS = {"u": 0, "v": 1, "p": 2, "phi": 3, "fu": 4, "fv": 5, "q": 6, "tu": 7, "tv": 8, "tp": 9,
              "cu_prev": 10, "cv_prev": 11}
FIELD_FAMILY = {"u": "u", "fu": "u", "tu": "u", "cu_prev": "u", "v": "v", "fv": "v", "tv": "v",
                "cv_prev": "v", "p": "p", "phi": "p", "q": "p", "tp": "p"}
NFIELDS = 12


class IBMError(RuntimeError):
    def __init__(self, func, status, msg=""):
        super().__init__("%s -> %s%s" % (func, STATUS_NAMES.get(status, status), (": " + msg) if msg else ""))
        self.status = status


class ibm_config(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int),
                ("xn", C.POINTER(C.c_double)), ("yn", C.POINTER(C.c_double)),
                ("Re", C.c_double), ("dt", C.c_double),
                ("omega_p", C.c_double), ("tol_p", C.c_double), ("maxit_p", C.c_int),
                ("omega_uv", C.c_double), ("tol_uv", C.c_double), ("maxit_uv", C.c_int),
                ("check_every", C.c_int), ("rank", C.c_int), ("nranks", C.c_int),
                ("nccl_id", C.c_void_p), ("device", C.c_int), ("sor_batch", C.c_int),
                ("loopback", C.c_int), ("sor_fuse", C.c_int)]


class ibm_step_stats(C.Structure):
    _fields_ = [("step", C.c_int), ("t_bar", C.c_double), ("it_uv", C.c_int), ("it_p", C.c_int),
                ("rho_uv", C.c_double), ("rho_p", C.c_double), ("cd", C.c_double), ("cl", C.c_double),
                ("ms", C.c_float * 8), ("status", C.c_int), ("launches", C.c_int)]


EXPORTS = ["ibm_workspace_size", "ibm_nccl_unique_id", "ibm_init", "ibm_set_body", "ibm_clear_body",
           "ibm_set_fields", "ibm_set_step", "ibm_step", "ibm_get_fields", "ibm_forces",
           "ibm_poisson_iterate", "ibm_query", "ibm_last_error", "ibm_destroy"]
IBM_QUERY_WF_M, IBM_QUERY_WF_L, IBM_QUERY_SLABS, IBM_QUERY_TB_M, IBM_QUERY_PEER_HALO = 0, 1, 2, 3, 4

_lib = None


def lib():
    """Loads the in-tree CUDA library; raises if it has not been built."""
    global _lib
    if _lib is None:
        # torch first: its bundled libnccl.so.2 must be the one the process loads
        # (libibm_b200.so links NCCL by soname and reuses whichever is loaded)
        import torch  # noqa: F401
        if not os.path.exists(LIB_PATH):
            raise ImportError("libibm_b200.so not built: run __graft_entry__.build() "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i, d = C.c_void_p, C.c_int, C.c_double
        L.ibm_workspace_size.argtypes = [C.POINTER(ibm_config), C.POINTER(C.c_size_t)]
        L.ibm_nccl_unique_id.argtypes = [C.c_char_p]
        L.ibm_init.argtypes = [C.POINTER(ibm_config), vp, C.c_size_t, vp, C.POINTER(vp)]
        L.ibm_set_body.argtypes = [vp, d, d, d, d, d, d]
        L.ibm_clear_body.argtypes = [vp]
        L.ibm_set_fields.argtypes = [vp, C.c_uint, C.POINTER(vp), i]
        L.ibm_set_step.argtypes = [vp, i, i]
        L.ibm_step.argtypes = [vp, i, C.POINTER(ibm_step_stats)]
        L.ibm_get_fields.argtypes = [vp, C.c_uint, C.POINTER(vp), i, C.POINTER(i), C.POINTER(i)]
        L.ibm_forces.argtypes = [vp, C.POINTER(d)]
        L.ibm_poisson_iterate.argtypes = [vp, i, C.POINTER(d)]
        L.ibm_query.argtypes = [vp, i, C.POINTER(i)]
        L.ibm_last_error.argtypes = [vp]
        L.ibm_last_error.restype = C.c_char_p
        L.ibm_destroy.argtypes = [vp]
        for name in EXPORTS:
            if name != "ibm_last_error":
                getattr(L, name).restype = i
        _lib = L
    return _lib


def _check(func, st, ctx=None, ok=(IBM_OK,)):
    if st not in ok:
        msg = lib().ibm_last_error(ctx).decode() if ctx else ""
        raise IBMError(func, st, msg)
    return st


def make_config(xn, yn, Re, dt, omega_p=1.5, tol_p=1e-6, maxit_p=10000, omega_uv=1.2, tol_uv=1e-8,
                maxit_uv=1000, check_every=1, rank=0, nranks=1, nccl_id=None, device=0, sor_batch=0,
                loopback=False, sor_fuse=0):
    xn = np.ascontiguousarray(xn, dtype=np.float64)
    yn = np.ascontiguousarray(yn, dtype=np.float64)
    cfg = ibm_config()
    cfg.nx, cfg.ny = len(xn) - 1, len(yn) - 1
    cfg.xn = xn.ctypes.data_as(C.POINTER(C.c_double))
    cfg.yn = yn.ctypes.data_as(C.POINTER(C.c_double))
    cfg.Re, cfg.dt = Re, dt
    cfg.omega_p, cfg.tol_p, cfg.maxit_p = omega_p, tol_p, maxit_p
    cfg.omega_uv, cfg.tol_uv, cfg.maxit_uv = omega_uv, tol_uv, maxit_uv
    cfg.check_every, cfg.rank, cfg.nranks = check_every, rank, nranks
    idbuf = None
    if nccl_id is not None:
        idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        cfg.nccl_id = C.cast(idbuf, C.c_void_p)
    cfg.device, cfg.sor_batch, cfg.loopback = device, sor_batch, int(bool(loopback))
    cfg.sor_fuse = int(sor_fuse)
    cfg._keep = (xn, yn, idbuf)  # keep host arrays alive for the call
    return cfg


# ---------------------------------------------------------------- C-ABI mirrors
def ibm_workspace_size(cfg: ibm_config) -> int:
    n = C.c_size_t(0)
    _check("ibm_workspace_size", lib().ibm_workspace_size(C.byref(cfg), C.byref(n)))
    return n.value


def ibm_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check("ibm_nccl_unique_id", lib().ibm_nccl_unique_id(buf))
    return buf.raw


def ibm_init(cfg: ibm_config, workspace_ptr: int, nbytes: int, stream_ptr: int) -> int:
    out = C.c_void_p(0)
    _check("ibm_init", lib().ibm_init(C.byref(cfg), C.c_void_p(workspace_ptr), nbytes,
                                      C.c_void_p(stream_ptr), C.byref(out)))
    return out.value


def ibm_set_body(ctx, a, b, x0, y0, h_bar, k):
    return _check("ibm_set_body", lib().ibm_set_body(ctx, a, b, x0, y0, h_bar, k), ctx)


def ibm_clear_body(ctx):
    return _check("ibm_clear_body", lib().ibm_clear_body(ctx), ctx)


def _ptr_array(ptrs):
    arr = (C.c_void_p * NFIELDS)()
    for bit, p in ptrs.items():
        arr[bit] = p
    return arr


def ibm_set_fields(ctx, mask, ptrs, where):
    return _check("ibm_set_fields", lib().ibm_set_fields(ctx, mask, _ptr_array(ptrs), where), ctx)


def ibm_set_step(ctx, step, have_history):
    return _check("ibm_set_step", lib().ibm_set_step(ctx, step, have_history), ctx)


def ibm_step(ctx, nsteps):
    stats = (ibm_step_stats * max(nsteps, 1))()
    st = lib().ibm_step(ctx, nsteps, stats)
    _check("ibm_step", st, ctx, ok=(IBM_OK, IBM_WARN_NOCONV, IBM_ERR_DIVERGED))
    return st, stats


def ibm_get_fields(ctx, mask, ptrs, where):
    j0, j1 = C.c_int(0), C.c_int(0)
    _check("ibm_get_fields", lib().ibm_get_fields(ctx, mask, _ptr_array(ptrs), where, C.byref(j0), C.byref(j1)), ctx)
    return j0.value, j1.value


def ibm_forces(ctx):
    out = (C.c_double * 3)()
    _check("ibm_forces", lib().ibm_forces(ctx, out), ctx)
    return tuple(out)


def ibm_poisson_iterate(ctx, iters):
    rho = C.c_double(0.0)
    st = lib().ibm_poisson_iterate(ctx, iters, C.byref(rho))
    _check("ibm_poisson_iterate", st, ctx, ok=(IBM_OK, IBM_ERR_DIVERGED))
    return st, rho.value


def ibm_query(ctx, key) -> int:
    out = C.c_int(0)
    _check("ibm_query", lib().ibm_query(ctx, key, C.byref(out)), ctx)
    return out.value


def ibm_last_error(ctx) -> str:
    return lib().ibm_last_error(ctx).decode()


def ibm_destroy(ctx):
    return _check("ibm_destroy", lib().ibm_destroy(ctx))


STATS_COLUMNS = ("t", "it_uv", "it_p", "rho_uv", "rho_p", "cd", "cl", "status")


def stats_array(stats, n):
    """(n, 8) array with the oracle's column order t, it_uv, it_p, rho_uv, rho_p, cd, cl, status."""
    out = np.zeros((n, 8))
    for k in range(n):
        s = stats[k]
        out[k] = (s.t_bar, s.it_uv, s.it_p, s.rho_uv, s.rho_p, s.cd, s.cl, s.status)
    return out


class Solver:
    """One solver instance on one CUDA device (one slab when nranks > 1)."""

    def __init__(self, xn, yn, Re, dt, device=0, stream=None, **kw):
        import torch  # plumbing only: device memory + stream

        if not torch.cuda.is_available():
            raise RuntimeError("paper_2402_17337_b200 needs a CUDA device (no CPU fallback)")
        self.torch = torch
        self.device = torch.device("cuda", device)
        self.cfg = make_config(xn, yn, Re, dt, device=device, **kw)
        self.nx, self.ny = self.cfg.nx, self.cfg.ny
        self.nranks, self.rank, self.loopback = self.cfg.nranks, self.cfg.rank, bool(self.cfg.loopback)
        nbytes = ibm_workspace_size(self.cfg)
        with torch.cuda.device(self.device):
            self.ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
            self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        base = self.ws.data_ptr()
        aligned = (base + 255) // 256 * 256
        self.ctx = ibm_init(self.cfg, aligned, nbytes, self.stream.cuda_stream)
        self.rows = self._rows()

    def _rows(self):
        if self.loopback or self.nranks == 1:
            return 0, self.ny
        from .dist import slab_rows
        return slab_rows(self.ny, self.nranks, self.rank)

    def shape(self, name):
        j0, j1 = self.rows
        fam = FIELD_FAMILY[name]
        last = (j1 == self.ny)
        if fam == "u":
            return (j1 - j0, self.nx + 1)
        if fam == "v":
            return (j1 - j0 + (1 if last else 0), self.nx)
        return (j1 - j0, self.nx)

    def close(self):
        if getattr(self, "ctx", None):
            ibm_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_body(self, a, b, x0, y0, h_bar, k):
        ibm_set_body(self.ctx, a, b, x0, y0, h_bar, k)

    def clear_body(self):
        ibm_clear_body(self.ctx)

    def set_fields(self, u=None, v=None, p=None, phi=None, restart=True):
        """Host (numpy) or device (torch) arrays of this rank's rows.  With
        restart=True (default, like the oracle) phi is zeroed unless given and
        the step counter and AB2 history are reset (ibm_set_step(0, 0))."""
        keep, ptrs, mask, where = [], {}, 0, None
        if restart and phi is None:
            on_dev = any(hasattr(a, "data_ptr") for a in (u, v, p))
            phi = (self.torch.zeros(self.shape("phi"), dtype=self.torch.float64, device=self.device)
                   if on_dev else np.zeros(self.shape("phi")))
        for name, arr in (("u", u), ("v", v), ("p", p), ("phi", phi)):
            if arr is None:
                continue
            if hasattr(arr, "data_ptr"):
                arr = arr.contiguous().to(dtype=self.torch.float64)
                w = IBM_DEVICE
                ptr = arr.data_ptr()
            else:
                arr = np.ascontiguousarray(arr, dtype=np.float64)
                w = IBM_HOST
                ptr = arr.ctypes.data
            if tuple(arr.shape) != self.shape(name):
                raise ValueError("%s: shape %s, expected %s" % (name, tuple(arr.shape), self.shape(name)))
            if where is None:
                where = w
            elif where != w:
                raise ValueError("set_fields: mix of host and device arrays")
            keep.append(arr)
            ptrs[FIELD_BITS[name]] = ptr
            mask |= 1 << FIELD_BITS[name]
        if mask:
            ibm_set_fields(self.ctx, mask, ptrs, where)
        if restart:
            ibm_set_step(self.ctx, 0, 0)

    def set_step(self, step, have_history):
        ibm_set_step(self.ctx, step, int(have_history))

    def step(self, nsteps=1):
        """Returns (status, stats[nsteps, 8]) like oracle.Oracle.step, plus raw records in .last_stats."""
        st, stats = ibm_step(self.ctx, nsteps)
        self.last_stats = stats
        return st, stats_array(stats, nsteps)

    def get(self, name, device=False):
        shape = self.shape(name)
        tag = name in ("tu", "tv", "tp")
        if device:
            out = self.torch.empty(shape, dtype=self.torch.uint8 if tag else self.torch.float64, device=self.device)
            ptr, where = out.data_ptr(), IBM_DEVICE
        else:
            out = np.zeros(shape, dtype=np.uint8 if tag else np.float64)
            ptr, where = out.ctypes.data, IBM_HOST
        ibm_get_fields(self.ctx, 1 << FIELD_BITS[name], {FIELD_BITS[name]: ptr}, where)
        return out

    def get_many(self, names):
        return {n: self.get(n) for n in names}

    def forces(self):
        return ibm_forces(self.ctx)

    def poisson_iterate(self, iters):
        return ibm_poisson_iterate(self.ctx, iters)

    def query(self, key):
        """Launch configuration chosen by the library: "wf_m" (Poisson iterations per
        HBM pass), "wf_L" (fused-pass segment length, 0 before tuning), "slabs"."""
        return ibm_query(self.ctx, {"wf_m": IBM_QUERY_WF_M, "wf_L": IBM_QUERY_WF_L,
                                    "slabs": IBM_QUERY_SLABS, "tb_m": IBM_QUERY_TB_M,
                                    "peer_halo": IBM_QUERY_PEER_HALO}[key])
