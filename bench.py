#!/usr/bin/env python
"""Benchmark of the B200 IBM hot path (one JSON line on rank 0).

Workload (BASELINE.json configs[3], input-scaling sweep, largest size that is
HBM-bound): plunging elliptic foil (t/c 0.12, Re 500, k 2 pi, h 0.16; P:33,
P:150) on an N x N uniform staggered grid over the paper's domain
[-7.5,24]x[-12.5,12.5], N = 8192 (dx ~ 0.0038 ~ the paper's 0.004), dt
1e-4, impulsive start, SOR omega 1.5/1.2, tol 1e-6/1e-8, maxit 10000/1000
(S:327).  A "step" is one time step of the whole hot path (classify,
predictor + forcing, velocity SOR, Poisson rhs, Poisson SOR to tol or maxit,
projection, forces) -- ibm_step(ctx, 1).

metric: Poisson+stencil grid-point updates/s
  = sum over steps of [it_p*Np + it_uv*(Nu+Nv) + 2*(Nu+Nv) + 2*Np] / time
  (SOR node updates + one node update per stencil pass: predictor, Poisson
  rhs, correction) -- DESIGN.md §7.  ms_per_step is reported beside it.

Multi-GPU (torchrun, N>1): the same grid split into N slabs along y (strong
scaling), NCCL halos + residual all-reduce; time = max over ranks.
--impl reference: the CPU oracle (oracle/) timed as it stands on the host
cores, on a bounded sample of the same workload (there is no reference
implementation to install: the paper ships no code).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import ibm_inputs as I  # noqa: E402

METRIC = "Poisson+stencil grid-point updates/s"
UNIT = "grid-point updates/s"
BYTES_PER_POISSON_UPDATE = 24  # phi read + b read + phi write per cell per HBM pass, fp64


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=8192, help="grid N x N on the paper domain")
    ap.add_argument("--maxit-p", type=int, default=10000)
    ap.add_argument("--maxit-uv", type=int, default=1000)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--cpu-sample-n", type=int, default=0, help="oracle sample grid (0 = auto)")
    ap.add_argument("--sor-fuse", type=int, default=0,
                    help="Poisson iterations fused per HBM pass (0 = library default 3)")
    ap.add_argument("--sor-batch", type=int, default=0,
                    help="> 0: host-launched SOR iterations in batches of this size instead of the graph WHILE loop")
    return ap.parse_args()


def node_counts(nx, ny):
    return (nx + 1) * ny, nx * (ny + 1), nx * ny


def updates_for(stats, nx, ny):
    Nu, Nv, Np = node_counts(nx, ny)
    it_uv, it_p = stats[:, 1].sum(), stats[:, 2].sum()
    n = stats.shape[0]
    return float(it_p * Np + it_uv * (Nu + Nv) + n * (2 * (Nu + Nv) + 2 * Np))


# ---------------------------------------------------------------- clocks sampler
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index, enabled=True):
        self.index, self.enabled, self.rows, self.proc = index, enabled, [], None

    def start(self):
        if not self.enabled:
            return
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.th.join(timeout=2)
        rows = [r for r in self.rows if len(r) >= 8]
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        pw = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[4 + k].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "power_w_median": float(np.median(pw)) if pw else None}


# ---------------------------------------------------------------- CPU oracle sample
def mem_available_gb():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable"):
                return int(line.split()[1]) / 1e6
    except Exception:
        pass
    return 8.0


def oracle_sample_n(n_req, requested):
    if requested:
        return requested
    # oracle: ~30 fp64 full arrays + SOR coefficient temporaries ~ 330 B/cell
    avail = mem_available_gb() * 1e9 * 0.4
    n = n_req
    while n > 512 and 330.0 * n * n > avail:
        n //= 2
    return n


ORACLE_SAMPLE_MAXIT_P, ORACLE_SAMPLE_MAXIT_UV = 20, 5


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_oracle_steps(n, steps, maxit_p, maxit_uv, omp=False):
    """One oracle instance (oracle_seq, or oracle_omp on every host core) on the
    N x N workload of the bench, each step with the SOR solves capped at
    maxit_p / maxit_uv iterations (a bounded sample).  Returns
    (updates/s, seconds, stats, per-step list, Poisson updates/s)."""
    if omp:
        os.environ["OMP_NUM_THREADS"] = str(host_cores())  # read when the OpenMP runtime starts
    from oracle import oracle as O
    O.build()
    cfg = I.cfg4(n=n, maxit_p=maxit_p, maxit_uv=maxit_uv)
    o = O.Oracle(cfg.xn, cfg.yn, omp=omp, **cfg.solver_kwargs())
    o.set_body(*cfg.body_args())
    o.set_fields(*I.initial_fields(cfg.nx, cfg.ny))
    o.timers()
    per = []
    psec = 0.0
    for _ in range(steps):
        t0 = time.perf_counter()
        st, stats = o.step(1)
        per.append((time.perf_counter() - t0, stats))
        psec += o.timers()[4]  # region "P solver" (Table 1 layout)
    secs = sum(p[0] for p in per)
    allstats = np.concatenate([p[1] for p in per])
    p_rate = float(allstats[:, 2].sum()) * cfg.nx * cfg.ny / max(psec, 1e-12)
    del o
    return updates_for(allstats, cfg.nx, cfg.ny) / secs, secs, allstats, per, p_rate


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(args):
    """The oracle as it stands on this host: oracle_omp on every core (the headline
    value) and oracle_seq on one core, each for one time step of the bench's own
    N x N workload with the SOR solves capped at 20 Poisson / 5 velocity
    iterations (the bounded sample; the GPU runs the uncapped solve)."""
    n = oracle_sample_n(args.n, args.cpu_sample_n)
    mp, mu = ORACLE_SAMPLE_MAXIT_P, ORACLE_SAMPLE_MAXIT_UV
    v1, s1, _, _, p1 = run_oracle_steps(n, 1, mp, mu, omp=False)
    cores = host_cores()
    vN, sN, _, _, pN = run_oracle_steps(n, 1, mp, mu, omp=True)
    return {"value": vN, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": "1 time step of the %dx%d foil workload (BJ configs[3]) with the SOR solves capped at "
                      "%d Poisson + %d velocity iterations; oracle_omp (same C source, -fopenmp, rows of one "
                      "colour split over %d threads, bitwise equal to oracle_seq) %.1f s; %s"
                      % (n, n, mp, mu, cores, sN, cpu_model()),
            "poisson_updates_per_s": pN,
            "seq": {"value": v1, "cores": 1, "seconds": s1, "poisson_updates_per_s": p1}}


# ---------------------------------------------------------------- reference arm = oracle
def run_reference(args, rank, world):
    if rank != 0:
        return
    n = oracle_sample_n(args.n, args.cpu_sample_n)
    mp, mu = ORACLE_SAMPLE_MAXIT_P, ORACLE_SAMPLE_MAXIT_UV
    total = args.warmup + args.steps
    cores = host_cores()
    v, secs, stats, per, p_rate = run_oracle_steps(n, total, mp, mu, omp=True)
    timed = per[args.warmup:]
    tsec = sum(p[0] for p in timed)
    tstats = np.concatenate([p[1] for p in timed])
    cfgd = I.cfg4(n=n)
    value = updates_for(tstats, cfgd.nx, cfgd.ny) / tsec
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tsec / max(args.steps, 1),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "cfg4-foil-%dx%d" % (args.n, args.n), "oracle_sample_n": n,
                       "maxit_p": mp, "maxit_uv": mu},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": "%d oracle_omp time steps of the %dx%d foil workload on %d host cores, SOR "
                                       "capped at %d Poisson + %d velocity iterations per step (%s)"
                                       % (args.steps, n, n, cores, mp, mu, cpu_model()),
                             "poisson_updates_per_s": p_rate},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- B200 arm
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2402_17337_b200 as P
    from paper_2402_17337_b200.dist import bootstrap_nccl_id, max_over_ranks, slab_of

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl_id = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        nccl_id = bootstrap_nccl_id(rank)

    cfg = I.cfg4(n=args.n, maxit_p=args.maxit_p, maxit_uv=args.maxit_uv)
    g = P.Solver(cfg.xn, cfg.yn, device=local, rank=rank, nranks=world, nccl_id=nccl_id, sor_batch=args.sor_batch,
                 sor_fuse=args.sor_fuse, **cfg.solver_kwargs())
    g.set_body(*cfg.body_args())
    j0, j1 = g.rows
    g.set_fields(*slab_of(*I.initial_fields(cfg.nx, cfg.ny), cfg.ny, world, rank))
    stream = g.stream

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()

    # warm-up
    if args.warmup:
        g.step(args.warmup)
    barrier()
    clocks = Clocks(local, enabled=(rank == 0 and not args.no_clocks))
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    st, stats = g.step(args.steps)
    e1.record(stream)
    barrier()
    clk = clocks.stop()
    t_ms = e0.elapsed_time(e1)
    raw = g.last_stats
    launches = int(sum(raw[k].launches for k in range(args.steps)))
    psor_ms = float(sum(raw[k].ms[3] for k in range(args.steps)))
    uvsor_ms = float(sum(raw[k].ms[1] for k in range(args.steps)))
    t_ms = max_over_ranks(t_ms, dev)
    updates = updates_for(stats, cfg.nx, cfg.ny)
    value = updates / (t_ms / 1e3)

    # roofline of the dominant kernel (the Poisson pass: k_sor_wf fusing m
    # red-black iterations per HBM pass, or k_sor with m = 1 on slabs):
    # algorithmic bytes per launch = 24 B x this rank's p cells (phi in, b in,
    # phi out once per pass); launch duration = CUDA events bracketing the
    # Poisson loop on the launch stream / passes (it_p / m per step)
    Np_local = cfg.nx * (j1 - j0)
    it_p = float(stats[:, 2].sum())
    fuse = g.query("wf_m")  # what the library chose (1 = one-iteration pass on thin slabs / mid grids)
    passes = float(sum(np.ceil(stats[:, 2] / fuse)))
    avg_iter_s = (psor_ms / 1e3) / max(it_p, 1.0)
    avg_launch_s = (psor_ms / 1e3) / max(passes, 1.0)
    achieved = BYTES_PER_POISSON_UPDATE * Np_local / avg_launch_s / 1e9
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peak, peak_src = float(peaks["hbm_gbs"]), "measured"
    except Exception:
        peak, peak_src = 6650.0, "fallback"
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        traffic = prof.get("k_sor_wf_poisson" if fuse > 1 else "k_sor_poisson", {}).get("dram_bytes_per_cell", None)
        if traffic is not None:
            traffic = float(traffic) * Np_local
    except Exception:
        pass

    # end to end through the C ABI with host buffers: per step the state comes
    # from pinned host memory (H2D) and the step's fields go back (D2H)
    e2e = None
    if not args.no_e2e:
        shapes = {n: g.shape(n) for n in ("u", "v", "p")}
        host = {n: torch.empty(shapes[n], dtype=torch.float64, pin_memory=True) for n in shapes}
        for n in host:
            host[n].copy_(g.get(n, device=True))
        import paper_2402_17337_b200.ibm as M
        ptrs = {M.FIELD_BITS[n]: host[n].data_ptr() for n in host}
        mask = sum(1 << M.FIELD_BITS[n] for n in host)
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        estats = []
        for _ in range(args.steps):
            M.ibm_set_fields(g.ctx, mask, ptrs, M.IBM_HOST)
            s2, st2 = g.step(1)
            estats.append(st2)
            M.ibm_get_fields(g.ctx, mask, ptrs, M.IBM_HOST)
        f1.record(stream)
        barrier()
        te = max_over_ranks(f0.elapsed_time(f1), dev)
        nbytes = sum(host[n].numel() * 8 for n in host)
        e2e = {"value": updates_for(np.concatenate(estats), cfg.nx, cfg.ny) / (te / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "ms_per_step": te / args.steps}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg4-foil-%dx%d" % (cfg.nx, cfg.ny), "nx": cfg.nx, "ny": cfg.ny,
                       "domain": list(I.PAPER_DOMAIN), "Re": cfg.Re, "dt": cfg.dt, "omega_p": cfg.omega_p,
                       "tol_p": cfg.tol_p, "maxit_p": cfg.maxit_p, "omega_uv": cfg.omega_uv,
                       "tol_uv": cfg.tol_uv, "maxit_uv": cfg.maxit_uv, "body": "foil a=0.5 b=0.06 h=0.16 k=2pi",
                       "l2": "inputs larger than L2 (%.1f GB workspace, 126 MB L2)" % (g.ws.numel() / 1e9),
                       "parallelism": "slab%d" % world,
                       "note": ("every Poisson solve stops at maxit_p (omega_p %.2f does not reach tol_p at this size): "
                                "ms_per_step is the time of a capped step, a throughput figure, not a converged "
                                "physical time step" % cfg.omega_p) if float(stats[:, 2].min()) >= cfg.maxit_p else
                               "Poisson solves converged"},
            "it_p": stats[:, 2].tolist(), "it_uv": stats[:, 1].tolist(),
            "poisson_ms_per_iteration": 1e3 * avg_iter_s, "poisson_ms_per_pass": 1e3 * avg_launch_s,
            "sor_fuse": fuse, "uv_sor_ms": uvsor_ms / args.steps,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": ("k_sor_wf<%d> (%d red-black Poisson iterations per HBM pass)" % (fuse, fuse)
                                    if fuse > 1 else "k_sor<0> (one red-black Poisson iteration per HBM pass)"),
                         "bytes_per_launch": BYTES_PER_POISSON_UPDATE * Np_local, "peak_source": peak_src,
                         # SURVEY 8(d) "effective algorithmic GB/s": the unfused pass's 24 B per cell per
                         # iteration over the time per iteration (exceeds HBM when iterations are fused)
                         "effective_per_iteration": {
                             "bytes_per_cell": BYTES_PER_POISSON_UPDATE,
                             "GBps": BYTES_PER_POISSON_UPDATE * Np_local / avg_iter_s / 1e9,
                             "frac": BYTES_PER_POISSON_UPDATE * Np_local / avg_iter_s / 1e9 / peak}},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    g.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
