"""Poisson SOR micro-benchmark (BJ configs[3] (i)): fixed iteration counts
(tolerance ignored) on the state reached after `presteps` full steps,
CUDA events on the solver stream.  Usage: microbench_sor.py N [presteps] [maxit_p] [sor_fuse]
GBs = 24 B x cells per iteration (the unfused pass's traffic); pass_GBs = 24 B x
cells per HBM pass (sor_fuse iterations) -- the fused kernel's own roofline figure."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import ibm_inputs as I
import paper_2402_17337_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
pre = int(sys.argv[2]) if len(sys.argv) > 2 else 1
mp = int(sys.argv[3]) if len(sys.argv) > 3 else 300
fuse = int(sys.argv[4]) if len(sys.argv) > 4 else 0
m = fuse if fuse else 3
cfg = I.cfg4(n=n, maxit_p=mp, maxit_uv=1000)
g = P.Solver(cfg.xn, cfg.yn, sor_fuse=fuse, **cfg.solver_kwargs())
g.set_body(*cfg.body_args())
g.set_fields(*I.initial_fields(cfg.nx, cfg.ny))
st, stats = g.step(pre)
raw = g.last_stats
res = {"n": n, "sor_fuse": m, "presteps": pre, "step_p_ms_per_it": [raw[k].ms[3] / max(raw[k].it_p, 1) for k in range(pre)]}
for iters in (10, 200):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(g.stream)
    t0 = time.perf_counter()
    g.poisson_iterate(iters)
    t1 = time.perf_counter()
    e1.record(g.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    res[iters] = {"ms_per_it": ms / iters, "host_ms_per_it": 1e3 * (t1 - t0) / iters,
                  "GBs": 24 * cfg.nx * cfg.ny / (ms / iters / 1e3) / 1e9,
                  "pass_GBs": 24 * cfg.nx * cfg.ny / (ms / iters * m / 1e3) / 1e9}
# SURVEY §8(d) cfg4(i) protocol: tolerance off, 20 warm-up iterations, then 5 repetitions of 200
# iterations, median (MICROBENCH_REPS=0 skips it)
reps = int(os.environ.get("MICROBENCH_REPS", "5"))
if reps:
    g.poisson_iterate(20)
    times = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(g.stream)
        g.poisson_iterate(200)
        e1.record(g.stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 200)
    med = float(np.median(times))
    res["protocol_8d"] = {"ms_per_it_median": med, "ms_per_it_all": times, "ms_per_pass": med * m,
                          "pass_GBs": 24 * cfg.nx * cfg.ny / (med * m / 1e3) / 1e9}
print(json.dumps(res))
