"""BJ configs[3]: input-scaling sweep N x N, N = 256 .. 8192, on one GPU.

For each N (plunging foil on the paper domain, impulsive start, tol_p 1e-6,
maxit_p 10^4): one warm-up step, then `--steps` timed steps (CUDA events) ->
grid-point updates/s (the bench metric), ms per step and Poisson iterations;
plus the Poisson micro-benchmark (200 fixed iterations on the state reached,
tolerance ignored) -> ms per iteration and algorithmic GB/s (24 B/cell) against
the measured HBM peak.  Writes one JSON document.

Usage: python scripts/sweep_sizes.py [--out profiles/r01_sweep.json] [--steps 2]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import ibm_inputs as I  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_sweep.json"))
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--sizes", default="256,512,1024,2048,4096,8192")
    args = ap.parse_args()
    import torch
    import paper_2402_17337_b200 as P
    from bench import updates_for

    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = 6650.0
    rows = []
    for n in [int(x) for x in args.sizes.split(",")]:
        cfg = I.cfg4(n=n)
        g = P.Solver(cfg.xn, cfg.yn, **cfg.solver_kwargs())
        g.set_body(*cfg.body_args())
        g.set_fields(*I.initial_fields(cfg.nx, cfg.ny))
        g.step(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(g.stream)
        st, stats = g.step(args.steps)
        e1.record(g.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        upd = updates_for(stats, cfg.nx, cfg.ny)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(g.stream)
        g.poisson_iterate(200)
        f1.record(g.stream)
        torch.cuda.synchronize()
        it_ms = f0.elapsed_time(f1) / 200
        gbs = 24.0 * cfg.nx * cfg.ny / (it_ms / 1e3) / 1e9
        rows.append({"n": n, "dt": cfg.dt, "updates_per_s": upd / (ms / 1e3), "ms_per_step": ms / args.steps,
                     "it_p": stats[:, 2].tolist(), "it_uv": stats[:, 1].tolist(),
                     "poisson_ms_per_iteration_200": it_ms, "poisson_GBs": gbs, "frac_of_peak": gbs / peak,
                     "working_set_MB": g.ws.numel() / 1e6,
                     "poisson_path": ("k_sor_wf<%d> fused pass" % g.query("wf_m")) if g.query("wf_m") > 1 else
                     ("k_sor_tb<%d> resident solve" % g.query("tb_m")) if g.query("tb_m") else "k_sor one-iteration pass"})
        print(json.dumps(rows[-1]), flush=True)
        g.close()
        del g
        torch.cuda.empty_cache()
    doc = {"what": "BJ configs[3] input-scaling sweep, 1 B200; updates/s = bench metric; GB/s = 24 B x cells / "
                   "Poisson iteration (200 back-to-back launches, CUDA events)", "peak_GBs": peak, "rows": rows}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(doc, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
