"""BJ configs[2] / SURVEY §8(f) f1: the plunging foil (Re = 500, k = 2 pi,
h = 0.16) on the paper's stretched production meshes M1/M2/M3
(6/12/18 lakh cells; reading R28 in DESIGN.md), dt = 1e-4,
impulsive start, run on the GPU through the C ABI.

Reports, per mesh level, the device time of the first `--steps` time steps
(the paper times the first 1000, Table 2), ms per step, the Poisson
and velocity SOR iteration counts, and the c_d / c_l history (CSV).  The
paper's OpenACC times on one V100 (SOL2) are printed beside them as
context -- another machine, another code, not a target.

Usage: python scripts/production_foil.py [--levels 1 2 3] [--steps 1000]
                                         [--out profiles/r01_production]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import ibm_inputs as I  # noqa: E402

# Table 2: first 1000 steps, seconds
PAPER_SOL2_1000 = {1: 244.4, 2: 378.0, 3: 368.3}   # OpenACC, 1 x V100 32 GB
PAPER_SOL0_1000 = {1: 13140.0, 2: 24663.0, 3: 39994.0}  # serial CPU


def run_level(level, steps, chunk=100, **kw):
    import torch
    import paper_2402_17337_b200 as P

    cfg = I.cfg3(level=level, steps=steps, **kw)
    g = P.Solver(cfg.xn, cfg.yn, **cfg.solver_kwargs())
    g.set_body(*cfg.body_args())
    g.set_fields(*I.initial_fields(cfg.nx, cfg.ny))
    rows, dev_ms, status = [], 0.0, 0
    t0 = time.time()
    for s in range(0, steps, chunk):
        n = min(chunk, steps - s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(g.stream)
        st, stats = g.step(n)
        e1.record(g.stream)
        torch.cuda.synchronize()
        dev_ms += e0.elapsed_time(e1)
        rows.append(stats)
        status = max(status, st)
        if st == 3:
            break
    wall = time.time() - t0
    S = np.concatenate(rows)
    done = len(S)
    g.close()
    return cfg, S, {
        "level": level, "mesh": "M%d" % level, "nx": cfg.nx, "ny": cfg.ny, "cells": cfg.nx * cfg.ny,
        "h_min": cfg.extra["h_min"], "steps_done": done, "status": int(status),
        "device_s": dev_ms / 1e3, "wall_s": wall, "ms_per_step": dev_ms / max(done, 1),
        "it_p_mean": float(S[:, 2].mean()), "it_p_max": float(S[:, 2].max()),
        "it_uv_mean": float(S[:, 1].mean()),
        "cell_steps_per_s": cfg.nx * cfg.ny * done / (dev_ms / 1e3),
        "poisson_updates_per_s": float(S[:, 2].sum()) * cfg.nx * cfg.ny / (dev_ms / 1e3),
        "cd_last": float(S[-1, 5]), "cl_last": float(S[-1, 6]),
        "paper_sol2_s_per_1000_steps_v100": PAPER_SOL2_1000[level],
        "paper_sol0_s_per_1000_steps_cpu": PAPER_SOL0_1000[level],
        "this_s_per_1000_steps": dev_ms / max(done, 1),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--levels", type=int, nargs="+", default=[1, 2, 3])
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--omega-p", type=float, default=None)
    ap.add_argument("--maxit-p", type=int, default=None)
    ap.add_argument("--chunk", type=int, default=100)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_production"))
    args = ap.parse_args()
    res = {"workload": "cfg3 plunging foil Re=500 k=2pi h=0.16 dt=1e-4, stretched paper-domain meshes (R28)",
           "context": "paper SOL2 = OpenACC on one V100 (Table 2, P:183); not a target", "levels": []}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    for lv in args.levels:
        kw = {} if args.omega_p is None else {"omega_p": args.omega_p}
        if args.maxit_p is not None:
            kw["maxit_p"] = args.maxit_p
        cfg, S, r = run_level(lv, args.steps, chunk=args.chunk, **kw)
        r["omega_p"] = cfg.omega_p
        r["maxit_p"] = cfg.maxit_p
        # plunge-cycle statistics (period 2 pi / k): cycle means, amplitude and the
        # rms change of the c_l history from one cycle to the next (SURVEY §8(c) force pins)
        T = 2 * np.pi / cfg.body.k
        per = int(round(T / cfg.dt))
        cyc = []
        for c0 in range(0, len(S) - per + 1, per):
            cl, cd = S[c0:c0 + per, 6], S[c0:c0 + per, 5]
            d = {"cycle": c0 // per + 1, "cl_mean": float(cl.mean()), "cd_mean": float(cd.mean()),
                 "cl_amplitude": float(0.5 * (cl.max() - cl.min()))}
            if c0 >= per:
                prev = S[c0 - per:c0, 6]
                d["cl_rms_change_vs_previous"] = float(np.sqrt(np.mean((cl - prev) ** 2)) / np.sqrt(np.mean(cl ** 2)))
            cyc.append(d)
        r["cycles"] = cyc
        res["levels"].append(r)
        np.savetxt("%s_M%d.csv" % (args.out, lv), np.c_[S[:, 0], S[:, 5], S[:, 6], S[:, 1], S[:, 2]],
                   delimiter=",", header="t_bar,cd,cl,it_uv,it_p", comments="")
        print(json.dumps(r), flush=True)
    json.dump(res, open(args.out + ".json", "w"), indent=1)


if __name__ == "__main__":
    main()
