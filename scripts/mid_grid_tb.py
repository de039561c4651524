"""Poisson iteration time on mid-size grids -- the resident temporally blocked
persistent solve (sor_tb.cu, IBM_SOR_TB = m iterations per grid barrier) against
the paths used before it (IBM_SOR_TB=0: launched one-iteration passes for
poisson_iterate, cooperative loop inside a step).  Fixed iteration counts
(tolerance ignored) on the state after one full step, CUDA events on the solver
stream.  Also checks that every variant produces bit-identical phi.
Usage: python scripts/mid_grid_tb.py [out.json]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import ibm_inputs as I
import paper_2402_17337_b200 as P


def t_iter(cfg, tb, iters=600):
    os.environ["IBM_SOR_TB"] = str(tb)
    g = P.Solver(cfg.xn, cfg.yn, **cfg.solver_kwargs())
    used = g.query("tb_m")
    g.set_body(*cfg.body_args())
    g.set_fields(*I.initial_fields(cfg.nx, cfg.ny, 0.01))
    st, stats = g.step(1)
    g.poisson_iterate(30)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(g.stream)
    g.poisson_iterate(iters)
    e1.record(g.stream)
    torch.cuda.synchronize()
    phi = g.get("phi")
    # one full step with a converging Poisson solve (tol) for the step-level time
    st2, s2 = g.step(1)
    g.close()
    return e0.elapsed_time(e1) / iters * 1e3, used, phi, float(s2[0, 2]), g.last_stats[0].ms[3] * 1e3 / max(s2[0, 2], 1)


cases = [("cfg2-cylinder-512x384", I.cfg2(maxit_p=3000)), ("cfg1-128x96", I.cfg1(maxit_p=3000)),
         ("M1-997x602", I.cfg3(1, maxit_p=3000)), ("M2-1443x832", I.cfg3(2, maxit_p=3000)),
         ("M3-1785x1008", I.cfg3(3, maxit_p=3000)),
         ("cfg4-1024", I.cfg4(1024, maxit_p=3000)), ("cfg4-2048", I.cfg4(2048, maxit_p=3000))]
if os.environ.get("MID_TB_CASES"):
    cases = cases[:int(os.environ["MID_TB_CASES"])]
out = []
for name, cfg in cases:
    r = {"case": name, "cells": cfg.nx * cfg.ny}
    ref = None
    for tb in (0, 2, 3, 4):
        us, used, phi, itp, step_us = t_iter(cfg, tb)
        r["tb%d" % tb] = {"us_per_it": us, "tb_m_used": used, "step_it_p": itp, "step_us_per_it": step_us}
        if ref is None:
            ref = phi
        else:
            r["tb%d" % tb]["phi_bitwise_equal"] = bool(np.array_equal(ref, phi))
    print(json.dumps(r), flush=True)
    out.append(r)
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
