"""Poisson iteration time on mid-size grids (production meshes M1-M3, cfg4 1024-4096):
fused pass (sor_fuse m, segment length via IBM_WF_ROWS) vs the automatic choice.
Usage: python scripts/mid_grid_sor.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ibm_inputs as I
import paper_2402_17337_b200 as P


def t_iter(cfg, fuse, rows, iters=300):
    if rows:
        os.environ["IBM_WF_ROWS"] = str(rows)
    else:
        os.environ.pop("IBM_WF_ROWS", None)
    g = P.Solver(cfg.xn, cfg.yn, sor_fuse=fuse, **cfg.solver_kwargs())
    g.set_body(*cfg.body_args())
    g.set_fields(*I.initial_fields(cfg.nx, cfg.ny))
    g.step(1)
    g.poisson_iterate(30)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(g.stream)
    g.poisson_iterate(iters)
    e1.record(g.stream)
    torch.cuda.synchronize()
    g.close()
    return e0.elapsed_time(e1) / iters * 1e3  # us


cases = [("M1", I.cfg3(1, maxit_p=50)), ("M2", I.cfg3(2, maxit_p=50)), ("M3", I.cfg3(3, maxit_p=50)),
         ("1024", I.cfg4(1024, maxit_p=50)), ("2048", I.cfg4(2048, maxit_p=50)), ("4096", I.cfg4(4096, maxit_p=50))]
for name, cfg in cases:
    r = {"case": name, "cells": cfg.nx * cfg.ny, "auto_us": t_iter(cfg, 0, 0)}
    for rows in (16, 32, 64):
        r["m3_L%d_us" % rows] = t_iter(cfg, 3, rows)
    r["m1_us"] = t_iter(cfg, 1, 0)
    print(json.dumps(r), flush=True)
