"""Validation case of the paper (Fig. Aerodynamic_coeffs) at trend level:
plunging elliptic foil (t/c = 0.12), Re = 500, k = 2 pi, h = 0.16
(k h ~ 1.0), impulsive start, run on the GPU through the C ABI for several
plunge periods T = 2 pi / k = 1.

The paper's force histories are figures, so no value can be
compared; what the physics fixes is checked instead (SURVEY §8(c) pins for the
forces): c_l periodic with the plunge period (cycle-to-cycle change of the
c_l history small once the start-up transient has decayed), mean c_l ~ 0 over
a cycle (the motion is symmetric about y = 0), and c_d periodic with half the
period (drag responds to |plunge velocity|).

Usage: python scripts/validate_foil.py [--grid cfg1|NxM] [--cycles 4] [--out profiles/r01_foil]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import ibm_inputs as I  # noqa: E402


def cycle_stats(t, y, period):
    """Per-cycle mean, amplitude, and the rms change between consecutive cycles
    (resampled on a common phase grid)."""
    n = int(np.floor(t[-1] / period + 1e-9))
    ph = np.linspace(0.0, period, 200, endpoint=False)
    cyc = [np.interp(k * period + ph, t, y) for k in range(n)]
    out = []
    for k, c in enumerate(cyc):
        d = None if k == 0 else float(np.sqrt(np.mean((c - cyc[k - 1]) ** 2)) / max(np.sqrt(np.mean(c ** 2)), 1e-300))
        out.append({"cycle": k + 1, "mean": float(c.mean()), "amp": float(0.5 * (c.max() - c.min())), "rel_change": d})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cycles", type=int, default=4)
    ap.add_argument("--nx", type=int, default=128)
    ap.add_argument("--ny", type=int, default=96)
    ap.add_argument("--dt", type=float, default=2e-3)
    ap.add_argument("--omega-p", type=float, default=None)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_foil"))
    args = ap.parse_args()
    import paper_2402_17337_b200 as P

    cfg = I.cfg1(nx=args.nx, ny=args.ny, perturb=0.0)
    cfg.dt = args.dt
    if args.omega_p is not None:
        cfg.omega_p = args.omega_p
    period = 2.0 * np.pi / cfg.body.k
    steps = int(round(args.cycles * period / cfg.dt))
    g = P.Solver(cfg.xn, cfg.yn, **cfg.solver_kwargs())
    g.set_body(*cfg.body_args())
    g.set_fields(*I.initial_fields(cfg.nx, cfg.ny))
    rows, status, t0 = [], 0, time.time()
    for s in range(0, steps, 250):
        st, stats = g.step(min(250, steps - s))
        rows.append(stats)
        status = max(status, st)
        if st == 3:
            break
    wall = time.time() - t0
    S = np.concatenate(rows)
    t, cd, cl = S[:, 0], S[:, 5], S[:, 6]
    cls, cds = cycle_stats(t, cl, period), cycle_stats(t, cd, period)
    last = slice(int(len(t) * (1 - 1.0 / max(args.cycles, 1))), None)
    res = {"config": cfg.describe(), "period": period, "steps_done": len(t), "status": int(status), "wall_s": wall,
           "cl_cycles": cls, "cd_cycles": cds,
           "cl_mean_last_cycle": float(np.mean(cl[last])), "cd_mean_last_cycle": float(np.mean(cd[last])),
           "cl_amp_last_cycle": float(0.5 * (cl[last].max() - cl[last].min())),
           "it_p_mean": float(S[:, 2].mean()), "it_p_max": float(S[:, 2].max()), "it_uv_mean": float(S[:, 1].mean()),
           "trend": "c_l periodic in T = 2 pi / k, cycle-mean c_l ~ 0, c_d at 2/T (P:150; figure only, P:154-155)"}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    np.savetxt(args.out + ".csv", np.c_[t, cl, cd, S[:, 1], S[:, 2]], delimiter=",",
               header="t_bar,cl,cd,it_uv,it_p", comments="")
    json.dump(res, open(args.out + ".json", "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k not in ("config",)}))


if __name__ == "__main__":
    main()
