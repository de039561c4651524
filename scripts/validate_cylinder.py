"""BJ configs[1] validation: stationary circular cylinder,
Re = 100, 512 x 384 uniform grid on [-8,24] x [-12,12] (16 cells per diameter),
dt = 0.02, 2000 steps (T = 40), run on the GPU through the C ABI.

Reports the force-coefficient history (CSV), the Strouhal number St = f D / U
from the zero crossings of c_l over the last periods, and the mean drag
coefficient over the same window -- a trend check against the textbook values
St ~ 0.16-0.17, mean C_d ~ 1.3-1.4 (external literature; the paper itself has
no cylinder case).  The shedding is triggered by the seeded perturbation of
ibm_inputs.initial_fields (amplitude --perturb).

Usage: python scripts/validate_cylinder.py [--steps 2000] [--out profiles/r01_cylinder]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import ibm_inputs as I  # noqa: E402


def strouhal(t, cl, D=1.0, U=1.0, window=0.5):
    """Mean frequency of c_l from upward zero crossings in the last `window`
    fraction of the record (linear interpolation of the crossing times)."""
    n0 = int(len(t) * (1.0 - window))
    tt, cc = t[n0:], cl[n0:] - np.mean(cl[n0:])
    ups = [tt[i] - cc[i] * (tt[i + 1] - tt[i]) / (cc[i + 1] - cc[i])
           for i in range(len(cc) - 1) if cc[i] < 0.0 <= cc[i + 1]]
    if len(ups) < 2:
        return None, ups
    period = (ups[-1] - ups[0]) / (len(ups) - 1)
    return D / (U * period), ups


def surface_pressure_force(p, tp, xn, yn):
    """Diagnostic: pressure force on the body from the active cells bordering the
    inactive (body) cells, p x face length summed over those faces; (c_d, c_l)."""
    act = tp == 0
    dx, dy = np.diff(xn), np.diff(yn)
    fx = fy = 0.0
    # x-faces: active cell west of a body cell pushes +x; east of it pushes -x
    w = act[:, :-1] & ~act[:, 1:]
    e = ~act[:, :-1] & act[:, 1:]
    fx += (p[:, :-1][w] * np.broadcast_to(dy[:, None], w.shape)[w]).sum()
    fx -= (p[:, 1:][e] * np.broadcast_to(dy[:, None], e.shape)[e]).sum()
    s_ = act[:-1, :] & ~act[1:, :]
    n_ = ~act[:-1, :] & act[1:, :]
    fy += (p[:-1, :][s_] * np.broadcast_to(dx[None, :], s_.shape)[s_]).sum()
    fy -= (p[1:, :][n_] * np.broadcast_to(dx[None, :], n_.shape)[n_]).sum()
    return 2.0 * fx, 2.0 * fy


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--perturb", type=float, default=0.05)
    ap.add_argument("--dt", type=float, default=0.02)
    ap.add_argument("--omega-p", type=float, default=1.9)
    ap.add_argument("--tol-p", type=float, default=1e-8)
    ap.add_argument("--nx", type=int, default=512)
    ap.add_argument("--ny", type=int, default=384)
    ap.add_argument("--maxit-p", type=int, default=10000)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_cylinder"))
    args = ap.parse_args()
    import paper_2402_17337_b200 as P

    cfg = I.cfg2(nx=args.nx, ny=args.ny, steps=args.steps, omega_p=args.omega_p, tol_p=args.tol_p,
                 maxit_p=args.maxit_p)
    cfg.dt = args.dt
    g = P.Solver(cfg.xn, cfg.yn, **cfg.solver_kwargs())
    g.set_body(*cfg.body_args())
    g.set_fields(*I.initial_fields(cfg.nx, cfg.ny, args.perturb))
    tb_m = g.query("tb_m")
    rows, t0 = [], time.time()
    chunk = 100
    status = 0
    for s in range(0, args.steps, chunk):
        st, stats = g.step(min(chunk, args.steps - s))
        rows.append(stats)
        status = max(status, st)
        if st == 3:
            break
    wall = time.time() - t0
    S = np.concatenate(rows)
    t, cd, cl = S[:, 0], S[:, 5], S[:, 6]
    St, ups = strouhal(t, cl)
    n0 = len(t) // 2
    cdp, clp = surface_pressure_force(g.get("p"), g.get("tp"), cfg.xn, cfg.yn)
    res = {"config": cfg.describe(), "steps_done": len(t), "status": int(status), "wall_s": wall,
           "cd_last": float(cd[-1]), "cd_surface_pressure_last": float(cdp), "cl_surface_pressure_last": float(clp),
           "St": St, "n_crossings": len(ups), "mean_cd_last_half": float(np.mean(cd[n0:])),
           "cl_amplitude_last_half": float(0.5 * (cl[n0:].max() - cl[n0:].min())),
           "poisson_path": "resident k_sor_tb, %d iterations per grid barrier" % tb_m if tb_m else "k_sor / k_sor_coop",
           "it_p_mean": float(S[:, 2].mean()), "it_p_max": float(S[:, 2].max()), "it_uv_mean": float(S[:, 1].mean()),
           "reference_trend": "St 0.16-0.17, mean Cd 1.3-1.4 (Re=100 cylinder, external literature)"}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    np.savetxt(args.out + ".csv", np.c_[t, cl, cd, S[:, 1], S[:, 2]], delimiter=",",
               header="t_bar,cl,cd,it_uv,it_p", comments="")
    json.dump(res, open(args.out + ".json", "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
