"""Diagnostic of the production-mesh foil runs (BJ configs[2], M1): where and
when the solution grows.  Steps in chunks, records max |u|, |v|, |p| and their
grid locations, SOR iteration counts and residuals, until NaN or --steps.
Usage: python scripts/production_diag.py [--level 1] [--steps 400] [--omega-p 1.97] [--maxit-p 100000]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import ibm_inputs as I
import paper_2402_17337_b200 as P

ap = argparse.ArgumentParser()
ap.add_argument("--level", type=int, default=1)
ap.add_argument("--steps", type=int, default=400)
ap.add_argument("--chunk", type=int, default=20)
ap.add_argument("--omega-p", type=float, default=1.97)
ap.add_argument("--maxit-p", type=int, default=100000)
ap.add_argument("--tol-p", type=float, default=1e-6)
ap.add_argument("--dt", type=float, default=1e-4)
ap.add_argument("--out", default=None)
a = ap.parse_args()
cfg = I.cfg3(level=a.level, omega_p=a.omega_p, maxit_p=a.maxit_p, tol_p=a.tol_p, dt=a.dt)
g = P.Solver(cfg.xn, cfg.yn, **cfg.solver_kwargs())
g.set_body(*cfg.body_args())
g.set_fields(*I.initial_fields(cfg.nx, cfg.ny))
xc, yc = 0.5 * (cfg.xn[1:] + cfg.xn[:-1]), 0.5 * (cfg.yn[1:] + cfg.yn[:-1])
log = []
done = 0
while done < a.steps:
    st, S = g.step(a.chunk)
    done += len(S)
    rec = {"step": done, "status": st, "it_p": S[:, 2].tolist(), "rho_p_last": float(S[-1, 4]),
           "it_uv_max": float(S[:, 1].max()), "cd": float(S[-1, 5]), "cl": float(S[-1, 6])}
    for n in ("u", "v", "p"):
        f = g.get(n)
        bad = ~np.isfinite(f)
        fa = np.where(bad, np.inf, np.abs(f))
        j, i = np.unravel_index(np.argmax(fa), f.shape)
        rec["max_" + n] = float(fa[j, i])
        rec["at_" + n] = [int(i), int(j), float(cfg.xn[min(i, cfg.nx)] if n == "u" else xc[min(i, cfg.nx - 1)]),
                          float(yc[min(j, cfg.ny - 1)] if n != "v" else cfg.yn[j])]
    print(json.dumps({k: v for k, v in rec.items() if k != "it_p"} | {"it_p_mean": float(np.mean(rec["it_p"]))}),
          flush=True)
    log.append(rec)
    if st == 3 or not np.isfinite(rec["max_u"]):
        break
if a.out:
    json.dump({"config": cfg.describe(), "tb_m": g.query("tb_m"), "log": log}, open(a.out, "w"), indent=1)
