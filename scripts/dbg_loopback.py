"""Debug helper: loopback slabs vs one slab with the fused Poisson pass, a few
fixed Poisson iterations, report where phi differs."""
import sys
sys.path.insert(0, '.')
import numpy as np
import ibm_inputs as I
import paper_2402_17337_b200 as P
cfg = I.cfg1(steps=1, maxit_p=1)
u0, v0, p0 = I.initial_fields(cfg.nx, cfg.ny, cfg.perturb, cfg.seed)
for y0 in (0.6, 0.25, 0.0, -0.25):
  for fuse in (2,):
    for iters in (2,):
        res = []
        for P_ in (1, 2):
            g = P.Solver(cfg.xn, cfg.yn, nranks=P_, loopback=(P_ > 1), sor_fuse=fuse, sor_batch=5, **cfg.solver_kwargs())
            ba = list(cfg.body_args()); ba[3] = y0
            g.set_body(*ba)
            g.set_fields(u0, v0, p0)
            g.step(1)
            g.poisson_iterate(iters)
            res.append((g.get("phi"), g.get("tp")))
            g.close()
        d = np.abs(res[0][0] - res[1][0])
        rows = np.where(d.max(axis=1) > 0)[0]
        brows = np.where(res[0][1].max(axis=1) > 0)[0]
        msg = "identical" if d.max() == 0 else "max %.3e rows %s cols %s" % (d.max(), rows.tolist()[:20], np.where(d.max(axis=0) > 0)[0].tolist()[:12])
        print("y0=%.2f body p-rows %s..%s fuse=%d iters=%d: %s" % (y0, brows.min(), brows.max(), fuse, iters, msg))
