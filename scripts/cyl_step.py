"""Two steps of BJ configs[1] (cylinder 512x384) -- a small-grid profiling target."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ibm_inputs as I
import paper_2402_17337_b200 as P
cfg = I.cfg2(steps=3)
g = P.Solver(cfg.xn, cfg.yn, **cfg.solver_kwargs())
g.set_body(*cfg.body_args())
g.set_fields(*I.initial_fields(cfg.nx, cfg.ny, 0.05))
st, stats = g.step(3)
print(stats[:, :3], [g.last_stats[k].ms[3] for k in range(3)])
