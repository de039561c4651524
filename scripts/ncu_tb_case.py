"""One resident mid-grid Poisson solve (k_sor_tb) on a BJ-shaped mesh for an ncu
capture: one full step, then a fixed-count solve (poisson_iterate).
Usage: python scripts/ncu_tb_case.py {M1|cyl} [iters]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ibm_inputs as I
import paper_2402_17337_b200 as P

case = sys.argv[1] if len(sys.argv) > 1 else "M1"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 400
cfg = I.cfg3(1, maxit_p=400) if case == "M1" else I.cfg2(maxit_p=400)
g = P.Solver(cfg.xn, cfg.yn, **cfg.solver_kwargs())
g.set_body(*cfg.body_args())
g.set_fields(*I.initial_fields(cfg.nx, cfg.ny, 0.01))
g.step(1)
g.poisson_iterate(iters)
print(case, "tb_m", g.query("tb_m"))
g.close()
