"""performance report in the layout of the paper's Table 1
(serial per-function times of one step) and Table 2,
for the CPU oracle on one core (oracle_seq: the analogue of the paper's serial
SOL0), the same oracle on every host core (oracle_omp: the analogue of the
OpenMP SOL1) and the B200 path (the SOL2 analogue), on the same
configuration and the same iteration counts; speedups S_SOLi = T_SOL0/T_SOLi
and S_relative = S_SOL2/S_SOL1 (Eqs. 6-7).

Regions (oracle: `Oracle.timers()`, wall clock per region; GPU: the CUDA-event
phase times of `ibm_step_stats.ms`):
  flagging            a1 classification + Poisson masks   (Table 1 "fluid/solid flagging")
  predictor+forcing   a2/a3 convection, Helmholtz rhs, IBM forcing targets
                      (contains Table 1's "body-force interpolation")
  U-V solver          a4 Helmholtz red-black SOR + outlet fill
  Poisson rhs         a5
  P solver            a6 Poisson red-black SOR
  correction          a7 projection + history rotation
  forces              a8
Amdahl: S(n) = 1 / ((1 - p) + p / n) with the paper's p = 0.998 gives
S_inf = 500; the measured whole-step ratio oracle / GPU is printed beside it.

Usage: python scripts/perf_report.py [--level 1] [--maxit-p 200] [--oracle-steps 2]
                                     [--gpu-steps 20] [--out profiles/r01_perf_report]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import ibm_inputs as I  # noqa: E402

REGIONS = ["flagging", "predictor+forcing", "U-V solver", "Poisson rhs", "P solver", "correction", "forces"]
# Table 1, seconds per step, SOL0 serial, i7 10th gen; mesh not stated
PAPER_T1 = {"P solver": 3.835, "flagging": 2.5515, "U-V solver": 0.5518, "body-force interpolation": 0.0758}
PAPER_P = 0.998
# Table 2: seconds for the first 1000 steps, [SOL0, SOL1, SOL2][mesh level]
PAPER_T2 = [{1: 13140.0, 2: 24663.0, 3: 39994.0}, {1: 4232.0, 2: 8175.0, 3: 11953.0}, {1: 244.4, 2: 378.0, 3: 368.3}]


def gpu_regions(ms):
    """ibm_step_stats.ms -> region seconds: [0] classify+predictor, [1] uv, [2] rhs, [3] p, [4] correct,
    [5] forces, [6] classification part of [0]."""
    return np.array([ms[6], ms[0] - ms[6], ms[1], ms[2], ms[3], ms[4], ms[5]]) / 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--level", type=int, default=1)
    ap.add_argument("--maxit-p", type=int, default=200)
    ap.add_argument("--oracle-steps", type=int, default=2)
    ap.add_argument("--gpu-steps", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_perf_report"))
    args = ap.parse_args()
    from oracle import oracle as O
    import paper_2402_17337_b200 as P

    cfg = I.cfg3(level=args.level, steps=args.oracle_steps, maxit_p=args.maxit_p)
    u0, v0, p0 = I.initial_fields(cfg.nx, cfg.ny)
    # oracle (single thread): the first oracle_steps steps
    o = O.Oracle(cfg.xn, cfg.yn, **cfg.solver_kwargs())
    o.set_body(*cfg.body_args())
    o.set_fields(u0, v0, p0)
    t0 = time.time()
    _, sto = o.step(args.oracle_steps)
    o_wall = (time.time() - t0) / args.oracle_steps
    o_reg = o.timers() / args.oracle_steps
    del o
    # oracle_omp on every host core (SOL1 analogue): bitwise the same steps
    cores = len(os.sched_getaffinity(0))
    os.environ["OMP_NUM_THREADS"] = str(cores)
    om = O.Oracle(cfg.xn, cfg.yn, omp=True, **cfg.solver_kwargs())
    om.set_body(*cfg.body_args())
    om.set_fields(u0, v0, p0)
    om.timers()
    t0 = time.time()
    _, stm = om.step(args.oracle_steps)
    m_wall = (time.time() - t0) / args.oracle_steps
    m_reg = om.timers() / args.oracle_steps
    assert np.array_equal(stm, sto), "oracle_omp differs from oracle_seq"
    del om
    # GPU: the same first steps (identical iteration counts), then more steps for a stable mean
    g = P.Solver(cfg.xn, cfg.yn, **cfg.solver_kwargs())
    g.set_body(*cfg.body_args())
    g.set_fields(u0, v0, p0)
    _, stg = g.step(args.oracle_steps)
    assert np.array_equal(stg[:, 1:3], sto[:, 1:3]), "iteration counts differ from the oracle"
    _, stg2 = g.step(args.gpu_steps)
    raw = g.last_stats
    g_reg = np.mean([gpu_regions(raw[k].ms) for k in range(args.gpu_steps)], axis=0)
    g_step = float(np.mean([raw[k].ms[7] for k in range(args.gpu_steps)])) / 1e3
    g.close()
    rows = []
    for name, a, am, b in zip(REGIONS, o_reg, m_reg, g_reg):
        rows.append({"region": name, "oracle_s": float(a), "oracle_pct": float(100 * a / o_reg.sum()),
                     "oracle_omp_s": float(am), "gpu_ms": float(1e3 * b), "gpu_pct": float(100 * b / g_reg.sum()),
                     "speedup": float(a / b) if b > 0 else None,
                     "S_SOL1": float(a / am) if am > 0 else None,
                     "S_rel": float(am / b) if b > 0 else None, "paper_sol0_s": PAPER_T1.get(name)})
    S = float(o_reg.sum() / g_reg.sum())
    S1 = float(o_reg.sum() / m_reg.sum())
    lv = args.level
    paper = {"T_SOL0": PAPER_T2[0][lv], "T_SOL1": PAPER_T2[1][lv], "T_SOL2": PAPER_T2[2][lv]}
    paper["S_SOL1"] = paper["T_SOL0"] / paper["T_SOL1"]
    paper["S_SOL2"] = paper["T_SOL0"] / paper["T_SOL2"]
    paper["S_rel"] = paper["S_SOL2"] / paper["S_SOL1"]
    res = {"config": {"workload": cfg.name, "nx": cfg.nx, "ny": cfg.ny, "maxit_p": args.maxit_p,
                      "it_p_per_step": stg2[:, 2].tolist()[:3], "it_uv_per_step": stg2[:, 1].tolist()[:3]},
           "oracle": {"cores": 1, "wall_s_per_step": o_wall, "regions_s_per_step": float(o_reg.sum())},
           "oracle_omp": {"cores": cores, "wall_s_per_step": m_wall, "regions_s_per_step": float(m_reg.sum())},
           "gpu": {"device": "B200", "step_ms": 1e3 * g_step, "regions_ms": float(1e3 * g_reg.sum())},
           "rows": rows, "speedup_whole_step": S,
           "S_SOL1": S1, "S_SOL2": S, "S_relative": S / S1,
           "paper_table2_eqs6_7": paper,
           "amdahl_paper": {"p": PAPER_P, "S_inf": 1.0 / (1.0 - PAPER_P)},
           "paper_table1_note": "Table 1 is SOL0 on an unstated mesh (P:109-112): shares, not seconds, compare",
           "paper_sol0_shares_pct": {k: 100 * v / 7.014 for k, v in PAPER_T1.items()}}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out + ".json", "w"), indent=1)
    lines = ["# Performance report (SURVEY §8(f) f4): %s, %d x %d, maxit_p = %d" % (cfg.name, cfg.nx, cfg.ny,
                                                                                       args.maxit_p), "",
             "SOL0 analogue = oracle_seq (plain C, one core of the GPU box's host); SOL1 analogue = oracle_omp",
             "(the same source with OpenMP, %d cores, bitwise-equal results asserted); SOL2 analogue = this build" % cores,
             "on one B200.  Same configuration and identical iteration counts (asserted).  Paper SOL0 shares from",
             "Table 1 (P:109-112, total 7.014 s over its four hotspots, mesh unstated) compare as SHARES.", "",
             "| region | SOL0 s/step | SOL0 % | SOL1 s/step | GPU ms/step | GPU % | S_SOL1 | S_SOL2 | S_rel | paper SOL0 % |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    f0 = lambda v: "%.0f" % v if v else "-"
    for r in rows:
        ps = res["paper_sol0_shares_pct"].get(r["region"])
        lines.append("| %s | %.4f | %.1f | %.4f | %.3f | %.1f | %s | %s | %s | %s |" % (
            r["region"], r["oracle_s"], r["oracle_pct"], r["oracle_omp_s"], r["gpu_ms"], r["gpu_pct"],
            "%.1f" % r["S_SOL1"] if r["S_SOL1"] else "-", f0(r["speedup"]), f0(r["S_rel"]),
            "%.1f" % ps if ps is not None else "-"))
    lines += ["", "Whole step: SOL0 %.3f s, SOL1 %.3f s, GPU %.3f ms: S_SOL1 = %.2f, S_SOL2 = %.0f, S_relative = %.0f "
              "(Eqs. 6-7, P:161-168)." % (o_reg.sum(), m_reg.sum(), 1e3 * g_reg.sum(), S1, S, S / S1),
              "Paper, M%d, first 1000 steps (Table 2, P:181-183; i7 / 16 threads / V100): S_SOL1 = %.2f, S_SOL2 = %.2f, "
              "S_relative = %.2f -- context, another machine and code." % (lv, paper["S_SOL1"], paper["S_SOL2"],
                                                                            paper["S_rel"]),
              "Amdahl with the paper's p = %.3f (P:101): S_inf = %.0f." % (PAPER_P, 1.0 / (1.0 - PAPER_P))]
    open(args.out + ".md", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
