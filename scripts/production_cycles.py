"""BJ configs[2] / SURVEY §8(f) f1: the paper's validation case (plunging foil,
Re = 500, k = 2 pi, h = 0.16) on the stretched production mesh M1 (P:198,
reading R28), dt = 1e-4, impulsive start, through the C ABI on one GPU.
Writes the per-step history (t, c_d, c_l, SOR iterations, residuals, step time)
as CSV while it runs and a summary JSON at the end: per-cycle means of c_d and
c_l, the rms change of the c_l history from one plunge cycle to the next, the
time per step over the first 1000 steps (cf. Table 2).  Stops at
--steps or after --max-minutes of wall time.
Usage: python scripts/production_cycles.py --out-prefix gpurun_out/f1 [--cycles 3]"""
import argparse, csv, json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import ibm_inputs as I
import paper_2402_17337_b200 as P

ap = argparse.ArgumentParser()
ap.add_argument("--level", type=int, default=1)
ap.add_argument("--cycles", type=float, default=3.0)
ap.add_argument("--chunk", type=int, default=100)
ap.add_argument("--omega-p", type=float, default=1.97)
ap.add_argument("--maxit-p", type=int, default=100000)
ap.add_argument("--tol-p", type=float, default=1e-6)
ap.add_argument("--max-minutes", type=float, default=150.0)
ap.add_argument("--out-prefix", default="gpurun_out/f1")
a = ap.parse_args()
cfg = I.cfg3(level=a.level, omega_p=a.omega_p, maxit_p=a.maxit_p, tol_p=a.tol_p)
body = cfg.body_args()
k = body[5]
period = 2 * math.pi / k
steps_per_cycle = int(round(period / cfg.dt))
total = int(round(a.cycles * steps_per_cycle))
g = P.Solver(cfg.xn, cfg.yn, **cfg.solver_kwargs())
g.set_body(*body)
g.set_fields(*I.initial_fields(cfg.nx, cfg.ny))
os.makedirs(os.path.dirname(a.out_prefix) or ".", exist_ok=True)
fcsv = open(a.out_prefix + ".csv", "w", newline="")
w = csv.writer(fcsv)
w.writerow(["step", "t_bar", "cd", "cl", "it_uv", "it_p", "rho_p", "status", "ms_step"])
t0 = time.time()
hist, status_counts, done, diverged = [], {}, 0, False
while done < total and (time.time() - t0) < 60 * a.max_minutes:
    n = min(a.chunk, total - done)
    st, S = g.step(n)
    raw = g.last_stats
    for q in range(len(S)):
        # stats columns (ibm.stats_array): t, it_uv, it_p, rho_uv, rho_p, cd, cl, status
        row = [done + q + 1, float(S[q, 0]), float(S[q, 5]), float(S[q, 6]), int(S[q, 1]), int(S[q, 2]),
               float(S[q, 4]), int(S[q, 7]), float(raw[q].ms[7])]
        w.writerow(row)
        hist.append(row)
    fcsv.flush()
    done += len(S)
    status_counts[st] = status_counts.get(st, 0) + 1
    if st == 3 or not np.all(np.isfinite(S[:, 5:7])):
        diverged = True
        break
H = np.array(hist, dtype=float)
summ = {"config": cfg.describe(), "tb_m": g.query("tb_m"), "steps_done": done, "steps_target": total,
        "steps_per_cycle": steps_per_cycle, "diverged": diverged, "wall_s": time.time() - t0,
        "status_counts": {str(k_): v for k_, v in status_counts.items()}}
if len(H):
    first = H[:1000]
    summ["first_1000"] = {"ms_per_step_mean": float(first[:, 8].mean()), "it_p_mean": float(first[:, 5].mean()),
                          "paper_sol2_s_per_step": 0.244, "paper_note": "OpenACC on one V100, M1, P:183 (context)"}
    summ["ms_per_step_mean"] = float(H[:, 8].mean())
    summ["it_p_mean"] = float(H[:, 5].mean())
    summ["capped_solves"] = int((H[:, 5] >= a.maxit_p).sum())
    cyc = []
    ncyc = done // steps_per_cycle
    for c in range(ncyc):
        seg = H[c * steps_per_cycle:(c + 1) * steps_per_cycle]
        cyc.append({"cycle": c + 1, "cd_mean": float(seg[:, 2].mean()), "cl_mean": float(seg[:, 3].mean()),
                    "cl_rms": float(np.sqrt(np.mean(seg[:, 3] ** 2))), "cd_min": float(seg[:, 2].min()),
                    "cd_max": float(seg[:, 2].max()), "cl_min": float(seg[:, 3].min()), "cl_max": float(seg[:, 3].max())})
    for c in range(1, ncyc):
        A = H[(c - 1) * steps_per_cycle:c * steps_per_cycle, 3]
        B = H[c * steps_per_cycle:(c + 1) * steps_per_cycle, 3]
        cyc[c]["cl_change_vs_prev_rel_rms"] = float(np.sqrt(np.mean((B - A) ** 2)) / max(np.sqrt(np.mean(B ** 2)), 1e-30))
    summ["cycles"] = cyc
json.dump(summ, open(a.out_prefix + ".json", "w"), indent=1)
print(json.dumps({k_: v for k_, v in summ.items() if k_ != "config"}), flush=True)
g.close()
