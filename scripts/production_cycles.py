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
ap.add_argument("--ckpt", default=None, help="checkpoint file: resumed from if present, rewritten at the end "
                "(u, v, p, phi, C^{n-1} and the step counter: a bit-exact continuation, test_checkpoint_restore)")
ap.add_argument("--history", default=None, help="CSV of the steps before the checkpoint (prepended to the summary)")
a = ap.parse_args()
cfg = I.cfg3(level=a.level, omega_p=a.omega_p, maxit_p=a.maxit_p, tol_p=a.tol_p)
body = cfg.body_args()
k = body[5]
period = 2 * math.pi / k
steps_per_cycle = int(round(period / cfg.dt))
total = int(round(a.cycles * steps_per_cycle))
g = P.Solver(cfg.xn, cfg.yn, **cfg.solver_kwargs())
g.set_body(*body)
hist, status_counts, done, diverged = [], {}, 0, False
if a.ckpt and os.path.exists(a.ckpt):
    import paper_2402_17337_b200.ibm as M
    z = np.load(a.ckpt)
    g.set_fields(z["u"], z["v"], z["p"], phi=z["phi"], restart=False)
    cu, cv = np.ascontiguousarray(z["cu_prev"]), np.ascontiguousarray(z["cv_prev"])
    M.ibm_set_fields(g.ctx, (1 << 10) | (1 << 11), {10: cu.ctypes.data, 11: cv.ctypes.data}, M.IBM_HOST)
    done = int(z["step"])
    g.set_step(done, True)
    print("resumed at step", done, flush=True)
else:
    g.set_fields(*I.initial_fields(cfg.nx, cfg.ny))
if a.history and os.path.exists(a.history):
    prev = np.genfromtxt(a.history, delimiter=",", skip_header=1)
    prev = prev[prev[:, 0] <= done]
    hist = [list(r) for r in prev]
os.makedirs(os.path.dirname(a.out_prefix) or ".", exist_ok=True)
fcsv = open(a.out_prefix + ".csv", "w", newline="")
w = csv.writer(fcsv)
w.writerow(["step", "t_bar", "cd", "cl", "it_uv", "it_p", "rho_p", "status", "ms_step"])
for r in hist:
    w.writerow(r)
t0 = time.time()
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
if a.ckpt and not diverged:
    snap = {n: g.get(n) for n in ("u", "v", "p", "phi", "cu_prev", "cv_prev")}
    np.savez(a.ckpt, step=done, **snap)
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
