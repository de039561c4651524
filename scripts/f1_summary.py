"""Summary of the production-mesh plunge-cycle run (scripts/production_cycles.py CSV):
per plunge cycle the means of c_d and c_l, the c_l rms, and the cycle-to-cycle
change of the c_l history, raw and after a 200-step running mean (the discrete-
forcing force history carries step-to-step spikes when cells change tag, the
spurious oscillations P:53's mass source q is meant to limit); time per step and
Poisson iterations, the first 1000 steps beside the paper's Table 2.
Usage: python scripts/f1_summary.py run.csv out.json"""
import json, sys
import numpy as np

d = np.genfromtxt(sys.argv[1], delimiter=",", names=True)
spc = 10000  # steps per plunge period (T = 2 pi / k = 1, dt = 1e-4)
k = 200
sm = lambda x: np.convolve(x, np.ones(k) / k, mode="same")
cl, cd = d["cl"], d["cd"]
cls, cds = sm(cl), sm(cd)
n = len(d) // spc
out = {"steps": int(len(d)), "t_end": float(d["t_bar"][-1]), "cycles_complete": n,
       "ms_per_step_mean": float(d["ms_step"].mean()), "it_p_mean": float(d["it_p"].mean()),
       "it_p_capped_1e5": int((d["it_p"] >= 100000).sum()), "it_uv_mean": float(d["it_uv"].mean()),
       "first_1000": {"ms_per_step_mean": float(d["ms_step"][:1000].mean()), "it_p_mean": float(d["it_p"][:1000].mean()),
                      "paper_sol2_s_per_step_M1": 0.244, "paper_note": "OpenACC, one V100, P:183 (context)"},
       "step_to_step_abs_dcl_median": float(np.median(np.abs(np.diff(cl)))), "cycles": []}
for c in range(n):
    s = slice(c * spc, (c + 1) * spc)
    r = {"cycle": c + 1, "cd_mean": float(cd[s].mean()), "cl_mean": float(cl[s].mean()),
         "cl_rms": float(np.sqrt(np.mean(cl[s] ** 2))), "cl_smoothed_min": float(cls[s].min()),
         "cl_smoothed_max": float(cls[s].max()), "cd_smoothed_min": float(cds[s].min()), "cd_smoothed_max": float(cds[s].max())}
    if c > 0:
        p = slice((c - 1) * spc, c * spc)
        r["cl_change_vs_prev_rel_rms_raw"] = float(np.sqrt(np.mean((cl[s] - cl[p]) ** 2)) / np.sqrt(np.mean(cl[s] ** 2)))
        r["cl_change_vs_prev_rel_rms_smoothed"] = float(np.sqrt(np.mean((cls[s] - cls[p]) ** 2)) / np.sqrt(np.mean(cls[s] ** 2)))
        r["cd_mean_change_vs_prev"] = float(cd[s].mean() - cd[p].mean())
    out["cycles"].append(r)
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
