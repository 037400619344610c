"""Time one device MaxCut solve on a synthetic graph (development probe, not the bench).

    python tools/probe_solve.py N DEG [time_limit] [random|delaunay] [reorder] [--out FILE]

Prints the report and writes the trace summarised per (stage, rank) segment to FILE
(JSON), so an escalation history can be read after the run.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_15049_b200 import driver, graphs, linops, problem  # noqa: E402

args = [a for a in sys.argv[1:]]
overrides = {}
while "--cfg" in args:            # --cfg key=value: a SolverConfig option (the reference's names)
    k = args.index("--cfg")
    key, val = args[k + 1].split("=", 1)
    overrides[key] = None if val == "None" else (int(val) if val.lstrip("-").isdigit() else float(val))
    del args[k:k + 2]
out = None
if "--out" in args:
    k = args.index("--out")
    out = args[k + 1]
    del args[k:k + 2]
n = int(float(args[0]))
deg = float(args[1])
tl = float(args[2]) if len(args) > 2 else 600.0
kind = args[3] if len(args) > 3 else "random"
reorder = len(args) > 4 and args[4] == "reorder"
t = time.perf_counter()
if kind == "completion":
    # matrix completion with n rows+cols split in half and deg*n/2 observations (configs[3] family)
    g = graphs.random_completion(n // 2, n - n // 2, int(deg * n / 2), seed=0)
elif kind == "delaunay":
    g = graphs.delaunay_like(n, seed=0)
elif kind == "path":
    g = graphs.path_like(n, extra=max(deg - 2.0, 0.0) / 2.0, seed=0)
else:
    g = graphs.random_sparse(n, deg=deg, seed=0)
t_g = time.perf_counter() - t
t = time.perf_counter()
p = problem.build_matrix_completion(g) if kind == "completion" else problem.build_maxcut(g)
t_p = time.perf_counter() - t
t = time.perf_counter()
ops = None if reorder else linops.build_operators(p)
torch.cuda.synchronize()
t_o = time.perf_counter() - t
print(f"{kind} reorder={reorder} n={n} m={p.m} gen {t_g:.2f}s build_problem {t_p:.2f}s "
      f"build_operators {t_o:.2f}s", flush=True)
t = time.perf_counter()
rep = driver.solve(p, driver.SolverConfig(time_limit=tl, reorder=reorder, **overrides), ops=ops)
print("options", overrides, flush=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t
print(f"solve {dt:.2f}s status {rep.status} obj {rep.objective:.10g} err1 {rep.err1:.2e} err3 {rep.err3:.2e} "
      f"err2 {rep.err2} rank {rep.rank_history} memcap {rep.memory_capped}/{rep.memory_rank_refused} "
      f"alm {rep.alm_outer_iterations}/{rep.alm_inner_iterations} "
      f"admm {rep.admm_steps} cg {rep.cg_iterations} reopt {rep.reopt_rounds} t_alm {rep.time_alm_s:.2f} "
      f"t_admm {rep.time_admm_s:.2f} launches {rep.gpu_launches} peak {rep.peak_bytes/2**30:.1f} GiB", flush=True)

segs = []
for row in rep.trace_rows:
    stage, k, obj, err1, metric, rho, rank, tt = row
    if not segs or segs[-1]["stage"] != stage or segs[-1]["rank"] != rank:
        segs.append({"stage": stage, "rank": rank, "first_row": k, "t_start": tt, "rows": 0})
    s = segs[-1]
    s["rows"] += 1
    s.update(t_end=tt, obj_end=obj, err1_end=err1, metric_end=metric, rho_end=rho)
gap_at = dict(rep.admm_gaps)
for s in segs:
    s["gap_end"] = gap_at.get(s["first_row"] + s["rows"] - 1)
for s in segs:
    print(f"  {s['stage']:4s} r={s['rank']:5d} rows {s['rows']:6d} t {s['t_start']:8.2f}-{s['t_end']:8.2f} "
          f"obj {s['obj_end']:.8g} err1 {s['err1_end']:.2e} metric {s['metric_end']:.2e} rho {s['rho_end']:.3g}"
          + (f" gap {s['gap_end']:.2e}" if s["gap_end"] is not None else ""))
if out:
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    with open(out, "w") as f:
        json.dump({"n": n, "deg": deg, "kind": kind, "reorder": reorder, "gen_s": t_g, "build_maxcut_s": t_p,
                   "build_operators_s": t_o, "solve_s": dt, "report": rep.to_json_dict(),
                   "rank_history": rep.rank_history, "memory_capped": rep.memory_capped,
                   "memory_rank_refused": rep.memory_rank_refused,
                   "alm": [rep.alm_outer_iterations, rep.alm_inner_iterations],
                   "admm_steps": rep.admm_steps, "cg": rep.cg_iterations, "segments": segs,
                   "admm_gaps": rep.admm_gaps[::max(1, len(rep.admm_gaps) // 400)],
                   "trace_sample": [list(r) for r in rep.trace_rows[::max(1, len(rep.trace_rows) // 400)]]},
                  f, indent=1)
