"""Time ALM inner iterations and ADMM steps of the device solver on synthetic MaxCut (dev probe).

    python tools/profile_alm.py N DEG ALM_ITERS ADMM_STEPS [RANK]
"""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_15049_b200 import admm, alm, driver, graphs, linops, problem  # noqa: E402
from paper_2407_15049_b200.device import padded_ld  # noqa: E402

n = int(float(sys.argv[1]))
deg = float(sys.argv[2])
iters = int(sys.argv[3])
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 0
p = problem.build_maxcut(graphs.random_sparse(n, deg=deg, seed=0))
ops = linops.build_operators(p)
dev = ops.dev
r = int(sys.argv[5]) if len(sys.argv) > 5 else driver.initial_rank(p.m, p.n)
ld = padded_ld(r)
rng = np.random.default_rng(0)
R = linops.to_factor(rng.standard_normal((n, r)) / math.sqrt(n * r), dev, ld)
rho = max(1.0, p.m / math.sqrt(p.nnz_a_full()))
dual = alm.DualVector(lam=dev.zeros(p.m), rho=rho)
core = alm.AlmCore(ops, n, ld)
# warm-up (compiles nothing, but touches every kernel once)
alm._inner(core, R.clone(), dual.lam, rho, 1.0, 1e-8, 3, None, 8, alm._RankRecorder(None, r))
torch.cuda.synchronize()
l0 = dev.launches
t = time.perf_counter()
res = alm._inner(core, R, dual.lam, rho, 1.0, 0.0, iters, None, 8, alm._RankRecorder(None, r))
torch.cuda.synchronize()
dt = time.perf_counter() - t
print(f"n={n} r={r} ld={ld}: {res.iterations} ALM inner iterations in {dt:.3f}s = "
      f"{1e3 * dt / max(res.iterations, 1):.2f} ms/iter, {(dev.launches - l0) / max(res.iterations, 1):.1f} launches/iter",
      flush=True)
if steps:
    del core, res
    torch.cuda.empty_cache()
    st = admm.AdmmState(U=R.clone(), V=R.clone(), dual=dual, r=r)
    hs = admm.HalfStep(ops, n, ld)
    pool = admm._Pool(dev, n, ld)
    admm.admm_step(st, ops, hs=hs, pool=pool)
    torch.cuda.synchronize()
    l0 = dev.launches
    t = time.perf_counter()
    cg = 0
    for _ in range(steps):
        s = admm.admm_step(st, ops, hs=hs, pool=pool)
        cg += s.cg_iters_u + s.cg_iters_v
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"ADMM: {steps} steps {cg} CG iterations in {dt:.3f}s = {1e3 * dt / steps:.2f} ms/step, "
          f"{1e3 * dt / max(cg, 1):.3f} ms/CG-iter, {(dev.launches - l0) / steps:.1f} launches/step", flush=True)
