"""Operator-layer and iteration timings on a synthetic matrix-completion instance (dev probe).

    python tools/probe_completion.py N2 N1 M
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

n2, n1, m = int(float(sys.argv[1])), int(float(sys.argv[2])), int(float(sys.argv[3]))
t = time.perf_counter()
o = graphs.random_completion(n2, n1, m, seed=0)
p = problem.build_matrix_completion(o)
t1 = time.perf_counter()
ops = linops.build_operators(p)
torch.cuda.synchronize()
print(f"n={p.n} m={p.m} gen {t1 - t:.1f}s build_operators {time.perf_counter() - t1:.1f}s "
      f"omega {ops.adj.omega.nnz} apat {ops.adj.apat.nnz} cpat {ops.c_mat.cpat.nnz}", flush=True)
dev = ops.dev
r = driver.initial_rank(p.m, p.n)
ld = padded_ld(r)
rng = np.random.default_rng(0)
U = linops.to_factor(rng.standard_normal((p.n, r)) / math.sqrt(p.n), dev, ld)
V = linops.to_factor(rng.standard_normal((p.n, r)) / math.sqrt(p.n), dev, ld)
lam = linops.to_vec(rng.standard_normal(p.m), dev)
out = dev.empty(p.n, ld)
y = dev.empty(p.m)


def timeit(name, fn, nbytes=None, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(dev.stream)
    for _ in range(reps):
        fn()
    e1.record(dev.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    extra = f" {nbytes / ms / 1e6:.0f} GB/s" if nbytes else ""
    print(f"{name}: {ms:.3f} ms{extra}", flush=True)


F = p.n * ld * 8
timeit("A(UV^T) constraint_eval", lambda: dev.constraint_eval(ops.cop.con, ld, U, V, y),
       p.m * 16 + 2 * p.m * (16 + 2 * ld * 8))
timeit("SDDMM K positions", lambda: dev.sddmm(ops.cop.imap, ops.cop.jmap, ld, U, V,
                                             torch.empty(ops.cop.ncols, dtype=torch.float64, device="cuda")))
timeit("S=C+A*(lam) SpMM (assemble+tiled)", lambda: dev.spmm(ops.adj.omega, V, ld, out=out, c_coeff=1.0, w1=lam),
       p.n * (8 + 8 * ld) + ops.adj.omega.nnz * (12 + 8 * ld))
hs = admm.HalfStep(ops, p.n, ld)
timeit("half-step apply (generic)", lambda: hs.apply(U, V, 1.5, out, dot_with=U, at=0))
dual = alm.DualVector(lam=lam.clone(), rho=2.0)
core = alm.AlmCore(ops, p.n, ld)
R = U.clone()
alm._inner(core, R.clone(), dual.lam, 2.0, 1.0, 0.0, 10, None, 8, alm._RankRecorder(None, r))   # warm-up: fills the history pool
torch.cuda.synchronize()
t = time.perf_counter()
res = alm._inner(core, R, dual.lam, 2.0, 1.0, 0.0, 10, None, 8, alm._RankRecorder(None, r))
torch.cuda.synchronize()
print(f"ALM inner: {1e3 * (time.perf_counter() - t) / max(res.iterations, 1):.2f} ms/iter", flush=True)
st = admm.AdmmState(U=U.clone(), V=V.clone(), dual=dual, r=r)
pool = admm._Pool(dev, p.n, ld)
admm.admm_step(st, ops, hs=hs, pool=pool)
torch.cuda.synchronize()
t = time.perf_counter()
cg = 0
for _ in range(3):
    s = admm.admm_step(st, ops, hs=hs, pool=pool)
    cg += s.cg_iters_u + s.cg_iters_v
torch.cuda.synchronize()
print(f"ADMM: {1e3 * (time.perf_counter() - t) / 3:.2f} ms/step, {cg / 3:.1f} CG its/step", flush=True)
