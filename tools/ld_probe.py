"""Time the C-pattern SpMM and a streaming pass at several factor leading dimensions
(row padding) on the bench instance: does aligning gathered rows to 64/128 bytes pay? Dev probe.

    python tools/ld_probe.py [n] [deg]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_15049_b200 import graphs, linops, problem  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
deg = float(sys.argv[2]) if len(sys.argv) > 2 else 6.0
p = problem.build_maxcut(graphs.random_sparse(n, deg=deg, seed=0))
ops = linops.build_operators(p)
dev = ops.dev
cpat = ops.c_mat.cpat
st = dev.stream
for ld in (26, 28, 32):
    X = torch.randn(n, ld, dtype=torch.float64, device=dev.dev)
    X[:, 25:] = 0.0
    out = torch.empty_like(X)
    for _ in range(3):
        dev.spmm(cpat, X, ld, out=out, c_coeff=1.0)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with torch.cuda.stream(st):
        ev[0].record()
        for _ in range(10):
            dev.spmm(cpat, X, ld, out=out, c_coeff=1.0)
        ev[1].record()
    torch.cuda.synchronize()
    t_spmm = ev[0].elapsed_time(ev[1]) / 10
    with torch.cuda.stream(st):
        ev[0].record()
        for _ in range(10):
            dev.lincomb(out, [X, out], [1.0, 0.5])
        ev[1].record()
    torch.cuda.synchronize()
    t_lc = ev[0].elapsed_time(ev[1]) / 10
    alg = n * (8 + 8 * 26) + cpat.nnz * (4 + 8 + 8 * 26)
    print(f"ld {ld}: spmm {t_spmm:.3f} ms ({alg / t_spmm / 1e6:.0f} GB/s of r=26 algorithmic bytes), "
          f"lincomb(2 in, 1 out) {t_lc:.3f} ms", flush=True)
    del X, out
