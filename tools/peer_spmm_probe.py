"""Cost of the peer-memory ghost mode in the SpMM on one GPU (dev tool).

One rank's share of an 8-way row split of the configs[2] graph (n = 1e7, deg 6): its
1.25e6 C rows, 7/8 of whose columns belong to other ranks, times the factor (ld 26), as
    local   global column ids on one whole factor (no ghosts: the ideal)
    halo    GHOST 1: remote rows from a packed halo buffer (the copy path's SpMM only)
    peer    GHOST 2: remote rows from 8 separate block allocations through the peer table
On one GPU the "peer" blocks are local memory, so this measures the kernel's decode and
register cost, not NVLink. Usage: python tools/peer_spmm_probe.py [variant .so ...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(libs):
    full = bool(libs) and libs[0] == "full"     # all 1e7 rows on one GPU: the unsharded variants only
    if full:
        libs = libs[1:]
    if libs:
        os.environ["CULORADS_LIB"] = libs[0]
    sys.path.insert(0, ROOT)
    import torch
    from paper_2407_15049_b200 import shard
    from paper_2407_15049_b200.device import Device
    from paper_2407_15049_b200.linops import DevicePattern, padded
    from tests.test_gpu_peer import _LocalHalo, _LocalPeers

    torch.cuda.set_device(0)
    dev = Device()
    ld = int(os.environ.get("PROBE_LD", "26"))
    n, deg, world, rank = 10_000_000, 6.0, (1 if full else 8), 0
    b = shard.block_bounds(n, world)
    lo, hi = b[rank], b[rank + 1]
    eu, ev = shard.random_graph_edges(n, deg, 0, dev.dev)
    indptr, cols, vals = shard.maxcut_rows(n, eu, ev, lo, hi)
    del eu, ev
    nl = hi - lo
    ptr = torch.zeros(nl + 1 + 16, dtype=torch.int64, device=dev.dev)
    ptr[:nl + 1] = indptr

    def pat(idx):
        return DevicePattern(nl, ptr[:nl + 1], padded(idx.to(torch.int32)), padded(vals), None, None, None)

    X = torch.randn(n, ld, dtype=torch.float64, device=dev.dev)
    blocks = [X[b[k]:b[k + 1]].clone() for k in range(world)]
    own = (cols >= lo) & (cols < hi)
    rem = torch.unique(cols[~own])
    hidx = cols - lo
    hidx[~own] = nl + torch.searchsorted(rem, cols[~own])
    p_local = pat(cols)
    p_halo = pat(hidx)
    p_halo.halo = _LocalHalo(nl, X[rem].contiguous())
    p_peer = pat(shard.encode_peer_columns(cols, lo, hi, b))
    p_peer.halo = _LocalPeers(b, lambda _X: blocks)
    out = torch.empty(nl, ld, dtype=torch.float64, device=dev.dev)
    Yl = torch.randn(nl, ld, dtype=torch.float64, device=dev.dev)
    x0 = torch.randn(nl, ld, dtype=torch.float64, device=dev.dev)
    r_ = torch.empty_like(x0)
    nlam = torch.randn(nl, dtype=torch.float64, device=dev.dev)
    aval = torch.ones(nl, dtype=torch.float64, device=dev.dev)
    ax_o, ln_o = torch.empty_like(aval), torch.empty_like(aval)
    res = {"ld": ld, "rows": nl, "slots": int(cols.numel()), "remote_frac": float((~own).sum()) / cols.numel(),
           "lib": libs[0] if libs else "default"}
    outs = {}
    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(dev.stream)
        for _ in range(20):
            fn()
        e1.record(dev.stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 20

    variants = [("local", p_local, X)] if full else [("local", p_local, X), ("halo", p_halo, blocks[rank]),
                                                        ("peer", p_peer, blocks[rank])]
    for name, P, Xa in variants:
        # fused epilogue (EPI 1: out = S X + 2 Y, two dots) and the diagonal-ADMM CG start (EPI 2)
        res[f"{name}_epi1_ms"] = timed(lambda: dev.spmm(P, Xa, ld, out=out, Y=(Yl,), ycoef=(2.0,), c_coeff=1.0,
                                                        dots=[("out", ("y", 0)), ("out", "out")], at=0))
        res[f"{name}_cg_init_ms"] = timed(lambda: dev.diag_admm_cg_init(P, Xa, x0, ld, 0.7, 3.0, nlam, aval, r_, 0))
        # the ALM line search's C D (alm_native.cu: Z = R, D, CR; dots <CD,R>, <CD,D>, <CR,D>)
        res[f"{name}_linesearch_ms"] = timed(lambda: dev.spmm(P, Xa, ld, out=out, Z=(x0, Xa if full else x0, Yl),
                                                              c_coeff=1.0, at=0,
                                                              dots=[("out", ("z", 0)), ("out", ("z", 1)),
                                                                    (("z", 2), ("z", 1))]))
        res[f"{name}_step_end_ms"] = timed(lambda: dev.diag_admm_step_end(P, x0, Xa, ld, aval, aval, nlam, 3.0,
                                                                          ax_o, ln_o, 0))
        fn = lambda: dev.spmm(P, Xa, ld, out=out, c_coeff=1.0)   # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(dev.stream)
        for _ in range(20):
            fn()
        e1.record(dev.stream)
        torch.cuda.synchronize()
        res[f"{name}_ms"] = e0.elapsed_time(e1) / 20
        outs[name] = out.clone()
    res["bit_identical"] = full or bool(torch.equal(outs["local"], outs["peer"]) and torch.equal(outs["halo"], outs["peer"]))
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
