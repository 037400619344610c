"""Rate of the diagonal-constraint CG kernels at n = 1e7, ld 26 (dev tool): cl_diag_cg_apply
(p <- r + beta p; Q = rho (a y Wf + p), y = a <p_i, Wf_i>; <p, Q>) and cl_diag_cg_step.
Usage: python tools/diag_cg_probe.py [variant .so]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(args):
    if args:
        os.environ["CULORADS_LIB"] = args[0]
    sys.path.insert(0, ROOT)
    import torch
    from paper_2407_15049_b200.device import Device
    torch.cuda.set_device(0)
    dev = Device()
    n, ld = 10_000_000, int(os.environ.get("PROBE_LD", "26"))
    F = lambda: torch.randn(n, ld, dtype=torch.float64, device="cuda")   # noqa: E731
    p, Wf, Q, r = F(), F(), F(), F()
    aval = torch.ones(n, dtype=torch.float64, device="cuda")
    res = {"lib": args[0] if args else "default", "n": n, "ld": ld}

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(dev.stream)
        for _ in range(10):
            fn()
        e1.record(dev.stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 10

    ms = timed(lambda: dev.diag_cg_apply(aval, ld, 2.0, p, Wf, Q, r=r, beta=0.5, at=0))
    res["cg_apply_ms"] = round(ms, 3)
    res["cg_apply_GBps"] = round(n * ld * 8 * 5 / ms / 1e6, 1)     # r, p, Wf read; p, Q written
    ms = timed(lambda: dev.diag_cg_apply(aval, ld, 2.0, p, Wf, Q, at=0))
    res["cg_apply_nor_ms"] = round(ms, 3)
    res["cg_apply_nor_GBps"] = round(n * ld * 8 * 3 / ms / 1e6, 1)  # p, Wf read; Q written
    coef = torch.empty(n, dtype=torch.float64, device="cuda")
    ms = timed(lambda: dev.diag_cg_apply_rows(aval, ld, 2.0, p, Wf, coef, r=r, beta=0.5, at=0))
    res["cg_apply_rows_ms"] = round(ms, 3)
    res["cg_apply_rows_GBps"] = round(n * ld * 8 * 4 / ms / 1e6, 1)   # r, p, Wf read; p written
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
