"""Rate of cl_diag_alm_update with a full L-BFGS history (dev tool).

The ALM inner iteration's second history pass (alm.py:306-318 step + gradient + Gram rows
of g and y against the 2*memory+1 = 17 history vectors): n = 1e7, ld 26, one stepping
(non-refresh) update with nh history vectors, CUDA-event mean over 10 launches.
Usage: python tools/diag_update_probe.py [variant .so]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(args):
    if args:
        os.environ["CULORADS_LIB"] = args[0]
    sys.path.insert(0, ROOT)
    import torch
    from paper_2407_15049_b200 import _lib
    from paper_2407_15049_b200.device import Device
    torch.cuda.set_device(0)
    dev = Device()
    n, ld = 10_000_000, int(os.environ.get("PROBE_LD", "26"))
    res = {"lib": args[0] if args else "default", "n": n, "ld": ld}
    F = lambda: torch.randn(n, ld, dtype=torch.float64, device="cuda")   # noqa: E731
    V = lambda: torch.rand(n, dtype=torch.float64, device="cuda")        # noqa: E731
    R, D, CR, CD, go, gn, y = F(), F(), F(), F(), F(), F(), F()
    H = [F() for _ in range(17)]
    ax, axo, q1, q2, lam, b, aval = V(), V(), V(), V(), V(), V(), V()
    for nh in (0, 4, 10, 17):
        a = _lib.DiagUpdateArgs()
        a.n, a.ld, a.aval, a.tau, a.rho, a.scale = n, ld, aval.data_ptr(), 1e-3, 2.0, 1.0
        a.R, a.D, a.CR, a.CD = R.data_ptr(), D.data_ptr(), CR.data_ptr(), CD.data_ptr()
        a.ax, a.ax_out, a.q1, a.q2 = ax.data_ptr(), axo.data_ptr(), q1.data_ptr(), q2.data_ptr()
        a.lam, a.b, a.g_old, a.g_new, a.y = lam.data_ptr(), b.data_ptr(), go.data_ptr(), gn.data_ptr(), y.data_ptr()
        a.nh = nh
        for h in range(nh):
            a.H[h] = H[h].data_ptr()
        a.refresh = 0
        for _ in range(3):
            dev.diag_update(a)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(dev.stream)
        for _ in range(10):
            dev.diag_update(a)
        e1.record(dev.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        byts = n * 8 * 6 + n * ld * 8 * (5 + nh + 4)     # m-vectors; R D CR CD g_old + H read, R CR g y written
        res[f"nh{nh}_ms"] = round(ms, 3)
        res[f"nh{nh}_GBps"] = round(byts / ms / 1e6, 1)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
