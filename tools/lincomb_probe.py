"""Rate of the L-BFGS direction pass (cl_lincomb, OUT_ALL dots) at n = 1e7, ld 26 (dev tool).
D = sum_j c_j H_j over nin history vectors with the Gram row <D, H_j> and <D, D>.
Usage: python tools/lincomb_probe.py [variant .so]"""
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
    N = 10_000_000 * 26
    H = [torch.randn(N, dtype=torch.float64, device="cuda") for _ in range(17)]
    out = torch.empty(N, dtype=torch.float64, device="cuda")
    res = {"lib": args[0] if args else "default"}
    for nin in (2, 8, 12, 17):
        fn = lambda: dev.lincomb(out, H[:nin], [0.5] * nin, dots=True, mode=_lib.CL_DOT_OUT_ALL)  # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(dev.stream)
        for _ in range(10):
            fn()
        e1.record(dev.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        res[f"nin{nin}_ms"] = round(ms, 3)
        res[f"nin{nin}_GBps"] = round(N * 8 * (nin + 1) / ms / 1e6, 1)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
