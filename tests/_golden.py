"""Helpers to rebuild problems from the golden fixtures (tests/golden/*.npz)."""

import json
import os

import numpy as np

from paper_2407_15049_b200.problem import SdpProblem, SymmetricSparse

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def problem_from(z):
    C = SymmetricSparse(int(z["n"]), z["c_rows"].astype(np.int64), z["c_cols"].astype(np.int64),
                        z["c_vals"].astype(np.float64))
    return SdpProblem(n=int(z["n"]), m=int(z["m"]), C=C, a_con=z["a_con"].astype(np.int64),
                      a_row=z["a_row"].astype(np.int64), a_col=z["a_col"].astype(np.int64),
                      a_val=z["a_val"].astype(np.float64), b=z["b"].astype(np.float64),
                      maximize=bool(z["maximize"]))


def cfg_of(z):
    return json.loads(str(z["cfg"]))


def solve_cases():
    return sorted(f[len("solve_"):-4] for f in os.listdir(GOLDEN) if f.startswith("solve_"))


def ops_cases():
    return sorted(f[len("ops_"):-4] for f in os.listdir(GOLDEN) if f.startswith("ops_"))
