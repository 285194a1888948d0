"""Helpers for the -m gpu parity tests (CUDA path vs reference golden vectors)."""

import numpy as np

from paper_2201_09212_b200.solver import SolverConfig
from paper_2201_09212_b200.system import make_packed


def packed(d):
    return make_packed(int(d["n"]), d["indptr"], d["indices"], d["data"], d["b"], d["col_i"], d["col_j"],
                       d["frames"], d["mu"], d["mu2"], d["phi"])


def config(d):
    return SolverConfig(**d["cfg"])


def relerr(a, b):
    a = np.asarray(a, float).ravel()
    b = np.asarray(b, float).ravel()
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))
