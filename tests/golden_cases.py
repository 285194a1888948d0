"""Loader for the committed golden fixtures (``tests/golden/*.npz``)."""

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    with open(os.path.join(GOLDEN, "INDEX.json")) as f:
        return json.load(f)


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    d = {k: z[k] for k in z.files}
    d["cfg"] = json.loads(str(d["cfg"]))
    d["name"] = name
    return d


def oracle_system(d):
    from oracle.vfpi_oracle import System

    return System(
        n=int(d["n"]), indptr=d["indptr"], indices=d["indices"], data=d["data"], b=d["b"],
        col_i=d["col_i"].astype(np.int64), col_j=d["col_j"].astype(np.int64),
        frames=d["frames"].reshape(-1, 3, 3), mu=d["mu"], mu2=d["mu2"], phi=d["phi"],
    )


def oracle_config(d):
    from oracle.vfpi_oracle import Config

    return Config(**d["cfg"])
