"""Load the golden fixtures written by tests/golden/make_golden.py."""

import os

import numpy as np

from oracle import stagflow_np as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return {k: z[k] for k in z.files}


def ogrid(case):
    dim = int(case["dim"])
    bounds = [case[f"bounds{a}"] for a in range(dim)]
    return O.OGrid(bounds, tuple(bool(p) for p in case["periodic"]), dtype=np.dtype(str(case["dtype"])))


def vel(case, prefix, dim):
    return [case[f"{prefix}{a}"].copy() for a in range(dim)]


def obcs(g):
    """Periodic, or channel walls on the non-periodic axis (the fixtures'
    only two boundary layouts)."""
    return [("P", "P") if p else (("D", 0.0), ("D", 0.0)) for p in g.periodic]


def _parse_side(txt):
    if txt.startswith("Periodic"):
        return "P"
    if txt.startswith("Symmetric"):
        return "S"
    return ("D", float(txt.split("=")[1].rstrip(")")))


def sides_bcs(case):
    """Oracle BCs from a fixture's ``sides`` (repr strings of the reference's
    Periodic / Dirichlet(values=v) / Symmetric)."""
    return [tuple(_parse_side(str(t)) for t in sd) for sd in case["sides"]]
