"""GPU channel statistics (stats.py:55-167, csrc/stats.cu) against golden
profiles produced by the reference's accumulate_stats on three snapshots of
a channel run with an LES closure (with and without eddy-viscosity profiles)."""

import numpy as np
import pytest

from _dev import grids, vel
from _golden import load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2604_18536_b200 as P

    return P


def _close(got, ref):
    # per column: relative to the column's scale; columns that are zero up to
    # round-off in the reference (the mean wall-normal velocity) against the
    # velocity scale of the profile
    vscale = float(np.max(np.abs(ref[:, 2:5])))
    for c in range(ref.shape[1]):
        scale = max(float(np.max(np.abs(ref[:, c]))), 1e-12 * vscale)
        assert float(np.max(np.abs(got[:, c] - ref[:, c]))) <= 1e-10 * scale + 1e-15 * vscale, c


def test_accumulate_stats_vs_reference_golden(P):
    c = load("stats_channel")
    bounds = [c[f"bounds{a}"] for a in range(3)]
    pg, og = grids(P, bounds, (True, False, True))
    bcs = P.BoundarySpec.channel(dim=3, wall_axis=1)
    snaps = [vel(P, pg, [c[f"snap{i}_{a}"] for a in range(3)]) for i in range(3)]
    nuts = [P.ScalarField(pg, c[f"nut{i}"]) for i in range(3)]
    nu = float(c["nu"])
    for tag, ns in (("plain", None), ("nut", nuts)):
        prof = P.accumulate_stats(snaps, bcs, nu, nut_snapshots=ns)
        assert prof.n_snapshots == 3
        assert prof.column_names()[:4] == ["y", "y_plus", "u0_mean", "u1_mean"]
        _close(prof.rows(), c[f"{tag}_rows"])
        assert abs(prof.u_tau - float(c[f"{tag}_u_tau"])) <= 1e-12 * float(c[f"{tag}_u_tau"])
    with pytest.raises(ValueError):
        P.accumulate_stats(snaps[:1], bcs, nu)
