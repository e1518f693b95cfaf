"""The statistics file formats (stats.py:170-228, csvio.py) byte for byte
against files the reference itself wrote (tests/golden/make_golden.py).  CPU."""

import os
import types

import numpy as np

from _golden import GOLDEN, load


def _mod():
    # host-only writers: the package imports without a GPU (no kernel runs here)
    from paper_2604_18536_b200 import stats

    return stats


def test_profile_csv_matches_reference(tmp_path):
    S = _mod()
    rows = load("stats_channel")["nut_rows"]
    d = 3
    prof = S.StatProfile(y=rows[:, 0], y_plus=rows[:, 1], u_mean=rows[:, 2:2 + d].T, rms=rows[:, 2 + d:2 + 2 * d].T,
                         u3=rows[:, 8], u4=rows[:, 9], uuv=rows[:, 10], uw=rows[:, 11], nut_over_nu=rows[:, 12],
                         u_tau=1.0, n_snapshots=3)
    out = tmp_path / "p.csv"
    S.write_profile_csv(out, prof)
    assert out.read_text() == open(os.path.join(GOLDEN, "stats_profile_ref.csv")).read()


def test_snapshot_roundtrip_matches_reference(tmp_path):
    S = _mod()
    arrays, t = S.read_snapshot(os.path.join(GOLDEN, "snapshot_ref"))
    assert t == 0.125 and len(arrays) == 3
    c = load("stats_channel")
    for a in range(3):
        assert np.array_equal(arrays[a], c[f"snap0_{a}"])
    base = tmp_path / "s"
    S.write_snapshot(base, types.SimpleNamespace(u=arrays), 0.125)
    for ext in (".bin", ".txt"):
        with open(str(base) + ext, "rb") as fh, open(os.path.join(GOLDEN, "snapshot_ref" + ext), "rb") as ref:
            assert fh.read() == ref.read()
