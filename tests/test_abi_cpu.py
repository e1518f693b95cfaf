"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/stagflow_b200.h declares, the ctypes struct layouts match the
C header, and the host-side grid tables equal the oracle's (bitwise)."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import stagflow_np as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "stagflow_b200.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(sfb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2604_18536_b200._native as N

    declared = _declared()
    assert declared, "no declarations parsed"
    lib = ctypes.CDLL(N.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(N.EXPORTED) == declared


def test_abi_version():
    import paper_2604_18536_b200._native as N

    assert N.lib.sfb_abi_version() == N.ABI_VERSION


def test_struct_layout_matches_header(tmp_path):
    import paper_2604_18536_b200._native as N

    prog = tmp_path / "layout.c"
    prog.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "stagflow_b200.h"\n'
        "int main(void){\n"
        'printf("%zu %zu %zu %zu\\n", sizeof(sfb_grid_desc), offsetof(sfb_grid_desc, tables),'
        " offsetof(sfb_grid_desc, width0), offsetof(sfb_grid_desc, val_hi));\n"
        'printf("%zu %zu %zu\\n", sizeof(sfb_stage_args), offsetof(sfb_stage_args, cb), offsetof(sfb_stage_args, force));\n'
        "return 0;}\n"
    )
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    got = [int(x) for x in out]
    G, S = N.GridDesc, N.StageArgs
    assert got[:4] == [ctypes.sizeof(G), G.tables.offset, G.width0.offset, G.val_hi.offset]
    assert got[4:] == [ctypes.sizeof(S), S.cb.offset, S.force.offset]


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("periodic", [(True, True, True), (True, False, True)])
def test_host_tables_match_oracle(dtype, periodic):
    import paper_2604_18536_b200 as P

    bounds = [O.uniform_bounds(0, 2.0, 7), O.tanh_bounds(0, 2.0, 9, 2.0), O.cosine_bounds(0, 1.0, 5)]
    pg = P.Grid(tuple(P.AxisCoords(b) for b in bounds), periodic, dtype=dtype)
    og = O.OGrid(bounds, periodic, dtype)
    packed = pg.packed_tables()
    off = 0
    for a in range(3):
        E = og.shape[a] + 2
        tabs = [og.dx[a], og.du[a], 1 / og.dx[a], 1 / og.du[a], og.w_lo[a], og.w_hi[a],
                og.own_hi[a], og.own_lo[a], og.tan_hi[a], og.tan_lo[a]]
        for t in tabs:
            np.testing.assert_array_equal(packed[off:off + E], np.asarray(t, dtype=dtype).astype(np.float64))
            off += E
        np.testing.assert_array_equal(pg.xb[a], og.xb[a])
        np.testing.assert_array_equal(pg.xc[a], og.xc[a])
    assert off == packed.size


def test_bcs_and_grid_validation():
    import paper_2604_18536_b200 as P

    with pytest.raises(ValueError):
        P.BoundarySpec([(P.Periodic(), P.Dirichlet(0.0))])
    with pytest.raises(P.ConfigurationError):
        P.Grid([P.uniform_grid(0, 1, 4)], (True,))
    with pytest.raises(ValueError):
        P.tanh_grid(0, 1, 4, -1.0)
    g = P.build_grid([P.uniform_grid(0, 1, 4), P.uniform_grid(0, 1, 5)], P.BoundarySpec.all_periodic(2))
    assert g.ext_shape == (6, 7) and g.uniform
    sig = P.plan.bcs_signature(P.BoundarySpec.channel())
    assert sig[2][0] == 1 and sig[0][0] == 0


def test_product_has_no_oracle_dependency():
    """The shipped package must not import the checker."""
    pkg = os.path.join(ROOT, "paper_2604_18536_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, re.M), fn
