"""CPU tests: the C ABI library loads and exports its header; host-side setup
(mesh text, macro-primitive graph, partitioners, stencil assembly) is bitwise
the reference's (checked against oracle/_ref, the reference library itself)."""
import ctypes

import numpy as np
import pytest

from oracle import ref as R
from paper_1805_10167_b200 import LIB_PATH, header_symbols
from paper_1805_10167_b200 import hytegrid as H

needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 45
    missing = [s for s in syms if not hasattr(lib, s)]
    assert missing == []


def test_abi_version():
    assert H.lib.hyb_abi_version() == 1


MESHES = [("unit_triangle", ()), ("unit_square", ()), ("unit_square_reversed", ()), ("square_ring8", ()),
          ("channel", (2, 1, 1.0, 1.0)), ("channel", (16, 16, 1.0, 1.0)), ("channel", (3, 2, 2.0, 1.5)),
          ("annulus", (8, 2, 1.0, 2.0)), ("annulus", (128, 32, 1.0, 2.0))]


@needs_ref
@pytest.mark.parametrize("kind,params", MESHES)
def test_meshgen_text_identical(kind, params):
    assert getattr(H.meshgen, kind)(*params) == R.meshgen(kind, *params)


def test_mesh_counts_match_survey_table():
    # SURVEY 8 config table (counts from the reference's own build_setup_graph)
    assert H.mesh_counts(H.meshgen.unit_square()) == (4, 5, 2)
    assert H.mesh_counts(H.meshgen.channel(16, 16)) == (289, 800, 512)
    assert H.mesh_counts(H.meshgen.annulus(128, 32, 1.0, 2.0)) == (4224, 12416, 8192)
    assert H.mesh_counts(H.meshgen.channel(64, 64)) == (4225, 12416, 8192)


def test_mesh_parse_errors_are_invalid_argument():
    with pytest.raises(H.InvalidArgument, match="line"):
        H.mesh_counts("3 1\n0 0 1\n1 0 1\n")  # truncated
    with pytest.raises(H.InvalidArgument, match="degenerate"):
        H.mesh_counts("3 1\n0 0 1\n1 0 1\n2 0 1\n0 1 2 0\n")
    with pytest.raises(H.InvalidArgument, match="twice"):
        H.mesh_counts("3 1\n0 0 1\n1 0 1\n0 1 1\n0 0 2 0\n")


def test_clockwise_triangle_is_flipped():
    cw = "3 1\n0 0 1\n0 1 1\n1 0 1\n0 1 2 0\n"
    # flipping keeps v0 and makes the triangle counter-clockwise: same graph as CCW input
    ccw = "3 1\n0 0 1\n0 1 1\n1 0 1\n0 2 1 0\n"
    for L in (2, 3):
        fid = 3 + 3
        assert np.array_equal(H.stencil_host(cw, L, fid), H.stencil_host(ccw, L, fid))


@needs_ref
@pytest.mark.parametrize("mesh", [H.meshgen.channel(16, 16), H.meshgen.channel(64, 64),
                                  H.meshgen.annulus(128, 32, 1.0, 2.0), H.meshgen.square_ring8()])
@pytest.mark.parametrize("ranks", [1, 2, 3, 4, 8])
def test_partitions_identical(mesh, ranks):
    assert np.array_equal(H.partition_round_robin(mesh, ranks), R.partition(mesh, ranks, 0))
    assert np.array_equal(H.partition_greedy_edgecut(mesh, ranks, 10), R.partition(mesh, ranks, 1, 10))


STENCIL_MESHES = {
    "tri": H.meshgen.unit_triangle(),
    "square": H.meshgen.unit_square(),
    "square_rev": H.meshgen.unit_square_reversed(),
    "ring8": H.meshgen.square_ring8(),
    "channel32": H.meshgen.channel(3, 2, 2.0, 1.5),
    "annulus": H.meshgen.annulus(8, 2, 1.0, 2.0),
    "annulus_perturbed": H.meshgen.perturb(H.meshgen.annulus(16, 4, 1.0, 2.0), 0.1, 2),
}


@needs_ref
@pytest.mark.parametrize("name", sorted(STENCIL_MESHES))
def test_stencils_bitwise(name):
    mesh = STENCIL_MESHES[name]
    nv, ne, nf = H.mesh_counts(mesh)
    for level in range(0, 6):
        s = R.RefSession(mesh, 1, level, level, 1)
        for pid in range(nv + ne + nf):
            if nv <= pid < nv + ne and level == 0:
                continue  # no interior line DoFs: the reference assembles nothing
            mine = H.stencil_host(mesh, level, pid)
            ref = s.stencil(pid, level)
            assert mine.shape == ref.shape and np.array_equal(mine, ref), (name, level, pid, mine, ref)


@needs_ref
@pytest.mark.parametrize("form", ["MASS", "DIV_X", "DIV_Y", "GRAD_X", "GRAD_Y", "PSPG"])
@pytest.mark.parametrize("name", ["square", "annulus_perturbed", "channel32", "ring8"])
def test_other_form_stencils_bitwise(name, form):
    """P1 MASS, DIV_X/Y, GRAD_X/Y and PSPG stencils (src/elements.cpp:31-76,
    src/operators.cpp:95-263) bitwise the reference's, every primitive, L0-4."""
    mesh = STENCIL_MESHES[name]
    nv, ne, nf = H.mesh_counts(mesh)
    f = H.FORMS[form]
    for level in range(0, 5):
        s = R.RefSession(mesh, 1, level, level, 1)
        s.set_form(f)
        for pid in range(nv + ne + nf):
            if nv <= pid < nv + ne and level == 0:
                continue
            mine = H.stencil_host(mesh, level, pid, form=f)
            ref = s.stencil(pid, level)
            assert mine.shape == ref.shape and np.array_equal(mine, ref), (name, form, level, pid, mine, ref)


def test_interior_stencil_of_structured_triangle():
    # reference tests/test_operators.cpp:58-82: {4,-1,-1,-1,-1,0,0}, level independent
    mesh = H.meshgen.unit_triangle()
    fid = 3 + 3
    for level in (2, 3, 4):
        w, nw, s, c, n, se, e, diag = H.stencil_host(mesh, level, fid)
        assert (w, nw, s, c, n, se, e) == (-1.0, 0.0, -1.0, 4.0, -1.0, 0.0, -1.0)
        assert diag == 4.0


def test_stencil_row_sums_vanish():
    # reference tests/test_operators.cpp:120-155 (partition of unity)
    mesh = H.meshgen.square_ring8()
    nv, ne, nf = H.mesh_counts(mesh)
    for pid in range(nv + ne + nf):
        st = H.stencil_host(mesh, 2, pid)
        assert abs(st[:-1].sum()) <= 1e-12


def test_edge_stencil_support_is_3_plus_2F():
    # reference tests/test_operators.cpp:109-118
    mesh = H.meshgen.square_ring8()
    nv, ne, nf = H.mesh_counts(mesh)
    sizes = {len(H.stencil_host(mesh, 2, nv + i)) - 1 for i in range(ne)}
    assert sizes == {5, 7}


def test_mass_stencil_row_sum_and_diagonal():
    # reference tests/test_operators.cpp:84-97
    mesh = H.meshgen.unit_triangle()
    for level in (1, 2, 3):
        h = 1.0 / (1 << level)
        st = H.stencil_host(mesh, level, 6, form=H.MASS)
        assert st[:-1].sum() == pytest.approx(h * h, rel=1e-12)
        assert st[-1] == pytest.approx(h * h / 2, rel=1e-12)


def test_perturbed_mesh_keeps_orientation_and_boundary():
    base = H.meshgen.annulus(128, 32, 1.0, 2.0)
    pert = H.meshgen.perturb(base, 0.1, 2)
    assert H.mesh_counts(pert) == H.mesh_counts(base)
    bl = [ln.split() for ln in base.splitlines()[2:2 + 4224]]
    pl = [ln.split() for ln in pert.splitlines()[2:2 + 4224]]
    moved = sum(1 for a, b in zip(bl, pl) if a[:2] != b[:2])
    assert moved == 4224 - 2 * 128  # every interior vertex, no boundary vertex
    assert all(a[2] == b[2] for a, b in zip(bl, pl))
