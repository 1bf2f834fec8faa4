"""CPU tests: pin the C restatement oracle (oracle/hyteg_oracle.c) against
(1) the committed golden vectors produced by the reference library itself
(tests/golden/reference_ops.npz, tests/golden/make_golden.py) and (2) the
reference library live (oracle/_ref) on more meshes, levels and BCs.
Bitwise for every operation; 1e-12 for V-cycle histories (the restatement's
coarse CG is matrix-free, the reference's uses the assembled matrix)."""
import os

import numpy as np
import pytest

from oracle import ref as R
from oracle import restatement as O
from tests.helpers import keyed_uniform

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_ops.npz")
MESHES = ["unit_square", "unit_square_reversed", "square_ring8", "channel21", "annulus82"]
BCS = {"dirichlet": {}, "mixed": {1: 4}}


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def mesh_of(golden, name):
    return golden[f"{name}/mesh"].tobytes().decode()


@pytest.mark.parametrize("name", MESHES)
@pytest.mark.parametrize("bc", sorted(BCS))
def test_restatement_matches_golden(golden, name, bc):
    mesh = mesh_of(golden, name)
    for level in range(0, 5):
        key = f"{name}/{bc}/L{level}/"
        lmin = max(level - 1, 0)
        o = O.Session(mesh, lmin, level, 4, BCS[bc])
        x, b, c = golden[key + "x"], golden[key + "b"], golden[key + "c"]
        assert np.array_equal(o.keyed_uniform(level, 101), x)  # same inputs as the reference got
        assert np.array_equal(o.flags(level), golden[key + "flags"])
        o.set(0, level, x)
        o.set(1, level, b)
        o.set(2, lmin, c)
        o.apply(0, 3, level)
        assert np.array_equal(o.get(3, level), golden[key + "apply"]), key
        o.set(3, level, b)
        o.apply(0, 3, level, 2)
        assert np.array_equal(o.get(3, level), golden[key + "apply_dirichlet_mask"]), key
        o.residual(1, 0, 3, level)
        assert np.array_equal(o.get(3, level), golden[key + "residual"]), key
        assert o.dot(0, 1, level) == golden[key + "dot_xb"][0]
        if level > lmin:
            o.restrict(0, 2, lmin)
            assert np.array_equal(o.get(2, lmin), golden[key + "restrict"]), key
            o.set(2, lmin, c)
            o.set(3, level, b)
            o.prolongate(2, 3, lmin, 5)
            assert np.array_equal(o.get(3, level), golden[key + "prolongate_smooth_mask"]), key
        o.jacobi(1, 0, 2.0 / 3.0, level)
        assert np.array_equal(o.get(0, level), golden[key + "jacobi"]), key
        o.set(0, level, x)
        o.gs(1, 0, level)
        assert np.array_equal(o.get(0, level), golden[key + "gs"]), key


@pytest.mark.parametrize("name", MESHES)
def test_restatement_stencils_match_golden(golden, name):
    mesh = mesh_of(golden, name)
    o = O.Session(mesh, 3, 3, 1)
    flat, lens = golden[f"{name}/stencils_L3"], golden[f"{name}/stencils_L3_len"]
    pos = 0
    for pid, n in enumerate(lens):
        assert np.array_equal(o.stencil(pid, 3), flat[pos:pos + n]), pid
        pos += n


def test_restatement_cfg1_history_matches_golden(golden):
    mesh = mesh_of(golden, "unit_square")
    o = O.Session(mesh, 0, 6, 7)
    o.set(0, 6, golden["cfg1/rhs"])
    res = o.vcycle_jacobi(0, 1, 6, 2, 2, 2.0 / 3.0, 1e-14, 10)
    ref = golden["cfg1/residuals"]
    assert np.max(np.abs(res - ref) / ref) <= 1e-12
    assert np.max(np.abs(o.get(1, 6) - golden["cfg1/x"])) <= 1e-13


def test_restatement_vcycle_with_coarse_system_matches_golden(golden):
    mesh = mesh_of(golden, "square_ring8")
    o = O.Session(mesh, 1, 5, 7)
    o.set(0, 5, keyed_uniform(mesh, 5, seed=31))
    o.set(1, 5, keyed_uniform(mesh, 5, seed=32))
    res = o.vcycle_jacobi(0, 1, 5, 2, 2, 2.0 / 3.0, 1e-12, 6)
    ref = golden["ring8_vcycle/residuals"]
    assert np.max(np.abs(res - ref) / ref) <= 1e-12
    assert np.max(np.abs(o.get(1, 5) - golden["ring8_vcycle/x"])) <= 1e-12


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("mesh_kind", [("channel", 3, 2, 2.0, 1.5), ("annulus", 16, 3, 1.0, 2.0)])
@pytest.mark.parametrize("level", [5, 6])
def test_restatement_matches_reference_live(mesh_kind, level):
    mesh = R.meshgen(*mesh_kind)
    for bc in BCS.values():
        r = R.RefSession(mesh, 3, level - 1, level, 4, bc)
        o = O.Session(mesh, level - 1, level, 4, bc)
        for fi, seed in ((0, 1), (1, 2)):
            v = keyed_uniform(mesh, level, seed)
            r.set(fi, level, v)
            o.set(fi, level, v)
        r.apply(0, 3, level)
        o.apply(0, 3, level)
        assert np.array_equal(r.get(3, level), o.get(3, level))
        r.jacobi(1, 0, 0.7, level)
        o.jacobi(1, 0, 0.7, level)
        assert np.array_equal(r.get(0, level), o.get(0, level))
        r.gs(1, 0, level)
        o.gs(1, 0, level)
        assert np.array_equal(r.get(0, level), o.get(0, level))
        r.restrict(0, 2, level - 1)
        o.restrict(0, 2, level - 1)
        assert np.array_equal(r.get(2, level - 1), o.get(2, level - 1))
        r.prolongate(2, 3, level - 1)
        o.prolongate(2, 3, level - 1)
        assert np.array_equal(r.get(3, level), o.get(3, level))
        assert r.dot(0, 1, level) == o.dot(0, 1, level)


def test_restatement_fmg_and_pcg_converge():
    """og_fmg / og_pcg have no reference counterpart: they compose the pinned
    primitives. Sanity: FMG reaches discretisation accuracy in one sweep and
    then converges monotonically; PCG's recurrence residual equals the true
    residual of its x."""
    from paper_1805_10167_b200 import hytegrid as H
    mesh = H.meshgen.channel(4, 4)
    o = O.Session(mesh, 2, 6, 11)
    o.set(0, 6, keyed_uniform(mesh, 6, seed=3, lo=-1e-3, hi=1e-3) + 1.0)
    fl = o.flags(6)
    b = o.get(0, 6)
    b[fl != 1] = 0.0
    o.set(0, 6, b)
    res = o.fmg(0, 1, 6, 0, 2, 2, 2.0 / 3.0, 1e-12, 1, 1e-10, 40)
    assert res[1] / res[0] < 0.1 and res[-1] <= 1e-10 * res[0]
    assert np.all(res[2:] < res[1:-1])
    o.set(0, 6, b)
    res = o.pcg(0, 1, 6, 1, 1, 2.0 / 3.0, 1e-12, 10)
    assert res[-1] / res[0] < 1e-6
    o.residual(0, 1, 2, 6)
    assert abs(np.sqrt(o.dot(2, 2, 6)) - res[-1]) <= 1e-6 * res[-1]


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("mesh_kind,lmin,L", [(("channel", 3, 2, 2.0, 1.5), 1, 5), (("annulus", 16, 3, 1.0, 2.0), 1, 5),
                                              (("channel", 16, 8, 1.0, 1.0), 2, 5)])
def test_device_coarse_solver_matches_reference_gridhierarchy(mesh_kind, lmin, L):
    """og_coarse_solver(1) -- the product's coarse solve restated: the
    constrained CSR of the min level and cg_solve's recurrence with the device
    kernels' dot shapes -- inside the reference GridHierarchy's own cycle
    (smooth_gs, min level >= 1) against GridHierarchy::solve itself. The matrix
    is the reference's, so only the dot order differs: <= 1e-10 per cycle.
    channel(16, 8) at level 2 has 2,145 DoFs: the register-resident
    (Chronopoulos-Gear) coarse kernel's path."""
    mesh = R.meshgen(*mesh_kind)
    b = keyed_uniform(mesh, L, seed=9)
    r = R.RefSession(mesh, 1, lmin, L, 2)
    fl = r.flags(0, L)
    b[fl != 1] = 0.0
    r.set(0, L, b)
    ref = r.gridhierarchy_solve(0, 1, L, 0.0, 4)
    for nsm in (148, 2):  # nsm 2: n > nsm * 512 forces the grid-kernel dot shape
        o = O.Session(mesh, lmin, L, 7)
        o.coarse_solver(1, nsm)
        o.set(0, L, b)
        mine = o.vcycle(0, 1, L, 1, 2, 2, 1.0, 1e-12, 4)
        assert np.max(np.abs(mine - ref) / ref) <= 1e-10, (nsm, mine, ref)


def _nz(coo):
    r, c, v = coo
    keep = v != 0.0
    return r[keep], c[keep], v[keep]


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("mesh_kind", [("unit_square",), ("square_ring8",), ("channel", 3, 2, 2.0, 1.5),
                                       ("annulus", 16, 3, 1.0, 2.0)])
@pytest.mark.parametrize("bc", ["dirichlet", "mixed"])
def test_coarse_matrix_bitwise_reference(mesh_kind, bc):
    """The min-level system the device coarse CG solves (hyb_coarse_matrix_host,
    csrc/coarse.cpp) and the one og_coarse_solver(1) restates are bitwise the
    reference GridHierarchy's constrained_matrix (assemble_global_sparse +
    constrain_dirichlet, src/solvers.cpp:358-364), stored zeros aside."""
    from paper_1805_10167_b200 import hytegrid as H
    mesh = R.meshgen(*mesh_kind)
    bcd = BCS[bc]
    for level in range(0, 4):
        ref = _nz(R.RefSession(mesh, 2, level, level, 1, bcd).coarse_matrix(level))
        dev = _nz(H.coarse_matrix_host(mesh, level, 0, bcd))
        og = _nz(O.Session(mesh, level, level, 1, bcd).coarse_matrix(0))
        for a, b in ((ref, dev), (ref, og)):
            for u, w in zip(a, b):
                assert np.array_equal(u, w), (mesh_kind, bc, level)
