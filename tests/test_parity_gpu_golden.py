"""GPU parity against the committed golden vectors (made by the reference
library, tests/golden/make_golden.py) and the C restatement oracle -- runs
without the reference tree or oracle/_ref. Bitwise for every operation;
V-cycle histories within 1e-8 relative per cycle (north star)."""
import os

import numpy as np
import pytest

from oracle import restatement as O
from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import keyed_uniform

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_ops.npz")
MESHES = ["unit_square", "unit_square_reversed", "square_ring8", "channel21", "annulus82"]
BCS = {"dirichlet": {}, "mixed": {1: 4}}


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


@pytest.mark.parametrize("name", MESHES)
@pytest.mark.parametrize("bc", sorted(BCS))
@pytest.mark.parametrize("ranks", [1, 2])
def test_device_matches_golden(golden, name, bc, ranks):
    mesh = golden[f"{name}/mesh"].tobytes().decode()
    for level in range(0, 5):
        key = f"{name}/{bc}/L{level}/"
        lmin = max(level - 1, 0)
        dom = H.DistributedDomain(mesh, ranks)
        ctl = H.Controller(dom)
        A = H.StencilOperator(dom, H.LAPLACE, lmin, level, BCS[bc])
        f = [H.ScalarFunction(f"f{i}", dom, lmin, level, BCS[bc]) for i in range(4)]
        x, b, c = golden[key + "x"], golden[key + "b"], golden[key + "c"]
        f[0].upload(level, x)
        f[1].upload(level, b)
        f[2].upload(lmin, c)
        assert np.array_equal(f[0].flags(level), golden[key + "flags"])
        H.apply(A, ctl, f[0], f[3], level)
        assert np.array_equal(f[3].download(level), golden[key + "apply"]), key
        f[3].upload(level, b)
        H.apply(A, ctl, f[0], f[3], level, H.DIRICHLET)
        assert np.array_equal(f[3].download(level), golden[key + "apply_dirichlet_mask"]), key
        H.residual(A, ctl, f[1], f[0], f[3], level)
        assert np.array_equal(f[3].download(level), golden[key + "residual"]), key
        d = H.dot(f[0], f[1], level)
        ref = golden[key + "dot_xb"][0]
        assert abs(d - ref) <= 1e-12 * max(1.0, abs(ref))
        if level > lmin:
            H.restrict_to_coarse(ctl, f[0], f[2], lmin)
            assert np.array_equal(f[2].download(lmin), golden[key + "restrict"]), key
            f[2].upload(lmin, c)
            f[3].upload(level, b)
            H.prolongate(ctl, f[2], f[3], lmin, H.SMOOTH_MASK)
            assert np.array_equal(f[3].download(level), golden[key + "prolongate_smooth_mask"]), key
        H.smooth_jacobi(A, ctl, f[1], f[0], 2.0 / 3.0, level)
        assert np.array_equal(f[0].download(level), golden[key + "jacobi"]), key


def test_device_cfg1_history_matches_golden(golden):
    """BASELINE config 1 history vs the reference's (golden), 1e-8 per cycle."""
    mesh = golden["unit_square/mesh"].tobytes().decode()
    dom = H.DistributedDomain(mesh, 1)
    ctl = H.Controller(dom)
    rhs = H.ScalarFunction("rhs", dom, 0, 6)
    x = H.ScalarFunction("x", dom, 0, 6)
    rhs.upload(6, golden["cfg1/rhs"])
    mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, 6, smoother="jacobi", omega=2.0 / 3.0, coarse_tol=1e-14)
    rep = mg.solve(rhs, x, 6, 0.0, 10)
    ref = golden["cfg1/residuals"]
    assert np.max(np.abs(np.array(rep.residuals) - ref) / ref) <= 1e-8
    assert np.max(np.abs(x.download(6) - golden["cfg1/x"])) <= 1e-10


@pytest.mark.parametrize("mesh_kind", [("channel", 3, 2, 2.0, 1.5), ("annulus", 16, 3, 1.0, 2.0)])
@pytest.mark.parametrize("ranks", [1, 3])
def test_device_matches_restatement_level6(mesh_kind, ranks):
    mesh = H.meshgen.channel(*mesh_kind[1:]) if mesh_kind[0] == "channel" else H.meshgen.annulus(*mesh_kind[1:])
    L = 6
    o = O.Session(mesh, L - 1, L, 4)
    dom = H.DistributedDomain(mesh, ranks)
    ctl = H.Controller(dom)
    A = H.StencilOperator(dom, H.LAPLACE, L - 1, L)
    f = [H.ScalarFunction(f"f{i}", dom, L - 1, L) for i in range(4)]
    x, b = keyed_uniform(mesh, L, 1), keyed_uniform(mesh, L, 2)
    o.set(0, L, x)
    o.set(1, L, b)
    H.interpolate_random(f[0], L, seed=1)
    H.interpolate_random(f[1], L, seed=2)
    H.apply(A, ctl, f[0], f[3], L)
    o.apply(0, 3, L)
    assert np.array_equal(f[3].download(L), o.get(3, L))
    for _ in range(2):
        H.smooth_jacobi(A, ctl, f[1], f[0], 2.0 / 3.0, L)
        o.jacobi(1, 0, 2.0 / 3.0, L)
    assert np.array_equal(f[0].download(L), o.get(0, L))
    H.restrict_to_coarse(ctl, f[0], f[2], L - 1)
    o.restrict(0, 2, L - 1)
    assert np.array_equal(f[2].download(L - 1), o.get(2, L - 1))
    H.prolongate_add(ctl, f[2], f[1], L - 1, H.SMOOTH_MASK)
    o.prolongate(2, 3, L - 1, H.SMOOTH_MASK)
    o.add_scaled(1, 1.0, 3, L, H.SMOOTH_MASK)
    assert np.array_equal(f[1].download(L), o.get(1, L))
