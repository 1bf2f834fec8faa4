"""CPU tests of the Stokes path's host pieces (no device): the min-level
monolithic matrix StokesMultigrid solves is bitwise the reference's
(constrained_stokes_matrix, src/solvers.cpp:578-592, checked against
oracle/_ref), and the coarse MINRES's hypot is glibc's (the reference's
minres_solve calls std::hypot, src/solvers.cpp:289)."""
import ctypes
import math

import numpy as np
import pytest

from oracle import ref as R
from paper_1805_10167_b200 import hytegrid as H

needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")

CHANNEL_U = {1: H.DIRICHLET, 2: H.DIRICHLET, 3: H.NEUMANN}   # channel_velocity_bc (tests/test_solvers.cpp:47-53)
ALL_NEUMANN = {1: H.NEUMANN, 2: H.NEUMANN, 3: H.NEUMANN}     # all_neumann (:39-45)


@needs_ref
@pytest.mark.parametrize("mesh,bcu,bcp,level", [
    ("channel21", CHANNEL_U, ALL_NEUMANN, 1),
    ("channel21", CHANNEL_U, ALL_NEUMANN, 2),
    ("channel42", CHANNEL_U, ALL_NEUMANN, 1),
    ("square", {}, ALL_NEUMANN, 1),
    ("square", {}, ALL_NEUMANN, 3),
    ("ring8", {1: H.DIRICHLET}, {1: H.DIRICHLET}, 2),
    ("annulus", {2: H.NEUMANN}, ALL_NEUMANN, 2),
])
def test_stokes_coarse_matrix_bitwise(mesh, bcu, bcp, level):
    text = {"channel21": H.meshgen.channel(2, 1), "channel42": H.meshgen.channel(4, 2, 2.0, 1.0),
            "square": H.meshgen.unit_square(), "ring8": H.meshgen.square_ring8(),
            "annulus": H.meshgen.annulus(8, 2, 1.0, 2.0)}[mesh]
    r, c, v = H.stokes_matrix_host(text, level, bcu, bcp)
    ref = R.RefStokes(text, 1, level, level, bcu, bcp)
    rr, rc, rv = ref.matrix(level)
    assert np.array_equal(r, rr) and np.array_equal(c, rc)
    assert np.array_equal(v.view(np.uint64), rv.view(np.uint64))


def test_coarse_hypot_is_glibc():
    libm = ctypes.CDLL("libm.so.6")
    libm.hypot.restype = ctypes.c_double
    libm.hypot.argtypes = [ctypes.c_double, ctypes.c_double]
    rng = np.random.default_rng(7)
    n = 200_000
    a = rng.uniform(-1, 1, n) * 10.0 ** rng.uniform(-12, 12, n)
    b = rng.uniform(-1, 1, n) * 10.0 ** rng.uniform(-12, 12, n)
    b[::3] = a[::3] * rng.uniform(0.5, 2, a[::3].size)   # comparable magnitudes: the correction branch
    b[1::97] = 0.0
    bad = 0
    for x, y in zip(a.tolist(), b.tolist()):
        if H.lib.hyb_coarse_hypot(x, y) != libm.hypot(x, y):
            bad += 1
    assert bad == 0
    # and it is not simply the correctly rounded value (glibc is not), so the pin means something
    assert H.lib.hyb_coarse_hypot(3.0, 4.0) == 5.0 and math.isclose(H.lib.hyb_coarse_hypot(1e-3, 1e-3), math.hypot(1e-3, 1e-3))
