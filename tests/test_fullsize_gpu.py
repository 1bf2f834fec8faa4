"""GPU parity at the benchmarked sizes (VERDICT r01 "do this" #1).

Config 2 (channel(16,16), 512 macro-faces) at levels 9 and 10 -- the face
kernel's column blocks with c0 > 0 (FS_COLS = 256) only occur there -- and
the config-3 mesh (perturbed annulus, 8192 faces) at level 8, every hot
operation compared BITWISE with the plain-C restatement (oracle/hyteg_oracle.c,
itself pinned bitwise to the reference library by tests/test_oracle_pins.py):

  apply (three masks), residual, weighted Jacobi, the reference's hybrid GS,
  restriction, prolongation, prolongate + add, and the two fused cycle
  kernels (residual + restriction; correction + first Jacobi sweep) against
  the composed restatement calls (src/operators.cpp:379-470,
  src/solvers.cpp:71-204, 418-427).

Inputs come from the same keyed generator on both sides (og_keyed_uniform ==
the device's hyb_interpolate_random, checked below), so no 2 GB vectors cross
numpy's RNG. Host RAM: about 6 restatement functions of 2.75 GB (levels 9-10).
"""
import numpy as np
import pytest

from oracle import restatement as O
from paper_1805_10167_b200 import hytegrid as H

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

OMEGA = 2.0 / 3.0


class Pair:
    """The same mesh / levels / functions on the device and in the restatement."""

    def __init__(self, mesh, lmin, lmax, nfuncs, bc=None):
        self.mesh, self.lmin, self.lmax = mesh, lmin, lmax
        self.dom = H.DistributedDomain(mesh, 1)
        self.ctl = H.Controller(self.dom)
        self.A = H.StencilOperator(self.dom, H.LAPLACE, lmin, lmax, bc)
        self.f = [H.ScalarFunction(f"f{i}", self.dom, lmin, lmax, bc) for i in range(nfuncs)]
        self.o = O.Session(mesh, lmin, lmax, nfuncs, bc)

    def rand(self, i, level, seed, stream=0):
        H.interpolate_random(self.f[i], level, seed, stream)
        v = self.o.keyed_uniform(level, seed, stream)
        self.o.set(i, level, v)
        return v

    def check(self, i, level, what):
        mine = self.f[i].download(level)
        want = self.o.get(i, level)
        if not np.array_equal(mine, want):
            bad = np.flatnonzero(mine != want)
            pytest.fail(f"{what}: {bad.size} of {mine.size} differ; first {bad[:5]}: {mine[bad[:5]]} vs "
                        f"{want[bad[:5]]}")
        return mine


@pytest.fixture(scope="module", params=[9, 10], ids=["L9", "L10"])
def cfg2(request):
    L = request.param
    p = Pair(H.meshgen.channel(16, 16), L - 1, L, 5)
    yield p, L
    del p


def test_cfg2_inputs_identical(cfg2):
    p, L = cfg2
    v = p.rand(0, L, seed=1, stream=0)
    assert np.array_equal(p.f[0].download(L), v)


def test_cfg2_apply_masks(cfg2):
    p, L = cfg2
    p.rand(0, L, seed=1, stream=0)
    p.rand(1, L, seed=1, stream=1)  # dst pre-filled: masked-out rows must stay
    for mask in (H.ALL_DOF_FLAGS, H.DIRICHLET, H.SMOOTH_MASK):
        H.apply(p.A, p.ctl, p.f[0], p.f[1], L, mask)
        p.o.apply(0, 1, L, mask)
        p.check(1, L, f"apply L{L} mask {mask}")


def test_cfg2_residual(cfg2):
    p, L = cfg2
    p.rand(0, L, seed=1, stream=1)  # rhs
    p.rand(1, L, seed=1, stream=0)  # x
    H.residual(p.A, p.ctl, p.f[0], p.f[1], p.f[2], L)
    p.o.residual(0, 1, 2, L)
    p.check(2, L, f"residual L{L}")


def test_cfg2_jacobi_two_sweeps(cfg2):
    p, L = cfg2
    p.rand(0, L, seed=3)
    p.rand(1, L, seed=4)
    for s in range(2):
        H.smooth_jacobi(p.A, p.ctl, p.f[0], p.f[1], OMEGA, L)
        p.o.jacobi(0, 1, OMEGA, L)
    p.check(1, L, f"jacobi L{L}")


def test_cfg2_gauss_seidel_sweep(cfg2):
    p, L = cfg2
    p.rand(0, L, seed=5)
    p.rand(1, L, seed=6)
    H.smooth_gs(p.A, p.ctl, p.f[0], p.f[1], L)
    p.o.gs(0, 1, L)
    p.check(1, L, f"smooth_gs L{L}")


def test_cfg2_transfers(cfg2):
    p, L = cfg2
    lc = L - 1
    p.rand(0, L, seed=11)
    p.rand(1, lc, seed=12)
    for mask in (H.ALL_DOF_FLAGS, H.SMOOTH_MASK):
        H.restrict_to_coarse(p.ctl, p.f[0], p.f[1], lc, mask)
        p.o.restrict(0, 1, lc, mask)
        p.check(1, lc, f"restrict {L}->{lc} mask {mask}")
        H.prolongate(p.ctl, p.f[1], p.f[0], lc, mask)
        p.o.prolongate(1, 0, lc, mask)
        p.check(0, L, f"prolongate {lc}->{L} mask {mask}")
    # fused prolongate + add (solvers.cpp:421-422) == prolongate into scratch + add_scaled
    p.rand(2, L, seed=13)
    H.prolongate_add(p.ctl, p.f[1], p.f[2], lc, H.SMOOTH_MASK)
    p.o.prolongate(1, 3, lc, H.SMOOTH_MASK)
    p.o.add_scaled(2, 1.0, 3, L, H.SMOOTH_MASK)
    p.check(2, L, f"prolongate_add {lc}->{L}")


def test_cfg2_fused_residual_restrict(cfg2):
    """hyb_residual_restrict == apply + assign + restrict_to_coarse (solvers.cpp:418-420)."""
    p, L = cfg2
    lc = L - 1
    p.rand(0, L, seed=71)  # rhs
    p.rand(1, L, seed=72)  # x
    H.residual_restrict(p.A, p.ctl, p.f[0], p.f[1], p.f[2], p.f[3], lc)
    p.o.residual(0, 1, 2, L)
    p.o.restrict(2, 3, lc, H.ALL_DOF_FLAGS)
    p.check(3, lc, f"residual_restrict {L}->{lc}")


def test_cfg2_fused_correction_jacobi(cfg2):
    """hyb_prolongate_add_jacobi == prolongate + add_scaled on the smooth mask +
    smooth_jacobi (solvers.cpp:421-427 with the Jacobi smoother)."""
    p, L = cfg2
    lc = L - 1
    p.rand(0, L, seed=81)   # rhs
    p.rand(1, L, seed=82)   # x
    p.rand(2, lc, seed=83)  # coarse correction
    H.prolongate_add_jacobi(p.A, p.ctl, p.f[2], p.f[0], p.f[1], OMEGA, lc)
    p.o.prolongate(2, 4, lc, H.SMOOTH_MASK)
    p.o.add_scaled(1, 1.0, 4, L, H.SMOOTH_MASK)
    p.o.jacobi(0, 1, OMEGA, L)
    p.check(1, L, f"prolongate_add_jacobi {lc}->{L}")


def test_cfg3_mesh_level8_coloured_and_jacobi():
    """Config-3 mesh (annulus(128,32) perturbed +-10%, seed 2; 8192 faces with
    per-face affine stencils, all six couplings non-zero) at level 8: the
    coloured GS kernel the config-3 cycle runs, plus residual and Jacobi."""
    mesh = H.meshgen.perturb(H.meshgen.annulus(128, 32, 1.0, 2.0), 0.1, 2)
    L = 8
    p = Pair(mesh, L, L, 3)
    p.rand(0, L, seed=2, stream=1)
    p.rand(1, L, seed=2, stream=2)
    for s in range(2):
        H.smooth_colored_gs(p.A, p.ctl, p.f[0], p.f[1], L)
        p.o.cgs(0, 1, L)
        p.check(1, L, f"cfg3 coloured GS L{L} sweep {s}")
    H.residual(p.A, p.ctl, p.f[0], p.f[1], p.f[2], L)
    p.o.residual(0, 1, 2, L)
    p.check(2, L, "cfg3 residual L8")
    H.smooth_jacobi(p.A, p.ctl, p.f[0], p.f[1], OMEGA, L)
    p.o.jacobi(0, 1, OMEGA, L)
    p.check(1, L, "cfg3 jacobi L8")


@pytest.mark.parametrize("L", [10, 11])
def test_coloured_gs_large_faces(L):
    """Faces with n >= 1024 run the eight-warp k_cgs_faces path:
    unit square at levels 10 and 11 against og_cgs, two sweeps."""
    mesh = H.meshgen.unit_square()
    p = Pair(mesh, L, L, 2)
    p.rand(0, L, seed=31)
    p.rand(1, L, seed=32)
    for s in range(2):
        H.smooth_colored_gs(p.A, p.ctl, p.f[0], p.f[1], L)
        p.o.cgs(0, 1, L)
        p.check(1, L, f"coloured GS unit square L{L} sweep {s}")
