"""GPU parity of the P1-P1-PSPG Stokes path (reference src/solvers.cpp:466-753)
through the C ABI against the reference's own StokesSystem / StokesMultigrid
(oracle/_ref), on the same inputs.

Bar: bitwise iterates. uzawa_smooth and stokes_residual are the reference's
call sequences on the bitwise kernels, and the coarse MINRES sums in the
reference's order with glibc's hypot, so every iterate of a solve equals the
reference's bit for bit. Residual norms in a solve history go through dot,
whose per-face partial is a fixed tree here and a sequential loop in the
reference (1e-12 for dots): histories agree within 1e-12
relative per cycle (north star: 1e-8)."""
import numpy as np
import pytest

from oracle import ref as R
from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import keyed_uniform

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")]

CHANNEL_U = {1: H.DIRICHLET, 2: H.DIRICHLET, 3: H.NEUMANN}   # tests/test_solvers.cpp:47-53
ALL_NEUMANN = {1: H.NEUMANN, 2: H.NEUMANN, 3: H.NEUMANN}     # :39-45

MESHES = {
    "channel21": lambda: H.meshgen.channel(2, 1),
    "channel42": lambda: H.meshgen.channel(4, 2, 2.0, 1.0),
    "channel44": lambda: H.meshgen.channel(4, 4),
    "square": H.meshgen.unit_square,
    "ring8": H.meshgen.square_ring8,
}


class StokesRig:
    def __init__(self, mesh, ranks, lmin, lmax, bcu, bcp, multigrid=True, project=False, omega=0.3):
        self.mesh, self.lmin, self.lmax = mesh, lmin, lmax
        self.dom = H.DistributedDomain(mesh, ranks)
        self.ctl = H.Controller(self.dom)
        if multigrid:
            self.S = H.StokesMultigrid(self.dom, self.ctl, lmin, lmax, bcu, bcp, project, omega)
        else:
            self.S = H.StokesSystem(self.dom, lmin, lmax, bcu, bcp)
        self.st = [H.StokesState(n, self.dom, lmin, lmax, bcu, bcp) for n in ("rhs", "x", "r")]
        self.ref = R.RefStokes(mesh, ranks, lmin, lmax, bcu, bcp, project=project, omega=omega)
        probe = R.RefSession(mesh, 1, lmax, lmax, nfuncs=2, bc=bcu)
        self.xy = probe.coords(lmax)
        self.flags_u = probe.flags(0, lmax)
        self.flags_p = R.RefSession(mesh, 1, lmax, lmax, nfuncs=1, bc=bcp).flags(0, lmax)

    def set(self, state, comp, level, v):
        self.st[state].components()[comp].upload(level, v)
        self.ref.set(state, comp, level, v)

    def check(self, state, level, what):
        for comp in range(3):
            mine = self.st[state].components()[comp].download(level)
            ref = self.ref.get(state, comp, level)
            if not np.array_equal(mine.view(np.uint64), ref.view(np.uint64)):
                bad = np.flatnonzero(mine != ref)
                pytest.fail(f"{what} comp {comp}: {bad.size}/{mine.size} differ, first {bad[:4]}: "
                            f"{mine[bad[:4]]} vs {ref[bad[:4]]}")

    def channel_rhs(self, level):
        """fill_channel_rhs (tests/test_solvers.cpp:495-500): Poiseuille on DIRICHLET velocity rows"""
        y = self.xy[:, 1]
        self.set(0, 0, level, np.where(self.flags_u & H.DIRICHLET, 4.0 * y * (1.0 - y), 0.0))
        self.set(0, 1, level, np.zeros(y.size))
        self.set(0, 2, level, np.zeros(y.size))


@pytest.mark.parametrize("mesh_name,bcu", [("channel21", CHANNEL_U), ("square", {}), ("ring8", {1: H.NEUMANN}),
                                           ("channel42", CHANNEL_U)])
@pytest.mark.parametrize("ranks", [1, 2, 3])
@pytest.mark.parametrize("level", [2, 3, 4])
def test_uzawa_and_residual_bitwise(mesh_name, bcu, ranks, level):
    mesh = MESHES[mesh_name]()
    rig = StokesRig(mesh, ranks, level, level, bcu, ALL_NEUMANN, multigrid=False)
    for comp in range(3):
        rig.set(0, comp, level, keyed_uniform(mesh, level, seed=11, stream=comp))
        rig.set(1, comp, level, keyed_uniform(mesh, level, seed=12, stream=comp))
    for sweep, omega in enumerate((0.3, 0.3, 0.7)):
        H.uzawa_smooth(rig.S, rig.ctl, rig.st[0], rig.st[1], level, omega)
        rig.ref.uzawa(level, omega)
        rig.check(1, level, f"uzawa sweep {sweep}")
    H.stokes_residual(rig.S, rig.ctl, rig.st[0], rig.st[1], rig.st[2], level)
    rig.ref.residual(level)
    rig.check(2, level, "stokes_residual")


def test_zero_damping_is_plain_gauss_seidel():
    """tests/test_solvers.cpp:620-648: omega = 0 and p = 0 leave p alone and
    sweep the velocities with plain hybrid Gauss-Seidel"""
    mesh, level = MESHES["channel21"](), 3
    rig = StokesRig(mesh, 2, level, level, CHANNEL_U, ALL_NEUMANN, multigrid=False)
    rig.channel_rhs(level)
    x, y = rig.xy[:, 0], rig.xy[:, 1]
    u1 = np.exp(0.3 * x - 0.2 * y) + 0.1 * x * y
    u2 = np.cos(1.3 * x) - 0.4 * y
    rig.set(1, 0, level, u1)
    rig.set(1, 1, level, u2)
    rig.set(1, 2, level, np.zeros(x.size))
    H.uzawa_smooth(rig.S, rig.ctl, rig.st[0], rig.st[1], level, 0.0)
    A = H.StencilOperator(rig.dom, H.LAPLACE, level, level, CHANNEL_U)
    c1, c2 = (H.ScalarFunction(n, rig.dom, level, level, CHANNEL_U) for n in ("c1", "c2"))
    c1.upload(level, u1)
    c2.upload(level, u2)
    H.smooth_gs(A, rig.ctl, rig.st[0].u1, c1, level)
    H.smooth_gs(A, rig.ctl, rig.st[0].u2, c2, level)
    assert np.array_equal(rig.st[1].u1.download(level), c1.download(level))
    assert np.array_equal(rig.st[1].u2.download(level), c2.download(level))
    assert H.max_abs(rig.st[1].p, level) == 0.0


SOLVES = [  # (mesh, ranks, lmin, lmax, tol, max_cycles): configurations where the reference's coarse MINRES converges
    ("channel42", 1, 1, 2, 1e-8, 15),
    ("channel42", 2, 1, 3, 1e-8, 15),
    ("channel42", 3, 2, 4, 1e-8, 15),
    ("channel44", 1, 2, 3, 1e-8, 15),
    ("channel44", 2, 1, 4, 1e-8, 8),
]


@pytest.mark.parametrize("mesh_name,ranks,lmin,lmax,tol,maxc", SOLVES)
def test_stokes_multigrid_solve_bitwise(mesh_name, ranks, lmin, lmax, tol, maxc):
    mesh = MESHES[mesh_name]()
    rig = StokesRig(mesh, ranks, lmin, lmax, CHANNEL_U, ALL_NEUMANN)
    rig.channel_rhs(lmax)
    ref_res, ref_conv = rig.ref.solve(lmax, tol, maxc)
    rep = rig.S.solve(rig.st[0], rig.st[1], lmax, tol, maxc)
    assert rep.converged == ref_conv
    res = np.array(rep.residuals)
    assert res.size == ref_res.size
    assert np.all(np.abs(res - ref_res) <= 1e-12 * ref_res), \
        f"history differs:\n{rep.history()}vs\n{H.SolveReport(ref_conv, len(ref_res) - 1, list(ref_res)).history()}"
    rig.check(1, lmax, "solution")
    assert rig.S.coarse_iterations() > 0


def test_cavity_with_pressure_projection():
    """tests/test_solvers.cpp:689-719: all-Dirichlet velocity, projected pressure mean"""
    mesh, level = MESHES["square"](), 3
    rig = StokesRig(mesh, 2, 1, level, {}, ALL_NEUMANN, project=True)
    x, y = rig.xy[:, 0], rig.xy[:, 1]
    probe = np.exp(0.3 * x - 0.2 * y) + 0.1 * x * y
    rig.set(0, 0, level, np.where(rig.flags_u & H.DIRICHLET, 0.0, probe))
    rig.set(0, 1, level, np.zeros(x.size))
    rig.set(0, 2, level, np.zeros(x.size))
    ref_res, ref_conv = rig.ref.solve(level, 1e-8, 20)
    rep = rig.S.solve(rig.st[0], rig.st[1], level, 1e-8, 20)
    assert rep.converged and ref_conv
    res = np.array(rep.residuals)
    assert res.size == ref_res.size and np.all(np.abs(res - ref_res) <= 1e-12 * ref_res)
    # the final mean-zero shift uses pressure_mean = dot(p, 1) / dot(1, 1): equal within the dot bar
    mine_p, ref_p = rig.st[1].p.download(level), rig.ref.get(1, 2, level)
    assert np.max(np.abs(mine_p - ref_p)) <= 1e-12 * np.max(np.abs(ref_p))
    for comp in (0, 1):
        assert np.array_equal(rig.st[1].components()[comp].download(level), rig.ref.get(1, comp, level))
    assert abs(rig.S.pressure_mean(rig.st[1].p, level)) <= 1e-9
    u1 = rig.st[1].u1.download(level)
    assert np.all(u1[(rig.flags_u & H.DIRICHLET) != 0] == 0.0)


def test_coarse_minres_failure_is_the_references():
    """channel(2,1) from min level 1: the reference's coarse MINRES stalls above
    1e-12 (its own tests fail there); the device solve fails the same
    way, with the same message and MINRES history"""
    mesh = MESHES["channel21"]()
    rig = StokesRig(mesh, 2, 1, 2, CHANNEL_U, ALL_NEUMANN)
    rig.channel_rhs(2)
    with pytest.raises(R.RefError) as ref_err:
        rig.ref.solve(2, 1e-10, 30)
    with pytest.raises(H.HybRuntimeError) as err:
        rig.S.solve(rig.st[0], rig.st[1], 2, 1e-10, 30)
    assert str(err.value) == str(ref_err.value).split("] ", 1)[1]


def test_stokes_argument_errors():
    mesh = MESHES["channel21"]()
    dom = H.DistributedDomain(mesh, 1)
    ctl = H.Controller(dom)
    with pytest.raises(H.InvalidArgument, match="min_level"):
        H.StokesMultigrid(dom, ctl, 0, 2, CHANNEL_U, ALL_NEUMANN)
    mg = H.StokesMultigrid(dom, ctl, 1, 2, CHANNEL_U, ALL_NEUMANN)
    s = H.StokesState("s", dom, 1, 2, CHANNEL_U, ALL_NEUMANN)
    with pytest.raises(H.OutOfRange):
        mg.vcycle(s, s, 3)
    with pytest.raises(H.InvalidArgument, match="negative"):
        mg.solve(s, s, 2, 1e-6, 3, -1, 2)
    bad = H.StokesState("b", dom, 1, 2, ALL_NEUMANN, ALL_NEUMANN)   # velocity BCs differ from the system's
    with pytest.raises(H.InvalidArgument, match="boundary conditions"):
        H.uzawa_smooth(mg, ctl, s, bad, 2)
