"""GPU parity: every hot-path operation through the C ABI against the
reference library itself (oracle/_ref), on the same seeded inputs.

Bar: bitwise for apply / residual / Jacobi / transfers / BLAS-1 (the kernels
reproduce the reference's term order without FMA); 1e-12 relative
for dot products (different but fixed per-primitive summation order); 1e-8
relative per cycle for V-cycle residual histories (north star)."""
import numpy as np
import pytest

from oracle import ref as R
from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import FIXTURES, keyed_uniform, probe

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")]

MIXED_BC = {1: H.NEUMANN}  # outer boundary free, others DIRICHLET (tests/test_operators.cpp:192-212)


class Rig:
    """Same mesh, ranks, levels and BCs on the device and in the reference."""

    def __init__(self, mesh, ranks, lmin, lmax, nfuncs=4, bc=None):
        self.mesh, self.lmin, self.lmax = mesh, lmin, lmax
        self.dom = H.DistributedDomain(mesh, ranks)  # round robin, as the reference tests
        self.ctl = H.Controller(self.dom)
        self.f = [H.ScalarFunction(f"f{i}", self.dom, lmin, lmax, bc) for i in range(nfuncs)]
        self.A = H.StencilOperator(self.dom, H.LAPLACE, lmin, lmax, bc)
        self.ref = R.RefSession(mesh, ranks, lmin, lmax, nfuncs, bc)

    def set(self, i, level, values):
        self.f[i].upload(level, values)
        self.ref.set(i, level, values)

    def rand(self, i, level, seed, stream=0):
        v = keyed_uniform(self.mesh, level, seed, stream)
        H.interpolate_random(self.f[i], level, seed, stream)
        self.ref.set(i, level, v)
        return v

    def same(self, i, level):
        mine, ref = self.f[i].download(level), self.ref.get(i, level)
        return np.array_equal(mine, ref), mine, ref


def assert_same(rig, i, level, what):
    ok, mine, ref = rig.same(i, level)
    if not ok:
        bad = np.flatnonzero(mine != ref)
        pytest.fail(f"{what}: {bad.size} of {mine.size} differ, first {bad[:5]}: {mine[bad[:5]]} vs {ref[bad[:5]]}")


CASES = [(m, r) for m in FIXTURES for r in (1, 2, 3)]


@pytest.mark.parametrize("mesh_name,ranks", CASES)
def test_device_rng_matches_host_restatement(mesh_name, ranks):
    rig = Rig(FIXTURES[mesh_name](), ranks, 3, 3, 1)
    v = rig.rand(0, 3, seed=7, stream=1)
    assert np.array_equal(rig.f[0].download(3), v)


@pytest.mark.parametrize("mesh_name,ranks", CASES)
@pytest.mark.parametrize("bc", [None, MIXED_BC], ids=["dirichlet", "mixed"])
def test_apply_bitwise(mesh_name, ranks, bc):
    mesh = FIXTURES[mesh_name]()
    for level in range(0, 6):
        rig = Rig(mesh, ranks, level, level, 2, bc)
        rig.rand(0, level, seed=1)
        rig.rand(1, level, seed=5)  # dst pre-filled: masked rows must stay untouched
        for mask in (H.ALL_DOF_FLAGS, H.DIRICHLET, H.SMOOTH_MASK):
            H.apply(rig.A, rig.ctl, rig.f[0], rig.f[1], level, mask)
            rig.ref.apply(0, 1, level, mask)
            assert_same(rig, 1, level, f"apply L{level} mask {mask}")


@pytest.mark.parametrize("mesh_name,ranks", CASES)
def test_residual_bitwise(mesh_name, ranks):
    mesh = FIXTURES[mesh_name]()
    for level in range(0, 7):
        rig = Rig(mesh, ranks, level, level, 3)
        rig.rand(0, level, seed=1)          # rhs
        rig.rand(1, level, seed=2)          # x
        H.residual(rig.A, rig.ctl, rig.f[0], rig.f[1], rig.f[2], level)
        rig.ref.residual(0, 1, 2, level)
        assert_same(rig, 2, level, f"residual L{level}")


@pytest.mark.parametrize("mesh_name,ranks", CASES)
@pytest.mark.parametrize("omega", [2.0 / 3.0, 0.7])
def test_jacobi_sweeps_bitwise(mesh_name, ranks, omega):
    mesh = FIXTURES[mesh_name]()
    for level in (1, 2, 4, 6):
        rig = Rig(mesh, ranks, level, level, 2, MIXED_BC if ranks == 2 else None)
        rig.rand(0, level, seed=3)
        rig.rand(1, level, seed=4)
        for sweep in range(3):
            H.smooth_jacobi(rig.A, rig.ctl, rig.f[0], rig.f[1], omega, level)
            rig.ref.jacobi(0, 1, omega, level)
            assert_same(rig, 1, level, f"jacobi L{level} sweep {sweep}")


@pytest.mark.parametrize("mesh_name,ranks", CASES)
def test_transfers_bitwise(mesh_name, ranks):
    mesh = FIXTURES[mesh_name]()
    for lc in range(0, 6):
        rig = Rig(mesh, ranks, lc, lc + 1, 3, MIXED_BC if ranks == 3 else None)
        rig.rand(0, lc + 1, seed=11)  # fine
        rig.rand(1, lc, seed=12)      # coarse
        for mask in (H.ALL_DOF_FLAGS, H.SMOOTH_MASK):
            H.restrict_to_coarse(rig.ctl, rig.f[0], rig.f[1], lc, mask)
            rig.ref.restrict(0, 1, lc, mask)
            assert_same(rig, 1, lc, f"restrict lc{lc} mask {mask}")
            H.prolongate(rig.ctl, rig.f[1], rig.f[0], lc, mask)
            rig.ref.prolongate(1, 0, lc, mask)
            assert_same(rig, 0, lc + 1, f"prolongate lc{lc} mask {mask}")
        # fused prolongate + add == prolongate into scratch + add_scaled(1.0)
        rig.rand(2, lc + 1, seed=13)
        H.prolongate_add(rig.ctl, rig.f[1], rig.f[2], lc, H.SMOOTH_MASK)
        rig.ref.prolongate(1, 0, lc, H.SMOOTH_MASK)
        rig.ref.add_scaled(2, 1.0, 0, lc + 1, H.SMOOTH_MASK)
        assert_same(rig, 2, lc + 1, f"prolongate_add lc{lc}")


@pytest.mark.parametrize("mesh_name,ranks", CASES)
def test_blas1_bitwise_and_dot(mesh_name, ranks):
    mesh = FIXTURES[mesh_name]()
    level = 4
    rig = Rig(mesh, ranks, level, level, 3, MIXED_BC)
    rig.rand(0, level, seed=21)
    rig.rand(1, level, seed=22)
    rig.rand(2, level, seed=23)
    for mask in (H.ALL_DOF_FLAGS, H.DIRICHLET, H.SMOOTH_MASK):
        H.assign(0.3, rig.f[0], -1.7, rig.f[1], rig.f[2], level, mask)
        rig.ref.assign(0.3, 0, -1.7, 1, 2, level, mask)
        assert_same(rig, 2, level, f"assign mask {mask}")
        H.add_scaled(rig.f[2], 2.5, rig.f[0], level, mask)
        rig.ref.add_scaled(2, 2.5, 0, level, mask)
        assert_same(rig, 2, level, f"add_scaled mask {mask}")
    d_mine = H.dot(rig.f[0], rig.f[1], level)
    d_ref = rig.ref.dot(0, 1, level)
    assert abs(d_mine - d_ref) <= 1e-12 * max(1.0, abs(d_ref))


def test_dot_counts_and_partition_invariance():
    # reference tests/test_functions.cpp:43-86: dot(1,1) counts owned DoFs
    mesh = H.meshgen.unit_square()
    dom = H.DistributedDomain(mesh, 1)
    f = H.ScalarFunction("one", dom, 3, 3)
    H.interpolate(f, 1.0, 3)
    assert H.dot(f, f, 3) == 81.0
    mesh = H.meshgen.square_ring8()
    vals = []
    for ranks in (1, 2, 4, 8):
        dom = H.DistributedDomain(mesh, ranks)
        f = H.ScalarFunction("f", dom, 5, 5)
        H.interpolate_random(f, 5, seed=9)
        vals.append(H.dot(f, f, 5))
    assert vals[1:] == vals[:-1]  # bitwise identical for every rank count


@pytest.mark.parametrize("ranks", [1, 2, 4])
def test_partition_invariance_of_jacobi_and_vcycle(ranks):
    # reference tests/test_operators.cpp:353-370, tests/test_solvers.cpp:464-487
    mesh = H.meshgen.square_ring8()
    out = []
    for rk in (1, ranks):
        dom = H.DistributedDomain(mesh, rk)
        mg = H.GridHierarchy(dom, H.Controller(dom), H.LAPLACE, 1, 4, smoother="jacobi")
        rhs = H.ScalarFunction("rhs", dom, 1, 4)
        x = H.ScalarFunction("x", dom, 1, 4)
        H.interpolate(rhs, probe, 4)
        H.interpolate(x, lambda a, b: np.cos(1.3 * a) - 0.4 * b, 4)
        mg.vcycle(rhs, x, 4)
        out.append(x.download(4))
    assert np.array_equal(out[0], out[1])


def test_interpolate_callable_matches_reference_coordinates():
    mesh = H.meshgen.square_ring8()
    rig = Rig(mesh, 2, 4, 4, 1)
    assert np.array_equal(rig.dom.coords(4), rig.ref.coords(4))
    H.interpolate(rig.f[0], probe, 4)
    xy = rig.ref.coords(4)
    assert np.array_equal(rig.f[0].download(4), probe(xy[:, 0], xy[:, 1]))


def test_flags_match_reference():
    for bc in (None, MIXED_BC, {1: H.NEUMANN, 2: H.NEUMANN, 3: H.NEUMANN}):
        rig = Rig(H.meshgen.channel(3, 2, 2.0, 1.5), 2, 3, 3, 1, bc)
        assert np.array_equal(rig.f[0].flags(3), rig.ref.flags(0, 3))


def test_vcycle_history_cfg1():
    """BASELINE config 1: unit square, L6 -> L0, Jacobi V(2,2) w=2/3, coarse CG
    to 1e-14, rhs U[-1,1] seed 0 on INNER, 10 cycles; per-cycle residual within
    1e-8 relative of the composed reference oracle."""
    mesh = H.meshgen.unit_square()
    L = 6
    rig = Rig(mesh, 1, 0, L, 2)
    rhs = keyed_uniform(mesh, L, seed=0)
    rhs[rig.f[0].flags(L) != H.INNER] = 0.0
    rig.set(0, L, rhs)
    mg = H.GridHierarchy(rig.dom, rig.ctl, H.LAPLACE, 0, L, smoother="jacobi", omega=2.0 / 3.0, coarse_tol=1e-14)
    rep = mg.solve(rig.f[0], rig.f[1], L, 0.0, 10)
    ref_hist = rig.ref.vcycle_jacobi(0, 1, L, 2, 2, 2.0 / 3.0, 1e-14, 10)
    mine = np.array(rep.residuals)
    assert mine.size == 11
    rel = np.abs(mine - ref_hist) / ref_hist
    assert rel.max() <= 1e-8, (mine, ref_hist)
    assert mine[-1] / mine[0] < 1e-4  # converging at ~0.3 per cycle
    xm, xr = rig.f[1].download(L), rig.ref.get(1, L)
    assert np.max(np.abs(xm - xr)) <= 1e-10 * np.max(np.abs(xr))


@pytest.mark.parametrize("mesh_name", ["square_rev", "ring8", "channel21"])
def test_vcycle_history_other_meshes(mesh_name):
    mesh = FIXTURES[mesh_name]()
    L = 5
    rig = Rig(mesh, 2, 1, L, 2)
    rig.rand(0, L, seed=31)
    rig.rand(1, L, seed=32)
    mg = H.GridHierarchy(rig.dom, rig.ctl, H.LAPLACE, 1, L, smoother="jacobi", omega=2.0 / 3.0, coarse_tol=1e-12)
    rep = mg.solve(rig.f[0], rig.f[1], L, 0.0, 6)
    ref_hist = rig.ref.vcycle_jacobi(0, 1, L, 2, 2, 2.0 / 3.0, 1e-12, 6)
    rel = np.abs(np.array(rep.residuals) - ref_hist) / ref_hist
    assert rel.max() <= 1e-8, (rep.residuals, ref_hist)


def test_harmonic_extension_of_linear_data():
    # reference tests/test_solvers.cpp:408-429 (Jacobi smoother here)
    mesh = H.meshgen.unit_square()
    L = 5
    dom = H.DistributedDomain(mesh, 3)
    ctl = H.Controller(dom)
    mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 1, L, smoother="jacobi")
    rhs = H.ScalarFunction("rhs", dom, 1, L)
    x = H.ScalarFunction("x", dom, 1, L)
    lin = lambda a, b: 1.5 + 2.0 * a - 0.75 * b  # noqa: E731
    H.interpolate(rhs, lin, L, H.DIRICHLET)
    rep = mg.solve(rhs, x, L, 1e-12, 60)
    assert rep.converged
    xy = dom.coords(L)
    assert np.max(np.abs(x.download(L) - lin(xy[:, 0], xy[:, 1]))) <= 1e-10


def test_errors_mirror_reference_exceptions():
    mesh = H.meshgen.unit_square()
    dom = H.DistributedDomain(mesh, 1)
    ctl = H.Controller(dom)
    A = H.StencilOperator(dom, H.LAPLACE, 2, 2)
    f = H.ScalarFunction("f", dom, 1, 2)
    g = H.ScalarFunction("g", dom, 1, 2)
    with pytest.raises(H.InvalidArgument):
        H.apply(A, ctl, f, f, 2)  # aliased
    with pytest.raises(H.OutOfRange):
        H.apply(A, ctl, f, g, 1)  # outside A's range
    with pytest.raises(H.InvalidArgument):
        H.smooth_jacobi(A, ctl, f, f, 0.5, 2)
    h = H.ScalarFunction("h", dom, 2, 2, {1: H.NEUMANN})
    H.apply(A, ctl, h, g, 2)  # src under other BCs is fine
    with pytest.raises(H.InvalidArgument):
        H.apply(A, ctl, g, h, 2)  # dst under other BCs is not
    with pytest.raises(H.OutOfRange):
        H.prolongate(ctl, f, g, 2)
    with pytest.raises(H.InvalidArgument):
        H.ScalarFunction("bad", dom, 3, 2)


def test_smoothers_keep_exact_solution_fixed():
    # reference tests/test_operators.cpp:287-310
    rig = Rig(H.meshgen.square_ring8(), 2, 2, 2, 3)
    H.interpolate(rig.f[0], probe, 2)
    H.apply(rig.A, rig.ctl, rig.f[0], rig.f[1], 2)  # consistent rhs
    want = rig.f[0].download(2)
    H.assign(1.0, rig.f[0], 0.0, rig.f[0], rig.f[2], 2)
    H.smooth_jacobi(rig.A, rig.ctl, rig.f[1], rig.f[2], 0.7, 2)
    assert np.array_equal(rig.f[2].download(2), want)


@pytest.mark.parametrize("mesh_name,ranks", [("ring8", 2), ("square_rev", 3), ("channel21", 1), ("tri", 2)])
@pytest.mark.parametrize("form", [H.LAPLACE, H.MASS], ids=["laplace", "mass"])
@pytest.mark.parametrize("bc", [None, MIXED_BC], ids=["dirichlet", "mixed"])
def test_diagonal_bitwise_reference(mesh_name, ranks, form, bc):
    """diagonal(A, d, level) (src/operators.cpp:484-505) against the reference's,
    bitwise, on every owned DoF (DIRICHLET rows included), levels 0-4."""
    mesh = FIXTURES[mesh_name]()
    for level in range(0, 5):
        dom = H.DistributedDomain(mesh, ranks)
        A = H.StencilOperator(dom, form, level, level, bc)
        d = H.ScalarFunction("d", dom, level, level, bc)
        H.diagonal(A, d, level)
        ref = R.RefSession(mesh, ranks, level, level, 1, bc)
        ref.diagonal(int(form), 0, level)
        mine, want = d.download(level), ref.get(0, level)
        assert np.array_equal(mine, want), (level, np.flatnonzero(mine != want)[:5])


def test_diagonal_annulus_perturbed_bitwise():
    """per-face affine stencils (config 3 family): non-trivial diagonals per face"""
    mesh = H.meshgen.perturb(H.meshgen.annulus(16, 4, 1.0, 2.0), 0.1, 2)
    dom = H.DistributedDomain(mesh, 3)
    A = H.StencilOperator(dom, H.LAPLACE, 4, 4)
    d = H.ScalarFunction("d", dom, 4, 4)
    H.diagonal(A, d, 4)
    ref = R.RefSession(mesh, 3, 4, 4, 1)
    ref.diagonal(0, 0, 4)
    assert np.array_equal(d.download(4), ref.get(0, 4))


@pytest.mark.slow
def test_cfg2_shape_vs_reference_level8():
    """BASELINE config 2 mesh (512 macro-faces) at level 8: apply and residual
    bitwise vs the reference on keyed U[-1,1] inputs (seed 1)."""
    mesh = H.meshgen.channel(16, 16)
    L = 8
    rig = Rig(mesh, 1, L, L, 3)
    rig.rand(0, L, seed=1, stream=0)
    rig.rand(1, L, seed=1, stream=1)
    H.apply(rig.A, rig.ctl, rig.f[0], rig.f[2], L)
    rig.ref.apply(0, 2, L)
    assert_same(rig, 2, L, "cfg2 apply L8")
    H.residual(rig.A, rig.ctl, rig.f[1], rig.f[0], rig.f[2], L)
    rig.ref.residual(1, 0, 2, L)
    assert_same(rig, 2, L, "cfg2 residual L8")


@pytest.mark.slow
def test_cfg2_full_size_properties():
    """Config 2 at full size (512 faces, level 10, 268,468,225 DoFs):
    size-independent checks -- residual == b - A x bitwise (fused vs composed),
    the stencil annihilates linear fields on interior rows, Jacobi fixes A^-1 b."""
    mesh = H.meshgen.channel(16, 16)
    L = 10
    dom = H.DistributedDomain(mesh, 1)
    ctl = H.Controller(dom)
    assert dom.owned_count(L)[0] == 268_468_225
    A = H.StencilOperator(dom, H.LAPLACE, L, L)
    x = H.ScalarFunction("x", dom, L, L)
    b = H.ScalarFunction("b", dom, L, L)
    y = H.ScalarFunction("y", dom, L, L)
    r = H.ScalarFunction("r", dom, L, L)
    H.interpolate_random(x, L, seed=1, stream=0)
    H.interpolate_random(b, L, seed=1, stream=1)
    H.apply(A, ctl, x, y, L)
    H.residual(A, ctl, b, x, r, L)
    H.assign(1.0, b, -1.0, y, y, L)
    assert np.array_equal(r.download(L), y.download(L))
    # linear field: interior rows vanish (reference tests/test_operators.cpp:265-285)
    H.interpolate(x, lambda a, c: 1.5 + 2.0 * a - 0.75 * c, L)
    H.apply(A, ctl, x, y, L)
    flags = y.flags(L)
    yv = y.download(L)
    assert np.max(np.abs(yv[flags == H.INNER])) <= 1e-12 * (1 << L) ** 0


def test_graph_replayed_vcycles_bitwise_equal_eager():
    """CUDA-graph replay of the V-cycle is the same computation as eager launches."""
    mesh = H.meshgen.channel(4, 4)
    L = 6
    out = []
    for graphs in (False, True):
        dom = H.DistributedDomain(mesh, 2)
        ctl = H.Controller(dom)
        mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, L, smoother="jacobi")
        mg.use_graphs(graphs)
        rhs = H.ScalarFunction("rhs", dom, 0, L)
        x = H.ScalarFunction("x", dom, 0, L)
        H.interpolate_random(rhs, L, seed=5, flag_mask=H.INNER)
        rep = mg.solve(rhs, x, L, 0.0, 6)
        out.append((x.download(L), rep.residuals, mg.use_graphs()))
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]
    assert out[0][2] == 0 and out[1][2] >= 4


MIXED = {1: H.DIRICHLET, 2: H.NEUMANN}  # channel: Dirichlet inflow side; ring8: Dirichlet outside, Neumann hole


@pytest.mark.parametrize("mesh_name", ["channel21", "ring8"])
@pytest.mark.parametrize("ranks", [1, 3])
def test_vcycle_history_mixed_bc(mesh_name, ranks):
    """Jacobi V(2,2) with Neumann rows (smoothed, transferred on the smooth
    mask) vs the reference's composed cycle under the same boundary map."""
    mesh = FIXTURES[mesh_name]()
    L = 5
    rig = Rig(mesh, ranks, 1, L, 2, MIXED)
    rig.rand(0, L, seed=33)
    mg = H.GridHierarchy(rig.dom, rig.ctl, H.LAPLACE, 1, L, MIXED, smoother="jacobi", omega=2.0 / 3.0,
                         coarse_tol=1e-12)
    rep = mg.solve(rig.f[0], rig.f[1], L, 0.0, 6)
    ref_hist = rig.ref.vcycle_jacobi(0, 1, L, 2, 2, 2.0 / 3.0, 1e-12, 6)
    rel = np.abs(np.array(rep.residuals) - ref_hist) / ref_hist
    assert rel.max() <= 1e-8, (rep.residuals, ref_hist)
    assert rep.residuals[-1] < 0.1 * rep.residuals[0]


@pytest.mark.parametrize("mesh_name", ["channel21", "ring8"])
def test_gridhierarchy_gs_mixed_bc_matches_reference(mesh_name):
    """The reference's own GridHierarchy (hybrid GS) with a Neumann boundary."""
    mesh = FIXTURES[mesh_name]()
    L = 5
    rig = Rig(mesh, 2, 1, L, 2, MIXED)
    rig.rand(0, L, seed=34)
    mg = H.GridHierarchy(rig.dom, rig.ctl, H.LAPLACE, 1, L, MIXED, smoother="gs", coarse_tol=1e-12)
    rep = mg.solve(rig.f[0], rig.f[1], L, 0.0, 6)
    ref_hist = rig.ref.gridhierarchy_solve(0, 1, L, 0.0, 6)
    mine = np.array(rep.residuals)
    assert np.max(np.abs(mine - ref_hist) / ref_hist) <= 1e-8, (mine, ref_hist)


def test_nccl_single_rank_communicator_path():
    """A one-process NCCL communicator (world size 1): dots and the V-cycle's
    coarse right-hand side go through ncclAllReduce, inside CUDA-graph capture
    for the cycles; results are bitwise those of the unconnected domain."""
    mesh = FIXTURES["ring8"]()
    L = 5
    out = []
    for connect in (False, True):
        dom = H.DistributedDomain(mesh, 1, local_ranks=[0])
        if connect:
            dom.connect_nccl(H.DistributedDomain.nccl_unique_id(), 0)
        ctl = H.Controller(dom)
        rhs = H.ScalarFunction("rhs", dom, 1, L)
        x = H.ScalarFunction("x", dom, 1, L)
        H.interpolate_random(rhs, L, seed=35, flag_mask=H.INNER)
        mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 1, L, smoother="jacobi")
        rep = mg.solve(rhs, x, L, 0.0, 5)  # cycles 2.. replay from a graph
        out.append((rep.residuals, H.dot(rhs, x, L), x.download(L), mg.use_graphs()))
    assert out[0][0] == out[1][0] and out[0][1] == out[1][1]
    assert np.array_equal(out[0][2], out[1][2])
    assert out[1][3] > 0  # graphs were replayed with the NCCL allreduce inside


@pytest.mark.parametrize("form", ["MASS", "DIV_X", "DIV_Y", "GRAD_X", "GRAD_Y", "PSPG"])
@pytest.mark.parametrize("mesh_name,ranks", [("square", 1), ("ring8", 2), ("channel21", 3), ("square_rev", 2)])
@pytest.mark.parametrize("bc", [None, MIXED_BC], ids=["dirichlet", "mixed"])
def test_apply_other_forms_bitwise(form, mesh_name, ranks, bc):
    """apply(A, ...) of the P1 MASS, DIV_X/Y, GRAD_X/Y and PSPG operators
    (src/elements.cpp:31-76) bitwise the reference's, every mask, L0-5; and
    r = b - A x for the same operator."""
    mesh = FIXTURES[mesh_name]()
    f = H.FORMS[form]
    for level in range(0, 6):
        rig = Rig(mesh, ranks, level, level, 3, bc)
        rig.A = H.StencilOperator(rig.dom, f, level, level, bc)
        rig.ref.set_form(f)
        rig.rand(0, level, seed=1)
        rig.rand(1, level, seed=5)
        for mask in (H.ALL_DOF_FLAGS, H.DIRICHLET, H.SMOOTH_MASK):
            H.apply(rig.A, rig.ctl, rig.f[0], rig.f[1], level, mask)
            rig.ref.apply(0, 1, level, mask)
            assert_same(rig, 1, level, f"{form} apply L{level} mask {mask}")
        rig.rand(2, level, seed=6)
        H.residual(rig.A, rig.ctl, rig.f[2], rig.f[0], rig.f[1], level)
        rig.ref.residual(2, 0, 1, level)
        assert_same(rig, 1, level, f"{form} residual L{level}")


@pytest.mark.parametrize("form", ["DIV_X", "GRAD_Y", "PSPG"])
def test_apply_other_forms_perturbed_annulus_level7(form):
    """non-right-angled faces (config 3 family) at level 7: the face kernel's
    full column blocks with all seven couplings of the non-symmetric stencils"""
    mesh = H.meshgen.perturb(H.meshgen.annulus(16, 4, 1.0, 2.0), 0.1, 2)
    f = H.FORMS[form]
    rig = Rig(mesh, 2, 7, 7, 2)
    rig.A = H.StencilOperator(rig.dom, f, 7, 7)
    rig.ref.set_form(f)
    rig.rand(0, 7, seed=3)
    H.apply(rig.A, rig.ctl, rig.f[0], rig.f[1], 7)
    rig.ref.apply(0, 1, 7)
    assert_same(rig, 1, 7, f"{form} apply annulus L7")
