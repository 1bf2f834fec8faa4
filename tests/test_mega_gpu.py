"""The coarse end of Jacobi V-cycles as one cooperative kernel (mega.cuh):
solves with it are bitwise the solves without it -- residual histories and
iterates -- for V(2,2) / V(1,1) / V(3,1), min levels 0 and 1, Dirichlet and
mixed boundaries, the whole cycle in the kernel (config 1) and only its coarse
end (top levels above the cutoff), FMG and PCG."""
import numpy as np
import pytest

from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import FIXTURES, keyed_uniform

pytestmark = pytest.mark.gpu


def solve(mesh, L, lmin, nu, mega, bc=None, max_n=64, cycles=6, how="solve"):
    dom = H.DistributedDomain(mesh, 1)
    ctl = H.Controller(dom)
    mg = H.GridHierarchy(dom, ctl, H.LAPLACE, lmin, L, bc=bc, smoother="jacobi",
                         coarse_tol=1e-14 if L <= 6 else 1e-12)
    mg.use_mega(mega, max_n)
    rhs, x = H.ScalarFunction("b", dom, lmin, L, bc), H.ScalarFunction("x", dom, lmin, L, bc)
    rhs.upload(L, keyed_uniform(mesh, L, 9))
    if how == "solve":
        rep = mg.solve(rhs, x, L, 0.0, cycles, *nu)
    elif how == "fmg":
        rep = mg.fmg(rhs, x, L, 1e-9, cycles, *nu)
    else:
        rep = mg.pcg(rhs, x, L, cycles, 0.0, *nu)
    return np.array(rep.residuals), x.download(L), mg.use_mega()


@pytest.mark.parametrize("mesh_name", ["square", "ring8", "channel21"])
@pytest.mark.parametrize("nu", [(2, 2), (1, 1), (3, 1)])
@pytest.mark.parametrize("lmin", [0, 1])
def test_mega_cycle_bitwise(mesh_name, nu, lmin):
    mesh = FIXTURES[mesh_name]()
    # a mixed case where the mesh has several boundary markers (an all-Neumann square is singular)
    mixed = {1: H.DIRICHLET, 2: H.DIRICHLET, 3: H.NEUMANN} if mesh_name == "channel21" else None
    for L, bc in ((6, None), (8, mixed)):
        on = solve(mesh, L, lmin, nu, True, bc)
        off = solve(mesh, L, lmin, nu, False, bc)
        assert on[2] > 0 and off[2] == 0
        assert np.array_equal(on[0], off[0]), (mesh_name, nu, lmin, L)
        assert np.array_equal(on[1], off[1]), (mesh_name, nu, lmin, L)


@pytest.mark.parametrize("how,nu", [("fmg", (2, 2)), ("pcg", (1, 1))])
def test_mega_fmg_pcg_bitwise(how, nu):
    mesh = H.meshgen.channel(4, 4)
    on = solve(mesh, 8, 0, nu, True, cycles=8, how=how)
    off = solve(mesh, 8, 0, nu, False, cycles=8, how=how)
    assert on[2] > 0
    assert np.array_equal(on[0], off[0]) and np.array_equal(on[1], off[1])


def test_mega_cutoffs():
    mesh = H.meshgen.channel(2, 2)
    ref = solve(mesh, 7, 0, (2, 2), False)
    for max_n in (4, 16, 128):
        got = solve(mesh, 7, 0, (2, 2), True, max_n=max_n)
        assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1]), max_n
