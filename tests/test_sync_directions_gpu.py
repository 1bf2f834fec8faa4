"""GPU: sync(c, f, level, span<Direction>) (src/function.cpp:234-237) --
the reference's relay directions one at a time and in any order -- and the
raw values(id, level) access, against the reference library. Every slot of
every primitive (owned and ghost) is set to distinct random values on both
sides, a direction sequence runs, and every slot must agree bitwise, except
an edge's halo row 0, which the device does not store (no P1 operation
reads it; the reference writes it only in FACE_TO_EDGE)."""
import numpy as np
import pytest

from oracle import ref as R
from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import FIXTURES

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")]

SEQUENCES = [[0], [1], [2], [3], [1, 2], [3, 0], [2, 1], [0, 1, 2, 3], [3, 2, 1, 0], [1, 1, 3]]


def _halo0_mask(mesh, pid, level, size):
    nv, ne, nf = H.mesh_counts(mesh)
    keep = np.ones(size, dtype=bool)
    if nv <= pid < nv + ne:
        n = 1 << level
        j = 0
        while (n + 1) + j * (2 * n + 1) < size:
            a = (n + 1) + j * (2 * n + 1)
            keep[a:a + n + 1] = False
            j += 1
    return keep


@pytest.mark.parametrize("mesh_name", ["square", "ring8", "channel21", "tri"])
@pytest.mark.parametrize("ranks", [1, 2, 3])
def test_sync_directions_bitwise(mesh_name, ranks):
    mesh = FIXTURES[mesh_name]()
    nv, ne, nf = H.mesh_counts(mesh)
    rng = np.random.default_rng(ranks)
    for level in (0, 1, 2, 4):
        for seq in SEQUENCES:
            dom = H.DistributedDomain(mesh, ranks)
            ctl = H.Controller(dom)
            f = H.ScalarFunction("f", dom, level, level)
            ref = R.RefSession(mesh, ranks, level, level, 1)
            for pid in range(nv + ne + nf):
                v = rng.uniform(-1, 1, ref.values(0, pid, level).size)
                ref.set_values(0, pid, level, v)
                f.set_values(pid, level, v)
            H.sync(ctl, f, level, seq)
            ref.sync_dirs(0, level, seq)
            for pid in range(nv + ne + nf):
                mine, want = f.values(pid, level), ref.values(0, pid, level)
                keep = _halo0_mask(mesh, pid, level, want.size)
                assert mine.size == want.size
                assert np.array_equal(mine[keep], want[keep]), (mesh_name, ranks, level, seq, pid)


def test_full_schedule_equals_sync_all():
    """the four directions in the reference's order reach sync_all's state"""
    mesh = FIXTURES["ring8"]()
    nv, ne, nf = H.mesh_counts(mesh)
    level = 3
    dom = H.DistributedDomain(mesh, 2)
    ctl = H.Controller(dom)
    a, b = H.ScalarFunction("a", dom, level, level), H.ScalarFunction("b", dom, level, level)
    rng = np.random.default_rng(7)
    for pid in range(nv + ne + nf):
        v = rng.uniform(-1, 1, a.values(pid, level).size)
        a.set_values(pid, level, v)
        b.set_values(pid, level, v)
    H.sync(ctl, a, level, H.FULL_SYNC_SCHEDULE)
    H.sync_all(ctl, b, level)
    for pid in range(nv + ne + nf):
        assert np.array_equal(a.values(pid, level), b.values(pid, level)), pid


def test_bad_direction_raises():
    dom = H.DistributedDomain(FIXTURES["square"](), 1)
    f = H.ScalarFunction("f", dom, 2, 2)
    with pytest.raises(H.InvalidArgument):
        H.sync(H.Controller(dom), f, 2, [4])
    with pytest.raises(H.OutOfRange):
        H.sync(H.Controller(dom), f, 3, [0])
