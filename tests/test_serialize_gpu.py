"""GPU: one primitive's field record (hyb_function_serialize) is byte-for-byte
the reference's DataCallbacks::serialize (src/field.cpp:157-175) of the same
field after sync_all, and deserialize inverts it (the checkpoint / migration
payload; reference tests/test_primitives.cpp:240-270 checks the
record survives a migration unchanged)."""
import numpy as np
import pytest

from oracle import ref as R
from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import FIXTURES, keyed_uniform

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")]

BCS = {"dirichlet": None, "mixed": {1: H.NEUMANN}, "free": {1: H.NEUMANN, 2: H.NEUMANN, 3: H.NEUMANN}}


def nprims(dom_mesh):
    return R._count(dom_mesh)


@pytest.mark.parametrize("mesh_name", ["square", "square_rev", "ring8", "channel21", "tri"])
@pytest.mark.parametrize("ranks", [1, 3])
@pytest.mark.parametrize("bc", ["dirichlet", "mixed", "free"])
def test_record_matches_the_reference_bytewise(mesh_name, ranks, bc):
    mesh = FIXTURES[mesh_name]()
    lmin, lmax = 0, 4
    bcd = BCS[bc]
    dom = H.DistributedDomain(mesh, ranks)
    f = H.ScalarFunction("u", dom, lmin, lmax, bcd)
    ref = R.RefSession(mesh, ranks, lmin, lmax, 1, bcd)
    for level in range(lmin, lmax + 1):
        v = keyed_uniform(mesh, level, seed=91 + level)
        f.upload(level, v)
        ref.set(0, level, v)
        ref.sync(0, level)
    for prim in range(nprims(mesh)):
        mine, want = f.serialize(prim), ref.serialize(0, prim)
        if mine != want:
            a, b = np.frombuffer(mine, np.uint8), np.frombuffer(want, np.uint8)
            k = int(np.flatnonzero(a[: min(a.size, b.size)] != b[: min(a.size, b.size)])[:1].tolist() or [-1])
            pytest.fail(f"prim {prim}: {a.size} vs {b.size} bytes, first difference at byte {k}")


@pytest.mark.parametrize("mesh_name", ["square", "ring8", "tri"])
@pytest.mark.parametrize("ranks", [1, 2])
def test_deserialize_inverts_serialize(mesh_name, ranks):
    mesh = FIXTURES[mesh_name]()
    lmin, lmax = 1, 5
    bcd = BCS["mixed"]
    dom = H.DistributedDomain(mesh, ranks)
    src = H.ScalarFunction("src", dom, lmin, lmax, bcd)
    dst = H.ScalarFunction("dst", dom, lmin, lmax, bcd)
    for level in range(lmin, lmax + 1):
        H.interpolate_random(src, level, seed=93, stream=level)
    recs = [src.serialize(p) for p in range(nprims(mesh))]
    for p, rec in enumerate(recs):
        dst.deserialize(p, rec)
    for level in range(lmin, lmax + 1):
        assert np.array_equal(src.download(level), dst.download(level)), level
    # ghosts came along too: the records agree without another exchange
    for p, rec in enumerate(recs):
        assert dst.serialize(p) == rec, p


def test_deserialize_rejects_foreign_records():
    mesh = FIXTURES["square"]()
    dom = H.DistributedDomain(mesh, 1)
    f = H.ScalarFunction("f", dom, 1, 3)
    g_levels = H.ScalarFunction("g", dom, 1, 4)
    g_bc = H.ScalarFunction("h", dom, 1, 3, {1: H.NEUMANN, 2: H.NEUMANN, 3: H.NEUMANN, 4: H.NEUMANN})
    H.interpolate_random(f, 3, seed=1)
    face = nprims(mesh) - 1
    rec = f.serialize(face)
    with pytest.raises(H.InvalidArgument):
        g_levels.deserialize(face, rec)          # level count differs
    with pytest.raises(H.InvalidArgument):
        g_bc.deserialize(face, rec)              # boundary flags differ
    with pytest.raises(H.InvalidArgument):
        f.deserialize(face, rec[:-1])            # truncated
    with pytest.raises(H.InvalidArgument):
        f.deserialize(face, rec + b"\0")         # trailing bytes
    with pytest.raises(H.InvalidArgument):
        f.deserialize(0, rec)                    # a vertex cannot take a face's record
    with pytest.raises(H.OutOfRange):
        f.serialize(nprims(mesh))
