"""GPU: stream-ordered host transfers (hyb_function_upload_async /
download_async). Downloads see exactly the state at their call even when later
operations overwrite the function; uploads are seen by later operations."""
import numpy as np
import pytest

from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import keyed_uniform

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ranks", [1, 2])
def test_async_pipeline_matches_synchronous(ranks):
    mesh = H.meshgen.channel(4, 4)
    L = 6
    dom = H.DistributedDomain(mesh, ranks)
    ctl = H.Controller(dom)
    A = H.StencilOperator(dom, H.LAPLACE, L, L)
    x, b, y, r = (H.ScalarFunction(nm, dom, L, L) for nm in ("x", "b", "y", "r"))
    n = dom.owned_count(L)[1]
    steps = 4
    xs = [H.PinnedBuffer(n) for _ in range(steps)]
    bs = [H.PinnedBuffer(n) for _ in range(steps)]
    ys = [H.PinnedBuffer(n) for _ in range(steps)]
    rs = [H.PinnedBuffer(n) for _ in range(steps)]
    for k in range(steps):
        xs[k].array[:] = keyed_uniform(mesh, L, seed=80 + k) if ranks == 1 else np.linspace(-1, 1, n) * (k + 1)
        bs[k].array[:] = np.cos(np.arange(n) * (k + 1))
    for k in range(steps):
        x.upload_async(L, xs[k].array)
        b.upload_async(L, bs[k].array)
        H.apply(A, ctl, x, y, L)
        H.residual(A, ctl, b, x, r, L)
        y.download_async(L, ys[k].array)
        r.download_async(L, rs[k].array)
    dom.synchronize()
    for k in range(steps):
        x.upload(L, xs[k].array, global_order=False)
        b.upload(L, bs[k].array, global_order=False)
        H.apply(A, ctl, x, y, L)
        H.residual(A, ctl, b, x, r, L)
        assert np.array_equal(ys[k].array, y.download(L, global_order=False)), k
        assert np.array_equal(rs[k].array, r.download(L, global_order=False)), k


def test_download_async_sees_state_at_call():
    mesh = H.meshgen.unit_square()
    L = 5
    dom = H.DistributedDomain(mesh, 1)
    f = H.ScalarFunction("f", dom, L, L)
    n = dom.owned_count(L)[1]
    before = keyed_uniform(mesh, L, seed=90)
    f.upload(L, before)
    out = H.PinnedBuffer(n)
    f.download_async(L, out.array)
    H.interpolate(f, 7.0, L)              # overwrites f right after the download was queued
    dom.synchronize()
    assert np.array_equal(out.array, before)
    assert np.all(f.download(L) == 7.0)


def test_async_argument_checks():
    dom = H.DistributedDomain(H.meshgen.unit_square(), 1)
    f = H.ScalarFunction("f", dom, 3, 3)
    with pytest.raises(H.InvalidArgument):
        f.upload_async(3, np.zeros(5))
    with pytest.raises(H.OutOfRange):
        f.download_async(4, np.zeros(5))
    with pytest.raises(ValueError):
        f.upload_async(3, np.zeros(dom.owned_count(3)[1], dtype=np.float32))
