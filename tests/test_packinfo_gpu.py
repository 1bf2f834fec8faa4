"""The PackInfo extension point (communication.hpp:24-34) driven by
Controller::sync (src/communication.cpp:126-173) through the C ABI: a
tracing PackInfo sees exactly the reference Controller's messages, in its
unpack order (same-rank pairs as local_copy, co-resident ranks through
messages), on 5 meshes x 1-4 ranks x every direction sequence."""
import struct

import numpy as np
import pytest

from oracle import ref as R
from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import FIXTURES

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")]


class TracePack(H.PackInfo):
    def __init__(self):
        self.log = []

    def pack(self, sender, receiver, direction, level):
        return struct.pack("<4Q", sender, receiver, direction, level)

    def unpack(self, receiver, sender, direction, level, data):
        self.log.append((receiver, sender, direction, level, *struct.unpack("<4Q", data)))
        return len(data)


SEQS = [[0, 1, 2, 3], [3, 2, 1, 0], [1], [2, 2], [0, 3, 1]]


@pytest.mark.parametrize("mesh_name", list(FIXTURES))
@pytest.mark.parametrize("ranks", [1, 2, 4])
def test_packinfo_schedule_matches_reference(mesh_name, ranks):
    mesh = FIXTURES[mesh_name]()
    dom = H.DistributedDomain(mesh, ranks)
    ctl = H.Controller(dom)
    info = TracePack()
    ctl.register_pack_info(7, info)
    for seq in SEQS:
        info.log.clear()
        ctl.sync(7, 2, seq)
        ref = R.controller_trace(mesh, ranks, 2, seq)
        assert np.array_equal(np.array(info.log, dtype=np.int64).reshape(-1, 8), ref), seq


def test_packinfo_errors():
    mesh = FIXTURES["square"]()
    dom = H.DistributedDomain(mesh, 2)
    ctl = H.Controller(dom)
    with pytest.raises(H.InvalidArgument, match="no PackInfo"):
        ctl.sync(3, 1, [0])

    class Greedy(TracePack):
        def unpack(self, receiver, sender, direction, level, data):
            return len(data) - 1  # leaves a byte unread

    ctl.register_pack_info(3, Greedy())
    with pytest.raises(H.LogicError, match="not fully consumed"):
        ctl.sync(3, 1, [1])

    class Broken(TracePack):
        def pack(self, sender, receiver, direction, level):
            raise ValueError("boom")

    ctl.register_pack_info(4, Broken())
    with pytest.raises(H.HybRuntimeError, match="pack failed"):
        ctl.sync(4, 1, [2])
    with pytest.raises(H.InvalidArgument, match="direction"):
        ctl.sync(4, 1, [5])
