"""Debug: Stokes V-cycles on the device vs the reference, cycle by cycle."""
import sys
import numpy as np
sys.path.insert(0, ".")
from tests.test_stokes_gpu import StokesRig, MESHES, CHANNEL_U, ALL_NEUMANN
from paper_1805_10167_b200 import hytegrid as H

for ranks, lmin, lmax in [(1, 1, 3), (2, 1, 3), (1, 2, 3), (2, 2, 3), (2, 1, 2)]:
    mesh = MESHES["channel42"]()
    rig = StokesRig(mesh, ranks, lmin, lmax, CHANNEL_U, ALL_NEUMANN)
    rig.channel_rhs(lmax)
    out = []
    for k in range(4):
        rig.S.vcycle(rig.st[0], rig.st[1], lmax, 2, 2)
        rig.ref.vcycle(lmax, 2, 2)
        diffs = []
        for comp in range(3):
            a = rig.st[1].components()[comp].download(lmax)
            b = rig.ref.get(1, comp, lmax)
            nd = int(np.sum(a != b))
            diffs.append((nd, float(np.max(np.abs(a - b)))))
        out.append(diffs)
    print(ranks, lmin, lmax, out, flush=True)
