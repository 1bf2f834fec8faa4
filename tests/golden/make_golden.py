#!/usr/bin/env python3
"""Regenerate tests/golden/*.npz from the reference library itself.

Runs the UNMODIFIED reference (oracle/_ref/libhyteg_ref.so, built from
/root/reference/proj/src by oracle/Makefile) on small seeded inputs and stores
inputs and outputs of every hot-path operation. Needs /root/reference only to
build oracle/_ref; the fixtures then travel with the repo so the restatement
and the CUDA path are pinned even where the reference tree is absent.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref as R  # noqa: E402
from tests.helpers import keyed_uniform  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

MESHES = {
    "unit_square": lambda: R.meshgen("unit_square"),
    "unit_square_reversed": lambda: R.meshgen("unit_square_reversed"),
    "square_ring8": lambda: R.meshgen("square_ring8"),
    "channel21": lambda: R.meshgen("channel", 2, 1, 1.0, 1.0),
    "annulus82": lambda: R.meshgen("annulus", 8, 2, 1.0, 2.0),
}
BCS = {"dirichlet": {}, "mixed": {1: 4}}  # mixed: marker 1 NEUMANN, others DIRICHLET


def ops_case(mesh, bc, level, ranks):
    lmin = max(level - 1, 0)
    s = R.RefSession(mesh, ranks, lmin, level, 4, bc)
    out = {}
    x = keyed_uniform(mesh, level, seed=101)
    b = keyed_uniform(mesh, level, seed=102)
    c = keyed_uniform(mesh, lmin, seed=103)
    out.update(x=x, b=b, c=c, flags=s.flags(0, level))
    s.set(0, level, x)
    s.set(1, level, b)
    s.set(2, lmin, c)
    s.apply(0, 3, level)
    out["apply"] = s.get(3, level)
    s.set(3, level, b)
    s.apply(0, 3, level, 2)
    out["apply_dirichlet_mask"] = s.get(3, level)
    s.residual(1, 0, 3, level)
    out["residual"] = s.get(3, level)
    out["dot_xb"] = np.array([s.dot(0, 1, level)])
    if level > lmin:
        s.restrict(0, 2, lmin)
        out["restrict"] = s.get(2, lmin)
        s.set(2, lmin, c)
        s.set(3, level, b)
        s.prolongate(2, 3, lmin, 5)
        out["prolongate_smooth_mask"] = s.get(3, level)
    s.jacobi(1, 0, 2.0 / 3.0, level)
    out["jacobi"] = s.get(0, level)
    s.set(0, level, x)
    s.gs(1, 0, level)
    out["gs"] = s.get(0, level)
    return out


def main():
    cases = {}
    for mname, mk in MESHES.items():
        mesh = mk()
        cases[f"{mname}/mesh"] = np.frombuffer(mesh.encode(), dtype=np.uint8)
        for bname, bc in BCS.items():
            for level in (0, 1, 2, 3, 4):
                for k, v in ops_case(mesh, bc, level, 2).items():
                    cases[f"{mname}/{bname}/L{level}/{k}"] = np.asarray(v)
        # stencils (level 3), all primitives
        s = R.RefSession(mesh, 1, 3, 3, 1)
        st = []
        nprim = R._count(mesh)
        for pid in range(nprim):
            st.append(s.stencil(pid, 3))
        cases[f"{mname}/stencils_L3"] = np.concatenate(st)
        cases[f"{mname}/stencils_L3_len"] = np.array([len(v) for v in st])
    # config 1: unit square L6 -> L0, Jacobi V(2,2) w=2/3, coarse CG 1e-14,
    # rhs U[-1,1] seed 0 on INNER (0 on DIRICHLET), x0 = 0, 10 cycles
    mesh = R.meshgen("unit_square")
    s = R.RefSession(mesh, 1, 0, 6, 2)
    rhs = keyed_uniform(mesh, 6, seed=0)
    rhs[s.flags(0, 6) != 1] = 0.0
    s.set(0, 6, rhs)
    cases["cfg1/rhs"] = rhs
    cases["cfg1/residuals"] = s.vcycle_jacobi(0, 1, 6, 2, 2, 2.0 / 3.0, 1e-14, 10)
    cases["cfg1/x"] = s.get(1, 6)
    # composed Jacobi V-cycle on a mesh with a real coarse system
    mesh = R.meshgen("square_ring8")
    s = R.RefSession(mesh, 1, 1, 5, 2)
    rhs, x0 = keyed_uniform(mesh, 5, seed=31), keyed_uniform(mesh, 5, seed=32)
    s.set(0, 5, rhs)
    s.set(1, 5, x0)
    cases["ring8_vcycle/residuals"] = s.vcycle_jacobi(0, 1, 5, 2, 2, 2.0 / 3.0, 1e-12, 6)
    cases["ring8_vcycle/x"] = s.get(1, 5)
    path = os.path.join(HERE, "reference_ops.npz")
    np.savez_compressed(path, **cases)
    print(f"wrote {path}: {len(cases)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
