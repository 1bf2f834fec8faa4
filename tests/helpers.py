"""Test helpers: host-side restatement of the device keyed RNG and fixtures.

keyed_uniform() reproduces the device generator (kernels.cu key_uniform) in
numpy, for owned DoFs in GlobalDoFMap order, so the oracle receives exactly
the values the GPU generated.
"""
from __future__ import annotations

import numpy as np

from paper_1805_10167_b200 import hytegrid as H

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def owned_keys(mesh_text: str, level: int) -> np.ndarray:
    """Canonical DoF keys (id << 40 ^ c << 20 ^ r) in GlobalDoFMap order."""
    nv, ne, nf = H.mesh_counts(mesh_text)
    n = 1 << level
    keys = [np.arange(nv, dtype=np.uint64) << np.uint64(40)]
    if n >= 2:
        k = np.arange(1, n, dtype=np.uint64)
        eids = np.arange(nv, nv + ne, dtype=np.uint64)
        keys.append(((eids[:, None] << np.uint64(40)) ^ (k[None, :] << np.uint64(20))).ravel())
    if n >= 3:
        rr, cc = [], []
        for r in range(1, n - 1):
            c = np.arange(1, n - r, dtype=np.uint64)
            cc.append(c)
            rr.append(np.full(c.size, r, dtype=np.uint64))
        cc, rr = np.concatenate(cc), np.concatenate(rr)
        fids = np.arange(nv + ne, nv + ne + nf, dtype=np.uint64)
        keys.append(((fids[:, None] << np.uint64(40)) ^ (cc[None, :] << np.uint64(20)) ^ rr[None, :]).ravel())
    return np.concatenate(keys)


def keyed_uniform(mesh_text: str, level: int, seed: int, stream: int = 0, lo: float = -1.0,
                  hi: float = 1.0) -> np.ndarray:
    with np.errstate(over="ignore"):
        sk = _mix64(_mix64(np.array([seed], dtype=np.uint64)) ^ (np.uint64(stream) * np.uint64(0xD1B54A32D192ED03)))
    h = _mix64(sk ^ _mix64(owned_keys(mesh_text, level)))
    u = (h >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return lo + (hi - lo) * u


FIXTURES = {
    "tri": H.meshgen.unit_triangle,
    "square": H.meshgen.unit_square,
    "square_rev": H.meshgen.unit_square_reversed,
    "ring8": H.meshgen.square_ring8,
    "channel21": lambda: H.meshgen.channel(2, 1),
}


def probe(x, y):
    """reference tests/test_operators.cpp:29"""
    return np.exp(0.3 * x - 0.2 * y) + 0.1 * x * y
