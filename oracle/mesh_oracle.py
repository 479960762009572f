"""Marching Cubes vertex oracle — TEST INFRASTRUCTURE ONLY (same rules as efunc_oracle.py: only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may use it).

NEXT-3: the paper evaluates O "at 512-resolution grid points. Then, we use
Marching Cubes on the resulting grid" (§4.1). What Marching Cubes fixes
independently of any case table is where its vertices are: one vertex on every lattice edge
whose two end nodes lie on different sides of the iso level (inside: O < iso), at the linear
interpolation of O along that edge. This module writes that definition out with plain numpy
over the lattice, in float64. The triangle table is not re-implemented here; the tests pin the
GPU triangles by topology (closed, consistently oriented, Euler characteristic of the shape).

Parity pins: tests/test_oracle.py::test_mc_vertices_* (brute-force triple loop on a tiny
lattice; vertices of an analytic sphere field lie within the linear-interpolation error of it).
"""
from __future__ import annotations

import numpy as np


def lattice_points(N: int, lo, hi) -> np.ndarray:
    """Node positions [N, N, N, 3] indexed (k, j, i) = (z, y, x): p = lo + (hi - lo) * (i, j, k)/(N - 1)."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    t = np.arange(N, dtype=np.float64) / (N - 1)
    x = lo[0] + (hi[0] - lo[0]) * t
    y = lo[1] + (hi[1] - lo[1]) * t
    z = lo[2] + (hi[2] - lo[2]) * t
    Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
    return np.stack([X, Y, Z], axis=-1)


def mc_vertices(O: np.ndarray, lo, hi, iso: float = 0.0) -> np.ndarray:
    """Vertices [V, 3] of Marching Cubes on the node values O [N, N, N] (z, y, x), one per
    sign-changing lattice edge: p0 + t (p1 - p0), t = (iso - O0) / (O1 - O0). Rows are in the
    order (axis x, y, z) then node index; callers compare as sets."""
    O = np.asarray(O, dtype=np.float64)
    P = lattice_points(O.shape[0], lo, hi)
    inside = O < iso
    out = []
    for ax in (2, 1, 0):  # x, y, z edges (array axis 2 is x)
        sl0 = [slice(None)] * 3
        sl1 = [slice(None)] * 3
        sl0[ax] = slice(0, -1)
        sl1[ax] = slice(1, None)
        s0, s1 = tuple(sl0), tuple(sl1)
        cross = inside[s0] != inside[s1]
        O0, O1 = O[s0][cross], O[s1][cross]
        p0, p1 = P[s0][cross], P[s1][cross]
        t = (iso - O0) / (O1 - O0)
        out.append(p0 + t[:, None] * (p1 - p0))
    return np.concatenate(out, axis=0) if out else np.zeros((0, 3))
