"""NEXT-3 inference: efunc_mesh = O on a lattice (§4.1), Marching
Cubes, vertex normals from one forward pass of Eq. func-normal (§4.5).

Pins: node values against the float64 oracle at sampled nodes; the vertex set against the
Marching Cubes vertex definition (oracle/mesh_oracle.py) on the same node values; the triangles by
topology (every directed edge once, its reverse once: a closed, consistently oriented surface;
Euler characteristic 2 for a sphere, 0 for a torus), outward winding; unit normals against the
oracle's G/|G| at sampled vertices.
"""
import numpy as np
import pytest

import oracle as orc
from oracle import mesh_oracle as mo
from workloads import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2505_21319_b200 as ef  # noqa: E402


def smooth_theta(R, shape, seed):
    """fitted_like_theta with exact values and gradients (no coefficient noise): O is a smooth
    approximation of the shape's SDF, so its zero set has the shape's topology."""
    th = synth.fitted_like_theta(R, shape, seed).astype(np.float64)
    k = orc.node_positions(R)
    kd = k + th[:, 5:8]
    th[:, 1] = shape.sdf(k)
    th[:, 2:5] = shape.grad(k)
    th[:, 9] = shape.sdf(kd)
    th[:, 10:13] = shape.grad(kd)
    return th.astype(np.float32)


def topology(tris, nv):
    t = tris.astype(np.int64)
    assert t.min() >= 0 and t.max() < nv
    assert np.all((t[:, 0] != t[:, 1]) & (t[:, 1] != t[:, 2]) & (t[:, 0] != t[:, 2]))
    e = np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]])
    code = e[:, 0] * nv + e[:, 1]
    u, c = np.unique(code, return_counts=True)
    assert c.max() == 1, "a directed edge is used twice: inconsistent orientation or non-manifold"
    rev = e[:, 1] * nv + e[:, 0]
    assert np.isin(rev, u).all(), "an edge without its twin: the surface is not closed"
    n_edges = len(u) // 2
    used = len(np.unique(t))
    return used - n_edges + len(t)  # Euler characteristic


def run_mesh(shape, R, N, lo, hi, seed=3):
    th = smooth_theta(R, shape, seed)
    m = ef.EFunc(R, th)
    verts, tris, nrm, lat = m.mesh(N, lo, hi, iso=0.0, want_lattice=True)
    torch.cuda.synchronize()
    return th, verts.cpu().numpy(), tris.cpu().numpy(), nrm.cpu().numpy(), lat.cpu().numpy()


def test_mesh_sphere_vertices_topology_normals():
    R, N, lo, hi = 16, 64, (-0.8, -0.8, -0.8), (0.8, 0.8, 0.8)
    sph = synth.Sphere(0.5)
    th, v, t, nrm, lat = run_mesh(sph, R, N, lo, hi)
    # node values vs the oracle at sampled nodes
    P = mo.lattice_points(N, lo, hi).reshape(-1, 3)
    idx = synth.rng(5).choice(N ** 3, 400, replace=False)
    f = orc.forward(th, R, P[idx].astype(np.float32))
    O_gpu = lat.reshape(-1)[idx]
    assert np.abs(O_gpu - f.O).max() / np.abs(f.O).max() <= 1e-5
    # vertex set = the Marching Cubes vertex definition on the same node values
    want = mo.mc_vertices(lat, lo, hi, 0.0)
    assert v.shape == want.shape
    from scipy.spatial import cKDTree
    d, _ = cKDTree(want).query(v)
    assert d.max() <= 2e-6, d.max()
    d2, _ = cKDTree(v).query(want)
    assert d2.max() <= 2e-6
    # closed, oriented, sphere topology
    assert topology(t, len(v)) == 2
    # winding: right-hand normals point outward (from O < 0 to O > 0)
    a, b, c = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
    fn = np.cross(b - a, c - a)
    assert (np.sum(fn * (a + b + c), axis=1) > 0).all()
    # unit normals = G/|G| at the vertices (Eq. func-normal)
    assert np.allclose(np.linalg.norm(nrm, axis=1), 1.0, atol=1e-6)
    sel = synth.rng(6).choice(len(v), 300, replace=False)
    g = orc.forward(th, R, v[sel]).G
    ref = g / np.linalg.norm(g, axis=1, keepdims=True)
    assert np.abs(nrm[sel] - ref).max() <= 2e-5
    # normals of a sphere point radially
    assert (np.sum(nrm * v, axis=1) > 0.9 * np.linalg.norm(v, axis=1)).all()


def test_mesh_torus_is_closed_genus_one():
    R, N, lo, hi = 32, 96, (-0.9, -0.9, -0.9), (0.9, 0.9, 0.9)
    th, v, t, nrm, lat = run_mesh(synth.Torus(), R, N, lo, hi)
    assert len(v) == len(mo.mc_vertices(lat, lo, hi, 0.0))
    assert topology(t, len(v)) == 0


def test_mesh_count_only_and_errors():
    R = 8
    m = ef.EFunc(R, smooth_theta(R, synth.Sphere(0.5), 1))
    verts, tris, nrm, _ = m.mesh(24, want_normals=False)
    assert nrm is None and len(verts) > 0 and len(tris) > 0
    with pytest.raises(ef.EfuncError):
        m.mesh(1)
    with pytest.raises(ef.EfuncError):
        m.mesh(16, lo=(0.0, 0.0, 0.0), hi=(0.0, 1.0, 1.0))
