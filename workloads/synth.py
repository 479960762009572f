"""Seeded synthetic inputs for the efunc fit step — shared by tests, the oracle side and bench.

Holds NONE of the method's arithmetic (no softmax, no RBF, no gradients, no optimizer):
only analytic signed-distance shapes, point sampling and parameter initialisation
recipes.  Recipe:

* queries: half uniform in [-1,1]^3, half near-surface = surface sample + N(0, sigma^2 I),
  sigma = 0.01 ("16384 points in the bounding volume and another 16384 points
  in the near-surface region"; sigma is reading R-11), target o = analytic SDF(q).
* shapes: sphere r=0.5 (C1), torus R0=0.5 r0=0.2 axis y (C2/C3/C4), CSG = min(torus,
  max(box 0.35, -sphere 0.45)).
* theta init: s0 = s1 = 7 (beta = e^7), c ~ N(0, 0.1^2), g = 0, Delta = 0
  (reading R-9); Delta is then set by mean-shift by the caller.
* "fitted-like" theta for parity tests: log-scales 7 + N(0, 0.3^2), c = sdf(k) + N(0, 0.01^2),
  g = grad sdf(k) + N(0, 0.05^2), Delta = surface projection of k - k + N(0, 0.003^2).
All draws use numpy Philox generators keyed by (seed, stream-id).
"""
from __future__ import annotations

import numpy as np

NCH = 13


def rng(seed: int, stream: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[seed & 0xFFFFFFFFFFFFFFFF, stream]))


# ----------------------------------------------------------------------------- shapes
class Shape:
    name = "shape"

    def sdf(self, p: np.ndarray) -> np.ndarray:
        raise NotImplementedError

    def grad(self, p: np.ndarray, eps: float = 1e-6) -> np.ndarray:
        p = np.asarray(p, np.float64)
        out = np.empty_like(p)
        for a in range(3):
            e = np.zeros(3); e[a] = eps
            out[:, a] = (self.sdf(p + e) - self.sdf(p - e)) / (2 * eps)
        return out

    def project(self, p: np.ndarray, iters: int = 8) -> np.ndarray:
        """Newton projection onto the zero level set."""
        p = np.array(p, np.float64)
        for _ in range(iters):
            gr = self.grad(p)
            n2 = np.maximum(np.sum(gr * gr, axis=1, keepdims=True), 1e-12)
            p = p - self.sdf(p)[:, None] * gr / n2
        return p

    def sample_surface(self, n: int, g: np.random.Generator) -> np.ndarray:
        out = []
        have = 0
        while have < n:
            p = g.uniform(-1, 1, size=(max(4 * n, 1024), 3))
            p = self.project(p)
            ok = (np.abs(self.sdf(p)) < 1e-7) & np.all(np.abs(p) <= 1.0, axis=1)
            out.append(p[ok]); have += int(ok.sum())
        return np.concatenate(out)[:n]


class Sphere(Shape):
    name = "sphere"

    def __init__(self, r: float = 0.5, center=(0.0, 0.0, 0.0)):
        self.r = r; self.c = np.asarray(center, np.float64)

    def sdf(self, p):
        return np.linalg.norm(np.asarray(p, np.float64) - self.c, axis=1) - self.r

    def sample_surface(self, n, g):
        v = g.normal(size=(n, 3))
        return self.c + self.r * v / np.linalg.norm(v, axis=1, keepdims=True)


class Torus(Shape):
    """Torus around the y axis: major radius R0, tube radius r0."""
    name = "torus"

    def __init__(self, R0: float = 0.5, r0: float = 0.2):
        self.R0 = R0; self.r0 = r0

    def sdf(self, p):
        p = np.asarray(p, np.float64)
        qx = np.sqrt(p[:, 0] ** 2 + p[:, 2] ** 2) - self.R0
        return np.sqrt(qx ** 2 + p[:, 1] ** 2) - self.r0

    def sample_surface(self, n, g):
        u = g.uniform(0, 2 * np.pi, size=4 * n + 64)
        v = g.uniform(0, 2 * np.pi, size=4 * n + 64)
        # area element is proportional to (R0 + r0 cos v): rejection sampling
        acc = g.uniform(0, 1, size=v.size) < (self.R0 + self.r0 * np.cos(v)) / (self.R0 + self.r0)
        u, v = u[acc][:n], v[acc][:n]
        rr = self.R0 + self.r0 * np.cos(v)
        return np.stack([rr * np.cos(u), self.r0 * np.sin(v), rr * np.sin(u)], axis=1)


class Box(Shape):
    name = "box"

    def __init__(self, half: float = 0.35):
        self.b = np.array([half, half, half])

    def sdf(self, p):
        d = np.abs(np.asarray(p, np.float64)) - self.b
        return np.linalg.norm(np.maximum(d, 0), axis=1) + np.minimum(np.max(d, axis=1), 0)

    def sample_surface(self, n, g):
        return _box_surface(self.b, n, g)


class Rotated(Shape):
    """A base shape turned by the rotation M (world = M @ local)."""

    def __init__(self, base: Shape, M: np.ndarray):
        self.base = base; self.M = np.asarray(M, np.float64); self.name = "rot_" + base.name

    def sdf(self, p):
        return self.base.sdf(np.asarray(p, np.float64) @ self.M)

    def sample_surface(self, n, g):
        return self.base.sample_surface(n, g) @ self.M.T


def _box_surface(b: np.ndarray, n: int, g: np.random.Generator) -> np.ndarray:
    """uniform samples on the surface of the box [-b, b]"""
    areas = np.array([b[1] * b[2], b[0] * b[2], b[0] * b[1]] * 2)
    face = g.choice(6, size=n, p=areas / areas.sum())
    p = g.uniform(-1, 1, size=(n, 3)) * b
    ax = face % 3
    p[np.arange(n), ax] = np.where(face < 3, 1.0, -1.0) * b[ax]
    return p


class CSG(Shape):
    """min(torus, max(box(0.35), -sphere(0.45)))."""
    name = "csg"

    def __init__(self):
        self.t = Torus(); self.b = Box(0.35); self.s = Sphere(0.45)

    def sdf(self, p):
        return np.minimum(self.t.sdf(p), np.maximum(self.b.sdf(p), -self.s.sdf(p)))

    def sample_surface(self, n, g):
        """boundary pieces of the three primitives (torus, box, sphere surfaces weighted by area)
        kept where they lie on the CSG surface"""
        areas = np.array([4 * np.pi ** 2 * self.t.R0 * self.t.r0, 24 * 0.35 ** 2, 4 * np.pi * 0.45 ** 2])
        out, have = [], 0
        while have < n:
            m = max(2 * n, 4096)
            k = g.multinomial(m, areas / areas.sum())
            c = np.concatenate([self.t.sample_surface(k[0], g), self.b.sample_surface(k[1], g),
                                self.s.sample_surface(k[2], g)])
            c = c[np.abs(self.sdf(c)) < 1e-9]
            out.append(c); have += len(c)
        p = np.concatenate(out)
        return p[g.permutation(len(p))[:n]]


SHAPES = {"sphere": Sphere, "torus": Torus, "box": Box, "csg": CSG}


def make_shape(name: str) -> Shape:
    return SHAPES[name]()


def c5_shapes(n: int, seed: int) -> list:
    """BASELINE config C5: n seeded shapes cycling torus / sphere / box / CSG, size parameter
    U[0.2, 0.6], each under a random rotation (QR of a Gaussian matrix)."""
    g = rng(seed, 55)
    out = []
    for i in range(n):
        r = g.uniform(0.2, 0.6)
        kind = i % 4
        if kind == 0:
            base = Torus(R0=r, r0=min(0.25, 0.4 * r))
        elif kind == 1:
            base = Sphere(r)
        elif kind == 2:
            base = Box(r / np.sqrt(2.0))
        else:
            base = CSG()
        Q, Rr = np.linalg.qr(g.normal(size=(3, 3)))
        Q = Q * np.sign(np.diag(Rr))
        if np.linalg.det(Q) < 0:
            Q[:, 0] = -Q[:, 0]
        out.append(Rotated(base, Q))
    return out


# ----------------------------------------------------------------------------- batches
def sample_batch(shape: Shape, J: int, seed: int, stream: int = 0, sigma: float = 0.01,
                 near_fraction: float = 0.5):
    """(q [J,3] float32, o [J] float32): J - J_near uniform in the cube, J_near near-surface."""
    g = rng(seed, 1000 + stream)
    jn = int(round(J * near_fraction))
    jv = J - jn
    qv = g.uniform(-1.0, 1.0, size=(jv, 3))
    qn = shape.sample_surface(jn, g) + g.normal(scale=sigma, size=(jn, 3)) if jn else np.zeros((0, 3))
    q = np.concatenate([qv, qn]).astype(np.float32)
    perm = g.permutation(J)
    q = q[perm]
    o = shape.sdf(q.astype(np.float64)).astype(np.float32)
    return np.ascontiguousarray(q), np.ascontiguousarray(o)


def sample_patch(shape: Shape, J: int, seed: int, radius: float = 0.06, sigma: float = 0.01):
    """(q, o): J near-surface points (surface sample + N(0, sigma^2)) confined to the surface patch
    within `radius` of one surface point: a full-density batch, every work item holds 32 queries
    (the near-surface density of C2/C3 at a size the float64 oracle finishes in seconds)."""
    g = rng(seed, 2000)
    centre = shape.sample_surface(1, g)[0]
    pts = []
    have = 0
    while have < J:
        p = shape.sample_surface(8 * J, g)
        p = p[np.linalg.norm(p - centre, axis=1) <= radius]
        pts.append(p)
        have += p.shape[0]
    q = (np.concatenate(pts)[:J] + g.normal(scale=sigma, size=(J, 3))).astype(np.float32)
    o = shape.sdf(q.astype(np.float64)).astype(np.float32)
    return np.ascontiguousarray(q), np.ascontiguousarray(o)


def surface_points(shape: Shape, N: int, seed: int) -> np.ndarray:
    """N surface samples (N = 16384 for mean-shift)."""
    return shape.sample_surface(N, rng(seed, 7)).astype(np.float32)


# ----------------------------------------------------------------------------- parameters
def _lattice_nodes(R: int) -> np.ndarray:
    t = (-1.0 + 2.0 * np.arange(R) / max(R - 1, 1)).astype(np.float32).astype(np.float64)
    if R == 1:
        t = np.zeros(1)
    z, y, x = np.meshgrid(t, t, t, indexing="ij")
    return np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1)


def init_theta(R: int, seed: int, c_std: float = 0.1, log_scale: float = 7.0) -> np.ndarray:
    """Paper init: all log-scales 7, c ~ N(0, c_std^2), g = 0, Delta = 0."""
    g = rng(seed, 11)
    th = np.zeros((R ** 3, NCH), np.float64)
    th[:, 0] = log_scale; th[:, 8] = log_scale
    th[:, 1] = g.normal(scale=c_std, size=R ** 3)
    th[:, 9] = g.normal(scale=c_std, size=R ** 3)
    return th.astype(np.float32)


def fitted_like_theta(R: int, shape: Shape, seed: int, offsets: np.ndarray | None = None,
                      log_scale_std: float = 0.3) -> np.ndarray:
    """A theta resembling a partially fitted state (all 13 channels non-trivial)."""
    g = rng(seed, 12)
    k = _lattice_nodes(R)
    n = R ** 3
    th = np.zeros((n, NCH), np.float64)
    sd = shape.sdf(k); gr = shape.grad(k)
    th[:, 0] = 7.0 + g.normal(scale=log_scale_std, size=n)
    th[:, 1] = sd + g.normal(scale=0.01, size=n)
    th[:, 2:5] = gr + g.normal(scale=0.05, size=(n, 3))
    if offsets is None:
        offsets = shape.project(k) - k + g.normal(scale=0.003, size=(n, 3))
    th[:, 5:8] = offsets
    kd = k + th[:, 5:8]
    th[:, 8] = 7.0 + g.normal(scale=log_scale_std, size=n)
    th[:, 9] = shape.sdf(kd) + g.normal(scale=0.01, size=n)
    th[:, 10:13] = shape.grad(kd) + g.normal(scale=0.05, size=(n, 3))
    return th.astype(np.float32)


def random_theta(R: int, seed: int, log_scale_mean: float = 7.0, log_scale_std: float = 0.5,
                 coef_std: float = 0.5, offset_std: float = 0.05) -> np.ndarray:
    """Fully random theta (every channel non-zero) for small-grid pins."""
    g = rng(seed, 13)
    n = R ** 3
    th = g.normal(scale=coef_std, size=(n, NCH))
    th[:, 0] = log_scale_mean + g.normal(scale=log_scale_std, size=n)
    th[:, 8] = log_scale_mean + g.normal(scale=log_scale_std, size=n)
    th[:, 5:8] = g.normal(scale=offset_std, size=(n, 3))
    return th.astype(np.float32)
