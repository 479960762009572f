"""Pins of oracle/variant_oracle.py (NEXT-4: Table 3 model families) against
things other than itself: the degree-1 / both-banks special case equals the separately written
efunc_oracle; partition of unity with a shared global quadratic (Eq. poly-func L400-405 + the
convex combination L347): O == P(q), G == grad P(q) exactly; degree 0 == the normalised RBF
(Eq. nrbf); G == central differences of O; dL/dtheta == central differences of the MSE loss; the
Table 3 parameter counts."""
import numpy as np
import pytest

import oracle as orc
from oracle import variant_oracle as vo
from workloads import synth


def rand_theta(R, banks, degree, seed, log_beta=2.0):
    g = synth.rng(seed, 40)
    lay = vo.layout(banks, degree)
    th = g.normal(scale=0.5, size=(R ** 3, lay["nch"]))
    for key in ("grid", "off"):
        if lay[key] is not None:
            th[:, lay[key]] = log_beta + g.normal(scale=0.3, size=R ** 3)
    if lay["delta"] is not None:
        th[:, lay["delta"]:lay["delta"] + 3] = g.normal(scale=0.1, size=(R ** 3, 3))
    return th


def test_table3_channel_counts():
    # Table 3: # Params at 32^3 for learnable-scale rows
    assert 32 ** 3 * vo.n_channels(vo.GRID, 0) == 65536      # G-5
    assert 32 ** 3 * vo.n_channels(vo.GRID, 1) == 163840     # G-6
    assert 32 ** 3 * vo.n_channels(vo.GRID, 2) == 360448     # G-7
    assert 32 ** 3 * vo.n_channels(vo.OFFSET, 1) == 262144   # Full-1
    assert 64 ** 3 * vo.n_channels(vo.OFFSET, 1) == 2097152  # Full-2
    assert 32 ** 3 * vo.n_channels(vo.BOTH, 1) == 425984     # Full-3 / Full-4
    assert vo.NCOEF[2] == 10 and vo.NCOEF[1] == 4 and vo.NCOEF[0] == 1  # "Deg 2, # 10"


def test_degree1_both_banks_equals_efunc_oracle():
    R = 3
    th = rand_theta(R, vo.BOTH, 1, 1)
    q = synth.rng(2).uniform(-1, 1, size=(23, 3))
    f = vo.forward(th, R, q, vo.BOTH, 1)
    f0 = orc.forward(th, R, q)
    np.testing.assert_allclose(f.O, f0.O, rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(f.G, f0.G, rtol=1e-12, atol=1e-13)
    r = synth.rng(3).normal(size=23)
    g = vo.backward(th, R, q, f, r, vo.BOTH, 1)
    g0 = orc.backward(th, R, q, f0, r)
    np.testing.assert_allclose(g, g0, rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("banks", [vo.GRID, vo.OFFSET, vo.BOTH])
def test_partition_of_unity_shared_quadratic(banks):
    """Every key carries the Taylor expansion of one global quadratic P at its own position, so the
    interpolant reproduces P and its gradient exactly (any beta, any offsets)."""
    R, degree = 3, 2
    gen = synth.rng(7)
    A0 = 0.3
    B = gen.normal(size=3)
    C = gen.normal(size=(3, 3)); C = 0.5 * (C + C.T)
    th = rand_theta(R, banks, degree, 8)
    lay = vo.layout(banks, degree)
    k = orc.node_positions(R)

    def fill(s0, pos):
        th[:, s0 + 1] = A0 + pos @ B + 0.5 * np.einsum("na,ab,nb->n", pos, C, pos)
        th[:, s0 + 2:s0 + 5] = B[None] + pos @ C
        for slot, (a, b) in enumerate(vo.H_IDX):
            th[:, s0 + 5 + slot] = C[a, b]
    if lay["grid"] is not None:
        fill(lay["grid"], k)
    if lay["off"] is not None:
        fill(lay["off"], k + th[:, lay["delta"]:lay["delta"] + 3])
    q = gen.uniform(-1.2, 1.2, size=(31, 3))
    f = vo.forward(th, R, q, banks, degree)
    P = A0 + q @ B + 0.5 * np.einsum("ja,ab,jb->j", q, C, q)
    np.testing.assert_allclose(f.O, P, atol=1e-12)
    np.testing.assert_allclose(f.G, B[None] + q @ C, atol=1e-11)


def test_degree0_is_normalised_rbf():
    R = 3
    th = rand_theta(R, vo.GRID, 0, 9)
    q = synth.rng(10).uniform(-1, 1, size=(11, 3))
    f = vo.forward(th, R, q, vo.GRID, 0)
    k = orc.node_positions(R)
    beta = np.exp(th[:, 0])
    a = beta[None] * np.sum((q[:, None] - k[None]) ** 2, axis=2)
    w = np.exp(-(a - a.min(axis=1, keepdims=True)))
    np.testing.assert_allclose(f.O, (w * th[None, :, 1]).sum(1) / w.sum(1), rtol=1e-13)


@pytest.mark.parametrize("banks,degree", [(vo.GRID, 2), (vo.OFFSET, 1), (vo.OFFSET, 2), (vo.BOTH, 2)])
def test_G_matches_central_differences(banks, degree):
    R = 3
    th = rand_theta(R, banks, degree, 11)
    q = synth.rng(12).uniform(-0.9, 0.9, size=(7, 3))
    f = vo.forward(th, R, q, banks, degree)
    eps = 1e-6
    for ax in range(3):
        dq = np.zeros(3); dq[ax] = eps
        fd = (vo.forward(th, R, q + dq, banks, degree).O - vo.forward(th, R, q - dq, banks, degree).O) / (2 * eps)
        np.testing.assert_allclose(f.G[:, ax], fd, atol=2e-7 * max(1.0, np.abs(fd).max()))


@pytest.mark.parametrize("banks,degree", [(vo.GRID, 2), (vo.OFFSET, 1), (vo.BOTH, 2), (vo.GRID, 0)])
def test_mse_gradient_matches_central_differences(banks, degree):
    R = 2
    th = rand_theta(R, banks, degree, 13)
    q = synth.rng(14).uniform(-1, 1, size=(9, 3))
    o = synth.rng(15).normal(size=9)

    def loss(t):
        return np.mean((vo.forward(t, R, q, banks, degree).O - o) ** 2)
    f = vo.forward(th, R, q, banks, degree)
    r = 2.0 * (f.O - o) / len(o)
    g = vo.backward(th, R, q, f, r, banks, degree)
    eps = 1e-6
    fd = np.zeros_like(th)
    for idx in np.ndindex(*th.shape):
        tp = th.copy(); tp[idx] += eps
        tm = th.copy(); tm[idx] -= eps
        fd[idx] = (loss(tp) - loss(tm)) / (2 * eps)
    np.testing.assert_allclose(g, fd, atol=1e-7 * max(1.0, np.abs(fd).max()))


def test_cosine_stack_b1_is_g6_and_weights():
    """Eq. cosine-series: B = 1 is Config G-6 (w_0 = 1); the weights are the
    separable cosines (reading R-C): w_b(0) = 1, w_b at the lattice point (1, 0, 0) is (-1)^b."""
    R = 3
    th = rand_theta(R, vo.GRID, 1, 50)
    q = synth.rng(51).uniform(-1, 1, size=(13, 3))
    S, GS, fs = vo.cosine_forward([th], R, q)
    f = vo.forward(th, R, q, vo.GRID, 1)
    np.testing.assert_allclose(S, f.O, rtol=0, atol=0)
    np.testing.assert_allclose(GS, f.G, rtol=0, atol=0)
    W, _ = vo.cosine_weights(np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]]), 4)
    np.testing.assert_allclose(W[:, 0], 1.0)
    np.testing.assert_allclose(W[:, 1], [1.0, -1.0, 1.0, -1.0], atol=1e-15)


def test_cosine_stack_gradients_match_central_differences():
    R, B = 2, 3
    ths = [rand_theta(R, vo.GRID, 1, 60 + b) for b in range(B)]
    q = synth.rng(61).uniform(-0.9, 0.9, size=(7, 3))
    o = synth.rng(62).normal(size=7)
    S, GS, fs = vo.cosine_forward(ths, R, q)
    eps = 1e-6
    for ax in range(3):
        dq = np.zeros(3); dq[ax] = eps
        fd = (vo.cosine_forward(ths, R, q + dq)[0] - vo.cosine_forward(ths, R, q - dq)[0]) / (2 * eps)
        np.testing.assert_allclose(GS[:, ax], fd, atol=1e-7 * max(1.0, np.abs(fd).max()))
    dS = 2.0 * (S - o) / len(o)
    g = vo.cosine_backward(ths, R, q, fs, dS)

    def loss(tt):
        return np.mean((vo.cosine_forward(tt, R, q)[0] - o) ** 2)
    for b in range(B):
        for idx in [(0, 0), (3, 1), (5, 2), (7, 4)]:
            tp = [t.copy() for t in ths]; tm = [t.copy() for t in ths]
            tp[b][idx] += eps; tm[b][idx] -= eps
            fd = (loss(tp) - loss(tm)) / (2 * eps)
            assert abs(g[b][idx] - fd) <= 1e-7 * max(1.0, abs(fd)), (b, idx, g[b][idx], fd)
