"""Pins for the CPU oracle (oracle/efunc_oracle.py) against things other than itself.

Each test names the paper passage / mathematical fact it pins. No GPU needed.
"""
import math
import os

import numpy as np
import pytest

import oracle as orc
from workloads import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden_lines(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return [ln.strip() for ln in fh if ln.strip() and not ln.startswith("#")]


# ----------------------------------------------------------------------------- layout / sizes
def test_param_counts_match_paper_tables():
    """Table 2 and Table 3 Full-4 (L803) parameter counts."""
    for ln in _golden_lines("param_counts.txt"):
        R, ch, val, kind = ln.split()
        n = orc.param_count(int(R), int(ch))
        val = int(val)
        if kind == "exact":
            assert n == val
        elif kind == "rounded_k":
            assert round(n / 1000) * 1000 == val
        elif kind == "rounded_m2":
            assert round(n / 1e4) * 1e4 == val


def test_lattice_endpoints_and_spacing():
    """Reading R-2: inclusive lattice on [-1,1]^3, h = 2/(R-1); node n = x + R(y + Rz)."""
    t = orc.lattice_1d(5)
    assert t[0] == -1.0 and t[-1] == 1.0 and t[2] == 0.0
    k = orc.node_positions(4)
    assert k.shape == (64, 3)
    n = 1 + 4 * (2 + 4 * 3)
    np.testing.assert_array_equal(k[n], [orc.lattice_1d(4)[1], orc.lattice_1d(4)[2], orc.lattice_1d(4)[3]])
    assert orc.lattice_1d(1).tolist() == [0.0]


# ----------------------------------------------------------------------------- forward pins
def _pou_theta(R, seed, A, B):
    """Every key carries the same global linear polynomial P(q) = A + B.q."""
    th = synth.random_theta(R, seed, log_scale_mean=3.0, log_scale_std=1.0).astype(np.float64)
    k = orc.node_positions(R)
    th[:, 1] = A + k @ B
    th[:, 2:5] = B
    th[:, 9] = A + (k + th[:, 5:8]) @ B
    th[:, 10:13] = B
    return th


@pytest.mark.parametrize("T", [None, 20.0, 3.0])
def test_partition_of_unity_reproduces_shared_linear_polynomial(T):
    """Softmax weights are a convex combination, so O = P(q) and dO/dq = B
    exactly for any beta/Delta and for any truncated key set (Eq. func-interp, func-normal)."""
    A, B = 0.3, np.array([0.7, -1.2, 0.4])
    th = _pou_theta(4, 1, A, B)
    q = synth.rng(2).uniform(-1.2, 1.2, size=(50, 3))
    f = orc.forward(th, 4, q, cutoff_T=T)
    np.testing.assert_allclose(f.O, A + q @ B, atol=1e-12)
    np.testing.assert_allclose(f.G, np.broadcast_to(B, f.G.shape), atol=1e-10)


def test_single_key_and_lambda():
    """One effective key: O = f(q - k), lambda = ln e_j = -beta ||q - k||^2.
    The offset key is moved 50 units away so its weight is exactly 0 in float64."""
    th = np.zeros((1, 13))
    th[0, 0] = 1.5; th[0, 1] = 0.25; th[0, 2:5] = [0.5, -1.0, 2.0]
    th[0, 5:8] = [50.0, 0, 0]; th[0, 8] = 5.0; th[0, 9] = 9.0
    q = np.array([[0.1, 0.2, -0.3], [0.0, 0.0, 0.0], [-0.5, 0.4, 0.9]])
    f = orc.forward(th, 1, q)
    np.testing.assert_allclose(f.O, 0.25 + q @ np.array([0.5, -1.0, 2.0]), rtol=1e-14)
    np.testing.assert_allclose(f.lam, -math.exp(1.5) * np.sum(q * q, axis=1), rtol=1e-14)
    np.testing.assert_allclose(f.G, np.broadcast_to([0.5, -1.0, 2.0], (3, 3)), atol=1e-13)


def test_degree0_reduces_to_normalized_rbf_via_scipy_softmax():
    """g = 0 turns Eq. func-interp into O^nrbf (Eq. nrbf); checked with
    scipy.special.softmax over the 2R^3 union keys as the textbook routine."""
    from scipy.special import softmax
    R = 3
    th = synth.random_theta(R, 5, log_scale_mean=2.0).astype(np.float64)
    th[:, 2:5] = 0; th[:, 10:13] = 0
    q = synth.rng(6).uniform(-1, 1, size=(7, 3))
    f = orc.forward(th, R, q)
    k = orc.node_positions(R)
    keys = np.concatenate([k, k + th[:, 5:8]])
    beta = np.exp(np.concatenate([th[:, 0], th[:, 8]]))
    vals = np.concatenate([th[:, 1], th[:, 9]])
    for j in range(q.shape[0]):
        p = softmax(-beta * np.sum((q[j] - keys) ** 2, axis=1))
        assert abs(f.O[j] - p @ vals) < 1e-13
        # range property
        assert vals.min() - 1e-15 <= f.O[j] <= vals.max() + 1e-15


def test_equal_constant_values_give_constant_field():
    """All degree-0 values equal v -> O == v everywhere."""
    th = synth.random_theta(3, 8).astype(np.float64)
    th[:, 2:5] = 0; th[:, 10:13] = 0; th[:, 1] = -0.7; th[:, 9] = -0.7
    f = orc.forward(th, 3, synth.rng(9).uniform(-1, 1, size=(20, 3)))
    np.testing.assert_allclose(f.O, -0.7, atol=1e-14)


def test_forward_against_mpmath_brute_force():
    """Independent 40-digit evaluation of Eq. func-offset by a per-key loop on a tiny grid,
    with G from mpmath numerical differentiation of that brute-force O."""
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.dps = 40
    R = 2
    th = synth.random_theta(R, 21, log_scale_mean=1.0, log_scale_std=0.5).astype(np.float64)
    t = [mpmath.mpf(float(v)) for v in orc.lattice_1d(R)]
    keys = []
    for n in range(R ** 3):
        x, y, z = n % R, (n // R) % R, n // (R * R)
        kn = [t[x], t[y], t[z]]
        row = [mpmath.mpf(float(v)) for v in th[n]]
        keys.append((kn, mpmath.e ** row[0], row[1], row[2:5]))
        kd = [kn[a] + row[5 + a] for a in range(3)]
        keys.append((kd, mpmath.e ** row[8], row[9], row[10:13]))

    def O_mp(qq):
        num = mpmath.mpf(0); den = mpmath.mpf(0)
        for kk, beta, c, g in keys:
            d = [qq[a] - kk[a] for a in range(3)]
            w = mpmath.e ** (-beta * sum(v * v for v in d))
            num += w * (c + sum(g[a] * d[a] for a in range(3)))
            den += w
        return num / den

    q = synth.rng(22).uniform(-1, 1, size=(3, 3))
    f = orc.forward(th, R, q)
    for j in range(3):
        qq = [mpmath.mpf(float(v)) for v in q[j]]
        assert abs(float(O_mp(qq)) - f.O[j]) < 1e-13
        for a in range(3):
            def fa(x, a=a):
                qv = list(qq); qv[a] = x
                return O_mp(qv)
            ga = float(mpmath.diff(fa, qq[a]))
            assert abs(ga - f.G[j, a]) < 1e-11 * max(1.0, abs(ga))


def test_query_gradient_matches_central_differences():
    """Eq. func-normal vs central differences of O."""
    R = 3
    th = synth.random_theta(R, 31, log_scale_mean=3.0, log_scale_std=0.5).astype(np.float64)
    q = synth.rng(32).uniform(-1, 1, size=(10, 3))
    f = orc.forward(th, R, q)
    eps = 1e-6
    for a in range(3):
        e = np.zeros(3); e[a] = eps
        fd = (orc.forward(th, R, q + e).O - orc.forward(th, R, q - e).O) / (2 * eps)
        np.testing.assert_allclose(f.G[:, a], fd, rtol=1e-7, atol=1e-8)


def test_mirror_symmetry_of_gradient():
    """Degree-0 values mirror-symmetric across x=0 with equal betas -> dO/dx = 0 on the plane
    (SPEC.md:L161). R=2 lattice is symmetric about x=0; the offset bank is moved 100 units away
    so its weights are exactly 0."""
    R = 2
    k = orc.node_positions(R)
    th = np.zeros((8, 13))
    th[:, 0] = 1.0; th[:, 8] = 1.0
    th[:, 5:8] = 100.0
    th[:, 1] = 0.3 * k[:, 1] + 0.1 * k[:, 2]
    q = np.array([[0.0, -0.3, 0.2], [0.0, 0.5, -0.9]])
    f = orc.forward(th, R, q)
    np.testing.assert_allclose(f.G[:, 0], 0.0, atol=1e-14)
    assert np.all(np.abs(f.G[:, 1]) > 1e-3)


# ----------------------------------------------------------------------------- losses
def test_mse_examples_from_golden():
    """Eq. loss hand-arithmetic examples."""
    for ln in _golden_lines("mse_examples.txt"):
        O, o, L, r = [np.array(s.split(), dtype=float) for s in ln.split(";")]
        L2, r2 = orc.mse_loss(O, o)
        assert abs(L2 - L[0]) < 1e-15
        np.testing.assert_allclose(r2, r, rtol=1e-15)
    with pytest.raises(ValueError):
        orc.mse_loss([1.0, 2.0], [1.0])


def test_eikonal_loss_zero_on_unit_gradients():
    G = np.array([[1.0, 0, 0], [0, 0.6, 0.8]])
    L, h = orc.eikonal_loss(G, 0.1)
    assert L == 0.0 and np.all(h == 0)
    L, h = orc.eikonal_loss(np.zeros((1, 3)), 0.1)
    assert abs(L - 0.1) < 1e-15 and np.all(h == 0)


# ----------------------------------------------------------------------------- backward pins
def _torch_loss(th_t, R, q_t, o_t, lam_e):
    """Independent float64 torch transcription of Eq. func-offset + MSE (+ Eikonal through
    autograd's create_graph) used only to differentiate by autograd."""
    import torch
    t = torch.tensor(orc.lattice_1d(R), dtype=torch.float64)
    z, y, x = torch.meshgrid(t, t, t, indexing="ij")
    k = torch.stack([x.reshape(-1), y.reshape(-1), z.reshape(-1)], 1)
    keys = torch.cat([k, k + th_t[:, 5:8]])
    beta = torch.exp(torch.cat([th_t[:, 0], th_t[:, 8]]))
    c = torch.cat([th_t[:, 1], th_t[:, 9]])
    g = torch.cat([th_t[:, 2:5], th_t[:, 10:13]])
    q_t = q_t.clone().requires_grad_(lam_e != 0)
    d = q_t[:, None, :] - keys[None]
    logits = -beta[None] * (d * d).sum(-1)
    p = torch.softmax(logits, dim=1)
    f = c[None] + (g[None] * d).sum(-1)
    O = (p * f).sum(1)
    L = ((O - o_t) ** 2).mean()
    if lam_e:
        G, = torch.autograd.grad(O.sum(), q_t, create_graph=True)
        L = L + lam_e * ((G.norm(dim=1) - 1) ** 2).mean()
    return L, O


@pytest.mark.parametrize("lam_e", [0.0, 0.1])
def test_backward_matches_torch_autograd(lam_e):
    """Alg. 2 + L569-598 (and the Eikonal second-order terms) vs float64 autograd."""
    torch = pytest.importorskip("torch")
    R = 3
    th = synth.random_theta(R, 41, log_scale_mean=2.5, log_scale_std=0.5).astype(np.float64)
    q, o = synth.sample_batch(synth.Sphere(0.5), 24, seed=42)
    q = q.astype(np.float64); o = o.astype(np.float64)
    th_t = torch.tensor(th, requires_grad=True)
    L_t, O_t = _torch_loss(th_t, R, torch.tensor(q), torch.tensor(o), lam_e)
    L_t.backward()
    f = orc.forward(th, R, q)
    L, r = orc.mse_loss(f.O, o)
    h = None
    if lam_e:
        LE, h = orc.eikonal_loss(f.G, lam_e)
        L += LE
    grad = orc.backward(th, R, q, f, r, h)
    assert abs(L - float(L_t.detach())) < 1e-12 * max(1, abs(L))
    ref = th_t.grad.numpy()
    for ch in range(13):
        scale = max(np.abs(ref[:, ch]).max(), 1e-30)
        assert np.abs(grad[:, ch] - ref[:, ch]).max() / scale < 1e-9, ch


def test_backward_matches_central_differences_all_channels():
    """dL/dtheta vs central differences of L through oracle.forward."""
    R = 2
    th = synth.random_theta(R, 51, log_scale_mean=2.0, log_scale_std=0.4).astype(np.float64)
    q, o = synth.sample_batch(synth.Sphere(0.5), 12, seed=52)
    q = q.astype(np.float64); o = o.astype(np.float64)
    lam_e = 0.1

    def loss(t):
        f = orc.forward(t, R, q)
        return orc.mse_loss(f.O, o)[0] + orc.eikonal_loss(f.G, lam_e)[0]

    f = orc.forward(th, R, q)
    _, r = orc.mse_loss(f.O, o)
    _, h = orc.eikonal_loss(f.G, lam_e)
    grad = orc.backward(th, R, q, f, r, h)
    eps = 1e-6
    fd = np.zeros_like(th)
    for n in range(th.shape[0]):
        for ch in range(13):
            tp = th.copy(); tp[n, ch] += eps
            tm = th.copy(); tm[n, ch] -= eps
            fd[n, ch] = (loss(tp) - loss(tm)) / (2 * eps)
    np.testing.assert_allclose(grad, fd, rtol=1e-5, atol=1e-8)


def test_backward_linear_invariants():
    """Sum_i dO/dc_i = 1 (softmax sums to 1), so sum_i dL/dc_i = sum_j r_j; zero upstream -> zero
    gradient; additivity over query subsets."""
    R = 3
    th = synth.fitted_like_theta(R, synth.Sphere(0.5), 61).astype(np.float64)
    q, o = synth.sample_batch(synth.Sphere(0.5), 40, seed=62)
    f = orc.forward(th, R, q)
    r = synth.rng(63).normal(size=40)
    g = orc.backward(th, R, q, f, r)
    assert abs(g[:, 1].sum() + g[:, 9].sum() - r.sum()) < 1e-12
    assert np.all(orc.backward(th, R, q, f, np.zeros(40)) == 0)
    fa = orc.forward(th, R, q[:17]); fb = orc.forward(th, R, q[17:])
    ga = orc.backward(th, R, q[:17], fa, r[:17]); gb = orc.backward(th, R, q[17:], fb, r[17:])
    np.testing.assert_allclose(ga + gb, g, rtol=1e-12, atol=1e-15)


def test_partition_of_unity_gradients():
    """Under PoU, dO/ds == 0 and dO/dDelta_n = -p_{I+n} B."""
    A, B = -0.1, np.array([0.2, 0.5, -0.3])
    R = 3
    th = _pou_theta(R, 71, A, B)
    q = synth.rng(72).uniform(-1, 1, size=(5, 3))
    f = orc.forward(th, R, q)
    for j in range(5):
        r = np.zeros(5); r[j] = 1.0
        g = orc.backward(th, R, q, f, r)
        np.testing.assert_allclose(g[:, 0], 0, atol=1e-13)
        np.testing.assert_allclose(g[:, 8], 0, atol=1e-13)
        # p of offset keys = dO/dc1
        np.testing.assert_allclose(g[:, 5:8], -g[:, 9:10] * B[None, :], atol=1e-13)


# ----------------------------------------------------------------------------- AdamW pins
def test_adamw_matches_torch_optim_adamw():
    """PAPER.md:L698 AdamW; torch.optim.AdamW (float64, foreach=False) is the textbook routine.
    The decay mask (reading R-10) is expressed with two param groups."""
    torch = pytest.importorskip("torch")
    hp = orc.AdamW(lr=1e-2, weight_decay=0.05)
    R = 2
    rs = synth.rng(81)
    th = rs.normal(size=(R ** 3, 13))
    mask = np.array([(hp.decay_mask >> c) & 1 for c in range(13)], bool)
    p_dec = torch.tensor(th[:, mask], requires_grad=True)
    p_nod = torch.tensor(th[:, ~mask], requires_grad=True)
    opt = torch.optim.AdamW([{"params": [p_dec], "weight_decay": hp.weight_decay},
                             {"params": [p_nod], "weight_decay": 0.0}],
                            lr=hp.lr, betas=(hp.beta1, hp.beta2), eps=hp.eps, foreach=False)
    m = np.zeros_like(th); v = np.zeros_like(th); cur = th.copy()
    for step in range(1, 6):
        g = rs.normal(size=th.shape) * (10.0 ** rs.integers(-6, 1, size=th.shape))
        p_dec.grad = torch.tensor(g[:, mask]); p_nod.grad = torch.tensor(g[:, ~mask])
        opt.step()
        cur, m, v = orc.adamw_step(cur, g, m, v, step, hp)
        np.testing.assert_allclose(cur[:, mask], p_dec.detach().numpy(), rtol=1e-13, atol=1e-15)
        np.testing.assert_allclose(cur[:, ~mask], p_nod.detach().numpy(), rtol=1e-13, atol=1e-15)


def test_adamw_closed_forms():
    """Zero grad + zero decay -> unchanged; zero grad + decay -> p(1 - lr wd); first step with
    g = 0.3 -> step = -lr g/(|g| + eps)."""
    hp0 = orc.AdamW(weight_decay=0.0)
    th = np.full((1, 13), 0.5)
    z = np.zeros_like(th)
    np.testing.assert_array_equal(orc.adamw_step(th, z, z, z, 1, hp0)[0], th)
    hp = orc.AdamW(weight_decay=0.01)
    out = orc.adamw_step(th, z, z, z, 1, hp)[0]
    mask = np.array([(hp.decay_mask >> c) & 1 for c in range(13)], bool)
    np.testing.assert_allclose(out[0, mask], 0.5 * (1 - hp.lr * 0.01), rtol=1e-15)
    np.testing.assert_allclose(out[0, ~mask], 0.5, rtol=1e-15)
    g = np.full_like(th, 0.3)
    out = orc.adamw_step(th, g, z, z, 1, hp0)[0]
    np.testing.assert_allclose(out - th, -hp0.lr * 0.3 / (0.3 + hp0.eps), rtol=1e-12)


# ----------------------------------------------------------------------------- mean shift pins
def test_mean_shift_single_point_and_symmetric_pair():
    """PAPER.md:L475 Eq.: N=1 -> k + Delta = s; two points symmetric about k -> midpoint
    (SPEC.md:L268-269)."""
    R = 3
    s = np.array([[0.3, -0.2, 0.9]])
    d = orc.mean_shift_offsets(R, s)
    np.testing.assert_allclose(orc.node_positions(R) + d, np.broadcast_to(s, (27, 3)), atol=1e-14)
    k = orc.node_positions(R)
    k13 = k[13]  # centre node (0,0,0)
    s2 = np.array([k13 + [0.1, 0.2, 0.0], k13 - [0.1, 0.2, 0.0]])
    d2 = orc.mean_shift_offsets(R, s2)
    np.testing.assert_allclose(d2[13], 0.0, atol=1e-14)


def test_mean_shift_moves_keys_to_sphere():
    """Mean shift pulls lattice keys towards the surface."""
    R = 8
    sph = synth.Sphere(0.5)
    s = synth.surface_points(sph, 2048, seed=3).astype(np.float64)
    d = orc.mean_shift_offsets(R, s)
    k = orc.node_positions(R)
    before = np.abs(np.linalg.norm(k, axis=1) - 0.5)
    after = np.abs(np.linalg.norm(k + d, axis=1) - 0.5)
    assert np.median(after) < 0.5 * np.median(before)
    assert np.mean(after < before) > 0.9


# ----------------------------------------------------------------------------- cutoff study
def test_cutoff_truncation_error_small_at_default_T():
    """Reading R-1: dropping pairs with a - m > 20 changes O and G by < 1e-7 (normwise) at
    the C1 geometry; T = inf reproduces the global sum."""
    R = 8
    sph = synth.Sphere(0.5)
    th = synth.fitted_like_theta(R, sph, 91).astype(np.float64)
    q, o = synth.sample_batch(sph, 400, seed=92)
    g = orc.forward(th, R, q)
    t = orc.forward(th, R, q, cutoff_T=20.0)
    assert np.abs(t.O - g.O).max() / np.abs(g.O).max() < 1e-7
    assert np.abs(t.G - g.G).max() / np.abs(g.G).max() < 1e-6
    assert t.kept.min() >= 1 and t.kept.max() < 2 * R ** 3
    ti = orc.forward(th, R, q, cutoff_T=float("inf"))
    np.testing.assert_allclose(ti.O, g.O, rtol=0, atol=0)


# ----------------------------------------------------------------------------- kept-pair count pins
def _node_theta(R, s=0.0):
    """beta = e^s on both banks, Delta = 0 (offset keys on the lattice), zero polynomials."""
    th = np.zeros((R ** 3, 13))
    th[:, 0] = s
    th[:, 8] = s
    return th


def test_kept_counts_lattice_points_at_a_node():
    """oracle.kept against the three-square counts r3(n) (tests/golden, OEIS A005875): with
    beta = 1, Delta = 0 and the query ON the centre node of R = 9 (h = 1/4, m_j = 0), the kept set of
    the cutoff a_ij - m_j <= T (reading R-1) is every key with |v|^2 <= T/h^2, twice (both banks).
    T sits halfway between shells, so a '<' vs '<=' slip or a missing shell shows."""
    r3 = {int(a): int(b) for a, b in (ln.split() for ln in _golden_lines("r3_sum_of_three_squares.txt"))}
    R, h = 9, 0.25
    th = _node_theta(R)
    q = np.zeros((1, 3))
    for n in range(16):
        T = (n + 0.5) * h * h
        f = orc.forward(th, R, q, cutoff_T=T)
        assert f.m[0] == 0.0
        assert int(f.kept[0]) == 2 * sum(r3[k] for k in range(n + 1)), n


def test_kept_counts_use_the_shifted_exponent():
    """Off a node the test is a_ij - m_j <= T (shifted, m_j = min_i a_ij), not a_ij <= T: at
    q = 0.3 h e_x the shifted and unshifted counts differ. Reference: integer-vector brute force."""
    import itertools
    R, h = 9, 0.25
    th = _node_theta(R)
    e = (0.3, 0.0, 0.0)
    q = np.array([[0.3 * h, 0.0, 0.0]])
    differs = 0
    for t in (0.45, 1.2, 2.05, 3.3):
        T = t * h * h
        f = orc.forward(th, R, q, cutoff_T=T)
        d2 = [sum((v[k] - e[k]) ** 2 for k in range(3)) for v in itertools.product(range(-4, 5), repeat=3)]
        m2 = min(d2)
        shifted = sum(1 for x in d2 if x - m2 <= t)
        unshifted = sum(1 for x in d2 if x <= t)
        assert int(f.kept[0]) == 2 * shifted, t
        differs += shifted != unshifted
    assert differs >= 2  # the pin discriminates shifted from unshifted exponents


def test_kept_and_values_against_python_loop_brute_force():
    """R = 2 and 3, random theta (beta spread, offsets) and out-of-domain queries: kept counts, O
    and lambda against a plain Python double loop over (query, key) with the math module."""
    for R, seed in ((2, 5), (3, 6)):
        th = synth.random_theta(R, seed, log_scale_mean=1.0, log_scale_std=0.7, offset_std=0.2).astype(np.float64)
        q = synth.rng(seed + 10).uniform(-1.4, 1.4, size=(12, 3))
        T = 2.5
        f = orc.forward(th, R, q, cutoff_T=T)
        g = orc.forward(th, R, q)
        t = [(-1.0 + 2.0 * i / (R - 1)) for i in range(R)]
        keys = []
        for z in range(R):
            for y in range(R):
                for x in range(R):
                    n = x + R * (y + R * z)
                    k = (float(np.float32(t[x])), float(np.float32(t[y])), float(np.float32(t[z])))
                    keys.append((k, math.exp(th[n, 0]), th[n, 1], th[n, 2:5]))
        for z in range(R):
            for y in range(R):
                for x in range(R):
                    n = x + R * (y + R * z)
                    k = keys[n][0]
                    kd = (k[0] + th[n, 5], k[1] + th[n, 6], k[2] + th[n, 7])
                    keys.append((kd, math.exp(th[n, 8]), th[n, 9], th[n, 10:13]))
        for j in range(q.shape[0]):
            a = []
            fv = []
            for (k, beta, c, gg) in keys:
                d = [q[j, 0] - k[0], q[j, 1] - k[1], q[j, 2] - k[2]]
                a.append(beta * (d[0] ** 2 + d[1] ** 2 + d[2] ** 2))
                fv.append(c + gg[0] * d[0] + gg[1] * d[1] + gg[2] * d[2])
            m = min(a)
            assert int(f.kept[j]) == sum(1 for x in a if x - m <= T)
            Z = sum(math.exp(-(x - m)) for x in a)
            O = sum(math.exp(-(x - m)) * v for x, v in zip(a, fv)) / Z
            assert abs(g.O[j] - O) <= 1e-12 * max(1.0, abs(O))
            assert abs(g.lam[j] - (-m + math.log(Z))) <= 1e-12 * max(1.0, abs(m))


def test_sharded_oracle_driver_equals_single_process():
    """oracle.parallel runs the oracle unchanged on query shards; per-query outputs concatenate and
    shard gradients add up to the full-batch gradient (additivity)."""
    from oracle import parallel as par
    R = 4
    th = synth.random_theta(R, 17, log_scale_mean=2.0).astype(np.float64)
    q = synth.rng(18).uniform(-1, 1, size=(37, 3))
    o = synth.rng(19).normal(size=37)
    f, L, g = par.fit_eval(th, R, q, o, lam_e=0.1, procs=3)
    f1 = orc.forward(th, R, q)
    Lm, r = orc.mse_loss(f1.O, o)
    Le, h = orc.eikonal_loss(f1.G, 0.1)
    g1 = orc.backward(th, R, q, f1, r, h)
    np.testing.assert_allclose(f.O, f1.O, rtol=0, atol=0)
    np.testing.assert_allclose(f.G, f1.G, rtol=0, atol=0)
    assert abs(L - (Lm + Le)) <= 1e-14 * (Lm + Le)
    np.testing.assert_allclose(g, g1, rtol=1e-12, atol=1e-14)


def test_mc_vertices_brute_force_tiny_lattice():
    """oracle.mesh_oracle.mc_vertices (Marching Cubes vertex placement) against a
    plain triple loop over every lattice edge of a random 4^3 field."""
    from oracle import mesh_oracle as mo
    N, lo, hi = 4, (-1.0, -0.5, 0.0), (1.0, 0.5, 2.0)
    O = synth.rng(31).normal(size=(N, N, N))
    got = mo.mc_vertices(O, lo, hi, iso=0.1)
    step = [(hi[a] - lo[a]) / (N - 1) for a in range(3)]
    want = []
    for k in range(N):
        for j in range(N):
            for i in range(N):
                for (di, dj, dk) in ((1, 0, 0), (0, 1, 0), (0, 0, 1)):
                    i1, j1, k1 = i + di, j + dj, k + dk
                    if i1 >= N or j1 >= N or k1 >= N:
                        continue
                    v0, v1 = O[k, j, i], O[k1, j1, i1]
                    if (v0 < 0.1) == (v1 < 0.1):
                        continue
                    t = (0.1 - v0) / (v1 - v0)
                    p0 = [lo[0] + i * step[0], lo[1] + j * step[1], lo[2] + k * step[2]]
                    p1 = [lo[0] + i1 * step[0], lo[1] + j1 * step[1], lo[2] + k1 * step[2]]
                    want.append([p0[a] + t * (p1[a] - p0[a]) for a in range(3)])
    want = np.array(want)
    assert got.shape == want.shape
    key = lambda a: np.lexsort(np.round(a, 12).T)  # noqa: E731
    np.testing.assert_allclose(got[key(got)], want[key(want)], atol=1e-12)


def test_mc_vertices_on_sphere_field_lie_on_the_sphere():
    """For O = |p| - r the vertices sit on the zero set up to the linear-interpolation error
    (|O| at a vertex <= h^2 / (2 r) on an edge of length h) and their count grows as N^2."""
    from oracle import mesh_oracle as mo
    r = 0.6
    for N in (17, 33):
        P = mo.lattice_points(N, (-1, -1, -1), (1, 1, 1))
        O = np.linalg.norm(P, axis=-1) - r
        v = mo.mc_vertices(O, (-1, -1, -1), (1, 1, 1))
        h = 2.0 / (N - 1)
        assert np.abs(np.linalg.norm(v, axis=1) - r).max() <= h * h / (2 * r) + 1e-12
        # every lattice line along an axis through the disc of radius r crosses the sphere twice:
        # 2 pi r^2 / h^2 crossing edges per axis
        est = 6 * math.pi * r * r / (h * h)
        assert 0.9 * est < len(v) < 1.1 * est, (len(v), est)
