"""GPU parity: libefunc (sm_100a, through the C ABI) vs the float64 CPU oracle.

Tolerances (north_star, read normwise per DESIGN.md reading R-T):
  values O, G        max|gpu - ref| / max|ref| <= 1e-5   (per component for G)
  parameter grads    per channel max|gpu - ref| / max|ref| <= 1e-4
  AdamW              rel 1e-6 (fp32 arithmetic vs float64)
The GPU evaluates the certified cutoff T = 20 (reading R-1); the oracle is the global sum.
"""
import numpy as np
import pytest

import oracle as orc
from workloads import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2505_21319_b200 as ef  # noqa: E402

TOL_VAL = 1e-5
TOL_GRAD = 1e-4


def nw(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def dev(x):
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def c1_case(seed=1, J=4096, R=8):
    sph = synth.Sphere(0.5)
    th = synth.fitted_like_theta(R, sph, seed)
    q, o = synth.sample_batch(sph, J, seed=seed + 100)
    return th, q, o


def check_grads(g, ref, tol=TOL_GRAD, floor=0.0):
    """Per channel normwise. floor > 0: a channel's scale is at least floor * (largest gradient of
    any channel), so a channel lying entirely beyond the certified cutoff is compared absolutely
    (e.g. the far offset bank of a 1-query batch: a dropped pair's term is at most
    e^-T (T + m) ~ 5e-8 of the largest terms at T = 20)."""
    big = float(np.abs(ref).max())
    for ch in range(13):
        scale = max(float(np.abs(ref[:, ch]).max()), floor * big, 1e-30)
        e = float(np.abs(np.asarray(g[:, ch], np.float64) - ref[:, ch]).max()) / scale
        assert e <= tol, (ch, e)


# ----------------------------------------------------------------------------- forward
@pytest.mark.parametrize("T", [20.0, float("inf")])
def test_forward_parity_c1(T):
    th, q, o = c1_case()
    m = ef.EFunc(8, th, cutoff_T=T)
    O, G, L = m.forward(dev(q), dev(o), loss=ef.LOSS_MSE, want_G=True)
    torch.cuda.synchronize()
    ref = orc.forward(th, 8, q)
    assert nw(O.cpu().numpy(), ref.O) <= TOL_VAL
    for a in range(3):
        assert nw(G.cpu().numpy()[:, a], ref.G[:, a]) <= TOL_VAL
    Lref, _ = orc.mse_loss(ref.O, o)
    assert abs(float(L.item()) - Lref) / Lref <= 1e-5


def test_partition_of_unity_on_gpu():
    """Shared linear polynomial is reproduced exactly for any truncated key set.
    R = 17 (h = 1/8), dyadic A, B and offsets make the float32 theta an EXACT partition-of-unity
    configuration, so O = P(q) and G = B up to arithmetic rounding only."""
    R = 17
    A, B = 0.25, np.array([0.5, -0.25, 0.125])
    th = synth.random_theta(R, 3, log_scale_mean=7.0, log_scale_std=0.3, offset_std=0.03).astype(np.float64)
    th[:, 5:8] = np.round(th[:, 5:8] * 4096.0) / 4096.0
    k = orc.node_positions(R)
    th[:, 1] = A + k @ B; th[:, 2:5] = B
    th[:, 9] = A + (k + th[:, 5:8]) @ B; th[:, 10:13] = B
    th = th.astype(np.float32)
    q = synth.rng(4).uniform(-1, 1, size=(50000, 3)).astype(np.float32)
    m = ef.EFunc(R, th)
    O, G, _ = m.forward(dev(q), want_G=True)
    exact = A + q.astype(np.float64) @ B
    eO = nw(O.cpu().numpy(), exact)
    eG = nw(G.cpu().numpy(), np.broadcast_to(B, (q.shape[0], 3)))
    assert eO <= 2e-6, eO
    # G's u-term 2((O - f0) S_u - S_uf)/Z takes O - f0 = M/Z before O is rounded (in fp32,
    # O - f0 would lose M/Z below ulp(O) and leave (M/Z) S_u unbalanced, ~5e-6 here)
    for a in range(3):
        eGa = nw(G.cpu().numpy()[:, a], np.full(q.shape[0], B[a]))
        assert eGa <= TOL_VAL, (a, eGa)
    assert eG <= TOL_VAL, eG


def test_eval_grad_matches_forward_and_oracle():
    th, q, o = c1_case(seed=5, J=1000)
    m = ef.EFunc(8, th)
    O, G = m.eval_grad(dev(q))
    ref = orc.forward(th, 8, q)
    assert nw(O.cpu().numpy(), ref.O) <= TOL_VAL
    assert nw(G.cpu().numpy(), ref.G) <= TOL_VAL


# ----------------------------------------------------------------------------- backward
@pytest.mark.parametrize("T", [20.0, float("inf")])
def test_backward_mse_parity_c1(T):
    th, q, o = c1_case(seed=7)
    m = ef.EFunc(8, th, cutoff_T=T)
    m.forward(dev(q), dev(o), loss=ef.LOSS_MSE)
    g = m.backward().cpu().numpy()
    f = orc.forward(th, 8, q)
    _, r = orc.mse_loss(f.O, o)
    check_grads(g, orc.backward(th, 8, q, f, r))


def test_backward_explicit_upstream_parity():
    th, q, o = c1_case(seed=9, J=2000)
    r = synth.rng(10).normal(size=2000).astype(np.float32)
    m = ef.EFunc(8, th)
    m.forward(dev(q))
    g = m.backward(dL_dO=dev(r)).cpu().numpy()
    f = orc.forward(th, 8, q)
    check_grads(g, orc.backward(th, 8, q, f, r.astype(np.float64)))


def test_backward_eikonal_parity():
    th, q, o = c1_case(seed=11, J=2048)
    m = ef.EFunc(8, th)
    O, G, L = m.forward(dev(q), dev(o), loss=ef.LOSS_MSE_EIKONAL, eikonal_lambda=0.1, want_G=True)
    g = m.backward().cpu().numpy()
    f = orc.forward(th, 8, q)
    Lm, r = orc.mse_loss(f.O, o)
    Le, h = orc.eikonal_loss(f.G, 0.1)
    assert abs(float(L.item()) - (Lm + Le)) / (Lm + Le) <= 1e-5
    check_grads(g, orc.backward(th, 8, q, f, r, h))


def test_backward_without_forward_is_state_error():
    th, q, o = c1_case(J=10)
    m = ef.EFunc(8, th)
    with pytest.raises(ef.EfuncError) as e:
        m.backward(dL_dO=dev(np.ones(10)))
    assert e.value.status == 2


# ----------------------------------------------------------------------------- AdamW / fit
def test_adamw_parity():
    R = 8
    th = synth.random_theta(R, 12)
    rs = synth.rng(13)
    m = ef.EFunc(R, th)
    hp = ef.AdamW(lr=1e-2, weight_decay=0.05)
    ohp = orc.AdamW(lr=1e-2, weight_decay=0.05)
    cur = th.astype(np.float64); mm = np.zeros_like(cur); vv = np.zeros_like(cur)
    for step in range(1, 4):
        g = (rs.normal(size=th.shape) * 10.0 ** rs.integers(-5, 0, size=th.shape)).astype(np.float32)
        m.adamw_step(dev(g), hp)
        cur, mm, vv = orc.adamw_step(cur, g, mm, vv, step, ohp)
        got = m.get_params()
        np.testing.assert_allclose(got, cur, rtol=2e-6, atol=1e-7)
    gm, gv, st = m.get_adam_state()
    assert st == 3
    # moments: fp32 rounding relative to the size of the gradients that built them
    assert np.abs(gm - mm).max() <= 1e-6 * np.abs(mm).max()
    assert np.abs(gv - vv).max() <= 1e-6 * np.abs(vv).max()


def test_fit_c1_ten_steps_resynced_and_free_running():
    """C1: 8^3 grid, 4096 sphere points, 10 AdamW steps. Step-by-step with re-sync (reading R-A)
    at 1e-4 on grads, plus a free-running loss trajectory."""
    R = 8
    sph = synth.Sphere(0.5)
    th0 = synth.init_theta(R, 21)
    s = synth.surface_points(sph, 4096, seed=22)
    th0[:, 5:8] = orc.mean_shift_offsets(R, s).astype(np.float32)
    hp = ef.AdamW(); ohp = orc.AdamW()
    m = ef.EFunc(R, th0)
    cur = th0.astype(np.float64); mm = np.zeros_like(cur); vv = np.zeros_like(cur)
    free = ef.EFunc(R, th0)
    losses_gpu, losses_ref = [], []
    for step in range(1, 11):
        q, o = synth.sample_batch(sph, 4096, seed=1000 + step)
        # re-synced step: both sides start from the oracle's theta_t and moments
        m.set_params(cur.astype(np.float32))
        m.set_adam_state(mm.astype(np.float32), vv.astype(np.float32), step - 1)
        _, _, L = m.forward(dev(q), dev(o), loss=ef.LOSS_MSE)
        g = m.backward().cpu().numpy()
        f = orc.forward(cur, R, q)
        Lr, r = orc.mse_loss(f.O, o)
        gref = orc.backward(cur, R, q, f, r)
        check_grads(g, gref)
        assert abs(float(L.item()) - Lr) / Lr <= 1e-5
        cur, mm, vv = orc.adamw_step(cur, gref, mm, vv, step, ohp)
        # free-running GPU fit
        losses_gpu.append(free.fit_step(torch.as_tensor(q).pin_memory(), torch.as_tensor(o).pin_memory(), hp))
        losses_ref.append(Lr)
    # free-running loss within 1e-3 relative (AdamW amplifies sign noise of near-zero grads)
    assert np.allclose(losses_gpu, losses_ref, rtol=1e-3)
    assert losses_gpu[-1] < losses_gpu[0]


# ----------------------------------------------------------------------------- full size (C2)
def test_c2_full_size_sampled_parity():
    """C2 geometry: 32^3 x 13, 2^20 torus points in the bench's launch configuration; outputs
    checked at sampled queries, gradients via a sampled upstream (linearity)."""
    R, J = 32, 1 << 20
    tor = synth.Torus()
    s = synth.surface_points(tor, 16384, seed=31)
    th = synth.init_theta(R, 32)
    q, o = synth.sample_batch(tor, J, seed=33)
    m = ef.EFunc(R, th)
    m.mean_shift_init(dev(s))
    th_gpu = m.get_params()
    # mean shift parity
    dref = orc.mean_shift_offsets(R, s.astype(np.float64))
    assert np.abs(th_gpu[:, 5:8] - dref).max() <= 1e-5
    qd, od = dev(q), dev(o)
    O, G, L = m.forward(qd, od, loss=ef.LOSS_MSE, want_G=True)
    idx = synth.rng(34).choice(J, size=1024, replace=False)
    ref = orc.forward(th_gpu, R, q[idx])
    assert nw(O.cpu().numpy()[idx], ref.O) <= TOL_VAL
    for a in range(3):
        assert nw(G.cpu().numpy()[idx, a], ref.G[:, a]) <= TOL_VAL
    # sampled upstream over the full batch
    sub = synth.rng(35).choice(J, size=512, replace=False)
    r = np.zeros(J, np.float32)
    r[sub] = synth.rng(36).normal(size=512).astype(np.float32)
    g = m.backward(dL_dO=dev(r)).cpu().numpy()
    fs = orc.forward(th_gpu, R, q[sub])
    check_grads(g, orc.backward(th_gpu, R, q[sub], fs, r[sub].astype(np.float64)))


def test_c2_pou_full_size():
    R, J = 32, 1 << 20
    A, B = -0.2, np.array([0.3, 0.1, -0.5])
    th = synth.fitted_like_theta(R, synth.Torus(), 41).astype(np.float64)
    k = orc.node_positions(R)
    th[:, 1] = A + k @ B; th[:, 2:5] = B
    th[:, 9] = A + (k + th[:, 5:8]) @ B; th[:, 10:13] = B
    q, o = synth.sample_batch(synth.Torus(), J, seed=42)
    m = ef.EFunc(R, th.astype(np.float32))
    O, G, _ = m.forward(dev(q), want_G=True)
    assert nw(O.cpu().numpy(), A + q.astype(np.float64) @ B) <= 2e-6
    # c_i = A + B.k_i rounded to float32 is PoU only up to ulp(c_i): f_i then differ by ~3e-8 and
    # G's u-term amplifies that by 2 beta |d| (the oracle sees the same float32 theta). So G is
    # compared with the oracle at sampled queries (1e-5 per component), and with B loosely.
    Gn = G.cpu().numpy()
    idx = synth.rng(44).choice(J, size=2048, replace=False)
    ref = orc.forward(th.astype(np.float32), R, q[idx])
    for a in range(3):
        assert nw(Gn[idx, a], ref.G[:, a]) <= TOL_VAL, a
        assert nw(Gn[:, a], np.full(J, B[a])) <= 3e-5, a
    # sum_i dL/dc_i = sum_j r_j (softmax sums to one)
    r = synth.rng(43).normal(size=J).astype(np.float32) / J
    g = m.backward(dL_dO=dev(r)).cpu().numpy().astype(np.float64)
    assert abs(g[:, 1].sum() + g[:, 9].sum() - r.astype(np.float64).sum()) <= 1e-4 * np.abs(r).sum()
    # the fused path (k_fit over the work items in their cost-class order) covers every query once:
    # O = P(q) at all 2^20 queries, and sum_i dL/dc_i = sum_j r_j = sum_j 2 (P(q_j) - o_j) / J
    gf, Of, _ = m.forward_backward(dev(q), dev(o), loss=ef.LOSS_MSE, want_O=True, want_loss=False)
    P = A + q.astype(np.float64) @ B
    assert nw(Of.cpu().numpy(), P) <= 2e-6
    rf = 2.0 * (P - o.astype(np.float64)) / J
    gf = gf.cpu().numpy().astype(np.float64)
    assert abs(gf[:, 1].sum() + gf[:, 9].sum() - rf.sum()) <= 1e-4 * np.abs(rf).sum()


# ----------------------------------------------------------------------------- edge cases
def test_empty_single_and_ragged():
    th, q, o = c1_case(seed=51, J=259)
    m = ef.EFunc(8, th)
    O, G, L = m.forward(dev(q[:0]), dev(o[:0]), loss=ef.LOSS_MSE, want_G=True)
    assert O.numel() == 0 and float(L.item()) == 0.0
    g = m.backward()
    assert float(g.abs().sum()) == 0.0
    for J in (1, 127, 128, 129, 259):
        O, G, _ = m.forward(dev(q[:J]), want_G=True)
        ref = orc.forward(th, 8, q[:J])
        assert nw(O.cpu().numpy(), ref.O) <= TOL_VAL


def test_out_of_domain_queries_and_small_grid():
    R = 2
    th = synth.random_theta(R, 61, log_scale_mean=1.0)
    q = synth.rng(62).uniform(-3, 3, size=(777, 3)).astype(np.float32)
    m = ef.EFunc(R, th)
    O, G, _ = m.forward(dev(q), want_G=True)
    ref = orc.forward(th, R, q)
    assert nw(O.cpu().numpy(), ref.O) <= TOL_VAL
    assert nw(G.cpu().numpy(), ref.G) <= TOL_VAL


def test_large_beta_spread_takes_exact_shift_path():
    """log-scales far from the init: the corner shift bound may overflow; the slow path must
    keep results exact."""
    R = 8
    th = synth.random_theta(R, 71, log_scale_mean=7.5, log_scale_std=1.5)
    q = synth.rng(72).uniform(-1, 1, size=(3000, 3)).astype(np.float32)
    m = ef.EFunc(R, th)
    O, G, _ = m.forward(dev(q), want_G=True)
    ref = orc.forward(th, R, q)
    assert nw(O.cpu().numpy(), ref.O) <= TOL_VAL
    for a in range(3):
        assert nw(G.cpu().numpy()[:, a], ref.G[:, a]) <= TOL_VAL, a


def test_nonfinite_query_reported():
    th, q, o = c1_case(J=100)
    q[17, 1] = np.nan
    m = ef.EFunc(8, th, sync_checks=True)
    with pytest.raises(ef.EfuncError) as e:
        m.forward(dev(q))
    assert e.value.status == 3
    m2 = ef.EFunc(8, th)
    m2.forward(dev(q))
    with pytest.raises(ef.EfuncError):
        m2.check()
    m2.check()  # flag cleared


def test_forward_bitwise_deterministic():
    th, q, o = c1_case(seed=81, J=50000)
    m = ef.EFunc(8, th)
    a = m.forward(dev(q), want_G=True)
    b = m.forward(dev(q), want_G=True)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def test_kept_pair_counter_matches_oracle():
    th, q, o = c1_case(seed=91, J=512)
    m = ef.EFunc(8, th)
    m.set_counting(True)
    m.forward(dev(q))
    st = m.stats()
    ref = orc.forward(th, 8, q, cutoff_T=20.0)
    assert abs(st["kept_pairs"] - ref.kept.sum()) <= 0.01 * ref.kept.sum()
    assert st["candidate_pairs"] >= st["kept_pairs"]


# ----------------------------------------------------------------------------- deterministic mode
def test_deterministic_backward_parity_and_bitwise_repeatability():
    """Deterministic mode (reading R-D): 64-bit fixed-point gradient accumulation; results match
    the oracle at 1e-4 and repeat bitwise across runs and handles."""
    th, q, o = c1_case(seed=101)
    m = ef.EFunc(8, th, deterministic=True)
    m.forward(dev(q), dev(o), loss=ef.LOSS_MSE)
    g1 = m.backward().cpu().numpy()
    f = orc.forward(th, 8, q)
    _, r = orc.mse_loss(f.O, o)
    check_grads(g1, orc.backward(th, 8, q, f, r))
    m.check()
    m2 = ef.EFunc(8, th, deterministic=True)
    m2.forward(dev(q), dev(o), loss=ef.LOSS_MSE)
    g2 = m2.backward().cpu().numpy()
    assert np.array_equal(g1, g2)


def test_deterministic_fit_bitwise_at_scale():
    """Three full fit steps at 32^3 x 13 with 2^18 torus points: bitwise identical theta twice."""
    R, J = 32, 1 << 18
    tor = synth.Torus()
    th0 = synth.init_theta(R, 7)
    s = dev(synth.surface_points(tor, 16384, seed=8))
    batches = [synth.sample_batch(tor, J, seed=200 + k) for k in range(3)]
    outs = []
    for _ in range(2):
        m = ef.EFunc(R, th0, deterministic=True)
        m.mean_shift_init(s)
        grad = torch.zeros(R ** 3, 13, device="cuda")
        for q, o in batches:
            grad.zero_()
            m.forward(dev(q), dev(o), loss=ef.LOSS_MSE, want_O=False)
            m.backward(grad=grad)
            m.adamw_step(grad)
        outs.append(m.get_params())
    assert np.array_equal(outs[0], outs[1])


def test_fit_step_graph_replay_bitwise_equals_eager():
    """efunc_fit_step with cfg.fit_graph (captured on the 2nd call, replayed after) gives bitwise the
    same theta, moments and loss trajectory as plain launches (deterministic mode), and the device-
    side AdamW step counter advances once per replay."""
    R, J = 16, 1 << 15
    tor = synth.Torus()
    th0 = synth.init_theta(R, 31)
    s = dev(synth.surface_points(tor, 4096, seed=32))
    batches = [synth.sample_batch(tor, J, seed=300 + k) for k in range(2)]
    qd = [dev(q) for q, _ in batches]
    od = [dev(o) for _, o in batches]
    # device-pointer fit_step: one q/o buffer pair per handle (the graph key includes the pointers)
    res = []
    for graph in (False, True):
        m = ef.EFunc(R, th0, deterministic=True, fit_graph=graph)
        m.mean_shift_init(s)
        qb, ob = torch.empty_like(qd[0]), torch.empty_like(od[0])
        lo = torch.zeros(1, device="cuda")
        losses = []
        for k in range(6):
            qb.copy_(qd[k % 2]); ob.copy_(od[k % 2])
            m.fit_step(qb, ob, ef.AdamW(), loss=ef.LOSS_MSE, loss_out=lo)
            losses.append(float(lo.item()))
        mm, vv, st = m.get_adam_state()
        res.append((m.get_params(), mm, vv, st, losses))
    (p0, m0, v0, s0, l0), (p1, m1, v1, s1, l1) = res
    assert s0 == s1 == 6
    assert np.array_equal(p0, p1) and np.array_equal(m0, m1) and np.array_equal(v0, v1)
    assert l0 == l1
    # host-io fit_step (pinned buffers, graph inside) also advances the step
    m = ef.EFunc(R, th0, fit_graph=True)
    for k in range(3):
        m.fit_step(torch.as_tensor(batches[k % 2][0]).pin_memory(), torch.as_tensor(batches[k % 2][1]).pin_memory())
    assert m.get_adam_state()[2] == 3


# ----------------------------------------------------------------------------- fused forward+backward
def test_forward_backward_single_query():
    """J = 1: one item with one query. The s-channel term -beta r p (f_i - O) dd of the dominant
    key is cancellation-limited in fp32 (O ~ f_i), so here the fused path is checked against the
    split path (same per-pair arithmetic) and against the oracle on the c and g channels."""
    th, q, o = c1_case(seed=91, J=4096)
    th = synth.random_theta(8, 92)
    q, o = q[:1], o[:1]
    m = ef.EFunc(8, th)
    g, O, L = m.forward_backward(dev(q), dev(o), loss=ef.LOSS_MSE, want_O=True)
    m.forward(dev(q), dev(o), loss=ef.LOSS_MSE)
    g2 = m.backward().cpu().numpy()
    g = g.cpu().numpy()
    assert np.abs(g - g2).max() <= 1e-6 * np.abs(g2).max()
    f = orc.forward(th, 8, q)
    _, r = orc.mse_loss(f.O, o)
    ref = orc.backward(th, 8, q, f, r)
    for ch in (1, 2, 3, 4, 9, 10, 11, 12):
        assert np.abs(g[:, ch] - ref[:, ch]).max() <= TOL_GRAD * max(np.abs(ref[:, ch]).max(), 1e-6 * np.abs(ref).max())


@pytest.mark.parametrize("J", [33, 259, 4096])
def test_forward_backward_fused_parity_c1(J):
    """efunc_forward_backward (k_fit: forward, MSE upstream and backward per item in one
    kernel) against the oracle's forward + Eq. loss + Alg. 2. Ragged tiny batches use a random
    theta: on a fitted theta with a handful of queries the s-channel sum sum_j r p (f - O) dd is
    cancellation-dominated (|f - O| ~ 1e-3 of |f|), beyond what fp32 f - O can resolve."""
    th, q, o = c1_case(seed=91, J=4096)
    if J < 4096:
        th = synth.random_theta(8, 92)
    q, o = q[:J], o[:J]
    m = ef.EFunc(8, th)
    g, O, L = m.forward_backward(dev(q), dev(o), loss=ef.LOSS_MSE, want_O=True)
    f = orc.forward(th, 8, q)
    Lref, r = orc.mse_loss(f.O, o)
    assert nw(O.cpu().numpy(), f.O) <= TOL_VAL
    # the loss inherits O's tolerance: |dL| <= 1e-5 L + 2 mean|O - o| * 1e-5 max|O| (reading R-T)
    tol_L = 1e-5 * Lref + 2.0 * np.abs(f.O - o).mean() * TOL_VAL * np.abs(f.O).max()
    assert abs(float(L.item()) - Lref) <= tol_L
    check_grads(g.cpu().numpy(), orc.backward(th, 8, q, f, r), floor=1e-6)
    with pytest.raises(ef.EfuncError):  # no saved state is left behind
        m.backward()


def test_forward_backward_fused_slow_paths():
    """Items the fused kernel hands to the split kernels: out-of-domain queries (no brick list)
    and a beta spread that overflows the corner shift bound."""
    R = 8
    th = synth.random_theta(R, 93, log_scale_mean=7.5, log_scale_std=1.5)
    rg = synth.rng(94)
    q = np.concatenate([rg.uniform(-1, 1, size=(2500, 3)), rg.uniform(-1.6, 1.6, size=(500, 3))]).astype(np.float32)
    o = rg.normal(scale=0.2, size=3000).astype(np.float32)
    m = ef.EFunc(R, th)
    g, O, L = m.forward_backward(dev(q), dev(o), loss=ef.LOSS_MSE, want_O=True)
    f = orc.forward(th, R, q)
    Lref, r = orc.mse_loss(f.O, o)
    assert nw(O.cpu().numpy(), f.O) <= TOL_VAL
    check_grads(g.cpu().numpy(), orc.backward(th, R, q, f, r))


def test_forward_backward_fused_matches_split_c2():
    """C2 at full size: the fused kernel and the split forward/backward compute the same sums
    (fp32, different order): gradients agree to 1e-5 normwise per channel, loss to 1e-6."""
    R, J = 32, 1 << 20
    tor = synth.Torus()
    th = synth.init_theta(R, 95)
    m = ef.EFunc(R, th)
    m.mean_shift_init(dev(synth.surface_points(tor, 16384, seed=96)))
    q, o = synth.sample_batch(tor, J, seed=97)
    qd, od = dev(q), dev(o)
    g1, O1, L1 = m.forward_backward(qd, od, loss=ef.LOSS_MSE, want_O=True)
    _, _, L2 = m.forward(qd, od, loss=ef.LOSS_MSE)
    g2 = m.backward().cpu().numpy()
    g1 = g1.cpu().numpy()
    for ch in range(13):
        assert nw(g1[:, ch], g2[:, ch]) <= 1e-5, ch
    assert abs(float(L1.item()) - float(L2.item())) <= 1e-6 * float(L2.item())
    # and the fused values at sampled queries against the oracle
    idx = synth.rng(98).choice(J, size=512, replace=False)
    ref = orc.forward(m.get_params(), R, q[idx])
    assert nw(O1.cpu().numpy()[idx], ref.O) <= TOL_VAL


def test_forward_backward_r16_parity():
    """A mid-size grid (16^3, several bricks per axis, many items) against the oracle."""
    R, J = 16, 6000
    tor = synth.Torus()
    th = synth.fitted_like_theta(R, tor, 99)
    q, o = synth.sample_batch(tor, J, seed=100)
    m = ef.EFunc(R, th)
    g, O, L = m.forward_backward(dev(q), dev(o), loss=ef.LOSS_MSE, want_O=True)
    f = orc.forward(th, R, q)
    Lref, r = orc.mse_loss(f.O, o)
    assert nw(O.cpu().numpy(), f.O) <= TOL_VAL
    check_grads(g.cpu().numpy(), orc.backward(th, R, q, f, r))


# ----------------------------------------------------------------------------- batched shapes (C5)
def test_batched_shapes_match_single_handles_and_oracle():
    """n_shapes = 3 in one handle (config C5's layout: [S][...] arrays) against three single
    handles on the same data, and shape 1 against the oracle."""
    R, J, S = 8, 1500, 3
    shapes = synth.c5_shapes(S, 7)
    ths = np.stack([synth.fitted_like_theta(R, sh, 10 + k) for k, sh in enumerate(shapes)])
    bs = [synth.sample_batch(sh, J, seed=20 + k) for k, sh in enumerate(shapes)]
    q = np.stack([b[0] for b in bs]); o = np.stack([b[1] for b in bs])
    mb = ef.EFunc(R, ths, n_shapes=S)
    gb, Ob, Lb = mb.forward_backward(dev(q), dev(o), loss=ef.LOSS_MSE, want_O=True)
    assert tuple(gb.shape) == (S, R ** 3, 13) and tuple(Ob.shape) == (S, J) and tuple(Lb.shape) == (S, 1)
    gb = gb.cpu().numpy(); Ob = Ob.cpu().numpy()
    for k in range(S):
        m1 = ef.EFunc(R, ths[k])
        g1, O1, L1 = m1.forward_backward(dev(q[k]), dev(o[k]), loss=ef.LOSS_MSE, want_O=True)
        # same kernels on the same data; the in-bin query order (atomic scatter) may differ, which
        # changes item composition and hence only the rounding of negligible candidate pairs
        assert nw(O1.cpu().numpy(), Ob[k]) <= 1e-6
        assert np.abs(g1.cpu().numpy() - gb[k]).max() <= 1e-5 * np.abs(gb[k]).max()
    f = orc.forward(ths[1], R, q[1])
    _, r = orc.mse_loss(f.O, o[1])
    assert nw(Ob[1], f.O) <= TOL_VAL
    check_grads(gb[1], orc.backward(ths[1], R, q[1], f, r))
    # AdamW and parameter access follow the same layout
    mb.adamw_step(torch.as_tensor(gb).cuda())
    th_after = mb.get_params()
    assert th_after.shape == (S, R ** 3, 13) and not np.array_equal(th_after, ths)


def test_fit_step_pipelined_host_io_matches_device_path():
    """host_io 2 (copies on the library's stream, double-buffered) gives the same trajectory as
    device-pointer fit steps on the same batches (same kernels, same order of steps)."""
    R, J = 8, 3000
    sph = synth.Sphere(0.5)
    th = synth.fitted_like_theta(R, sph, 5)
    batches = [synth.sample_batch(sph, J, seed=60 + i) for i in range(4)]
    ma, mb = ef.EFunc(R, th, fit_graph=False), ef.EFunc(R, th, fit_graph=False)
    ma.set_params(th); mb.set_params(th)
    la = []
    for q, o in batches:
        lo = torch.zeros(1, device="cuda")
        ma.fit_step(dev(q), dev(o), loss_out=lo)
        la.append(float(lo.item()))
    hq = [torch.as_tensor(q).pin_memory() for q, _ in batches]
    ho = [torch.as_tensor(o).pin_memory() for _, o in batches]
    outs = [mb.fit_step(hq[i], ho[i], pipelined=True) for i in range(4)]
    mb.sync()
    lb = [float(x[0]) for x in outs]
    assert np.allclose(la, lb, rtol=1e-5, atol=0)
    # float atomics reorder between the two runs: a near-zero gradient may flip sign and AdamW then
    # moves that entry by up to 2 lr per step; everything else agrees to rounding
    d = np.abs(ma.get_params() - mb.get_params())
    assert d.max() <= 2 * 6e-4 * len(batches) + 1e-6
    assert np.mean(d > 1e-5) <= 1e-3


# ----------------------------------------------------------------------------- C4 geometry (64^3)
def test_c4a_grid_sampled_parity():
    """C4a geometry: 64^3 x 13 grid (2 x 2 x 2-cell bricks), 2^22 torus points through the fused
    fit path; values at sampled queries and the gradient of a sampled upstream against the
    oracle (global sums over all 2 x 64^3 keys)."""
    R, J = 64, 1 << 22
    tor = synth.Torus()
    th = synth.init_theta(R, 64)
    m = ef.EFunc(R, th)
    m.mean_shift_init(dev(synth.surface_points(tor, 16384, seed=65)))
    thg = m.get_params()
    q, o = synth.sample_batch(tor, J, seed=66)
    qd, od = dev(q), dev(o)
    g, O, L = m.forward_backward(qd, od, loss=ef.LOSS_MSE, want_O=True)
    idx = synth.rng(67).choice(J, size=96, replace=False)
    ref = orc.forward(thg, R, q[idx])
    assert nw(O.cpu().numpy()[idx], ref.O) <= TOL_VAL
    sub = synth.rng(68).choice(J, size=64, replace=False)
    r = np.zeros(J, np.float32)
    r[sub] = synth.rng(69).normal(size=64).astype(np.float32)
    m.forward(qd)
    gs = m.backward(dL_dO=dev(r)).cpu().numpy()
    fs = orc.forward(thg, R, q[sub])
    check_grads(gs, orc.backward(thg, R, q[sub], fs, r[sub].astype(np.float64)))
    # a few bricks inside dense offset-key clusters exceed the 16384-entry list cap; their items
    # take the enumerate path (exact, slower)
    assert m.stats()["list_overflow"] <= 0.01 * 32 ** 3


@pytest.mark.parametrize("R", [8, 16])
def test_forward_backward_dense_mode_parity(R):
    """cutoff_T = inf (the paper's dense definition, every pair): the fused kernel walks all 2R^3
    keys per item; against the oracle's global sums."""
    tor = synth.Torus()
    th = synth.fitted_like_theta(R, tor, 101)
    q, o = synth.sample_batch(tor, 3000, seed=102)
    m = ef.EFunc(R, th, cutoff_T=float("inf"))
    g, O, L = m.forward_backward(dev(q), dev(o), loss=ef.LOSS_MSE, want_O=True)
    f = orc.forward(th, R, q)
    Lref, r = orc.mse_loss(f.O, o)
    assert nw(O.cpu().numpy(), f.O) <= TOL_VAL
    check_grads(g.cpu().numpy(), orc.backward(th, R, q, f, r))
    assert m.stats()["candidate_pairs"] == 3000 * 2 * R ** 3


# ----------------------------------------------------------------------------- fused Eikonal (C3)
@pytest.mark.parametrize("J", [33, 4096])
def test_forward_backward_eikonal_fused_parity(J):
    """k_fit_eik (forward with G, MSE + Eikonal upstreams, second-order backward per item)
    against the oracle: O, G and the loss, and all 13 gradient channels."""
    th, q, o = c1_case(seed=111, J=4096)
    if J < 4096:
        th = synth.random_theta(8, 112)
    q, o = q[:J], o[:J]
    m = ef.EFunc(8, th)
    g, O, L = m.forward_backward(dev(q), dev(o), loss=ef.LOSS_MSE_EIKONAL, eikonal_lambda=0.1, want_O=True)
    f = orc.forward(th, 8, q)
    Lm, r = orc.mse_loss(f.O, o)
    Le, h = orc.eikonal_loss(f.G, 0.1)
    assert nw(O.cpu().numpy(), f.O) <= TOL_VAL
    assert abs(float(L.item()) - (Lm + Le)) <= 1e-5 * (Lm + Le) + 2e-5 * np.abs(f.O - o).mean() * np.abs(f.O).max()
    check_grads(g.cpu().numpy(), orc.backward(th, 8, q, f, r, h), floor=1e-6)


def test_forward_backward_eikonal_fused_slow_paths():
    R = 8
    th = synth.random_theta(R, 113, log_scale_mean=7.5, log_scale_std=1.5)
    rg = synth.rng(114)
    q = np.concatenate([rg.uniform(-1, 1, size=(2500, 3)), rg.uniform(-1.6, 1.6, size=(500, 3))]).astype(np.float32)
    o = rg.normal(scale=0.2, size=3000).astype(np.float32)
    m = ef.EFunc(R, th)
    g, O, L = m.forward_backward(dev(q), dev(o), loss=ef.LOSS_MSE_EIKONAL, eikonal_lambda=0.1, want_O=True)
    f = orc.forward(th, R, q)
    _, r = orc.mse_loss(f.O, o)
    _, h = orc.eikonal_loss(f.G, 0.1)
    assert nw(O.cpu().numpy(), f.O) <= TOL_VAL
    check_grads(g.cpu().numpy(), orc.backward(th, R, q, f, r, h), floor=1e-6)


def test_forward_backward_eikonal_fused_matches_split_c3():
    """C3 geometry at full size (2^22 torus points): fused vs split (forward with G + Eikonal
    backward) agree to 1e-5 per channel."""
    R, J = 32, 1 << 22
    tor = synth.Torus()
    m = ef.EFunc(R, synth.init_theta(R, 115))
    m.mean_shift_init(dev(synth.surface_points(tor, 16384, seed=116)))
    q, o = synth.sample_batch(tor, J, seed=117)
    qd, od = dev(q), dev(o)
    g1, _, L1 = m.forward_backward(qd, od, loss=ef.LOSS_MSE_EIKONAL, eikonal_lambda=0.1)
    _, _, L2 = m.forward(qd, od, loss=ef.LOSS_MSE_EIKONAL, eikonal_lambda=0.1, want_G=True)
    g2 = m.backward().cpu().numpy()
    g1 = g1.cpu().numpy()
    for ch in range(13):
        assert nw(g1[:, ch], g2[:, ch]) <= 1e-5, ch
    assert abs(float(L1.item()) - float(L2.item())) <= 1e-6 * float(L2.item())


def test_c4b_grid_128_functional_parity():
    """C4b geometry (128^3 x 13 = 27M parameters): at T = 20 the brick lists overflow the list cap
    (the cutoff ball holds ~35k keys per brick), so every item takes the enumerate path; values
    and sampled-upstream gradients still match the oracle."""
    R, J = 128, 1 << 14
    tor = synth.Torus()
    th = synth.init_theta(R, 128)
    m = ef.EFunc(R, th)
    m.mean_shift_init(dev(synth.surface_points(tor, 16384, seed=129)))
    thg = m.get_params()
    q, o = synth.sample_batch(tor, J, seed=130)
    g, O, L = m.forward_backward(dev(q), dev(o), loss=ef.LOSS_MSE, want_O=True)
    idx = synth.rng(131).choice(J, size=32, replace=False)
    ref = orc.forward(thg, R, q[idx])
    assert nw(O.cpu().numpy()[idx], ref.O) <= TOL_VAL
    sub = idx[:16]
    r = np.zeros(J, np.float32)
    r[sub] = synth.rng(132).normal(size=16).astype(np.float32)
    m.forward(dev(q))
    gs = m.backward(dL_dO=dev(r)).cpu().numpy()
    fs = orc.forward(thg, R, q[sub])
    check_grads(gs, orc.backward(thg, R, q[sub], fs, r[sub].astype(np.float64)))


# ----------------------------------------------------------------------------- degree 0 (NEXT-4)
def test_degree0_variant_parity_and_frozen_g():
    """degree = 0 (Table 3 G-0, f = c): the g channels are zeroed at creation and never updated;
    values and the c / s / Delta gradients match the oracle on the same theta with g = 0."""
    th, q, o = c1_case(seed=121, J=3000)
    m = ef.EFunc(8, th, degree=0)
    th0 = th.copy()
    th0[:, 2:5] = 0.0
    th0[:, 10:13] = 0.0
    assert np.array_equal(m.get_params(), th0)
    g, O, L = m.forward_backward(dev(q), dev(o), loss=ef.LOSS_MSE, want_O=True)
    f = orc.forward(th0, 8, q)
    _, r = orc.mse_loss(f.O, o)
    ref = orc.backward(th0, 8, q, f, r)
    assert nw(O.cpu().numpy(), f.O) <= TOL_VAL
    g = g.cpu().numpy()
    for ch in (0, 1, 5, 6, 7, 8, 9):
        assert nw(g[:, ch], ref[:, ch]) <= TOL_GRAD, ch
    for _ in range(3):
        m.fit_step(dev(q), dev(o))
    p = m.get_params()
    assert np.all(p[:, 2:5] == 0.0) and np.all(p[:, 10:13] == 0.0)
    assert not np.array_equal(p[:, 1], th0[:, 1])


def test_batched_shapes_pipelined_host_io():
    """n_shapes = 2 with pipelined host I/O: each shape's fit step and loss read-back through the
    batched handle equals two single-shape handles stepping the same batches."""
    R, J, S = 8, 2000, 2
    shapes = synth.c5_shapes(S, 17)
    ths = np.stack([synth.fitted_like_theta(R, sh, 30 + k) for k, sh in enumerate(shapes)])
    batches = []
    for i in range(3):
        bs = [synth.sample_batch(sh, J, seed=40 + 10 * i + k) for k, sh in enumerate(shapes)]
        batches.append((np.stack([b[0] for b in bs]), np.stack([b[1] for b in bs])))
    mb = ef.EFunc(R, ths, n_shapes=S, fit_graph=False)
    outs = [mb.fit_step(torch.as_tensor(q).pin_memory(), torch.as_tensor(o).pin_memory(), pipelined=True)
            for q, o in batches]
    mb.sync()
    for k in range(S):
        m1 = ef.EFunc(R, ths[k], fit_graph=False)
        for i, (q, o) in enumerate(batches):
            lo = torch.zeros(1, device="cuda")
            m1.fit_step(dev(q[k]), dev(o[k]), loss_out=lo)
            assert abs(float(lo.item()) - float(outs[i][k])) <= 1e-5 * float(lo.item())
        d = np.abs(m1.get_params() - mb.get_params()[k])
        assert np.mean(d > 1e-5) <= 1e-3


@pytest.mark.parametrize("R", [2, 3])
def test_forward_backward_tiny_grids(R):
    """R = 2, 3 (one or a few cells; the out-of-domain queries go to the split kernels) through
    the fused call, and J = 0."""
    th = synth.random_theta(R, 140 + R, log_scale_mean=1.0)
    rg = synth.rng(150 + R)
    q = rg.uniform(-1.5, 1.5, size=(700, 3)).astype(np.float32)
    o = rg.normal(scale=0.3, size=700).astype(np.float32)
    m = ef.EFunc(R, th)
    g, O, L = m.forward_backward(dev(q), dev(o), loss=ef.LOSS_MSE, want_O=True)
    f = orc.forward(th, R, q)
    _, r = orc.mse_loss(f.O, o)
    assert nw(O.cpu().numpy(), f.O) <= TOL_VAL
    check_grads(g.cpu().numpy(), orc.backward(th, R, q, f, r), floor=1e-6)
    g0, _, L0 = m.forward_backward(dev(q[:0]), dev(o[:0]), loss=ef.LOSS_MSE)
    assert float(g0.abs().sum()) == 0.0 and float(L0.item()) == 0.0


def test_forward_backward_large_beta_accuracy():
    """Large scales (s ~ 9 +- 0.5, beta ~ 8e3, as after long fits) at 32^3: the fused kernel's
    item-local expansion of the exponent keeps O and all 13 gradient channels within tolerance
    of the oracle (full batch, every query's upstream)."""
    R, J = 32, 2000
    tor = synth.Torus()
    th = synth.fitted_like_theta(R, tor, 160)
    rg = synth.rng(161)
    th[:, 0] = 9.0 + rg.normal(scale=0.5, size=R ** 3)
    th[:, 8] = 9.0 + rg.normal(scale=0.5, size=R ** 3)
    th = th.astype(np.float32)
    q, o = synth.sample_batch(tor, J, seed=162)
    m = ef.EFunc(R, th)
    g, O, L = m.forward_backward(dev(q), dev(o), loss=ef.LOSS_MSE, want_O=True)
    f = orc.forward(th, R, q)
    _, r = orc.mse_loss(f.O, o)
    assert nw(O.cpu().numpy(), f.O) <= TOL_VAL
    check_grads(g.cpu().numpy(), orc.backward(th, R, q, f, r))


# ----------------------------------------------------------------------------- fitting (end to end)
def test_fit_linear_field_to_zero_and_torus_loss_drops():
    """The fit loop through the fused path (SURVEY §8(c) "Fit loop" pin): a linear target is
    exactly representable (partition of unity), so the MSE falls by more than an order of
    magnitude within 200 steps; on the torus at 32^3 (paper lr 6e-4) the loss falls by a third within 300 steps of
    2^18 points."""
    R = 16
    A, B = 0.1, np.array([0.3, -0.2, 0.4])
    rg = synth.rng(170)
    m = ef.EFunc(R, synth.init_theta(R, 171))
    hp = ef.AdamW(lr=3e-3)
    lo = torch.zeros(1, device="cuda")
    losses = []
    for k in range(200):
        q = rg.uniform(-1, 1, size=(1 << 14, 3)).astype(np.float32)
        o = (A + q.astype(np.float64) @ B).astype(np.float32)
        m.fit_step(dev(q), dev(o), hp, loss_out=lo)
        losses.append(float(lo.item()))
    assert np.mean(losses[-10:]) < 0.05 * np.mean(losses[:10]), (losses[0], losses[-1])
    tor = synth.Torus()
    m2 = ef.EFunc(32, synth.init_theta(32, 172))
    m2.mean_shift_init(dev(synth.surface_points(tor, 16384, seed=173)))
    tl = []
    for k in range(300):
        q, o = synth.sample_batch(tor, 1 << 18, seed=2000 + k)
        m2.fit_step(dev(q), dev(o), loss_out=lo)
        tl.append(float(lo.item()))
    assert np.mean(tl[-20:]) < 0.65 * np.mean(tl[:20]), (np.mean(tl[:20]), np.mean(tl[-20:]))


def test_eval_grad_padded_lattice_many_out_of_domain_queries():
    """A lattice over a padded box: ~35% of the queries lie outside [-1,1]^3 and share
    the out-of-domain bin. The stable sort (LSD radix, O(n) per pass) keeps this fast, and the
    outside queries (exact-shift split kernels) match the oracle."""
    import time
    R, N = 16, 96
    th = synth.fitted_like_theta(R, synth.Torus(), 181)
    t = np.linspace(-1.15, 1.15, N, dtype=np.float32)
    z, y, x = np.meshgrid(t, t, t, indexing="ij")
    q = np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1).astype(np.float32)
    outside = np.any(np.abs(q) > 1.0, axis=1)
    assert outside.mean() > 0.3
    m = ef.EFunc(R, th)
    qd = dev(q)
    m.eval_grad(qd)  # warm-up (sizes the workspaces)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    O, G = m.eval_grad(qd)
    torch.cuda.synchronize()
    assert time.perf_counter() - t0 < 5.0
    rs = synth.rng(182)
    idx = np.concatenate([rs.choice(np.where(outside)[0], 150, replace=False),
                          rs.choice(np.where(~outside)[0], 150, replace=False)])
    ref = orc.forward(th, R, q[idx])
    assert nw(O.cpu().numpy()[idx], ref.O) <= TOL_VAL
    for a in range(3):
        assert nw(G.cpu().numpy()[idx, a], ref.G[:, a]) <= TOL_VAL
