"""NEXT-4: the Table 3 model families on the GPU against the float64
variant oracle (oracle/variant_oracle.py): degree-2 polynomials of Eq. poly-func,
O over the fixed grid alone (Eq. func-interp), O^Delta with learnable keys alone (Eq. func-with-offset,
PAPER.md:L442-447) and their union (Eq. func-offset). Tolerances as everywhere (reading R-T):
normwise 1e-5 on O and each G component, 1e-4 per gradient channel."""
import numpy as np
import pytest

import oracle as orc
from oracle import variant_oracle as vo
from workloads import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2505_21319_b200 as ef  # noqa: E402

VARIANT = {vo.BOTH: ef.VARIANT_COMBINED, vo.GRID: ef.VARIANT_GRID, vo.OFFSET: ef.VARIANT_OFFSET}


def nw(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def dev(x):
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def variant_theta(R, shape, banks, degree, seed, h_scale=0.5):
    """A fitted-looking theta in the variant layout: s ~ 7 +- 0.3, c = sdf + noise, g = grad sdf +
    noise, H a random symmetric square, offsets = surface projection + noise."""
    g = synth.rng(seed, 77)
    lay = vo.layout(banks, degree)
    n = R ** 3
    th = np.zeros((n, lay["nch"]))
    k = orc.node_positions(R)

    def fill(s0, pos):
        th[:, s0] = 7.0 + g.normal(scale=0.3, size=n)
        th[:, s0 + 1] = shape.sdf(pos) + g.normal(scale=0.01, size=n)
        if degree >= 1:
            th[:, s0 + 2:s0 + 5] = shape.grad(pos) + g.normal(scale=0.05, size=(n, 3))
        if degree >= 2:
            th[:, s0 + 5:s0 + 11] = g.normal(scale=h_scale, size=(n, 6))
    if lay["grid"] is not None:
        fill(lay["grid"], k)
    if lay["off"] is not None:
        d = shape.project(k) - k + g.normal(scale=0.003, size=(n, 3))
        th[:, lay["delta"]:lay["delta"] + 3] = d
        fill(lay["off"], k + d)
    return th.astype(np.float32)


def check_grads(g, ref, tol=1e-4):
    for ch in range(ref.shape[1]):
        scale = max(float(np.abs(ref[:, ch]).max()), 1e-30)
        e = float(np.abs(g[:, ch] - ref[:, ch]).max()) / scale
        assert e <= tol, (ch, e)


CASES = [
    (vo.GRID, 2, 8, 2048),      # Table 3 G-7
    (vo.GRID, 2, 16, 4096),
    (vo.BOTH, 2, 8, 2048),      # O^{+Delta} with degree 2 (25 channels)
    (vo.GRID, 1, 8, 2048),      # G-6 (fused path)
    (vo.GRID, 0, 8, 2048),      # G-5
    (vo.OFFSET, 1, 8, 2048),    # Full-1 (dense)
    (vo.OFFSET, 2, 8, 1024),
]


@pytest.mark.parametrize("banks,degree,R,J", CASES)
def test_variant_forward_backward_matches_oracle(banks, degree, R, J):
    sph = synth.Sphere(0.5)
    th = variant_theta(R, sph, banks, degree, 3)
    q, o = synth.sample_batch(sph, J, seed=11)
    m = ef.EFunc(R, th, degree=degree, variant=VARIANT[banks])
    assert m.nch == vo.n_channels(banks, degree)
    O, G, L = m.forward(dev(q), dev(o), loss=ef.LOSS_MSE, want_G=True)
    grad = m.backward()
    torch.cuda.synchronize()
    f = vo.forward(th, R, q, banks, degree)
    assert nw(O.cpu().numpy(), f.O) <= 1e-5
    Gg = G.cpu().numpy()
    # O^Delta alone (no fixed keys) extrapolates far from its surface keys: there the softmax weights
    # of a query ~1 away from every key (m_j ~ 1e3 nats) move by 2 beta |d| |delta k| ~ 2e-4 relative
    # under the fp32 rounding of the key positions k_n + Delta_n themselves, so G is compared at 1e-5
    # on the queries within 0.1 of the surface and at 1e-4 on the far field (reading R-V2)
    near = np.abs(sph.sdf(q.astype(np.float64))) <= 0.1 if banks == vo.OFFSET else np.ones(J, bool)
    for ax in range(3):
        assert nw(Gg[near, ax], f.G[near, ax]) <= 1e-5, ax
        assert nw(Gg[:, ax], f.G[:, ax]) <= (1e-4 if banks == vo.OFFSET else 1e-5), ax
    r = 2.0 * (f.O - o) / J
    gref = vo.backward(th, R, q, f, r, banks, degree)
    check_grads(grad.cpu().numpy(), gref)
    Lr = np.mean((f.O - o) ** 2)
    assert abs(float(L.item()) - Lr) <= 1e-5 * Lr
    # the fused call (k_fit for degree <= 1, forward + backward for degree 2) on the same batch
    m2 = ef.EFunc(R, th, degree=degree, variant=VARIANT[banks])
    g2, O2, _ = m2.forward_backward(dev(q), dev(o), loss=ef.LOSS_MSE, want_O=True)
    torch.cuda.synchronize()
    assert nw(O2.cpu().numpy(), f.O) <= 1e-5
    check_grads(g2.cpu().numpy(), gref)


@pytest.mark.parametrize("banks", [vo.GRID, vo.BOTH])
def test_degree2_partition_of_unity_on_gpu(banks):
    """Every key carries one global quadratic P's Taylor expansion at its position: the GPU
    interpolant returns P(q) and grad P(q) (fp32 rounding only), for any beta and offsets."""
    R, degree = 12, 2
    gen = synth.rng(21)
    A0, B = 0.2, gen.normal(size=3)
    Cm = gen.normal(scale=0.5, size=(3, 3)); Cm = 0.5 * (Cm + Cm.T)
    th = variant_theta(R, synth.Sphere(0.5), banks, degree, 5).astype(np.float64)
    lay = vo.layout(banks, degree)
    k = orc.node_positions(R)

    def fill(s0, pos):
        th[:, s0 + 1] = A0 + pos @ B + 0.5 * np.einsum("na,ab,nb->n", pos, Cm, pos)
        th[:, s0 + 2:s0 + 5] = B[None] + pos @ Cm
        for slot, (a, b) in enumerate(vo.H_IDX):
            th[:, s0 + 5 + slot] = Cm[a, b]
    th32 = th.astype(np.float32)
    if lay["grid"] is not None:
        fill(lay["grid"], k)
    if lay["off"] is not None:
        fill(lay["off"], k + th32[:, lay["delta"]:lay["delta"] + 3].astype(np.float64))
    th32 = th.astype(np.float32)
    q = gen.uniform(-0.95, 0.95, size=(4096, 3)).astype(np.float32)
    m = ef.EFunc(R, th32, degree=degree, variant=VARIANT[banks])
    O, G = m.eval_grad(dev(q))
    torch.cuda.synchronize()
    qd = q.astype(np.float64)
    P = A0 + qd @ B + 0.5 * np.einsum("ja,ab,jb->j", qd, Cm, qd)
    assert nw(O.cpu().numpy(), P) <= 2e-6
    GB = B[None] + qd @ Cm
    Gg = G.cpu().numpy()
    for ax in range(3):
        assert nw(Gg[:, ax], GB[:, ax]) <= 1e-5, ax


def test_variant_fit_loop_and_api():
    """G-7 (grid keys, degree 2, learnable scale) fits a sphere through efunc_fit_step; layout
    checks; mean shift needs an offset bank."""
    R = 16
    sph = synth.Sphere(0.5)
    th = variant_theta(R, sph, vo.GRID, 2, 9, h_scale=0.0)
    th[:, 1] += 0.05  # start off the target
    m = ef.EFunc(R, th, degree=2, variant=ef.VARIANT_GRID)
    assert m.get_params().shape == (R ** 3, 11)
    batches = [synth.sample_batch(sph, 8192, seed=40 + i) for i in range(4)]
    lo = torch.zeros(1, device="cuda")
    losses = []
    for s in range(60):
        q, o = batches[s % 4]
        m.fit_step(dev(q), dev(o), hp=ef.AdamW(lr=2e-3), loss_out=lo)
        losses.append(float(lo.item()))
    assert losses[-1] < 0.5 * losses[0], (losses[0], losses[-1])
    with pytest.raises(ef.EfuncError):
        m.mean_shift_init(dev(synth.surface_points(sph, 64, 1)))
    with pytest.raises(ef.EfuncError):  # degree 2 has no Eikonal terms
        m.forward(dev(batches[0][0]), dev(batches[0][1]), loss=ef.LOSS_MSE_EIKONAL)
    # the offset-only variant takes the mean-shift initialisation
    m2 = ef.EFunc(8, variant_theta(8, sph, vo.OFFSET, 1, 2), degree=1, variant=ef.VARIANT_OFFSET)
    m2.mean_shift_init(dev(synth.surface_points(sph, 2048, 3)))
    th2 = m2.get_params()
    assert th2.shape == (512, 8)
    k = orc.node_positions(8)
    ref = orc.mean_shift_offsets(8, synth.surface_points(sph, 2048, 3))
    assert np.abs(th2[:, 0:3] - ref).max() <= 1e-4
