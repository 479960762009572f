"""NEXT-4 cosine-series stacks (§4.4, Eq. cosine-series) on the GPU: S, dS/dq and
the per-band parameter gradients of the MSE loss of S against the float64 oracle
(oracle/variant_oracle.py cosine_forward / cosine_backward); a short fit. Tolerances as everywhere
(reading R-T)."""
import numpy as np
import pytest

from oracle import variant_oracle as vo
from workloads import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2505_21319_b200 as ef  # noqa: E402


def nw(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def dev(x):
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def band_thetas(R, B, shape, seed):
    """G-6 bands [s, c, g]: band 0 carries the shape's SDF, the others small random corrections."""
    g = synth.rng(seed, 88)
    k = synth._lattice_nodes(R)
    th = np.zeros((B, R ** 3, 5))
    for b in range(B):
        th[b, :, 0] = 5.5 + g.normal(scale=0.3, size=R ** 3)
        amp = 1.0 if b == 0 else 0.05
        th[b, :, 1] = amp * shape.sdf(k) + g.normal(scale=0.01, size=R ** 3)
        th[b, :, 2:5] = amp * shape.grad(k) + g.normal(scale=0.05, size=(R ** 3, 3))
    return th.astype(np.float32)


@pytest.mark.parametrize("B", [1, 3])
def test_cosine_stack_matches_oracle(B):
    R, J = 8, 2048
    sph = synth.Sphere(0.5)
    th = band_thetas(R, B, sph, 4)
    q, o = synth.sample_batch(sph, J, seed=5)
    st = ef.CosineStack(R, B, th)
    S, GS, L = st.forward(dev(q), dev(o), want_G=True)
    grad = st.backward()
    torch.cuda.synchronize()
    Sr, GSr, fs = vo.cosine_forward([t for t in th], R, q)
    assert nw(S.cpu().numpy(), Sr) <= 1e-5
    G = GS.cpu().numpy()
    for ax in range(3):
        assert nw(G[:, ax], GSr[:, ax]) <= 1e-5, ax
    Lr = np.mean((Sr - o) ** 2)
    assert abs(float(L.item()) - Lr) <= 1e-5 * Lr
    gr = vo.cosine_backward([t for t in th], R, q, fs, 2.0 * (Sr - o) / J)
    g = grad.cpu().numpy().reshape(B, R ** 3, 5)
    for b in range(B):
        for ch in range(5):
            assert nw(g[b, :, ch], gr[b][:, ch]) <= 1e-4, (b, ch)


def test_cosine_stack_fit_and_errors():
    R, B = 16, 3
    sph = synth.Sphere(0.5)
    th = band_thetas(R, B, sph, 6)
    th[0, :, 1] += 0.05
    st = ef.CosineStack(R, B, th)
    batches = [synth.sample_batch(sph, 8192, seed=70 + i) for i in range(4)]
    losses = []
    for s in range(40):
        q, o = batches[s % 4]
        _, _, L = st.forward(dev(q), dev(o))
        g = st.backward()
        st.adamw_step(g, ef.AdamW(lr=2e-3))
        losses.append(float(L.item()))
    assert losses[-1] < 0.5 * losses[0], (losses[0], losses[-1])
    lib = ef.load_library()
    assert lib.efunc_cosine_combine(None, 4, 0, None, None, None, 0, None, None, None, None, None) == 1  # B < 1
