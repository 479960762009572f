"""Edge cases of the round-2 paths against the float64 oracles: the fused deterministic kernel with
items that take the fixed-point slow path, dense mode with queries whose Z underflows, degree-2 and
O^Delta-only variants with empty, single and out-of-domain queries, and a mesh without a surface.
Tolerances as everywhere (reading R-T)."""
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
from test_gpu_variants import variant_theta  # noqa: E402


def nw(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def dev(x):
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def check_grads(g, ref, tol=1e-4):
    for ch in range(ref.shape[1]):
        scale = max(float(np.abs(ref[:, ch]).max()), 1e-30)
        assert float(np.abs(g[:, ch] - ref[:, ch]).max()) / scale <= tol, ch


def test_deterministic_fused_with_slow_items_bitwise_and_parity():
    """Deterministic mode runs k_fit with 64-bit fixed-point sums; out-of-domain queries go to the
    split kernels' fixed-point list backward with the same unit. Two handles agree bitwise and the
    gradient matches the oracle."""
    R = 8
    sph = synth.Sphere(0.5)
    th = synth.fitted_like_theta(R, sph, 31)
    q, o = synth.sample_batch(sph, 3000, seed=32)
    q[:200] *= 1.6  # a slice of the batch outside [-1, 1]^3
    o = sph.sdf(q.astype(np.float64)).astype(np.float32)
    outs = []
    for _ in range(2):
        m = ef.EFunc(R, th, deterministic=True)
        g, O, L = m.forward_backward(dev(q), dev(o), loss=ef.LOSS_MSE, want_O=True)
        torch.cuda.synchronize()
        outs.append((g.cpu().numpy(), O.cpu().numpy(), float(L.item())))
        m.check()
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2]
    f = orc.forward(th, R, q)
    _, r = orc.mse_loss(f.O, o)
    assert nw(outs[0][1], f.O) <= 1e-5
    check_grads(outs[0][0], orc.backward(th, R, q, f, r))


def test_dense_mode_with_far_queries_and_tiny_batches():
    """cutoff_T = inf: out-of-domain queries take the split kernels; batches of 1 and 33 queries."""
    R = 8
    tor = synth.Torus()
    th = synth.fitted_like_theta(R, tor, 41)
    for J, far in ((1, 0), (33, 0), (2000, 40)):
        q, o = synth.sample_batch(tor, J, seed=42 + J)
        if far:
            # outside [-1, 1]^3 (their items take the split kernels) but not so far that the
            # s-gradient, ~ a (f - O) with a in the thousands of nats, is cancellation-limited in fp32
            q[:far] = synth.rng(43).uniform(1.02, 1.3, size=(far, 3)) * np.sign(q[:far])
            o = tor.sdf(q.astype(np.float64)).astype(np.float32)
        m = ef.EFunc(R, th, cutoff_T=float("inf"))
        g, O, L = m.forward_backward(dev(q), dev(o), loss=ef.LOSS_MSE, want_O=True)
        torch.cuda.synchronize()
        f = orc.forward(th, R, q)
        _, r = orc.mse_loss(f.O, o)
        assert nw(O.cpu().numpy(), f.O) <= 1e-5, J
        gref = orc.backward(th, R, q, f, r)
        if J > 1:
            check_grads(g.cpu().numpy(), gref)
        else:
            # one query: the s and Delta channels are cancellation-limited in fp32 (their terms carry
            # f_i - O with O ~ f_i), as in test_forward_backward_single_query: the c and g channels
            # against the oracle, all channels against the dense split path (same pair arithmetic)
            gg = g.cpu().numpy()
            for ch in (1, 2, 3, 4, 9, 10, 11, 12):
                assert np.abs(gg[:, ch] - gref[:, ch]).max() <= 1e-4 * max(np.abs(gref[:, ch]).max(),
                                                                           1e-6 * np.abs(gref).max()), ch
            m.forward(dev(q), dev(o), loss=ef.LOSS_MSE)
            g2 = m.backward().cpu().numpy()
            assert np.abs(gg - g2).max() <= 1e-5 * np.abs(g2).max()


@pytest.mark.parametrize("banks,degree", [(vo.GRID, 2), (vo.OFFSET, 1), (vo.BOTH, 2)])
def test_variants_empty_single_and_out_of_domain(banks, degree):
    R = 6
    sph = synth.Sphere(0.5)
    th = variant_theta(R, sph, banks, degree, 51)
    variant = {vo.BOTH: ef.VARIANT_COMBINED, vo.GRID: ef.VARIANT_GRID, vo.OFFSET: ef.VARIANT_OFFSET}[banks]
    m = ef.EFunc(R, th, degree=degree, variant=variant)
    # empty batch
    q0 = torch.zeros(0, 3, device="cuda")
    O0, _, _ = m.forward(q0)
    assert O0.numel() == 0
    for J in (1, 500):
        q = synth.rng(52 + J).uniform(-1.4, 1.4, size=(J, 3)).astype(np.float32)  # partly out of domain
        o = sph.sdf(q.astype(np.float64)).astype(np.float32)
        g, O, _ = m.forward_backward(dev(q), dev(o), loss=ef.LOSS_MSE, want_O=True)
        torch.cuda.synchronize()
        f = vo.forward(th, R, q, banks, degree)
        assert nw(O.cpu().numpy(), f.O) <= 1e-5, J
        gref = vo.backward(th, R, q, f, 2.0 * (f.O - o) / J, banks, degree)
        # the far offset bank of a 1-query batch is compared relative to the largest gradient
        big = float(np.abs(gref).max())
        for ch in range(gref.shape[1]):
            scale = max(float(np.abs(gref[:, ch]).max()), (1e-3 if J == 1 else 0.0) * big, 1e-30)
            assert float(np.abs(g.cpu().numpy()[:, ch] - gref[:, ch]).max()) / scale <= 1e-4, (J, ch)


def test_mesh_without_surface_and_minimal_lattice():
    R = 8
    sph = synth.Sphere(0.5)
    m = ef.EFunc(R, synth.fitted_like_theta(R, sph, 61))
    v, t, n, lat = m.mesh(8, iso=5.0, want_lattice=True)  # O < 5 everywhere: no crossing
    assert v.shape[0] == 0 and t.shape[0] == 0
    assert lat.shape == (8, 8, 8)
    v2, t2, _, _ = m.mesh(2, lo=(-0.1, -0.1, -0.1), hi=(0.9, 0.9, 0.9))  # one cube across the sphere
    assert v2.shape[0] >= 3 and t2.shape[0] >= 1


@pytest.mark.parametrize("R,J", [(8, 2000), (16, 3000)])
def test_dense_eikonal_fused_parity(R, J):
    """cutoff_T = inf with the MSE + Eikonal loss: the key-sliced dense kernels (k_dense_eik_*)
    against the oracle's global sums: O, G via eval, the loss and all 13 gradient channels; a few
    out-of-domain queries take the split kernels."""
    tor = synth.Torus()
    th = synth.fitted_like_theta(R, tor, 71)
    q, o = synth.sample_batch(tor, J, seed=72)
    q[:20] = synth.rng(73).uniform(1.02, 1.2, size=(20, 3)) * np.sign(q[:20])
    o = tor.sdf(q.astype(np.float64)).astype(np.float32)
    m = ef.EFunc(R, th, cutoff_T=float("inf"))
    g, O, L = m.forward_backward(dev(q), dev(o), loss=ef.LOSS_MSE_EIKONAL, eikonal_lambda=0.1, want_O=True)
    torch.cuda.synchronize()
    f = orc.forward(th, R, q)
    Lm, r = orc.mse_loss(f.O, o)
    Le, h = orc.eikonal_loss(f.G, 0.1)
    assert nw(O.cpu().numpy(), f.O) <= 1e-5
    assert abs(float(L.item()) - (Lm + Le)) <= 1e-5 * (Lm + Le)
    check_grads(g.cpu().numpy(), orc.backward(th, R, q, f, r, h))
    assert m.stats()["candidate_pairs"] == J * 2 * R ** 3


def test_tensor_core_fit_path_parity():
    """The A/B tensor-core fit kernel (k_fit_tc: mma.sync, 3xTF32 contractions; EFUNC_FIT_TC=1, read
    once per process) on the fused-path oracle checks: C1 parity, the full-density R = 32 batch and
    the deterministic bitwise test, in a child process."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, EFUNC_FIT_TC="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_gpu_parity.py"),
                        os.path.join(root, "tests", "test_gpu_bench_configs.py"),
                        "-k", "fused_parity_c1 or full_density_r32 and not eik or deterministic_fit_bitwise"],
                       env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and " failed" not in r.stdout
