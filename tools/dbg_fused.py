"""Debug: per-channel gradient error of the fused path vs the oracle at small J (random theta)."""
import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
import oracle as orc, paper_2505_21319_b200 as ef
from workloads import synth
sph = synth.Sphere(0.5); th = synth.random_theta(8, 92); q, o = synth.sample_batch(sph, 4096, seed=191)
for J in (1, 33):
    qq, oo = q[:J], o[:J]
    m = ef.EFunc(8, th)
    g, O, L = m.forward_backward(torch.as_tensor(qq).cuda(), torch.as_tensor(oo).cuda(), loss=ef.LOSS_MSE, want_O=True)
    g = g.cpu().numpy()
    f = orc.forward(th, 8, qq); Lr, r = orc.mse_loss(f.O, oo); gr = orc.backward(th, 8, qq, f, r)
    big = np.abs(gr).max()
    for c in range(13):
        e = np.abs(g[:, c] - gr[:, c]); i = int(e.argmax())
        print(J, c, f"maxref/big {np.abs(gr[:, c]).max()/big:.3e} err/big {e.max()/big:.3e} at {i} gpu {g[i, c]:.6e} ref {gr[i, c]:.6e}")
