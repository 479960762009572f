"""Debug: OFFSET/1 G NaNs (dense split forward)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_21319_b200 as ef
from oracle import variant_oracle as vo
from workloads import synth
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_variants import variant_theta, dev, nw
for banks, deg in ((vo.OFFSET, 1), (vo.OFFSET, 2), (vo.GRID, 2)):
    R, J = 8, 2048
    sph = synth.Sphere(0.5)
    th = variant_theta(R, sph, banks, deg, 3)
    q, o = synth.sample_batch(sph, J, seed=11)
    m = ef.EFunc(R, th, degree=deg, variant={1: 1, 2: 2, 3: 0}[banks])
    O, G, L = m.forward(dev(q), dev(o), loss=ef.LOSS_MSE, want_G=True)
    torch.cuda.synchronize()
    Gg = G.cpu().numpy(); Og = O.cpu().numpy()
    bad = np.where(~np.isfinite(Gg).all(axis=1))[0]
    f = vo.forward(th, R, q, banks, deg)
    print(banks, deg, "nan rows", len(bad), bad[:10], "stats", m.stats())
    for j in bad[:5]:
        print(" q", q[j], "O", Og[j], f.O[j], "G", Gg[j], f.G[j])
    fin = np.isfinite(Gg).all(axis=1)
    for ax in range(3):
        e = np.abs(Gg[fin, ax] - f.G[fin, ax]); k = np.argmax(e)
        print(" ax", ax, "nw", e.max() / np.abs(f.G[:, ax]).max(), "worst q", q[fin][k], Gg[fin][k], f.G[fin][k])
