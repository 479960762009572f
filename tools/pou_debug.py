import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as orc
import paper_2505_21319_b200 as ef
from workloads import synth
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
O, G, _ = m.forward(torch.as_tensor(q).cuda(), want_G=True)
G = G.cpu().numpy(); O = O.cpu().numpy()
err = np.abs(G - B[None]).max(axis=1)
idx = np.argsort(-err)[:10]
np.savez("gpurun_out/pou_debug.npz", q=q[idx], G=G[idx], err=err[idx], th=th)
print("max err", err[idx[:5]], "queries", q[idx[:3]])
ref = orc.forward(th, R, q[idx[:5]])
print("oracle G", ref.G, "gpu G", G[idx[:5]])
print("oracle O-P", ref.O - (A + q[idx[:5]].astype(np.float64) @ B), "gpu O-P", O[idx[:5]] - (A + q[idx[:5]].astype(np.float64) @ B))
