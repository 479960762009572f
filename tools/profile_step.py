"""Run a few C2/C3 fit steps (no timing) for ncu launch lists / captures."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_21319_b200 as ef  # noqa: E402
from workloads import synth  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--steps", type=int, default=3)
p.add_argument("--R", type=int, default=32)
p.add_argument("--J", type=int, default=1 << 20)
p.add_argument("--eikonal", action="store_true")
p.add_argument("--split", action="store_true", help="forward + backward instead of forward_backward")
p.add_argument("--dense", action="store_true", help="cutoff_T = inf (every pair)")
p.add_argument("--near", type=float, default=0.5, help="near-surface fraction of the batch")
a = p.parse_args()
tor = synth.Torus()
m = ef.EFunc(a.R, synth.init_theta(a.R, 1234), cutoff_T=float("inf") if a.dense else 20.0)
m.mean_shift_init(torch.as_tensor(synth.surface_points(tor, 16384, 1234)).cuda())
q, o = synth.sample_batch(tor, a.J, seed=99, near_fraction=a.near)
qd, od = torch.as_tensor(q).cuda(), torch.as_tensor(o).cuda()
grad = torch.zeros(a.R ** 3, 13, device="cuda")
loss = ef.LOSS_MSE_EIKONAL if a.eikonal else ef.LOSS_MSE
for s in range(a.steps):
    grad.zero_()
    if a.split:
        m.forward(qd, od, loss=loss, want_O=False, want_loss=False)
        m.backward(grad=grad)
    else:
        m.forward_backward(qd, od, loss=loss, grad=grad, want_loss=False)
    m.adamw_step(grad)
torch.cuda.synchronize()
print("done", m.stats())
