"""k_fit time by query population (diagnostic, not a bench number): C2 grid (32^3, torus, mean-shift
offsets), 2^20 queries with near-surface fraction 0 / 0.5 / 1; per population the warm k_fit time
(library CUDA events), items, candidate pairs and the executed candidate lane-op rate
(28 lane-ops per candidate pair: forward 9 + backward 19).

  python tools/kfit_mix.py [--J 1048576] [--reps 10]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_21319_b200 as ef  # noqa: E402
from workloads import synth  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--J", type=int, default=1 << 20)
p.add_argument("--reps", type=int, default=10)
a = p.parse_args()
tor = synth.Torus()
th = synth.init_theta(32, 1234)
m = ef.EFunc(32, th)
m.mean_shift_init(torch.as_tensor(synth.surface_points(tor, 16384, 1234)).cuda())
m.set_timing(a.reps)
out = []
for frac in (0.0, 0.5, 1.0):
    q, o = synth.sample_batch(tor, a.J, seed=99, near_fraction=frac)
    qd, od = torch.as_tensor(q).cuda(), torch.as_tensor(o).cuda()
    grad = torch.zeros(32 ** 3, 13, device="cuda")
    for _ in range(3):
        m.forward_backward(qd, od, loss=ef.LOSS_MSE, grad=grad, want_loss=False)
    torch.cuda.synchronize()
    m.set_timing(a.reps)
    for _ in range(a.reps):
        m.forward_backward(qd, od, loss=ef.LOSS_MSE, grad=grad, want_loss=False)
    torch.cuda.synchronize()
    ms = sorted(m.kernel_ms(a.reps))[a.reps // 2]
    st = m.stats()
    cp = st["candidate_pairs"]
    out.append({"near_fraction": frac, "k_fit_ms": ms, "items": st["items"], "cand_per_point": cp / a.J,
                "queries_per_item": a.J / st["items"],
                "cand_Tlaneops_per_s": 28 * cp / (ms * 1e-3) / 1e12})
for r in out:
    print(json.dumps(r))
