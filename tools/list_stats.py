"""Print brick-list / candidate statistics for the C2 workload (diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_21319_b200 as ef  # noqa: E402
from workloads import synth  # noqa: E402

R, J = int(sys.argv[1]) if len(sys.argv) > 1 else 32, 1 << 20
tor = synth.Torus()
m = ef.EFunc(R, synth.init_theta(R, 1234))
m.mean_shift_init(torch.as_tensor(synth.surface_points(tor, 16384, 1234)).cuda())
q, o = synth.sample_batch(tor, J, seed=99)
qd, od = torch.as_tensor(q).cuda(), torch.as_tensor(o).cuda()
m.set_counting(True)
m.forward(qd, od, loss=ef.LOSS_MSE)
s = m.stats()
print({k: (v / J if k in ("candidate_pairs", "kept_pairs") else v) for k, v in s.items()})
