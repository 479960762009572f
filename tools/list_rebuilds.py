"""How often the brick lists are rebuilt during C2 fitting (Verlet skin), and the cost per build."""
import sys; sys.path.insert(0, "/root/repo")
import torch
import paper_2505_21319_b200 as ef
from workloads import synth
tor = synth.Torus()
m = ef.EFunc(32, synth.init_theta(32, 1234))
m.mean_shift_init(torch.as_tensor(synth.surface_points(tor, 16384, 1234)).cuda())
bs = [synth.sample_batch(tor, 1 << 20, seed=i) for i in range(4)]
qd = [torch.as_tensor(q).cuda() for q, _ in bs]
od = [torch.as_tensor(o).cuda() for _, o in bs]
lo = torch.zeros(1, device="cuda")
b0 = m.stats()["list_builds"]
for k in range(200):
    m.fit_step(qd[k % 4], od[k % 4], loss_out=lo)
torch.cuda.synchronize()
print("list builds in 200 steps:", m.stats()["list_builds"] - b0)
