"""C5 diagnostics: per shape, brick-list overflow and slow-path items of the fused path."""
import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2505_21319_b200 as ef
from workloads import synth
R, J, SEED = 32, 1 << 20, 1234
for k, sh in enumerate(synth.c5_shapes(8, SEED)):
    m = ef.EFunc(R, synth.init_theta(R, SEED + k))
    m.mean_shift_init(torch.as_tensor(synth.surface_points(sh, 16384, SEED)).cuda())
    q, o = synth.sample_batch(sh, J, seed=5)
    g, _, _ = m.forward_backward(torch.as_tensor(q).cuda(), torch.as_tensor(o).cuda())
    st = m.stats()
    m.set_counting(True); m.forward(torch.as_tensor(q).cuda(), torch.as_tensor(o).cuda(), loss=ef.LOSS_MSE)
    st2 = m.stats()
    print(k, sh.name, {x: st[x] for x in ("items", "list_entries", "list_overflow", "overflow_items")},
          "cand/pt", round(st["candidate_pairs"] / J, 1), "kept/pt", round(st2["kept_pairs"] / J, 1))
