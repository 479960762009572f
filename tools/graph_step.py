"""Experiment: the C2 fit step captured in a CUDA graph (one per input batch) vs eager launches.
Timing only (the captured AdamW bias correction is frozen at capture): not a bench number."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_21319_b200 as ef  # noqa: E402
from workloads import synth  # noqa: E402

J = 1 << 20
tor = synth.Torus()
m = ef.EFunc(32, synth.init_theta(32, 1234))
m.mean_shift_init(torch.as_tensor(synth.surface_points(tor, 16384, 1234)).cuda())
hp = ef.AdamW()
batches = [synth.sample_batch(tor, J, seed=99 + i) for i in range(4)]
qd = [torch.as_tensor(q).cuda() for q, _ in batches]
od = [torch.as_tensor(o).cuda() for _, o in batches]
grad = torch.zeros(32 ** 3, 13, device="cuda")


def step(i):
    grad.zero_()
    m.forward(qd[i % 4], od[i % 4], loss=ef.LOSS_MSE, want_O=False, want_loss=False)
    m.backward(grad=grad)
    m.adamw_step(grad, hp)


def timeit(fn, n=50):
    for i in range(5):
        fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n):
        fn(i)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


print("eager ms/step", timeit(step))
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
graphs = []
with torch.cuda.stream(s):
    for i in range(3):
        step(i)
    for i in range(4):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step(i)
        graphs.append(g)
torch.cuda.current_stream().wait_stream(s)
print("graph ms/step", timeit(lambda i: graphs[i % 4].replay()))
