"""Warm per-kernel timings of the C2/C3 fit step via the CUDA activity trace (torch.profiler / CUPTI),
plus the idle time between kernels on the stream (launch gaps). Not a bench number: diagnostics.

  python tools/step_kernels.py [--config c2|c3] [--steps 5]
"""
import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2505_21319_b200 as ef  # noqa: E402
from workloads import synth  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="c2")
p.add_argument("--steps", type=int, default=5)
p.add_argument("--split", action="store_true", help="forward + backward instead of forward_backward")
p.add_argument("--graph", action="store_true", help="replay one CUDA graph per batch (as bench.py)")
a = p.parse_args()
J = (1 << 20) if a.config == "c2" else (1 << 22)
loss = ef.LOSS_MSE if a.config == "c2" else ef.LOSS_MSE_EIKONAL
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
    if a.split:
        m.forward(qd[i % 4], od[i % 4], loss=loss, want_O=False, want_loss=False)
        m.backward(grad=grad)
    else:
        m.forward_backward(qd[i % 4], od[i % 4], loss=loss, grad=grad, want_loss=False)
    m.adamw_step(grad, hp)


for i in range(10):
    step(i)
torch.cuda.synchronize()
run = step
if a.graph:
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    graphs = []
    with torch.cuda.stream(cap):
        for i in range(4):
            step(i)
    torch.cuda.synchronize()
    for i in range(4):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            step(i)
        graphs.append(g)
    run = lambda i: graphs[i % 4].replay()  # noqa: E731
    for i in range(8):
        run(i)
    torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(a.steps):
        run(i)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
agg = collections.OrderedDict()
for e in ev:
    agg.setdefault(e.name.split("(")[0], []).append(e.time_range.end - e.time_range.start)
busy = sum(e.time_range.end - e.time_range.start for e in ev)
span = ev[-1].time_range.end - ev[0].time_range.start
print(f"{a.config}: {a.steps} steps, span {span / a.steps:.1f} us/step, kernels+copies busy {busy / a.steps:.1f} us/step, "
      f"gaps {(span - busy) / a.steps:.1f} us/step, {len(ev) / a.steps:.1f} activities/step")
print("| kernel | per step | mean us | us/step | share |")
print("|---|---|---|---|---|")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"| `{k[:60]}` | {len(v) / a.steps:.1f} | {sum(v) / len(v):.1f} | {sum(v) / a.steps:.1f} | {100 * sum(v) / busy:.1f}% |")

# one step's activities in order (start offset, duration, gap before)
t0 = ev[0].time_range.start
per = len(ev) // a.steps
print("\nlast step, in order: start_us dur_us gap_us name")
prev_end = None
for e in ev[-per:]:
    st, en = e.time_range.start, e.time_range.end
    gap = 0 if prev_end is None else st - prev_end
    print(f"{st - ev[-per].time_range.start:9.1f} {en - st:8.1f} {gap:7.1f}  {e.name.split('(')[0][:60]}")
    prev_end = en
