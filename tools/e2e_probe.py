"""Probe the pipelined host-I/O fit step (host_io 2): per-step wall time in steady state, with and
without the loss read-back, against the device-resident graph step (diagnostics)."""
import sys, time; sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2505_21319_b200 as ef
from workloads import synth
R, J = 32, 1 << 20
tor = synth.Torus()
m = ef.EFunc(R, synth.init_theta(R, 1234))
m.mean_shift_init(torch.as_tensor(synth.surface_points(tor, 16384, 1234)).cuda())
bs = [synth.sample_batch(tor, J, seed=i) for i in range(4)]
hq = [torch.as_tensor(q).pin_memory() for q, _ in bs]
ho = [torch.as_tensor(o).pin_memory() for _, o in bs]
qd = [torch.as_tensor(q).cuda() for q, _ in bs]
od = [torch.as_tensor(o).cuda() for _, o in bs]
lo = torch.zeros(1, device="cuda")
for mode in ("device", "pipelined", "sync_host"):
    for k in range(6):
        if mode == "device": m.fit_step(qd[k % 4], od[k % 4], loss_out=lo)
        elif mode == "pipelined": m.fit_step(hq[k % 4], ho[k % 4], pipelined=True)
        else: m.fit_step(hq[k % 4], ho[k % 4])
    m.sync(); torch.cuda.synchronize()
    t = time.perf_counter(); n = 100
    for k in range(n):
        if mode == "device": m.fit_step(qd[k % 4], od[k % 4], loss_out=lo)
        elif mode == "pipelined": m.fit_step(hq[k % 4], ho[k % 4], pipelined=True)
        else: m.fit_step(hq[k % 4], ho[k % 4])
    m.sync(); torch.cuda.synchronize()
    print(mode, f"{(time.perf_counter() - t) / n * 1e3:.3f} ms/step")
# overlap check: device-pointer steps on the current stream while a side stream copies 16.8 MB
side = torch.cuda.Stream()
dq = torch.empty_like(qd[0]); do_ = torch.empty_like(od[0])
torch.cuda.synchronize()
t = time.perf_counter(); n = 50
for k in range(n):
    with torch.cuda.stream(side):
        dq.copy_(hq[k % 4], non_blocking=True); do_.copy_(ho[k % 4], non_blocking=True)
    m.fit_step(qd[k % 4], od[k % 4], loss_out=lo)
torch.cuda.synchronize()
print("device step + side-stream copy", f"{(time.perf_counter() - t) / n * 1e3:.3f} ms/step")
print("current stream handle", torch.cuda.current_stream().cuda_stream)
# pipelined without the loss read-back (no D2H, no host callback)
import ctypes as C
from paper_2505_21319_b200 import efunc as efm
lc = efm.Loss(ef.LOSS_MSE, 0.1, 0); p = ef.AdamW().c()
for k in range(6):
    m.lib.efunc_fit_step(m.h, hq[k % 4].data_ptr(), ho[k % 4].data_ptr(), J, C.byref(lc), C.byref(p), None, None, 2, 0)
m.sync(); torch.cuda.synchronize()
t = time.perf_counter(); n = 100
for k in range(n):
    m.lib.efunc_fit_step(m.h, hq[k % 4].data_ptr(), ho[k % 4].data_ptr(), J, C.byref(lc), C.byref(p), None, None, 2, 0)
m.sync(); torch.cuda.synchronize()
print("pipelined, no loss read-back", f"{(time.perf_counter() - t) / n * 1e3:.3f} ms/step")
s2 = torch.cuda.Stream()
with torch.cuda.stream(s2):
    for k in range(6):
        m.fit_step(hq[k % 4], ho[k % 4], pipelined=True)
    m.sync(); torch.cuda.synchronize()
    t = time.perf_counter(); n = 100
    for k in range(n):
        m.fit_step(hq[k % 4], ho[k % 4], pipelined=True)
    m.sync(); torch.cuda.synchronize()
print("pipelined on a non-default stream", f"{(time.perf_counter() - t) / n * 1e3:.3f} ms/step")
