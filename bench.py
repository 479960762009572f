#!/usr/bin/env python
"""bench.py — efunc fit-step throughput (points/s) on B200, BASELINE.json's metric.

A step = one pass of the whole hot path over one batch: query binning,
forward + MSE epilogue, backward, gradient all-reduce (N > 1), AdamW + key rebuild.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c1] [--impl ours|reference]

N > 1: one rank per GPU over NCCL. Under torchrun (WORLD_SIZE set) the ranks come from the
environment; `python bench.py --gpus N` without torchrun re-launches itself under
torch.distributed.run with N local ranks. Every rank processes its own 2^20-point batch per step
(weak scaling) and the 1.7 MB gradient is all-reduced inside the step's CUDA graph (NCCL
collectives are graph-capturable). Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fit-step points/sec (fwd+bwd+AdamW) at 32^3×13 grid, 1/2/4/8 B200; % roofline"
CONFIGS = {
    # name: (R, points per GPU per step, shape, loss, workload label)
    "c2": (32, 1 << 20, "torus", "mse", "C2: 32^3x13 grid, torus SDF, 2^20 points/step/GPU, MSE"),
    "c3": (32, 1 << 22, "torus", "mse_eikonal", "C3: 32^3x13 grid, torus SDF, 2^22 points/step/GPU, MSE+0.1 Eikonal"),
    "c1": (8, 4096, "sphere", "mse", "C1: 8^3x13 grid, sphere SDF, 4096 points/step"),
    "c4a": (64, 1 << 24, "torus", "mse",
            "C4a: 64^3x13 grid, torus SDF, 2^24 points/step in total sharded over the GPUs, MSE"),
    "c4b": (128, 1 << 24, "torus", "mse",
            "C4b: 128^3x13 grid, torus SDF, 2^24 points/step in total sharded over the GPUs, MSE"),
    "c5": (32, 1 << 20, "c5", "mse",
           "C5: 8 independent 32^3x13 shapes per GPU (seeded rotated tori/spheres/boxes/CSG), 2^20 points/step per shape, MSE"),
}
C5_SHAPES_PER_GPU = 8
# strong scaling: these configs fix the global batch; each of N ranks takes 1/N of it
STRONG = {"c4a": 1 << 24, "c4b": 1 << 24}
SEED = 1234
POOL = 8                       # distinct batches cycled through; 8 x 16.8 MB > 126 MB L2 at C2
SM_COUNT, FP32_LANES, SM_MAX_MHZ = 148, 128, 1965.0
# algorithmic FP32 lane-ops per kept pair (FFMA = 1 op): SURVEY App. C, DESIGN.md §5 (direct form;
# the kernels' own instruction counts are not the numerator)
OPS_FWD = 12            # d(3), |d|^2(3), exponent(1), f(3), Z(1), M(1)
OPS_FWD_G = 23          # + S_g(3), w beta(1), S_u(3), w beta f(1), S_uf(3) (Eq. func-normal)
OPS_BWD_GRID, OPS_BWD_OFF = 18, 21
OPS_BWD_EIK_GRID, OPS_BWD_EIK_OFF = 33, 42
PEAKS_FILE = os.path.join(ROOT, "profiles", "fp32_peaks.json")
# Table 4 of the paper (GPU and precision unstated): J = 16384, I = 32^3
PAPER_T4 = {"J": 16384, "I": "32^3", "fwd_ms": 3.064, "bwd_ms": 10.561, "memory_MB": 1.68,
            "fwd_bwd_points_per_s": 16384 / (3.064e-3 + 10.561e-3), "gpu": "unstated",
            "source": "PAPER.md:L842-848 (Table 4); dense global sums, no AdamW"}


def fp32_peak():
    """(peak T lane-op/s, basis): the measured FFMA rate (profiles/fp32_peaks.json, written from
    tools/ubench_fp32.cu on a B200), else the nominal unit-count figure (fallback)."""
    try:
        d = json.load(open(PEAKS_FILE))
        return float(d[d["peak_used"]]), f"measured ({d['peak_used']}, profiles/fp32_peaks.json: {d['source']})"
    except Exception:
        return SM_COUNT * FP32_LANES * SM_MAX_MHZ * 1e6 / 1e12, "fallback: nominal 148 SM x 128 FP32 lanes x 1965 MHz"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=None,
                   help="GPUs (ranks); without torchrun, N > 1 re-launches under torch.distributed.run")
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--eager", action="store_true", help="N=1: plain launches instead of a CUDA graph per step")
    p.add_argument("--split", action="store_true", help="efunc_forward + efunc_backward instead of the fused call")
    p.add_argument("--deterministic", action="store_true",
                   help="deterministic mode (stable sorts, 64-bit fixed-point gradient sums in the fused kernel)")
    return p.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.samples = []
        self.proc = None
        self.active = False

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits",
                 "-i", self.gpu_id, "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        threading.Thread(target=self._reader, daemon=True).start()

    def _reader(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.samples.append((self.active, parts))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sel = [s for a, s in self.samples if a] or [s for _, s in self.samples]
        if not sel:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no nvidia-smi samples"], "samples": 0}
        sm = [float(s[0]) for s in sel if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in sel if s[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for s in sel for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sel)}


# ----------------------------------------------------------------------------- oracle legs
# queries per oracle sample (float64 global sums, all host cores): the paper's Table-4 batch
# (J = 16384) at 32^3 MSE; scaled down where a query costs more
CPU_SAMPLE = {"c1": 4096, "c2": 16384, "c3": 8192, "c4a": 1024, "c4b": 128, "c5": 16384}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class OracleStep:
    """One oracle fit step (float64 global sum over all 2R^3 keys: forward, MSE (+ Eikonal) loss,
    backward, AdamW) on n queries of the workload, sharded over the host cores by
    oracle.parallel (the oracle as it stands; shard gradients summed in fixed order). The oracle's
    cost does not depend on theta's values, so the paper init is used with Delta = 0."""

    def __init__(self, R, shape, loss_kind):
        import oracle as orc
        from oracle import parallel as par
        from workloads import synth
        self.orc, self.par, self.synth = orc, par, synth
        self.R, self.shape, self.lam = R, shape, (0.1 if loss_kind == "mse_eikonal" else 0.0)
        self.th = synth.init_theta(R, SEED).astype(np.float64)
        self.cores = par.host_cores()

    def run(self, n, seed):
        q, o = self.synth.sample_batch(self.shape, n, seed=seed)
        t0 = time.perf_counter()
        _, L, g = self.par.fit_eval(self.th, self.R, q, o, lam_e=self.lam, procs=self.cores)
        z = np.zeros_like(g)
        self.orc.adamw_step(self.th, g, z, z, 1, self.orc.AdamW())
        return time.perf_counter() - t0


def cpu_baseline(config, R, shape, loss_kind):
    st = OracleStep(R, shape, loss_kind)
    n = CPU_SAMPLE[config]
    t = st.run(n, seed=SEED + 777)
    return {"value": n / t, "unit": "points/s", "cores": st.cores, "kind": "oracle", "cpu": cpu_model(),
            "sample": f"{n} queries of the {R}^3 workload, one full fit step (global-support float64 forward + "
                      f"loss + backward + AdamW), oracle.parallel over {st.cores} processes; {t:.1f} s"}


def run_reference(args, rank, world):
    """The reference arm (task tier framing): the CPU oracle as it stands, timed on the host cores,
    on our arm's config/metric; each step a bounded sample of the workload."""
    R, J, shape_name, loss_kind, label = CONFIGS[args.config]
    if rank != 0:
        return
    from workloads import synth
    shape = synth.c5_shapes(1, SEED)[0] if shape_name == "c5" else synth.make_shape(shape_name)
    st = OracleStep(R, shape, loss_kind)
    # size the per-step sample so that warmup + steps take about two minutes in total
    n0 = 4 * st.cores
    rate = n0 / st.run(n0, seed=SEED - 1)
    n = int(max(st.cores, min(CPU_SAMPLE[args.config], 120.0 * rate / max(1, args.steps + args.warmup))))
    for w in range(args.warmup):
        st.run(n, seed=SEED + w)
    t = 0.0
    for k in range(args.steps):
        t += st.run(n, seed=SEED + 100 + k)
    v = n * args.steps / t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": label, "R": R, "sample_points_per_step": n},
            "cpu_baseline": {"value": v, "unit": "points/s", "cores": st.cores, "kind": "oracle", "cpu": cpu_model(),
                             "sample": f"{n} queries per step of the {R}^3 workload (float64 global sum, "
                                       f"oracle.parallel over {st.cores} processes)"},
            "e2e": {"value": v, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our path
def run_ours(args, rank, world, local_rank, nccl):
    import torch
    import torch.distributed as dist

    import paper_2505_21319_b200 as ef
    from paper_2505_21319_b200 import dist as edist
    from workloads import synth

    R, J, shape_name, loss_kind, label = CONFIGS[args.config]
    if args.config in STRONG:
        J = STRONG[args.config] // world
    dev = local_rank
    torch.cuda.set_device(dev)
    loss = ef.LOSS_MSE if loss_kind == "mse" else ef.LOSS_MSE_EIKONAL
    # C5: S independent shapes per GPU in one batched handle (replicas: no collective);
    # otherwise one shape, data parallel over the ranks
    S = C5_SHAPES_PER_GPU if shape_name == "c5" else 1
    if S > 1:
        shapes = synth.c5_shapes(S * world, SEED)[rank * S:(rank + 1) * S]
        J_global = J  # every shape's loss is its own batch mean
    else:
        shapes = [synth.make_shape(shape_name)]
        J_global = edist.global_batch(J, world)
    shape = shapes[0]
    # EFUNC_BENCH_NCCL1=1 at world 1: the N > 1 step (NCCL all-reduce captured in the step graph)
    # on one rank, a code-path check of the collective's capture (not a multi-GPU measurement)
    reduce_grad = (world > 1 or nccl) and S == 1

    # input pool (> L2); each rank draws its own points
    pool = max(2, min(POOL, int(np.ceil(160e6 / (16 * J * S)))))

    def draw(i):
        bs = [synth.sample_batch(sh, J, seed=edist.rank_seed(SEED + 97 * k, rank, i)) for k, sh in enumerate(shapes)]
        if S == 1:
            return bs[0]
        return np.stack([b[0] for b in bs]), np.stack([b[1] for b in bs])
    host = [draw(i) for i in range(pool)]
    qd = [torch.as_tensor(q).cuda(dev) for q, _ in host]
    od = [torch.as_tensor(o).cuda(dev) for _, o in host]
    surf = np.stack([synth.surface_points(sh, 16384, SEED) for sh in shapes])
    surf_d = torch.as_tensor(surf if S > 1 else surf[0]).cuda(dev)
    torch.cuda.synchronize()

    # model: paper init (s = 7, c ~ N(0, 0.1^2), g = 0) + mean-shift offsets on the GPU. The device
    # memory the library holds (parameters, optimizer state, key records, brick lists, work queues)
    # is the drop in free memory across creation and the first step (workspaces size on first use).
    free0 = torch.cuda.mem_get_info(dev)[0]
    th0 = np.stack([synth.init_theta(R, SEED + k) for k in range(S)]) if S > 1 else synth.init_theta(R, SEED)
    m = ef.EFunc(R, th0, device=dev, n_shapes=S, deterministic=args.deterministic)
    m.mean_shift_init(surf_d)
    hp = ef.AdamW()
    grad = m._grad_zeros()
    # EFUNC_BENCH_P2P=1 (with an NCCL group): the gradient lives in torch symmetric memory and the
    # library's fold adds it into every rank's copy (NVLS multimem.red through the multicast
    # address, else red.v4 over the NVLink peer mappings; efunc_set_grad_peers) between two
    # symmetric-memory barriers, instead of the NCCL all-reduce after the fold
    p2p = None
    if nccl and S == 1 and os.environ.get("EFUNC_BENCH_P2P") == "1":
        import torch.distributed._symmetric_memory as symm_mem
        gsym = symm_mem.empty(grad.numel(), device=f"cuda:{dev}", dtype=torch.float32)
        p2p = symm_mem.rendezvous(gsym, dist.group.WORLD.group_name)
        m.set_grad_peers(p2p.buffer_ptrs, p2p.multicast_ptr)
        grad = gsym.view(grad.shape)

    def reduce_pre():  # every rank's copy is zero before any rank adds into it
        if p2p is not None:
            p2p.barrier(channel=0)

    def reduce_post():  # the sum is complete in this rank's copy
        if p2p is not None:
            p2p.barrier(channel=1)
        elif reduce_grad:
            edist.allreduce_grad(grad)

    # fused path (default): efunc_forward_backward runs the fused fit kernel k_fit for the MSE loss;
    # --split: efunc_forward + efunc_backward (k_item_lists, k_forward_keys, k_backward)
    def step_calls(i):
        grad.zero_()
        reduce_pre()
        if args.split:
            m.forward(qd[i], od[i], loss=loss, J_global=J_global, want_O=False, want_loss=False)
            m.backward(grad=grad)
        else:
            m.forward_backward(qd[i], od[i], loss=loss, J_global=J_global, grad=grad, want_loss=False)
        reduce_post()
        m.adamw_step(grad, hp)

    # The step is replayed from a CUDA graph per input batch (the same ABI calls captured once; the
    # AdamW step counter is device-side; with N > 1 the NCCL all-reduce is captured inside the
    # graph). The library records CUDA events around the dominant kernel (k_fit, or k_backward on
    # the split path) of every step: slot = batch index. gloo (shared-GPU code-path runs) cannot be
    # captured: plain launches there.
    use_graph = (world == 1 or nccl) and not args.eager
    graphs, launches_per_step = [], None
    m.set_timing(pool)
    cap = torch.cuda.Stream(device=dev)
    cap.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(cap):
        for i in range(pool):  # sizes every workspace (and warms NCCL) before capture
            step_calls(i)
    torch.cuda.synchronize()
    lib_bytes = free0 - torch.cuda.mem_get_info(dev)[0]
    graph_note = None
    if use_graph:
        l0 = m.stats()["launches"]
        try:
            for i in range(pool):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cap):
                    step_calls(i)
                graphs.append(g)
            launches_per_step = (m.stats()["launches"] - l0) / pool
        except Exception as e:  # a collective that cannot be captured: plain launches, said in config
            if world == 1:
                raise
            torch.cuda.synchronize()
            graphs, use_graph = [], False
            graph_note = f"graph capture failed ({type(e).__name__}); eager launches"

    def step(i):
        if use_graph:
            graphs[i].replay()
        else:
            step_calls(i)

    # kept-pair census (algorithmic work per point), outside the timed region
    m.set_counting(True)
    m.forward(qd[0], od[0], loss=loss, J_global=J_global, want_O=False, want_loss=False)
    st = m.stats()
    m.set_counting(False)
    kept = st["kept_pairs"]; kept_off = st["kept_pairs_offset"]; cand = st["candidate_pairs"]
    n_pts = J * S  # points per step per GPU

    for w in range(args.warmup):
        step(w % pool)
    torch.cuda.synchronize()

    uuid = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
    clk = ClockSampler(uuid)
    clk.start()
    time.sleep(0.3)
    # soak so the sampler sees the loaded clock, then the timed region. The soak length is a step
    # count every rank agrees on (a step holds an all-reduce when N > 1: ranks must issue the same
    # number of collectives)
    torch.cuda.synchronize()
    ts = time.perf_counter()
    step(0)
    step(0)
    torch.cuda.synchronize()
    n_soak = int(np.ceil(0.5 / max((time.perf_counter() - ts) / 2, 1e-5)))
    if world > 1:
        tn = torch.tensor([n_soak], dtype=torch.int64, device=f"cuda:{dev}")
        dist.all_reduce(tn, op=dist.ReduceOp.MIN)
        n_soak = int(tn[0])
    for _ in range(min(n_soak, 5000)):
        step(0)
    torch.cuda.synchronize()
    launches0 = m.stats()["launches"]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk.active = True
    t0.record()
    for k in range(args.steps):
        step((args.warmup + k) % pool)
    t1.record()
    torch.cuda.synchronize()
    clk.active = False
    if world > 1:
        dist.barrier()
    launches = m.stats()["launches"] - launches0
    sec = t0.elapsed_time(t1) / 1e3
    if use_graph:
        launches = launches_per_step * args.steps
    # the dominant kernel's CUDA-event time in the last `pool` steps of the timed region
    bwd_ms = float(np.nanmean(m.kernel_ms(pool)))
    if world > 1:
        tt = torch.tensor([sec, bwd_ms], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        sec, bwd_ms = float(tt[0]), float(tt[1])
    time.sleep(0.1)
    clk.stop()
    clocks = clk.summary()
    value = (J_global if S == 1 else n_pts * world) * args.steps / sec

    if p2p is not None and world == 1:
        m.set_grad_peers([], 0)  # the single-rank e2e path (efunc_fit_step) folds into its own workspace
    # e2e: same steps through the public API with pinned host inputs, H2D + loss D2H inside
    e2e = None
    if not args.no_e2e:
        hq = [torch.as_tensor(q).pin_memory() for q, _ in host]
        ho = [torch.as_tensor(o).pin_memory() for _, o in host]
        if world == 1:
            # efunc_fit_step with pipelined host I/O: every step copies its pinned host batch in
            # (on the library's copy stream, overlapping the previous step's compute) and reads its
            # loss back; the clock stops after efunc_sync, i.e. after the last loss arrived
            for w in range(3):
                m.fit_step(hq[w % pool], ho[w % pool], hp, loss=loss, pipelined=True)
            m.sync()
            torch.cuda.synchronize()
            e0 = time.perf_counter()
            for k in range(args.steps):
                m.fit_step(hq[k % pool], ho[k % pool], hp, loss=loss, pipelined=True)
            m.sync()
            esec = time.perf_counter() - e0
        else:
            # every step: H2D of its pinned batch, the fused step, the all-reduce, AdamW, and a
            # non-blocking D2H of its loss into a pinned slot (read on the host after the loop, no
            # per-step host sync)
            qbuf = torch.empty_like(qd[0]); obuf = torch.empty_like(od[0])
            lpin = torch.zeros(args.steps + 3, S).pin_memory()

            def estep(i, slot):
                qbuf.copy_(hq[i], non_blocking=True)
                obuf.copy_(ho[i], non_blocking=True)
                grad.zero_()
                reduce_pre()
                _, _, L = m.forward_backward(qbuf, obuf, loss=loss, J_global=J_global, grad=grad)
                reduce_post()
                m.adamw_step(grad, hp)
                lpin[slot].copy_(L.view(-1), non_blocking=True)
            for w in range(3):
                estep(w % pool, args.steps + w)
            torch.cuda.synchronize()
            dist.barrier()
            e0 = time.perf_counter()
            for k in range(args.steps):
                estep(k % pool, k)
            torch.cuda.synchronize()
            esec = time.perf_counter() - e0
            tt = torch.tensor([esec], dtype=torch.float64, device=f"cuda:{dev}")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            esec = float(tt[0])
        e2e = {"value": (J_global if S == 1 else n_pts * world) * args.steps / esec, "unit": "points/s",
               "h2d_bytes_per_step": int(n_pts * 16), "d2h_bytes_per_step": 4 * S}

    # paper context (Table 4, J = 16384 at 32^3): our forward, backward and fused fwd+bwd on the
    # first 16384 points of a batch (eager launches, CUDA events, after warm-up)
    if p2p is not None:
        m.set_grad_peers([], 0)  # the Table-4 context below runs on rank 0 alone: local folds only
    t4 = None
    if R == 32 and S == 1 and rank == 0:
        nq = PAPER_T4["J"]
        q4, o4 = qd[0][:nq].contiguous(), od[0][:nq].contiguous()
        g4 = m._grad_zeros()

        def tms(fn, reps=20):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                fn()
            b.record()
            torch.cuda.synchronize()
            return a.elapsed_time(b) / reps
        fwd_ms = tms(lambda: m.forward(q4, o4, loss=loss, want_O=False, want_loss=False))

        def fb():
            m.forward(q4, o4, loss=loss, want_O=False, want_loss=False)
            m.backward(grad=g4)
        fb_ms = tms(fb)
        fused_ms = tms(lambda: m.forward_backward(q4, o4, loss=loss, grad=g4, want_loss=False))
        # the paper's own setting: dense global sums (cutoff_T = inf), same theta and batch
        md = ef.EFunc(R, m.get_params(), device=dev, cutoff_T=float("inf"))
        gd = md._grad_zeros()
        dense_ms = tms(lambda: md.forward_backward(q4, o4, loss=loss, grad=gd, want_loss=False), reps=10)
        dense_ops = nq * R ** 3 * ((OPS_FWD + OPS_BWD_GRID) + (OPS_FWD + OPS_BWD_OFF))
        del md
        t4 = {"paper": PAPER_T4, "ours_fwd_ms": fwd_ms, "ours_bwd_ms": fb_ms - fwd_ms,
              "ours_fused_fwd_bwd_ms": fused_ms, "ours_fused_points_per_s": nq / (fused_ms * 1e-3),
              "ours_dense_fused_fwd_bwd_ms": dense_ms,
              "ours_dense_frac_of_fp32_peak": dense_ops / (dense_ms * 1e-3) / (fp32_peak()[0] * 1e12),
              "note": "ours: certified cutoff T = 20 (reading R-1), this batch's loss, eager launches incl. "
                      "binning; ours_dense: every pair (cutoff_T = inf, k_dense_* kernels), frac on "
                      "direct-form lane-ops of all pairs; the paper: dense global sums on an unstated GPU"}

    if rank != 0:
        return
    # roofline of the dominant kernel: algorithmic lane-ops per launch / its time. k_fit (fused,
    # MSE) does the forward and the backward of every kept pair; k_backward only the backward.
    fused = not args.split
    kname = ("k_fit" if loss_kind == "mse" else "k_fit_eik") if fused else "k_backward"
    if loss_kind == "mse":
        ops = OPS_BWD_GRID * (kept - kept_off) + OPS_BWD_OFF * kept_off
    else:
        ops = OPS_BWD_EIK_GRID * (kept - kept_off) + OPS_BWD_EIK_OFF * kept_off
    if fused:
        ops += (OPS_FWD if loss_kind == "mse" else OPS_FWD_G) * kept
    peak, peak_basis = fp32_peak()
    step_ms = 1e3 * sec / args.steps
    if S > 1:
        # the shapes run concurrently on forked streams: their kernel events overlap, so the
        # per-kernel sum overstates the time; use the whole step (a lower bound on the rate)
        bwd_ms = min(bwd_ms, step_ms)
    achieved = ops / (bwd_ms * 1e-3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(f"{args.config}:{kname}")
        except Exception:
            traffic = None
    nominal = SM_COUNT * FP32_LANES * SM_MAX_MHZ * 1e6 / 1e12
    roof = {"bound": "alu", "kernel": kname, "achieved": achieved, "peak": peak,
            "unit": "T fp32 lane-op/s", "frac": achieved / peak, "traffic": traffic,
            "ops_per_launch": ops, "launch_ms": bwd_ms,
            "launch_ms_source": (f"CUDA events the library records around {kname} on the launch stream "
                                 "(efunc_set_timing; external event nodes inside each batch's step graph), "
                                 "mean over the final steps of the timed region") if S == 1 else
                                ("the whole step's time: the S shapes' kernels run concurrently on forked "
                                 "streams, so per-kernel events overlap (lower bound on the kernel rate)"),
            "share_of_step": bwd_ms * 1e-3 / (sec / args.steps),
            "peak_basis": peak_basis, "frac_of_nominal": achieved / nominal,
            "frac_of_step": ops / (sec / args.steps) / 1e12 / peak,
            "ops_basis": "direct-form lane-ops per kept pair (SURVEY App. C): fwd 12 (O) / 23 (O+G), "
                         "bwd 18/21 (MSE grid/offset), 33/42 (MSE+Eikonal)",
            "kept_pairs_per_point": kept / n_pts, "candidate_pairs_per_point": cand / n_pts}
    if clocks.get("sm_mhz"):
        roof["frac_at_observed_clock"] = achieved / (peak * clocks["sm_mhz"] / SM_MAX_MHZ)
    line = {"metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sec / args.steps, "higher_is_better": True,
            "scaling": "strong" if args.config in STRONG else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": label, "R": R, "points_per_step_per_gpu": n_pts,
                       "global_batch": J_global if S == 1 else n_pts * world, "shapes_per_gpu": S,
                       "cutoff_T": 20.0, "parallelism": f"dp{world}" if S == 1 else f"replicas{world}",
                       "launch": ("cuda-graph per step" + ((" (fused fold + peer reduction and its barriers inside)"
                                                             if p2p is not None else " (NCCL all-reduce inside)")
                                                            if reduce_grad else ""))
                                 if use_graph else (graph_note or "eager"),
                       "collective": (("fused fold + " + ("NVLS multimem.red" if p2p.multicast_ptr else
                                                            f"red.v4 into {len(p2p.buffer_ptrs)} peer copies")
                                       + " of the R^3 x 13 gradient (torch symmetric memory, 2 barriers)")
                                      if p2p is not None else
                                      "NCCL all_reduce (sum, fp32) of the R^3 x 13 gradient" if nccl else
                                      "gloo all_reduce (shared-GPU code-path run, not a measurement)")
                                     if reduce_grad else None,
                       "deterministic": bool(args.deterministic),
                       "path": "split forward/backward" if args.split else
                               f"efunc_forward_backward (fused {'k_fit' if loss_kind == 'mse' else 'k_fit_eik'})",
                       "l2": f"inputs larger than L2: pool of {pool} batches x {n_pts * 16 / 1e6:.1f} MB cycled"},
            "roofline": roof, "clocks": clocks, "gpu_launches": int(launches), "e2e": e2e,
            "gpu_memory": {"library_bytes": int(lib_bytes),
                           "params_and_adamw_bytes": int(3 * S * R ** 3 * 13 * 4),
                           "note": "library_bytes: drop in free device memory across efunc_create + mean shift + "
                                   "the first fit steps (parameters, AdamW moments, gradient accumulators, key "
                                   "records, brick lists, query sort and work-item buffers sized for this J)"}}
    if t4 is not None:
        line["paper_table4"] = t4
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, R, shape, loss_kind)
    print(json.dumps(line), flush=True)


def relaunch(n):
    """`python bench.py --gpus N` without torchrun: run this script under torch.distributed.run with N
    local ranks (127.0.0.1 rendezvous) and return its exit code."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if os.environ.get("EFUNC_BENCH_WATCHDOG"):  # debugging aid: every rank dumps its stacks and exits
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["EFUNC_BENCH_WATCHDOG"]), exit=True)
    if "WORLD_SIZE" not in os.environ and (args.gpus or 1) > 1:
        sys.exit(relaunch(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus is not None and args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    args.gpus = world
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    # EFUNC_BENCH_SHARED_GPU=1 (code-path check only, not a measurement): every rank on the GPUs
    # that exist (ranks share them) and gloo for the collectives (NCCL refuses a shared GPU)
    shared = os.environ.get("EFUNC_BENCH_SHARED_GPU") == "1"
    dev = local_rank
    nccl = False
    if world == 1 and os.environ.get("EFUNC_BENCH_NCCL1") == "1":
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
        nccl = True
    if world > 1:
        import torch
        import torch.distributed as dist
        if shared:
            dev = local_rank % torch.cuda.device_count()
            torch.cuda.set_device(dev)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
            nccl = True
    try:
        run_ours(args, rank, world, dev, nccl)
    finally:
        if world > 1 or nccl:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
