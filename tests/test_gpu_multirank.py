"""Data-parallel path with libefunc in more than one rank, on the one GPU this build
has: 2 processes share cuda:0 and all-reduce over gloo. Each rank runs the fused fit kernel on its
shard with the loss scaled by 1/J_global; the all-reduced gradient must equal the oracle's
full-batch gradient (the loss is a batch mean; additivity SPEC.md:L225).
Also: `python bench.py --gpus 2` spawns its own ranks when WORLD_SIZE is unset."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_2505_21319_b200 as ef
    from paper_2505_21319_b200 import dist as edist
    from workloads import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    R, J = 8, 2048
    sph = synth.Sphere(0.5)
    th = synth.fitted_like_theta(R, sph, 5)
    q, o = synth.sample_batch(sph, J, seed=edist.rank_seed(9, rank))
    m = ef.EFunc(R, th)
    g, _, L = m.forward_backward(torch.as_tensor(q).cuda(), torch.as_tensor(o).cuda(), loss=ef.LOSS_MSE,
                                 J_global=edist.global_batch(J, world))
    gc = g.cpu()
    lc = L.cpu().to(torch.float64)
    edist.allreduce_grad(gc)
    edist.allreduce_grad(lc)
    if rank == 0:
        out.put((gc.numpy(), float(lc[0])))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_allreduced_gradient_equals_oracle_full_batch():
    import oracle as orc
    from paper_2505_21319_b200 import dist as edist
    from workloads import synth
    ctx = mp.get_context("spawn")
    qq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, qq)) for r in range(2)]
    for p in procs:
        p.start()
    g, L = qq.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    R, J = 8, 2048
    sph = synth.Sphere(0.5)
    th = synth.fitted_like_theta(R, sph, 5).astype(np.float64)
    qs, os_ = zip(*[synth.sample_batch(sph, J, seed=edist.rank_seed(9, k)) for k in range(2)])
    qa, oa = np.concatenate(qs), np.concatenate(os_)
    f = orc.forward(th, R, qa)
    La, ra = orc.mse_loss(f.O, oa)
    ga = orc.backward(th, R, qa, f, ra)
    for ch in range(13):
        e = np.abs(g[:, ch] - ga[:, ch]).max() / np.abs(ga[:, ch]).max()
        assert e <= 1e-4, (ch, e)
    assert abs(L - La) <= 1e-5 * La + 2e-5 * np.abs(f.O - oa).mean() * np.abs(f.O).max()


def test_bench_gpus_2_spawns_ranks_without_torchrun():
    """`python bench.py --gpus 2` (no torchrun, WORLD_SIZE unset) re-launches under
    torch.distributed.run; with EFUNC_BENCH_SHARED_GPU=1 both ranks share this GPU over gloo (a
    code-path check, not a measurement) and rank 0 prints one line with n_gpus = 2."""
    env = dict(os.environ, EFUNC_BENCH_SHARED_GPU="1", EFUNC_BENCH_WATCHDOG="150")
    env.pop("WORLD_SIZE", None)
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        # files, not pipes: a leftover grandchild holding a pipe open must not stall the test
        with open(os.path.join(td, "out"), "w") as fo, open(os.path.join(td, "err"), "w") as fe:
            rc = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "c1",
                                 "--steps", "5", "--warmup", "3"], env=env, stdout=fo, stderr=fe, timeout=300,
                                cwd=ROOT).returncode
        out = open(os.path.join(td, "out")).read()
        err = open(os.path.join(td, "err")).read()
    assert rc == 0, err[-3000:]
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "dp2"
    assert d["config"]["global_batch"] == 2 * 4096
    assert d["value"] > 0 and d["e2e"]["value"] > 0


def test_bench_nccl_allreduce_captured_in_step_graph_single_rank():
    """EFUNC_BENCH_NCCL1=1: bench.py's N > 1 step (the NCCL all-reduce of the gradient captured
    inside each batch's CUDA graph) on a one-rank NCCL group: checks that the collective captures
    and replays with this torch/NCCL, which the multi-GPU scaling run depends on."""
    env = dict(os.environ, EFUNC_BENCH_NCCL1="1", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()),
               EFUNC_BENCH_WATCHDOG="150")
    env.pop("WORLD_SIZE", None)
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        with open(os.path.join(td, "out"), "w") as fo, open(os.path.join(td, "err"), "w") as fe:
            rc = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c1", "--steps", "5",
                                 "--warmup", "3", "--no-cpu-baseline"], env=env, stdout=fo, stderr=fe,
                                timeout=300, cwd=ROOT).returncode
        out = open(os.path.join(td, "out")).read()
        err = open(os.path.join(td, "err")).read()
    assert rc == 0, err[-3000:]
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out
    d = json.loads(lines[0])
    assert d["config"]["launch"] == "cuda-graph per step (NCCL all-reduce inside)", d["config"]
    assert d["config"]["collective"].startswith("NCCL all_reduce")
    assert d["value"] > 0


def test_bench_fused_peer_reduction_single_rank():
    """EFUNC_BENCH_P2P=1 on a one-rank NCCL group: the gradient in torch symmetric memory, the
    library's fold adding it into every rank's copy (efunc_set_grad_peers: here the rank's own copy)
    between two symmetric-memory barriers, all captured in the step graph. The code path of the
    fused fold + peer reduction; its sum over ranks is the gloo-checked algebra above."""
    env = dict(os.environ, EFUNC_BENCH_NCCL1="1", EFUNC_BENCH_P2P="1", MASTER_ADDR="127.0.0.1",
               MASTER_PORT=str(_free_port()), EFUNC_BENCH_WATCHDOG="150")
    env.pop("WORLD_SIZE", None)
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        with open(os.path.join(td, "out"), "w") as fo, open(os.path.join(td, "err"), "w") as fe:
            rc = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c1", "--steps", "5",
                                 "--warmup", "3", "--no-cpu-baseline"], env=env, stdout=fo, stderr=fe,
                                timeout=300, cwd=ROOT).returncode
        out = open(os.path.join(td, "out")).read()
        err = open(os.path.join(td, "err")).read()
    assert rc == 0, err[-3000:]
    d = json.loads([ln for ln in out.splitlines() if ln.startswith("{")][0])
    assert d["config"]["collective"].startswith("fused fold + "), d["config"]
    assert d["value"] > 0


def test_fused_peer_fold_equals_local_fold():
    """efunc_set_grad_peers with this device's own buffer as the only peer: the fused fold adds the
    same gradient the local fold writes (up to the order of the float atomics in the fit kernel)."""
    import paper_2505_21319_b200 as ef
    from workloads import synth
    R, J = 16, 1 << 14
    tor = synth.Torus()
    th = synth.fitted_like_theta(R, tor, 3)
    q, o = synth.sample_batch(tor, J, seed=4)
    qd, od = torch.as_tensor(q).cuda(), torch.as_tensor(o).cuda()
    m = ef.EFunc(R, th)
    g0, _, _ = m.forward_backward(qd, od, loss=ef.LOSS_MSE)
    buf = torch.zeros_like(g0)
    m.set_grad_peers([buf.data_ptr()], 0)
    gdummy = torch.zeros_like(g0)
    m.forward_backward(qd, od, loss=ef.LOSS_MSE, grad=gdummy)
    torch.cuda.synchronize()
    m.set_grad_peers([], 0)
    assert float(gdummy.abs().max()) == 0.0  # the local grad is untouched
    # float reds in a different order: equal up to rounding of the atomic sums
    scale = float(g0.abs().max())
    assert float((buf - g0).abs().max()) <= 1e-5 * scale
