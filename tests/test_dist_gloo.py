"""Multi-process (gloo, world_size 2, CPU) check of the data-parallel algebra used by bench.py:
each rank computes its shard's gradient with the loss scaled by 1/J_global, the gradients are
all-reduced through paper_2505_21319_b200.dist, and the result equals the full-batch gradient.
The per-shard gradients come from the CPU oracle (test infrastructure)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import oracle as orc
    from paper_2505_21319_b200 import dist as edist
    from workloads import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    R, J = 3, 40
    sph = synth.Sphere(0.5)
    th = synth.fitted_like_theta(R, sph, 5).astype(np.float64)
    q, o = synth.sample_batch(sph, J, seed=edist.rank_seed(9, rank))
    Jg = edist.global_batch(J, world)
    f = orc.forward(th, R, q)
    L, r = orc.mse_loss(f.O, o, J_global=Jg)
    g = torch.tensor(orc.backward(th, R, q, f, r))
    lt = torch.tensor([L], dtype=torch.float64)
    edist.allreduce_grad(g)
    edist.allreduce_grad(lt)
    if rank == 0:
        qs, os_ = zip(*[synth.sample_batch(sph, J, seed=edist.rank_seed(9, k)) for k in range(world)])
        qa, oa = np.concatenate(qs), np.concatenate(os_)
        fa = orc.forward(th, R, qa)
        La, ra = orc.mse_loss(fa.O, oa)
        ga = orc.backward(th, R, qa, fa, ra)
        out.put((float(np.abs(g.numpy() - ga).max() / np.abs(ga).max()), abs(float(lt[0]) - La) / La))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_gradient_allreduce_equals_full_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    eg, el = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert eg < 1e-12 and el < 1e-12


def test_rank_seeds_distinct_and_global_batch():
    from paper_2505_21319_b200 import dist as edist
    seeds = {edist.rank_seed(1234, r, s) for r in range(8) for s in range(100)}
    assert len(seeds) == 800
    assert edist.global_batch(1 << 20, 8) == 1 << 23
    rank, world, local = edist.world()
    assert world >= 1 and 0 <= rank < world
