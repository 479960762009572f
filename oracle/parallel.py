"""Query-sharded driver of the float64 oracle — TEST INFRASTRUCTURE ONLY (same rules as
efunc_oracle.py: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may use it).

It runs the oracle functions AS THEY STAND on contiguous query shards in worker processes and
merges the results in shard order. Nothing of the method is re-implemented here: the split is
exact because every per-query quantity (Alg. 1) depends on that query alone
and the loss is a batch mean whose parameter gradient is a sum over queries (Eq. loss,
PAPER.md:L486-490; additivity SPEC.md:L225), so shard gradients add up to the full-batch one
(up to float64 summation order).
"""
from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

from . import efunc_oracle as orc


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _shard_fit(args):
    theta, R, q, o, lam_e, J_global, cutoff_T, want_grad = args
    f = orc.forward(theta, R, q, cutoff_T=cutoff_T)
    out = {"O": f.O, "G": f.G, "lam": f.lam, "m": f.m, "ubar": f.ubar, "kept": f.kept}
    if o is None:
        return out
    L, r = orc.mse_loss(f.O, o, J_global)
    h = None
    if lam_e:
        LE, h = orc.eikonal_loss(f.G, lam_e, J_global)
        L += LE
    out["loss"] = L
    if want_grad:
        out["grad"] = orc.backward(theta, R, q, f, r, h)
    return out


def fit_eval(theta, R: int, q, o=None, lam_e: float = 0.0, J_global: int | None = None,
             cutoff_T: float | None = None, want_grad: bool = True, procs: int | None = None):
    """Forward (+ MSE / Eikonal loss and the backward when o is given) of the oracle over q, sharded
    over `procs` worker processes. Returns (Forward, loss or None, grad or None)."""
    q = np.asarray(q, np.float64).reshape(-1, 3)
    J = q.shape[0]
    Jg = J if J_global is None else J_global
    procs = max(1, min(procs or host_cores(), J))
    bounds = np.linspace(0, J, procs + 1).astype(int)
    jobs = [(theta, R, q[a:b], None if o is None else np.asarray(o, np.float64)[a:b], lam_e, Jg, cutoff_T, want_grad)
            for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
    if len(jobs) == 1:
        parts = [_shard_fit(jobs[0])]
    else:
        with mp.get_context("fork").Pool(len(jobs)) as pool:
            parts = pool.map(_shard_fit, jobs)
    cat = {k: np.concatenate([p[k] for p in parts]) for k in ("O", "G", "lam", "m", "ubar", "kept")}
    fwd = orc.Forward(cat["O"], cat["G"], cat["lam"], cat["m"], cat["ubar"], cat["kept"])
    loss = grad = None
    if o is not None:
        loss = float(sum(p["loss"] for p in parts))
        if want_grad:
            grad = parts[0]["grad"].copy()
            for p in parts[1:]:
                grad += p["grad"]
    return fwd, loss, grad
