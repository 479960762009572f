"""Dense inference on this build ("256^3 points in about 5 seconds"):
efunc_eval_grad (O and dO/dq, Eq. func-normal) over a regular 256^3 lattice of query points in
[-1,1]^3, in chunks, for a 32^3 x 13 grid fitted for a few hundred steps to the torus.

  python tools/inference.py [--res 256] [--chunk 4194304] [--fit-steps 300]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_21319_b200 as ef  # noqa: E402
from workloads import synth  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--res", type=int, default=256)
    p.add_argument("--chunk", type=int, default=1 << 22)
    p.add_argument("--fit-steps", type=int, default=300)
    p.add_argument("--mesh", type=str, default="256,512", help="lattice sizes for efunc_mesh timing ('' = none)")
    a = p.parse_args()
    tor = synth.Torus()
    m = ef.EFunc(32, synth.init_theta(32, 1))
    m.mean_shift_init(torch.as_tensor(synth.surface_points(tor, 16384, 2)).cuda())
    batches = [synth.sample_batch(tor, 1 << 20, seed=10 + i) for i in range(4)]
    qd = [torch.as_tensor(q).cuda() for q, _ in batches]
    od = [torch.as_tensor(o).cuda() for _, o in batches]
    lo = torch.zeros(1, device="cuda")
    for k in range(a.fit_steps):
        m.fit_step(qd[k % 4], od[k % 4], loss_out=lo)
    torch.cuda.synchronize()
    n = a.res
    lin = torch.linspace(-1.0, 1.0, n, device="cuda")
    zz, yy, xx = torch.meshgrid(lin, lin, lin, indexing="ij")
    pts = torch.stack([xx, yy, zz], dim=-1).reshape(-1, 3).contiguous()
    N = pts.shape[0]
    O = torch.empty(N, device="cuda")
    G = torch.empty(N, 3, device="cuda")

    def run():
        for s in range(0, N, a.chunk):
            e = min(N, s + a.chunk)
            Oc, Gc = m.eval_grad(pts[s:e])
            O[s:e] = Oc
            G[s:e] = Gc
    run()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    run()
    ev1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    gpu_ms = ev0.elapsed_time(ev1)
    sdf = torch.as_tensor(tor.sdf(pts.cpu().numpy().astype(np.float64)), dtype=torch.float32, device="cuda")
    err = float((O - sdf).abs().mean())
    gn = float((G.norm(dim=1) - 1).abs().mean())
    res = {"points": N, "grid": "32^3x13 fitted %d steps" % a.fit_steps, "gpu_ms": gpu_ms, "wall_s": wall,
           "points_per_s": N / (gpu_ms / 1e3), "mean_abs_sdf_err": err, "mean_abs_grad_norm_minus_1": gn,
           "paper": "256^3 in about 5 s (PAPER.md:L853, unknown GPU)"}
    # NEXT-3: efunc_mesh = lattice O + Marching Cubes + vertex normals
    # on a grid whose keys carry the torus SDF and its gradient (a "fitted-like" state; the short fit
    # above is far from converged), so the mesh is the torus and its statistics mean something
    mf = ef.EFunc(32, synth.fitted_like_theta(32, tor, 1))
    meshes = []
    for nres in [int(x) for x in a.mesh.split(",") if x]:
        mf.mesh(nres)  # warm-up (allocations, table upload)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        v, t, nrm, _ = mf.mesh(nres)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        vd = v.double().cpu().numpy()
        err_v = float(np.abs(tor.sdf(vd)).mean())
        # normal vs the analytic torus gradient at the vertices
        gt = tor.grad(vd)
        cosv = float(np.mean(np.sum(gt * nrm.double().cpu().numpy(), axis=1) / np.linalg.norm(gt, axis=1)))
        meshes.append({"N": nres, "lattice_points": nres ** 3, "verts": int(v.shape[0]), "tris": int(t.shape[0]),
                       "wall_s": dt, "mean_abs_sdf_at_verts": err_v, "mean_cos_normal_vs_analytic": cosv,
                       "theta": "fitted_like_theta(32, torus): c = sdf + N(0, 0.01^2), g = grad sdf + N(0, 0.05^2)", "note": "one synchronous efunc_mesh call: lattice O in z-slabs of 2^23 points (value-only "
                               "forward), Marching Cubes count/scan/emit, normals from one eval_grad pass"})
    res["mesh"] = meshes
    res["paper_mesh"] = "O at 512^3 then Marching Cubes (PAPER.md:L680); normals from one forward pass (L962-971)"
    print(json.dumps(res))


if __name__ == "__main__":
    main()
