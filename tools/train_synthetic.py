"""NEXT-4: a synthetic training run through the library's training iteration (paper_2605_13794_b200.
train.Trainer: bgs_batch_step with supervised views, selective Adam, density control, the scoring
passes and the L_max(t) schedule of P:342 / P:204, scaled to a short run).

Ground truth: an aerial-city scene (synthetic.gen_city) rendered by the library's forward at V
cameras.  Initialisation (SfM-like): a seeded 40% subset of the ground-truth Gaussians with
perturbed means, grey colour, opacity 0.3 and 1.3x scales.  The loss must fall.

    python tools/train_synthetic.py [--iters 3000] [--n 300000] [--out profiles/r02_train_curve.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_13794_b200.bgs as B  # noqa: E402
import synthetic as S  # noqa: E402
from paper_2605_13794_b200.train import Schedule, Trainer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=3000)
    ap.add_argument("--n", type=int, default=300_000)
    ap.add_argument("--W", type=int, default=576)
    ap.add_argument("--H", type=int, default=432)
    ap.add_argument("--views", type=int, default=32)
    ap.add_argument("--scale", type=float, default=0.075, help="schedule scale (P:342 steps x scale)")
    ap.add_argument("--tau", type=float, default=2e-4)
    ap.add_argument("--d0-factor", type=float, default=64.0,
                    help="LOD reference distance d0 = factor x median camera distance (R19).  The generator's "
                         "levels are not redundant (each Gaussian covers its own surface), so at factor 1 the "
                         "Eq.4 distance term drops visible surface; at 64 only L_max(t) binds")
    ap.add_argument("--unlock", type=float, default=0.045,
                    help="L_max unlock start as a fraction of the paper's 2,000 x (scale/0.075) ... "
                         "0.045 x 2000 = 90: every level unlocked (90 x 2^4 = 1440) before the window ends")
    ap.add_argument("--out", default="gpurun_out/train_curve.json")
    a = ap.parse_args()
    dev = "cuda:0"
    torch.cuda.set_device(0)
    gt = S.gen_city("rubble", n=a.n, W=a.W, H=a.H, V=a.views, seed=21)
    ctx = B.Context(0, 1, 0)
    g_gt = B.GaussianPlanes.from_scene(gt, dev)
    targets = []
    H, W = a.H, a.W
    rad = torch.zeros(gt.n, dtype=torch.int32, device=dev)
    for cam in gt.cameras:
        rgb = torch.zeros(3, H, W, device=dev)
        T = torch.zeros(H, W, device=dev)
        nc = torch.zeros(H, W, dtype=torch.int32, device=dev)
        B.bgs_view_step(ctx, g_gt, B.camera(cam), None, None, 0, rad, rgb, T, nc, None, None, None)
        targets.append(rgb)
    torch.cuda.synchronize()
    # SfM-like initialisation
    rng = np.random.Generator(np.random.PCG64(5))
    idx = np.sort(rng.choice(gt.n, size=int(0.4 * gt.n), replace=False))
    means = gt.means[idx] + rng.normal(0, 1, (idx.size, 3)) * 0.5 * gt.scales[idx].max(1, keepdims=True)
    scales = gt.scales[idx] * 1.3
    quats = gt.quats[idx]
    opac = np.full(idx.size, 0.3, np.float32)
    sh = np.zeros((idx.size, 48), np.float32)
    sh[:, :3] = rng.normal(0, 0.1, (idx.size, 3))
    lod = gt.lod[idx]
    ml = np.concatenate([means, np.log(opac / (1 - opac))[:, None]], 1).astype(np.float32)
    ls = np.zeros((idx.size, 4), np.float32)
    ls[:, :3] = np.log(scales)
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(dev)
    tp = B.TrainParams(t(ml), t(quats), t(ls), t(sh))
    lod_t = torch.from_numpy(np.ascontiguousarray(lod, np.uint8)).to(dev)
    sched = Schedule(k_levels=gt.k_levels).scaled(a.scale)
    sched.unlock_first = max(1, int(round(2000 * a.unlock)))
    dp = B.densify_params(a.tau, 0.01 * 1000.0, 0.005, 1.6, 11, gt.k_levels)
    tr = Trainer(ctx, tp, lod_t, gt.cameras, targets, gt.d0 * a.d0_factor, sched, batch=4, lam=0.2, beta=10.0, seed=7, densify=dp,
                 device=dev)
    logs = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    plain_ms, plain_n = 0.0, 0
    for it in range(1, a.iters + 1):
        ev0.record(tr.stream)
        lg = tr.step(it)
        ev1.record(tr.stream)
        if not lg.event:
            torch.cuda.synchronize()
            plain_ms += ev0.elapsed_time(ev1)
            plain_n += 1
        if it % 10 == 0 or lg.event or it == 1:
            logs.append(dict(t=lg.t, loss=lg.loss, l1=lg.l1, ssim=lg.ssim, n=lg.n_gaussians, l_max=lg.l_max,
                             gate=lg.gate, event=lg.event))
        if lg.event:
            print(it, lg.event, f"loss {lg.loss:.4f}", flush=True)
    wall = time.perf_counter() - t0
    first = np.mean([x["loss"] for x in logs[:5]])
    last = np.mean([x["loss"] for x in logs[-5:]])
    out = {"what": "NEXT-4 synthetic training run (paper_2605_13794_b200.train.Trainer)",
           "scene": f"gen_city rubble-shaped, {gt.n} ground-truth Gaussians, {a.W}x{a.H}, {a.views} cameras; "
                    f"init: 40% subset, perturbed means, grey SH, opacity 0.3, 1.3x scales",
           "schedule": vars(sched), "d0_factor": a.d0_factor, "iters": a.iters, "batch": 4, "lambda": 0.2, "beta": 10.0, "tau": a.tau,
           "loss_first": first, "loss_last": last, "falls": bool(last < first),
           "iter_ms_device_mean": plain_ms / max(plain_n, 1), "iters_per_s_device": 1000.0 * plain_n / plain_ms,
           "wall_s": wall, "final_gaussians": tr.n, "log": logs}
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "log"}), flush=True)


if __name__ == "__main__":
    main()
