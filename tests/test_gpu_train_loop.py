"""NEXT-4 training iteration (paper_2605_13794_b200.train.Trainer) on a small synthetic scene: every
schedule event of P:342 fires on its step (density control inside the window, stochastic pruning at T1,
mass pruning at T2, the gate engaged outside the window with L_max(t) from S:398) and the loss falls
from a perturbed start towards the ground truth the library rendered."""
import numpy as np
import pytest
import torch

import synthetic as S

pytestmark = pytest.mark.gpu


def test_trainer_schedule_and_loss():
    import paper_2605_13794_b200.bgs as B
    from paper_2605_13794_b200.train import Schedule, Trainer
    dev = "cuda:0"
    gt = S.gen_city("rubble", n=60_000, W=192, H=144, V=8, seed=31)
    ctx = B.Context(0, 1, 0)
    g_gt = B.GaussianPlanes.from_scene(gt, dev)
    H, W = 144, 192
    targets = []
    rad = torch.zeros(gt.n, dtype=torch.int32, device=dev)
    for cam in gt.cameras:
        rgb = torch.zeros(3, H, W, device=dev)
        T = torch.zeros(H, W, device=dev)
        nc = torch.zeros(H, W, dtype=torch.int32, device=dev)
        B.bgs_view_step(ctx, g_gt, B.camera(cam), None, None, 0, rad, rgb, T, nc, None, None, None)
        targets.append(rgb)
    torch.cuda.synchronize()
    rng = np.random.Generator(np.random.PCG64(2))
    idx = np.sort(rng.choice(gt.n, size=gt.n // 2, replace=False))
    means = gt.means[idx] + rng.normal(0, 1, (idx.size, 3)) * 0.3 * gt.scales[idx].max(1, keepdims=True)
    opac = np.full(idx.size, 0.3, np.float32)
    sh = np.zeros((idx.size, 48), np.float32)
    ml = np.concatenate([means, np.log(opac / (1 - opac))[:, None]], 1).astype(np.float32)
    ls = np.zeros((idx.size, 4), np.float32)
    ls[:, :3] = np.log(gt.scales[idx] * 1.2)
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(dev)
    tp = B.TrainParams(t(ml), t(gt.quats[idx]), t(ls), t(sh))
    lod = torch.from_numpy(np.ascontiguousarray(gt.lod[idx], np.uint8)).to(dev)
    sched = Schedule(dc_start=10, dc_end=60, dc_every=10, t1=40, t2=80, unlock_first=5, k_levels=gt.k_levels)
    dp = B.densify_params(2e-4, 10.0, 0.005, 1.6, 5, gt.k_levels)
    tr = Trainer(ctx, tp, lod, gt.cameras, targets, gt.d0 * 64, sched, batch=4, lam=0.2, beta=10.0, seed=3,
                 densify=dp, device=dev)
    logs = [tr.step(it) for it in range(1, 101)]
    events = {lg.t: lg.event for lg in logs if lg.event}
    assert sorted(t for t, e in events.items() if "densify" in e) == [10, 20, 30, 40, 50, 60]
    assert "scoring (stochastic)" in events[40] and "scoring (mass)" in events[80]
    assert all(lg.gate == sched.gate_enabled(lg.t) and lg.l_max == sched.l_max(lg.t) for lg in logs)
    assert [lg.l_max for lg in logs][:4] == [0, 0, 0, 0] and logs[-1].l_max == gt.k_levels - 1
    first = np.mean([lg.loss for lg in logs[:5]])
    last = np.mean([lg.loss for lg in logs[-5:]])
    assert last < 0.8 * first, (first, last)
    assert np.isfinite([lg.loss for lg in logs]).all()
    ctx.close()
