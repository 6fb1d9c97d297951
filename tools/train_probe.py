"""Run a few supervised Rubble views (bgs_train_view_step + bgs_densify_accumulate), then one
bgs_adam_step and one bgs_densify_apply, for ncu launch lists / captures of the training-step
kernels (tools only; never a bench number)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synthetic as S  # noqa: E402
import paper_2605_13794_b200.bgs as B  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "rubble"
nviews = int(sys.argv[2]) if len(sys.argv) > 2 else 3
scene = S.gen_city(cfg, V=8)
g = B.GaussianPlanes.from_scene(scene, "cuda")
ctx = B.Context(0, 1, 0)
cam0 = scene.cameras[0]
H, W = cam0["H"], cam0["W"]
n = scene.n
radius = torch.zeros(n, dtype=torch.int32, device="cuda")
rgb, T = torch.zeros(3, H, W, device="cuda"), torch.zeros(H, W, device="cuda")
nc, dl = torch.zeros(H, W, dtype=torch.int32, device="cuda"), torch.zeros(3, H, W, device="cuda")
tgt = torch.from_numpy(S.target_image(H, W)).cuda()
lo = torch.zeros(5, dtype=torch.float64, device="cuda")
grads = g.zeros_grads()
st = torch.cuda.Stream()
stat = torch.zeros(n, device="cuda")
cnt = torch.zeros(n, dtype=torch.int32, device="cuda")
with torch.cuda.stream(st):
    for v in range(nviews):
        B.bgs_train_view_step(ctx, g, B.camera(scene.cameras[v % 8]), None, None, 0, radius,
                              B.supervision(tgt, 0.2, 0.25, 0.0025, lo), rgb, T, nc, dl, grads, None, st)
        B.bgs_densify_accumulate(ctx, n, None, stat, cnt, st)
    o = g.mean_opac[:, 3].clamp(1e-6, 1 - 1e-6)
    tp = B.TrainParams(torch.cat([g.mean_opac[:, :3], torch.log(o / (1 - o))[:, None]], 1).contiguous(),
                       g.quat.clone(), torch.log(g.scale.clamp_min(1e-30)).contiguous(), g.sh.clone())
    act = B.GaussianPlanes(torch.empty_like(g.mean_opac), torch.empty_like(g.quat), torch.empty_like(g.scale), tp.sh,
                           g.lod)
    B.bgs_adam_step(ctx, tp, grads, act, None, B.adam_hparams(step=1), st)
    cap = 2 * n + 1
    tout = B.TrainParams(*(torch.empty(cap, c, device="cuda") for c in (4, 4, 4, 48)))
    lod_out = torch.empty(cap, dtype=torch.uint8, device="cuda")
    n_new = B.bgs_densify_apply(ctx, tp, g.lod, stat, cnt, B.densify_params(5e-5, 10.0, 0.005, 1.6, 1), tout,
                                lod_out, None, st)
    st.synchronize()
print("densify rows", n, "->", n_new)
print(lo.cpu().tolist())
