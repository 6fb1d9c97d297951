"""Run a few supervised Rubble views (bgs_train_view_step) for ncu launch lists of the loss
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
with torch.cuda.stream(st):
    for v in range(nviews):
        B.bgs_train_view_step(ctx, g, B.camera(scene.cameras[v % 8]), None, None, 0, radius,
                              B.supervision(tgt, 0.2, 0.25, 0.0025, lo), rgb, T, nc, dl, grads, None, st)
    st.synchronize()
print(lo.cpu().tolist())
