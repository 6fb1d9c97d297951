"""A few Rubble views through bgs_view_step (a1-a11, world 1, Z-ordered shard) for ncu captures of the
view kernels (tools only; never a bench number).  python tools/view_probe.py [views] [config]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synthetic as S  # noqa: E402
import paper_2605_13794_b200.bgs as B  # noqa: E402

nviews = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = sys.argv[2] if len(sys.argv) > 2 else "rubble"
with_imp = len(sys.argv) > 3 and sys.argv[3] == "imp"
scene = S.gen_city(cfg, V=64)
g = B.GaussianPlanes.from_scene(scene, "cuda")
ctx = B.Context(0, 1, 0)
perm = B.spatial_order(ctx, g)
g = B.GaussianPlanes(g.mean_opac[perm].contiguous(), g.quat[perm].contiguous(), g.scale[perm].contiguous(),
                     g.sh[perm].contiguous(), g.lod[perm].contiguous())
cam0 = scene.cameras[0]
H, W = cam0["H"], cam0["W"]
n = scene.n
radius = torch.zeros(n, dtype=torch.int32, device="cuda")
rgb, T = torch.zeros(3, H, W, device="cuda"), torch.zeros(H, W, device="cuda")
nc = torch.zeros(H, W, dtype=torch.int32, device="cuda")
dl = torch.from_numpy(S.grad_image(H, W)).cuda()
grads = g.zeros_grads()
imp = None
if with_imp:
    imp = B.importance_out(torch.zeros(n, dtype=torch.float64, device="cuda"), torch.zeros(n, dtype=torch.int32, device="cuda"),
                           torch.zeros(n, dtype=torch.int32, device="cuda"),
                           torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda"))
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for v in range(nviews):
        B.bgs_view_step(ctx, g, B.camera(scene.cameras[(5 + v) % 64]), None, None, 0, radius, rgb, T, nc, dl, grads,
                        imp, st)
    st.synchronize()
print("ok", ctx.query())
