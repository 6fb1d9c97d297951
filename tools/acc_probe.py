import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
import synthetic as S
import paper_2605_13794_b200.bgs as B
cfg = sys.argv[1]
scene = S.gen_city(cfg)
g = B.GaussianPlanes.from_scene(scene, "cuda")
ctx = B.Context(0, 1, 0)
cam = scene.cameras[int(sys.argv[2]) if len(sys.argv) > 2 else 1]
H, W = cam["H"], cam["W"]
n = scene.n
radius = torch.zeros(n, dtype=torch.int32, device="cuda")
rgb, T = torch.zeros(3, H, W, device="cuda"), torch.zeros(H, W, device="cuda")
nc = torch.zeros(H, W, dtype=torch.int32, device="cuda")
dl = torch.from_numpy(S.grad_image(H, W)).cuda()
grads = g.zeros_grads()
s = torch.zeros(n, dtype=torch.float64, device="cuda"); cr = torch.zeros(n, dtype=torch.int32, device="cuda"); cv = torch.zeros(n, dtype=torch.int32, device="cuda")
cull = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
for imp in (False, True):
    B.bgs_view_step(ctx, g, B.camera(cam), None, None, 0, radius, rgb, T, nc, dl, grads,
                    B.importance_out(s, cr, cv, cull) if imp else None)
    torch.cuda.synchronize()
    acc = ctx.debug_buffer("acc")
    q = ctx.query()
    print("imp", imp, "dtype", acc.dtype, acc.numel(), "R", q["R"], "F", q["F"])
    av = acc.view(torch.int32).view(-1, 12)[:, 9].cpu().numpy().view(np.uint32)
    print(" a: min", av.min(), "max", av.max(), "sum", av.astype(np.int64).sum(), "n>1e7", (av > 10_000_000).sum())
    print(" E", int(nc.sum(dtype=torch.int64).item()))
    tsum = acc.view(torch.int32).view(-1, 12)[:, 9].sum(dtype=torch.int64).item()
    print(" torch sum", tsum)
    big = np.flatnonzero(av > (1 << 20))
    print(" big a:", len(big), big[:10], av[big[:10]])
    if len(big):
        f = acc.view(torch.float32).view(-1, 12)[torch.from_numpy(big[:5]).cuda()].cpu().numpy()
        print(" rows", f)
