"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): one tiny view
through every stage (a1..a12, world 1), two views in flight on two contexts, the batched step
(eager and graph), the in-process group at M = 2 and the NEXT-1/3/4 calls, so every kernel of
libbgs runs at least once under the tool.

    compute-sanitizer --tool racecheck python tools/sanitize_probe.py
"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_13794_b200.bgs as B  # noqa: E402
import synthetic as S  # noqa: E402


def main():
    dev = "cuda:0"
    torch.cuda.set_device(0)
    sc = S.gen_tiny(n=3000, W=128, H=96, seed=3)
    cams = [S.make_camera(128, 96, np.eye(3), np.array([0.05 * k, 0.0, 0.0])) for k in range(4)]
    H, W = 96, 128
    g = B.GaussianPlanes.from_scene(sc, dev)
    grads = g.zeros_grads()
    n = sc.n
    nw = (n + 31) // 32
    s = torch.zeros(n, dtype=torch.float64, device=dev)
    cr = torch.zeros(n, dtype=torch.int32, device=dev)
    cv = torch.zeros(n, dtype=torch.int32, device=dev)
    dl = torch.from_numpy(S.grad_image(H, W)).to(dev)

    def bufs():
        return dict(radius=torch.zeros(n, dtype=torch.int32, device=dev), rgb=torch.zeros(3, H, W, device=dev),
                    T=torch.zeros(H, W, device=dev), nc=torch.zeros(H, W, dtype=torch.int32, device=dev),
                    cull=torch.zeros(nw, dtype=torch.int32, device=dev))

    # two views in flight (two contexts, two streams, shared gradients / importance outputs)
    ctxs = [B.Context(0, 1, 0) for _ in range(2)]
    bb = [bufs() for _ in range(2)]
    st = [torch.cuda.Stream(dev) for _ in range(2)]
    for k in range(2):
        b = bb[k]
        B.bgs_view_step(ctxs[k], g, B.camera(cams[k]), None, None, 0, b["radius"], b["rgb"], b["T"], b["nc"], dl,
                        grads, B.importance_out(s, cr, cv, b["cull"]), st[k])
    torch.cuda.synchronize()
    # supervised step + Adam + density control + simplification on ctx 0
    ctx = ctxs[0]
    tgt = torch.from_numpy(S.target_image(H, W)).to(dev)
    lo = torch.zeros(5, dtype=torch.float64, device=dev)
    dls = torch.zeros(3, H, W, device=dev)
    b = bb[0]
    B.bgs_train_view_step(ctx, g, B.camera(cams[0]), None, None, 0, b["radius"], B.supervision(tgt, 0.2, 1.0, 0.01, lo),
                          b["rgb"], b["T"], b["nc"], dls, grads, None)
    stat = torch.zeros(n, dtype=torch.float32, device=dev)
    cnt = torch.zeros(n, dtype=torch.int32, device=dev)
    B.bgs_densify_accumulate(ctx, n, None, stat, cnt)
    vis = torch.zeros(nw, dtype=torch.int32, device=dev)
    B.bgs_visibility_mask(ctx, n, b["radius"], vis)
    o = g.mean_opac[:, 3].clamp(1e-6, 1 - 1e-6)
    tp = B.TrainParams(torch.cat([g.mean_opac[:, :3], torch.log(o / (1 - o))[:, None]], 1).contiguous(),
                       g.quat.clone(), torch.log(g.scale).contiguous(), g.sh.clone())
    tp.log_scale[:, 3] = 0
    act = B.GaussianPlanes(torch.zeros_like(g.mean_opac), torch.zeros_like(g.quat), torch.zeros_like(g.scale), tp.sh,
                           g.lod)
    B.bgs_adam_step(ctx, tp, grads, act, vis, B.adam_hparams(step=1))
    cap = 2 * n + 1
    tout = B.TrainParams(*(torch.empty(cap, c, device=dev) for c in (4, 4, 4, 48)))
    lod_out = torch.empty(cap, dtype=torch.uint8, device=dev)
    act2 = B.GaussianPlanes(torch.empty(cap, 4, device=dev), torch.empty(cap, 4, device=dev),
                            torch.empty(cap, 4, device=dev), tout.sh, lod_out)
    B.bgs_densify_apply(ctx, tp, g.lod, stat, cnt, B.densify_params(1e-9, 0.05, 0.005, 1.6, 7), tout, lod_out, act2)
    phi = torch.zeros(n, dtype=torch.float64, device=dev)
    keep = torch.zeros(n, dtype=torch.uint8, device=dev)
    B.bgs_score_phi(ctx, n, cr, cv, phi)
    B.bgs_prune_stochastic(ctx, n, s, n // 2, 11, keep)
    B.bgs_prune_mass_cut(ctx, n, s, 99, 100, keep)
    out_g = B.GaussianPlanes(torch.empty(n + 1, 4, device=dev), torch.empty(n + 1, 4, device=dev),
                             torch.empty(n + 1, 4, device=dev), torch.empty(n + 1, 48, device=dev),
                             torch.empty(n + 1, dtype=torch.uint8, device=dev))
    B.bgs_redistribute(ctx, g, keep, out_g)
    torch.cuda.synchronize()
    # batched step: eager, then graph (twice: the first graph batch may fall back while arenas grow)
    bctx = B.Context(0, 1, 0)
    vb = [bufs() for _ in range(4)]
    views = [B.batch_view(B.camera(cams[k]), vb[k]["radius"], vb[k]["rgb"], vb[k]["T"], vb[k]["nc"], dl,
                          cull_out=vb[k]["cull"]) for k in range(4)]
    imp = B.importance_out(s, cr, cv, vb[0]["cull"])
    for flags in (0, B.BGS_GRAPH, B.BGS_GRAPH):
        B.bgs_batch_step(bctx, g, views, None, flags, grads, imp)
    torch.cuda.synchronize()
    bctx.close()
    # in-process group, M = 2, per-view and batched
    grp = B.Context.local_group(2, 0)
    errs = []

    def run(r):
        try:
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream(dev)
            with torch.cuda.stream(stream):
                sh = sc.shard(r, 2)
                gg = B.GaussianPlanes.from_scene(sh, dev)
                gr = gg.zeros_grads()
                m = sh.n
                mb = dict(radius=torch.zeros(m, dtype=torch.int32, device=dev), rgb=torch.zeros(3, H, W, device=dev),
                          T=torch.zeros(H, W, device=dev), nc=torch.zeros(H, W, dtype=torch.int32, device=dev))
                ss = torch.zeros(m, dtype=torch.float64, device=dev)
                c1 = torch.zeros(m, dtype=torch.int32, device=dev)
                c2 = torch.zeros(m, dtype=torch.int32, device=dev)
                cu = torch.zeros((m + 31) // 32, dtype=torch.int32, device=dev)
                B.bgs_view_step(grp[r], gg, B.camera(cams[0]), None, None, 0, mb["radius"], mb["rgb"], mb["T"],
                                mb["nc"], dl, gr, B.importance_out(ss, c1, c2, cu), stream)
                # each view of a batch needs its own output buffers (the views run concurrently)
                vb2 = [dict(radius=torch.zeros(m, dtype=torch.int32, device=dev), rgb=torch.zeros(3, H, W, device=dev),
                            T=torch.zeros(H, W, device=dev), nc=torch.zeros(H, W, dtype=torch.int32, device=dev))
                       for _ in range(2)]
                vv = [B.batch_view(B.camera(cams[k]), vb2[k]["radius"], vb2[k]["rgb"], vb2[k]["T"], vb2[k]["nc"], dl)
                      for k in range(2)]
                B.bgs_batch_step(grp[r], gg, vv, None, 0, gr, None, stream)
                stream.synchronize()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for c in grp + ctxs:
        c.close()
    if errs:
        raise errs[0]
    torch.cuda.synchronize()
    print("sanitize probe ok")


if __name__ == "__main__":
    main()
