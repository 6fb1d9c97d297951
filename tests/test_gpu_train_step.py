"""NEXT-4 supervised view step through the C ABI: bgs_train_view_step(_host_async) equals the
composition of its parity-tested parts (bgs_view_step with the dL/dC that bgs_loss_photo
writes, plus bgs_loss_scale), and the host-buffer variant returns the device variant's loss.

Gradients are fp32 atomics (order-dependent): compared within 1e-5 |g| + 1e-6 max|g|; loss
values are deterministic (fixed-order sums): compared exactly.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import synthetic as S  # noqa: E402

pytestmark = pytest.mark.gpu
LAM, BINV, BETA = 0.2, 0.25, 0.01


def _setup(scene, B):
    dev = "cuda:0"
    g = B.GaussianPlanes.from_scene(scene, dev)
    cam = scene.cameras[0]
    H, W = cam["H"], cam["W"]
    n = scene.n
    bufs = dict(radius=torch.zeros(n, dtype=torch.int32, device=dev), rgb=torch.zeros(3, H, W, device=dev),
                T=torch.zeros(H, W, device=dev), nc=torch.zeros(H, W, dtype=torch.int32, device=dev),
                dl=torch.zeros(3, H, W, device=dev))
    tgt = torch.from_numpy(S.target_image(H, W)).to(dev)
    return g, B.camera(cam), bufs, tgt


def _close(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.all(np.abs(a - b) <= 1e-5 * np.abs(b) + 1e-6 * np.abs(b).max())


def test_train_step_equals_its_parts(tiny_scene):
    import paper_2605_13794_b200.bgs as B
    g, cam, b, tgt = _setup(tiny_scene, B)
    ctx = B.Context(0, 1, 0)
    st = torch.cuda.Stream()
    try:
        with torch.cuda.stream(st):
            # fused step
            gr1 = g.zeros_grads()
            lo1 = torch.zeros(5, dtype=torch.float64, device="cuda")
            sup = B.supervision(tgt, LAM, BINV, BETA, lo1)
            B.bgs_train_view_step(ctx, g, cam, None, None, 0, b["radius"], sup, b["rgb"], b["T"], b["nc"], b["dl"],
                                  gr1, None, st)
            st.synchronize()
            rgb1, dl1 = b["rgb"].clone(), b["dl"].clone()
            # parts: forward, explicit loss, backward with that dL/dC, explicit Eq.8
            gr2 = g.zeros_grads()
            B.bgs_project(ctx, g, cam, None, None, 0, b["radius"], st)
            B.bgs_route(ctx, None, st)
            B.bgs_sort_tiles(ctx, st)
            B.bgs_raster_fwd(ctx, 0, b["rgb"], b["T"], b["nc"], st)
            dl2 = torch.zeros_like(b["dl"])
            lo2 = torch.zeros(5, dtype=torch.float64, device="cuda")
            B.bgs_loss_photo(ctx, b["rgb"], tgt, LAM, BINV, dl2, lo2[:3], st)
            B.bgs_raster_bwd(ctx, dl2, b["T"], b["nc"], st)
            B.bgs_route_reverse(ctx, st)
            B.bgs_project_bwd(ctx, g, cam, gr2, st)
            B.bgs_loss_scale(ctx, g, BETA, gr2, lo2[3:], st)
            st.synchronize()
        assert torch.equal(rgb1, b["rgb"]) and torch.equal(dl1, dl2)
        assert torch.equal(lo1, lo2), (lo1, lo2)
        assert lo1[4].item() > 0 and 0 < lo1[2].item() < 1
        for k in ("mean_opac", "quat", "scale", "sh"):
            assert _close(getattr(gr1, k).cpu().numpy(), getattr(gr2, k).cpu().numpy()), k
        assert getattr(gr1, "scale").abs().sum().item() > 0
    finally:
        ctx.close()


def test_train_step_host_async_matches_device(tiny_scene):
    import paper_2605_13794_b200.bgs as B
    g, cam, b, tgt = _setup(tiny_scene, B)
    ctx = B.Context(0, 1, 0)
    st = torch.cuda.Stream()
    try:
        with torch.cuda.stream(st):
            gr1 = g.zeros_grads()
            lo1 = torch.zeros(5, dtype=torch.float64, device="cuda")
            B.bgs_train_view_step(ctx, g, cam, None, None, 0, b["radius"], B.supervision(tgt, LAM, BINV, BETA, lo1),
                                  b["rgb"], b["T"], b["nc"], b["dl"], gr1, None, st)
            gr2 = g.zeros_grads()
            tgt_h = tgt.cpu().pin_memory()
            lo_h = torch.full((5,), -1.0, dtype=torch.float64).pin_memory()
            B.bgs_train_view_step_host_async(ctx, g, cam, None, None, 0, b["radius"], tgt_h, LAM, BINV, BETA, lo_h,
                                             gr2, None, st)
            st.synchronize()
        assert torch.equal(lo_h, lo1.cpu()), (lo_h, lo1)
        for k in ("mean_opac", "quat", "scale", "sh"):
            assert _close(getattr(gr1, k).cpu().numpy(), getattr(gr2, k).cpu().numpy()), k
    finally:
        ctx.close()
