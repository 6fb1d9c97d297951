"""NEXT-4 supervision through the C ABI vs oracle/loss.py (Eq.7, Eq.8).

Both sides see the same rendered image (the CUDA path's own forward, parity-tested in
test_gpu_parity.py) and the same seeded target.  Tolerances: loss terms within
2e-6 relative (fp32 window sums, fp64 accumulation of the means); dl/drgb within
1e-3 |g| + 1e-4 max|g| per element (fp32 statistics; sigma^2 = E[x^2] - mu^2 loses ~1e-5
relative to cancellation in flat regions); world > 1: dl/drgb bit-identical to world 1 on the
owned pixels (same full image, same per-CTA arithmetic), loss within 1e-12 (summation order).
Eq.8: |V| exact, L_scale within 1e-12, the gradient exactly float(beta/|V|) on the argmin axis.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import synthetic as S  # noqa: E402
from gpu_helpers import GpuStep  # noqa: E402
from oracle import loss as OL  # noqa: E402

pytestmark = pytest.mark.gpu
LAM = 0.2
BINV = 0.25


def _check_photo(gs, tgt, lam=LAM, binv=BINV):
    x = gs.img.astype(np.float64)
    l, l1, ssim = OL.photo_loss(x, tgt, lam)
    lo = gs.loss[0]
    assert abs(lo[1] - l1) <= 2e-6 * abs(l1) + 1e-12, (lo, l1)
    assert abs(lo[2] - ssim) <= 2e-6 * abs(ssim) + 1e-12, (lo, ssim)
    assert abs(lo[0] - l) <= 2e-6 * abs(l) + 1e-12, (lo, l)
    g = OL.photo_loss_grad(x, tgt, lam, binv)
    d = np.abs(gs.dl_loss - g)
    tol = 1e-3 * np.abs(g) + 1e-4 * np.abs(g).max()
    assert np.all(d <= tol), (d.max(), np.abs(g).max(), np.unravel_index(np.argmax(d - tol), d.shape))


@pytest.fixture(scope="module")
def tiny_loss(tiny_scene):
    cam = tiny_scene.cameras[0]
    tgt = S.target_image(cam["H"], cam["W"])
    gs = GpuStep(tiny_scene, cam, M=1, target=tgt, lam=LAM, batch_inv=BINV, beta=0.5)
    yield tiny_scene, cam, tgt, gs
    gs.close()


def test_photo_loss_parity(tiny_loss):
    _, _, tgt, gs = tiny_loss
    _check_photo(gs, tgt)


@pytest.mark.parametrize("lam", [0.0, 1.0])
def test_photo_loss_lambda_ends(tiny_scene, lam):
    cam = tiny_scene.cameras[0]
    tgt = S.target_image(cam["H"], cam["W"], seed=4)
    gs = GpuStep(tiny_scene, cam, M=1, target=tgt, lam=lam, batch_inv=1.0, importance=False)
    try:
        _check_photo(gs, tgt, lam, 1.0)
    finally:
        gs.close()


def test_photo_loss_ragged_image():
    sc = S.gen_small(21, 400, 250, 181)
    cam = sc.cameras[0]
    tgt = S.target_image(cam["H"], cam["W"], seed=2)
    gs = GpuStep(sc, cam, M=1, target=tgt, lam=LAM, batch_inv=BINV)
    try:
        _check_photo(gs, tgt)
    finally:
        gs.close()


@pytest.mark.parametrize("M", [2, 3])
def test_photo_loss_world_invariance(tiny_loss, M):
    sc, cam, tgt, g1 = tiny_loss
    gm = GpuStep(sc, cam, M=M, target=tgt, lam=LAM, batch_inv=BINV, beta=0.5)
    try:
        assert np.array_equal(gm.img, g1.img)
        assert np.array_equal(gm.dl_loss, g1.dl_loss)  # owned pixels stitched: every pixel once
        for r in range(M):
            assert np.allclose(gm.loss[r], g1.loss[0], rtol=1e-12, atol=0)
            assert np.allclose(gm.loss_scale[r], g1.loss_scale[0], rtol=1e-12, atol=0)
        assert np.array_equal(gm.g_scale_reg, g1.g_scale_reg)
    finally:
        gm.close()


def test_photo_loss_identical_target(tiny_scene):
    cam = tiny_scene.cameras[0]
    g0 = GpuStep(tiny_scene, cam, M=1, importance=False)
    img = g0.img.copy()
    g0.close()
    gs = GpuStep(tiny_scene, cam, M=1, target=img, lam=LAM, batch_inv=1.0, importance=False)
    try:
        assert abs(gs.loss[0][0]) < 1e-6 and gs.loss[0][1] == 0.0
        ref = np.abs(OL.photo_loss_grad(img, S.target_image(cam["H"], cam["W"]), LAM)).max()
        assert np.abs(gs.dl_loss).max() < 1e-3 * ref
    finally:
        gs.close()


def test_scale_regulariser_parity(tiny_loss):
    sc, _, _, gs = tiny_loss
    L, nv, g = OL.scale_reg(sc.scales, gs.radius, 0.5)
    lo = gs.loss_scale[0]
    assert lo[1] == nv and nv > 0
    assert abs(lo[0] - L) <= 1e-12 * L
    want = np.zeros((sc.n, 4), np.float32)
    want[:, :3] = g.astype(np.float32)
    nz = g != 0
    want[:, :3][nz] = np.float32(0.5 / nv)
    assert np.array_equal(gs.g_scale_reg, want)


def test_photo_loss_full_size():
    """BASELINE image size (1152x864, the bench's Rubble views) with many 32x32 loss tiles and a ragged
    last tile row (864 = 27 x 32; 1152 = 36 x 32): loss terms and the gradient on every pixel."""
    sc = S.gen_small(23, 3000, 1152, 864, spread=2.0)
    cam = sc.cameras[0]
    tgt = S.target_image(cam["H"], cam["W"], seed=8)
    gs = GpuStep(sc, cam, M=1, target=tgt, lam=LAM, batch_inv=BINV, importance=False)
    try:
        assert gs.img.max() > 0.05  # something rendered
        _check_photo(gs, tgt)
    finally:
        gs.close()
