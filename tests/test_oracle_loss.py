"""Pins of the NEXT-4 supervision oracle (oracle/loss.py) against what the paper and the
mathematics fix: Eq.7 with the 3DGS SSIM (reading R34), Eq.8 (R35)."""
import numpy as np
import pytest
from scipy import ndimage

from oracle import loss as OL


def _imgs(H=23, W=31, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.random((3, H, W))
    y = np.clip(x + 0.2 * rng.standard_normal((3, H, W)), 0, 1)
    return x, y


def test_window_is_normalised_symmetric_gaussian():
    g = OL.gaussian_window()
    assert g.shape == (11,) and abs(g.sum() - 1) < 1e-15
    assert np.allclose(g, g[::-1], rtol=0, atol=0)
    # successive ratios of a sigma = 1.5 Gaussian: g[c+1]/g[c] = exp(-1/4.5)
    assert abs(g[6] / g[5] - np.exp(-1 / 4.5)) < 1e-15
    assert abs(g[7] / g[5] - np.exp(-4 / 4.5)) < 1e-15


def test_identical_images_give_zero_loss_and_zero_gradient():
    x, _ = _imgs()
    l, l1, ssim = OL.photo_loss(x, x, 0.2)
    assert l1 == 0.0 and abs(ssim - 1.0) < 1e-14 and abs(l) < 1e-14
    g = OL.photo_loss_grad(x, x, 0.2)
    assert np.max(np.abs(g)) < 1e-12  # SSIM is maximal at y = x; sign(0) = 0 for L1


def test_constant_images_closed_form():
    """Interior pixels (>= 5 from the border) of constant images a, b: sigma terms vanish and
    S = (2ab + C1) / (a^2 + b^2 + C1)."""
    a, b = 0.7, 0.3
    x = np.full((3, 20, 24), a)
    y = np.full((3, 20, 24), b)
    m = OL.ssim_terms(x, y)["map"][:, 5:-5, 5:-5]
    want = (2 * a * b + OL.C1) / (a * a + b * b + OL.C1)
    assert np.allclose(m, want, rtol=1e-12, atol=0)
    # the zero padding lowers the window means at the border, so the border differs
    assert not np.allclose(OL.ssim_terms(x, y)["map"][:, 0, 0], want)


def test_ssim_map_matches_scipy_correlate():
    """Independent filtering routine (scipy.ndimage.correlate, constant-zero mode)."""
    x, y = _imgs(seed=3)
    g = OL.gaussian_window()
    w = np.outer(g, g)

    def f(im):
        return ndimage.correlate(im, w, mode="constant", cval=0.0)

    m = np.empty_like(x)
    for c in range(3):
        mx, my = f(x[c]), f(y[c])
        sx, sy, sxy = f(x[c] ** 2) - mx ** 2, f(y[c] ** 2) - my ** 2, f(x[c] * y[c]) - mx * my
        m[c] = (2 * mx * my + OL.C1) * (2 * sxy + OL.C2) / ((mx ** 2 + my ** 2 + OL.C1) * (sx + sy + OL.C2))
    assert np.allclose(OL.ssim_terms(x, y)["map"], m, rtol=1e-12, atol=1e-14)


def test_l1_closed_forms():
    x, _ = _imgs()
    y = x - 0.125
    l, l1, _ = OL.photo_loss(x, y, 0.0)
    assert abs(l1 - 0.125) < 1e-15 and abs(l - 0.125) < 1e-15
    g = OL.photo_loss_grad(x, y, 0.0, batch_inv=0.25)
    assert np.allclose(g, 0.25 / x.size)


@pytest.mark.parametrize("lam", [0.0, 0.2, 1.0])
def test_gradient_matches_finite_differences(lam):
    x, y = _imgs(H=17, W=19, seed=5)
    g = OL.photo_loss_grad(x, y, lam)
    rng = np.random.default_rng(1)
    pts = [(0, 0, 0), (2, 16, 18), (1, 8, 0), (0, 3, 9)] + [tuple(int(v) for v in rng.integers((3, 17, 19)))
                                                             for _ in range(8)]
    h = 1e-6
    for c, i, j in pts:
        xp, xm = x.copy(), x.copy()
        xp[c, i, j] += h
        xm[c, i, j] -= h
        fd = (OL.photo_loss(xp, y, lam)[0] - OL.photo_loss(xm, y, lam)[0]) / (2 * h)
        assert abs(fd - g[c, i, j]) <= 1e-7 * max(1e-3, abs(g).max()), (c, i, j, fd, g[c, i, j])


def test_scale_regulariser_hand_example():
    s = np.array([[1.0, 2.0, 3.0, 0], [0.5, 0.2, 0.9, 0], [4.0, 4.0, 4.0, 0], [0.3, 0.1, 0.1, 0]])
    r = np.array([1, 0, 3, 2])
    L, nv, g = OL.scale_reg(s, r, beta=0.6)
    assert nv == 3 and abs(L - (1.0 + 4.0 + 0.1) / 3) < 1e-15
    want = np.zeros((4, 3))
    want[0, 0] = want[2, 0] = want[3, 1] = 0.6 / 3  # ties: first minimal axis
    assert np.array_equal(g, want)
    L0, n0, g0 = OL.scale_reg(s, np.zeros(4), beta=1.0)
    assert L0 == 0.0 and n0 == 0 and not g0.any()
