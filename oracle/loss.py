"""NEXT-4 supervision oracle: the loss of Eq.7-8, plain numpy in fp64.

TEST INFRASTRUCTURE ONLY: imported by tests/ (and nothing in the product package).  It shares
no code with paper_2605_13794_b200/csrc/loss.cu.

Definitions followed (readings R34, R35 in DESIGN.md §2):
  Eq.7  l_v = (1 - lambda) ||I^ - I||_1 + lambda (1 - SSIM(I^, I))
        ||.||_1 and SSIM are means over the 3 H W elements; L_photo = (1/B) sum_b l_b.
  SSIM  the 3DGS form: per channel, window w = outer(g, g), g the normalised 11-tap Gaussian of
        sigma 1.5, "same"-size filtering with zero padding, C1 = 0.01^2, C2 = 0.03^2:
          mu_x = w * x, sigma_x^2 = w * x^2 - mu_x^2, sigma_xy = w * (x y) - mu_x mu_y
          S(p) = (2 mu_x mu_y + C1)(2 sigma_xy + C2) / ((mu_x^2 + mu_y^2 + C1)(sigma_x^2 + sigma_y^2 + C2))
  Eq.8  L_scale = (1/|V|) sum_{i in V} min_j sigma_ij, V = {i : radius_i > 0}

Pins (tests/test_oracle_loss.py): identical images, constant-image closed form, the SSIM map
against scipy.ndimage.correlate, finite differences of the loss, L1 closed forms, Eq.8 hand
examples.
"""
from __future__ import annotations

import numpy as np

C1 = 0.01 ** 2
C2 = 0.03 ** 2
WIN = 11
SIGMA = 1.5


def gaussian_window(size: int = WIN, sigma: float = SIGMA) -> np.ndarray:
    """Normalised 1-D Gaussian window g[k] ~ exp(-(k - c)^2 / (2 sigma^2)), k = 0..size-1."""
    c = size // 2
    g = np.array([np.exp(-((k - c) ** 2) / (2.0 * sigma * sigma)) for k in range(size)], np.float64)
    return g / g.sum()


def filter_same(img: np.ndarray, g: np.ndarray) -> np.ndarray:
    """out[p] = sum_{u,v} g[u] g[v] img[p + (u - c, v - c)], zero outside the image (one 2-D
    plane), written as the plain sum over the size^2 window offsets."""
    H, W = img.shape
    c = len(g) // 2
    pad = np.zeros((H + 2 * c, W + 2 * c), np.float64)
    pad[c:c + H, c:c + W] = img
    out = np.zeros((H, W), np.float64)
    for u in range(len(g)):
        for v in range(len(g)):
            out += g[u] * g[v] * pad[u:u + H, v:v + W]
    return out


def ssim_terms(x: np.ndarray, y: np.ndarray):
    """Per-channel window statistics and the SSIM map of (x, y), both [3][H][W] fp64."""
    g = gaussian_window()
    mu_x = np.stack([filter_same(x[c], g) for c in range(3)])
    mu_y = np.stack([filter_same(y[c], g) for c in range(3)])
    sx2 = np.stack([filter_same(x[c] * x[c], g) for c in range(3)]) - mu_x * mu_x
    sy2 = np.stack([filter_same(y[c] * y[c], g) for c in range(3)]) - mu_y * mu_y
    sxy = np.stack([filter_same(x[c] * y[c], g) for c in range(3)]) - mu_x * mu_y
    l_num = 2 * mu_x * mu_y + C1
    c_num = 2 * sxy + C2
    l_den = mu_x * mu_x + mu_y * mu_y + C1
    c_den = sx2 + sy2 + C2
    smap = (l_num * c_num) / (l_den * c_den)
    return dict(mu_x=mu_x, mu_y=mu_y, sx2=sx2, sy2=sy2, sxy=sxy, l_num=l_num, c_num=c_num, l_den=l_den,
                c_den=c_den, map=smap)


def photo_loss(x, y, lam: float):
    """Eq.7 of one view: (l_v, L1_v, SSIM_v)."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    l1 = float(np.mean(np.abs(x - y)))
    ssim = float(np.mean(ssim_terms(x, y)["map"]))
    return (1.0 - lam) * l1 + lam * (1.0 - ssim), l1, ssim


def photo_loss_grad(x, y, lam: float, batch_inv: float = 1.0) -> np.ndarray:
    """batch_inv * d l_v / d x (reverse mode through the steps of ssim_terms; sign(0) = 0)."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    n = x.size
    t = ssim_terms(x, y)
    g = gaussian_window()
    # d S(p) / d (mu_x, sigma_x^2, sigma_xy) at every p
    den = t["l_den"] * t["c_den"]
    d_mu_x = 2 * t["mu_y"] * t["c_num"] / den - t["map"] * 2 * t["mu_x"] / t["l_den"]
    d_sx2 = -t["map"] / t["c_den"]
    d_sxy = 2 * t["l_num"] / den
    # adjoints of the filtered quantities: mu_x enters directly, through sigma_x^2 = E[xx] - mu_x^2
    # and through sigma_xy = E[xy] - mu_x mu_y
    adj_mu_x = d_mu_x - 2 * t["mu_x"] * d_sx2 - t["mu_y"] * d_sxy
    adj_exx = d_sx2
    adj_exy = d_sxy
    # the filter is symmetric, so its adjoint is the same zero-padded filter
    dS = np.stack([filter_same(adj_mu_x[c], g) + 2 * x[c] * filter_same(adj_exx[c], g)
                   + y[c] * filter_same(adj_exy[c], g) for c in range(3)])
    d_l1 = np.sign(x - y)
    return batch_inv * ((1.0 - lam) * d_l1 / n - lam * dS / n)


def scale_reg(scales, radius, beta: float):
    """Eq.8 of one view: (L_scale, |V|, grad) with grad[i, argmin_j] = beta / |V| (first minimal
    axis among ties) for i in V."""
    s = np.asarray(scales, np.float64)[:, :3]
    vis = np.asarray(radius) > 0
    nv = int(vis.sum())
    grad = np.zeros_like(s)
    if nv == 0:
        return 0.0, 0, grad
    mins = s.min(axis=1)
    L = float(mins[vis].sum() / nv)
    arg = np.argmin(s, axis=1)  # numpy: first occurrence of the minimum
    idx = np.flatnonzero(vis)
    grad[idx, arg[idx]] = beta / nv
    return L, nv, grad
