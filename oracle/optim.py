"""NEXT-3 optimizer oracle: activations, their chain rule and Adam, plain numpy in fp64.

TEST INFRASTRUCTURE ONLY: imported by tests/ (never by the product package); shares no code with
paper_2605_13794_b200/csrc/adam.cu.

Definitions followed (readings R13, R38):
  activations (the 3DGS parameterisation; the render ABI takes activated values, R13):
    opacity = sigmoid(logit), s = exp(log s), q = q_raw / |q_raw|, mean and SH identity
  Adam (Kingma & Ba, bias-corrected), per parameter group learning rate:
    m = b1 m + (1 - b1) g;  v = b2 v + (1 - b2) g^2
    p = p - lr (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)
  groups (R38): mean, opacity, rotation, scale, SH coefficient 0 (DC) and SH coefficients 1..15.

Pins (tests/test_oracle_optim.py): torch.optim.Adam on the same raw parameters and gradients,
finite differences of the chain rule, the first-step closed form |update| = lr (eps = 0).
"""
from __future__ import annotations

import numpy as np


def activate(mean_logit, quat_raw, log_scale):
    """Raw planes [n,4] -> activated (mean_opac, quat, scale) [n,4] (scale w = 0)."""
    ml = np.asarray(mean_logit, np.float64)
    q = np.asarray(quat_raw, np.float64)
    ls = np.asarray(log_scale, np.float64)
    mo = ml.copy()
    mo[:, 3] = 1.0 / (1.0 + np.exp(-ml[:, 3]))
    qa = q / np.linalg.norm(q, axis=1, keepdims=True)
    sc = np.zeros_like(ls)
    sc[:, :3] = np.exp(ls[:, :3])
    return mo, qa, sc


def raw_grads(mean_logit, quat_raw, log_scale, g_mo, g_q, g_s):
    """Gradients w.r.t. the activated planes -> gradients w.r.t. the raw planes."""
    ml = np.asarray(mean_logit, np.float64)
    q = np.asarray(quat_raw, np.float64)
    ls = np.asarray(log_scale, np.float64)
    g_mo = np.asarray(g_mo, np.float64)
    g_q = np.asarray(g_q, np.float64)
    g_s = np.asarray(g_s, np.float64)
    o = 1.0 / (1.0 + np.exp(-ml[:, 3]))
    r_ml = g_mo.copy()
    r_ml[:, 3] = g_mo[:, 3] * o * (1.0 - o)            # d sigmoid = o (1 - o)
    nrm = np.linalg.norm(q, axis=1, keepdims=True)
    qh = q / nrm
    r_q = (g_q - qh * np.sum(qh * g_q, axis=1, keepdims=True)) / nrm  # (I - qh qh^T) / |q|
    r_s = np.zeros_like(ls)
    r_s[:, :3] = g_s[:, :3] * np.exp(ls[:, :3])        # d exp = exp
    return r_ml, r_q, r_s


def adam_update(p, m, v, g, lr, b1, b2, eps, t):
    """One bias-corrected Adam update of arrays p, m, v (copies returned); lr broadcastable."""
    m = b1 * m + (1.0 - b1) * g
    v = b2 * v + (1.0 - b2) * g * g
    mh = m / (1.0 - b1 ** t)
    vh = v / (1.0 - b2 ** t)
    return p - lr * mh / (np.sqrt(vh) + eps), m, v


def sh_lr(n: int, lr_dc: float, lr_rest: float) -> np.ndarray:
    """Per-element learning rate of the [n,48] SH plane: floats 0..2 (coefficient 0) take lr_dc."""
    lr = np.full((n, 48), lr_rest)
    lr[:, :3] = lr_dc
    return lr


def adam_step(params: dict, state: dict, grads_act: dict, h: dict, visible=None):
    """The whole step of bgs_adam_step.  params: mean_logit, quat_raw, log_scale [n,4], sh [n,48];
    state: m / v dicts with the same keys; grads_act: mean_opac, quat, scale [n,4], sh [n,48] (w.r.t.
    the activated parameters); h: lr_* / beta1 / beta2 / eps / step; visible: optional bool [n]
    (rows with False untouched).  Returns (params, state, activated dict)."""
    n = params["mean_logit"].shape[0]
    rows = np.ones(n, bool) if visible is None else np.asarray(visible, bool)
    r_ml, r_q, r_s = raw_grads(params["mean_logit"], params["quat_raw"], params["log_scale"],
                               grads_act["mean_opac"], grads_act["quat"], grads_act["scale"])
    g = {"mean_logit": r_ml, "quat_raw": r_q, "log_scale": r_s, "sh": np.asarray(grads_act["sh"], np.float64)}
    lr_ml = np.empty((n, 4))
    lr_ml[:, :3] = h["lr_mean"]
    lr_ml[:, 3] = h["lr_opacity"]
    lrs = {"mean_logit": lr_ml, "quat_raw": np.full((n, 4), h["lr_quat"]),
           "log_scale": np.full((n, 4), h["lr_scale"]), "sh": sh_lr(n, h["lr_sh_dc"], h["lr_sh_rest"])}
    out_p, out_m, out_v = {}, {}, {}
    for k in ("mean_logit", "quat_raw", "log_scale", "sh"):
        p = np.asarray(params[k], np.float64).copy()
        m = np.asarray(state["m"][k], np.float64).copy()
        v = np.asarray(state["v"][k], np.float64).copy()
        gk = g[k]
        if k == "log_scale":
            gk = gk.copy()
            gk[:, 3] = 0.0
        pn, mn, vn = adam_update(p[rows], m[rows], v[rows], gk[rows], lrs[k][rows], h["beta1"], h["beta2"],
                                 h["eps"], h["step"])
        if k == "log_scale":  # the unused 4th lane (parameter and moments) stays as it was
            pn[:, 3], mn[:, 3], vn[:, 3] = p[rows, 3], m[rows, 3], v[rows, 3]
        p[rows], m[rows], v[rows] = pn, mn, vn
        out_p[k], out_m[k], out_v[k] = p, m, v
    mo, qa, sc = activate(out_p["mean_logit"], out_p["quat_raw"], out_p["log_scale"])
    return out_p, {"m": out_m, "v": out_v}, {"mean_opac": mo, "quat": qa, "scale": sc, "sh": out_p["sh"]}
