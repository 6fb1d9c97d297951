"""Pins of the NEXT-3 optimizer oracle (oracle/optim.py): an independent Adam (torch.optim.Adam on
CPU, float64), finite differences of the activation chain rule, the first-step closed form."""
import numpy as np
import pytest

from oracle import optim as OP

torch = pytest.importorskip("torch")

H = dict(lr_mean=1.6e-4, lr_opacity=0.05, lr_quat=1e-3, lr_scale=5e-3, lr_sh_dc=2.5e-3, lr_sh_rest=1.25e-4,
         beta1=0.9, beta2=0.999, eps=1e-15)


def _rand(n=37, seed=0):
    rng = np.random.default_rng(seed)
    params = {"mean_logit": rng.standard_normal((n, 4)), "quat_raw": rng.standard_normal((n, 4)),
              "log_scale": np.c_[rng.uniform(-5, -1, (n, 3)), np.zeros(n)], "sh": rng.standard_normal((n, 48))}
    grads = {"mean_opac": rng.standard_normal((n, 4)), "quat": rng.standard_normal((n, 4)),
             "scale": np.c_[rng.standard_normal((n, 3)), np.zeros(n)], "sh": rng.standard_normal((n, 48))}
    return params, grads


def test_chain_rule_matches_finite_differences():
    params, _ = _rand(9, 1)
    rng = np.random.default_rng(2)
    W = [rng.standard_normal((9, 4)) for _ in range(3)]
    W[2][:, 3] = 0

    def f(ml, q, ls):
        mo, qa, sc = OP.activate(ml, q, ls)
        return float(np.sum(W[0] * mo) + np.sum(W[1] * qa) + np.sum(W[2] * sc))

    r = OP.raw_grads(params["mean_logit"], params["quat_raw"], params["log_scale"], *W)
    base = [params["mean_logit"], params["quat_raw"], params["log_scale"]]
    h = 1e-6
    for k in range(3):
        for i in range(9):
            for j in range(3 if k == 2 else 4):
                a = [b.copy() for b in base]
                c = [b.copy() for b in base]
                a[k][i, j] += h
                c[k][i, j] -= h
                fd = (f(*a) - f(*c)) / (2 * h)
                assert abs(fd - r[k][i, j]) < 1e-7 * max(1.0, abs(fd)), (k, i, j, fd, r[k][i, j])


@pytest.mark.parametrize("steps", [1, 3])
def test_adam_matches_torch(steps):
    params, grads = _rand()
    n = params["mean_logit"].shape[0]
    # torch: the same raw parameters, one param tensor per learning-rate group
    groups = {"mean": params["mean_logit"][:, :3], "opac": params["mean_logit"][:, 3:], "quat": params["quat_raw"],
              "scale": params["log_scale"][:, :3], "dc": params["sh"][:, :3], "rest": params["sh"][:, 3:]}
    lr = {"mean": H["lr_mean"], "opac": H["lr_opacity"], "quat": H["lr_quat"], "scale": H["lr_scale"],
          "dc": H["lr_sh_dc"], "rest": H["lr_sh_rest"]}
    tp = {k: torch.tensor(v.copy(), dtype=torch.float64, requires_grad=True) for k, v in groups.items()}
    opt = torch.optim.Adam([{"params": [tp[k]], "lr": lr[k]} for k in tp], betas=(H["beta1"], H["beta2"]),
                           eps=H["eps"])
    state = {"m": {k: np.zeros_like(v) for k, v in params.items()},
             "v": {k: np.zeros_like(v) for k, v in params.items()}}
    p = params
    for t in range(1, steps + 1):
        # gradients w.r.t. the activated parameters -> raw, for both sides at the current point
        r_ml, r_q, r_s = OP.raw_grads(p["mean_logit"], p["quat_raw"], p["log_scale"], grads["mean_opac"],
                                      grads["quat"], grads["scale"])
        rg = {"mean": r_ml[:, :3], "opac": r_ml[:, 3:], "quat": r_q, "scale": r_s[:, :3], "dc": grads["sh"][:, :3],
              "rest": grads["sh"][:, 3:]}
        for k in tp:
            tp[k].grad = torch.tensor(rg[k], dtype=torch.float64)
        opt.step()
        p, state, act = OP.adam_step(p, state, grads, dict(H, step=t))
    got = {"mean": p["mean_logit"][:, :3], "opac": p["mean_logit"][:, 3:], "quat": p["quat_raw"],
           "scale": p["log_scale"][:, :3], "dc": p["sh"][:, :3], "rest": p["sh"][:, 3:]}
    for k in tp:
        assert np.allclose(got[k], tp[k].detach().numpy(), rtol=1e-12, atol=1e-15), k
    assert np.array_equal(p["log_scale"][:, 3], params["log_scale"][:, 3])
    assert np.allclose(act["scale"][:, :3], np.exp(p["log_scale"][:, :3]))
    assert np.allclose(np.linalg.norm(act["quat"], axis=1), 1.0)
    assert n == 37


def test_first_step_closed_form_and_visibility():
    """t = 1, eps = 0: m_hat = g, v_hat = g^2, so every element moves by exactly -lr sign(g);
    rows outside the visible mask are untouched."""
    params, grads = _rand(8, 3)
    h = dict(H, eps=0.0, step=1)
    vis = np.array([1, 0, 1, 1, 0, 1, 1, 1], bool)
    state = {"m": {k: np.zeros_like(v) for k, v in params.items()},
             "v": {k: np.zeros_like(v) for k, v in params.items()}}
    p, st, _ = OP.adam_step(params, state, grads, h, visible=vis)
    d = p["sh"] - params["sh"]
    g = grads["sh"]
    assert np.allclose(d[vis][:, :3], -h["lr_sh_dc"] * np.sign(g[vis][:, :3]), rtol=1e-12)
    assert np.allclose(d[vis][:, 3:], -h["lr_sh_rest"] * np.sign(g[vis][:, 3:]), rtol=1e-12)
    for k in p:
        assert np.array_equal(p[k][~vis], params[k][~vis]) and not st["m"][k][~vis].any()
