"""NEXT-3 fused Adam (bgs_adam_step) through the C ABI vs oracle/optim.py (fp64) on the same seeded
raw parameters and activated-parameter gradients, three steps, with and without a visibility mask.

Tolerances (fp32 kernel, fp64 oracle): raw parameters |d| <= 1e-6 |p| + 1e-3 lr (the update of one
step is ~lr; fp32 rounding of m/sqrt(v) ~1e-6 relative, of p ~6e-8 |p|), moments within 1e-5
relative + 1e-6 of the plane's largest (m = b1 m + (1 - b1) g cancels near 0), activated planes within 2e-6 relative (fast-math exp in the sigmoid / exp).
Rows outside the mask, and the unused 4th lane of the scale plane, are bit-identical to their
input; gradients of updated rows are zeroed.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import optim as OP  # noqa: E402

pytestmark = pytest.mark.gpu
H = dict(lr_mean=1.6e-4, lr_opacity=0.05, lr_quat=1e-3, lr_scale=5e-3, lr_sh_dc=2.5e-3, lr_sh_rest=1.25e-4,
         beta1=0.9, beta2=0.999, eps=1e-15)


def _inputs(n, seed):
    rng = np.random.default_rng(seed)
    f = np.float32
    params = {"mean_logit": rng.standard_normal((n, 4)).astype(f), "quat_raw": rng.standard_normal((n, 4)).astype(f),
              "log_scale": np.c_[rng.uniform(-5, -1, (n, 3)), rng.standard_normal(n)].astype(f),
              "sh": rng.standard_normal((n, 48)).astype(f)}
    grads = [{"mean_opac": rng.standard_normal((n, 4)).astype(f), "quat": rng.standard_normal((n, 4)).astype(f),
              "scale": np.c_[rng.standard_normal((n, 3)), np.zeros(n)].astype(f),
              "sh": rng.standard_normal((n, 48)).astype(f)} for _ in range(3)]
    return params, grads


@pytest.mark.parametrize("masked", [False, True])
def test_adam_parity(masked):
    import paper_2605_13794_b200.bgs as B
    import synthetic as S
    n = 10007
    params, grads = _inputs(n, 5 + masked)
    vis = np.random.default_rng(9).random(n) < 0.6 if masked else None
    dev = "cuda"
    tp = B.TrainParams(*(torch.from_numpy(params[k]).to(dev) for k in ("mean_logit", "quat_raw", "log_scale", "sh")))
    act = B.GaussianPlanes(torch.zeros(n, 4, device=dev), torch.zeros(n, 4, device=dev), torch.zeros(n, 4, device=dev),
                           tp.sh, torch.zeros(n, dtype=torch.uint8, device=dev))
    gp = B.GradPlanes(*(torch.zeros(n, c, device=dev) for c in (4, 4, 4, 48)))
    vis_dev = None if vis is None else torch.from_numpy(S.pack_bits(vis).astype(np.int32)).to(dev)
    ctx = B.Context(0, 1, 0)
    p = {k: v.astype(np.float64) for k, v in params.items()}
    st = {"m": {k: np.zeros_like(v) for k, v in p.items()}, "v": {k: np.zeros_like(v) for k, v in p.items()}}
    try:
        for t in range(1, 4):
            g = grads[t - 1]
            for k, name in (("mean_opac", "mean_opac"), ("quat", "quat"), ("scale", "scale"), ("sh", "sh")):
                getattr(gp, name).copy_(torch.from_numpy(g[k]))
            B.bgs_adam_step(ctx, tp, gp, act, vis_dev, B.adam_hparams(**H, step=t))
            torch.cuda.synchronize()
            p, st, a = OP.adam_step(p, st, g, dict(H, step=t), visible=vis)
            rows = np.ones(n, bool) if vis is None else vis
            for k, name in (("mean_opac", "mean_opac"), ("quat", "quat"), ("scale", "scale"), ("sh", "sh")):
                gg = getattr(gp, name).cpu().numpy()
                assert not gg[rows].any(), k                      # zeroed
                assert np.array_equal(gg[~rows], g[k][~rows]), k  # untouched
        lr_of = {"mean_logit": np.r_[[H["lr_mean"]] * 3, H["lr_opacity"]], "quat_raw": H["lr_quat"],
                 "log_scale": H["lr_scale"], "sh": OP.sh_lr(n, H["lr_sh_dc"], H["lr_sh_rest"])}
        for k, t_ in (("mean_logit", tp.mean_logit), ("quat_raw", tp.quat_raw), ("log_scale", tp.log_scale),
                      ("sh", tp.sh)):
            got = t_.cpu().numpy().astype(np.float64)
            assert np.all(np.abs(got - p[k]) <= 1e-6 * np.abs(p[k]) + 1e-3 * lr_of[k]), k
            if vis is not None:
                assert np.array_equal(t_.cpu().numpy()[~vis], params[k][~vis]), k
            j = ["mean_logit", "quat_raw", "log_scale", "sh"].index(k)
            for mom in ("m", "v"):
                gm = (tp.m if mom == "m" else tp.v)[j].cpu().numpy().astype(np.float64)
                assert np.all(np.abs(gm - st[mom][k]) <= 1e-5 * np.abs(st[mom][k]) + 1e-6 * np.abs(st[mom][k]).max()), (k, mom)
        assert np.array_equal(tp.log_scale.cpu().numpy()[:, 3], params["log_scale"][:, 3])
        rows = np.ones(n, bool) if vis is None else vis
        for k, t_ in (("mean_opac", act.mean_opac), ("quat", act.quat), ("scale", act.scale)):
            got = t_.cpu().numpy().astype(np.float64)[rows]
            assert np.allclose(got, a[k][rows], rtol=2e-6, atol=1e-7), k
    finally:
        ctx.close()


def test_adam_edge_cases():
    """Empty shard is a no-op; step 0 and betas outside [0, 1) are refused; a too-small act is refused."""
    import paper_2605_13794_b200.bgs as B
    dev = "cuda"
    ctx = B.Context(0, 1, 0)
    try:
        e = B.TrainParams(*(torch.zeros(0, c, device=dev) for c in (4, 4, 4, 48)))
        act0 = B.GaussianPlanes(*(torch.zeros(0, c, device=dev) for c in (4, 4, 4, 48)),
                                torch.zeros(0, dtype=torch.uint8, device=dev))
        g0 = B.GradPlanes(*(torch.zeros(0, c, device=dev) for c in (4, 4, 4, 48)))
        B.bgs_adam_step(ctx, e, g0, act0, None, B.adam_hparams(step=1))
        n = 5
        p = B.TrainParams(*(torch.ones(n, c, device=dev) for c in (4, 4, 4, 48)))
        g = B.GradPlanes(*(torch.ones(n, c, device=dev) for c in (4, 4, 4, 48)))
        small = B.GaussianPlanes(*(torch.zeros(n - 1, c, device=dev) for c in (4, 4, 4, 48)),
                                 torch.zeros(n - 1, dtype=torch.uint8, device=dev))
        for h, what in ((B.adam_hparams(step=0), "step"), (B.adam_hparams(beta1=1.0), "betas")):
            with pytest.raises(B.BgsError) as err:
                B.bgs_adam_step(ctx, p, g, small, None, h)
            assert "INVALID" in str(err.value), what
        with pytest.raises(B.BgsError) as err:
            B.bgs_adam_step(ctx, p, g, small, None, B.adam_hparams(step=1))
        assert "CAPACITY" in str(err.value)
        assert float(p.mean_logit.sum().item()) == 4.0 * n  # nothing written on refusal
    finally:
        ctx.close()


def test_adam_full_size_sampled():
    """The Rubble shard size (6M rows), three steps; 20000 sampled rows against the oracle."""
    import paper_2605_13794_b200.bgs as B
    n = 6_000_000
    gen = torch.Generator(device="cuda").manual_seed(3)
    dev = "cuda"

    def rnd(*shape):
        return torch.randn(*shape, device=dev, generator=gen)

    tp = B.TrainParams(rnd(n, 4), rnd(n, 4), torch.cat([rnd(n, 3) * 0.5 - 3.0, torch.zeros(n, 1, device=dev)], 1),
                       rnd(n, 48))
    idx = torch.randperm(n, generator=torch.Generator().manual_seed(5))[:20000].sort().values
    p = {k: getattr(tp, k)[idx.to(dev)].double().cpu().numpy() for k in ("mean_logit", "quat_raw", "log_scale", "sh")}
    st = {"m": {k: np.zeros_like(v) for k, v in p.items()}, "v": {k: np.zeros_like(v) for k, v in p.items()}}
    act = B.GaussianPlanes(torch.zeros(n, 4, device=dev), torch.zeros(n, 4, device=dev), torch.zeros(n, 4, device=dev),
                           tp.sh, torch.zeros(n, dtype=torch.uint8, device=dev))
    gp = B.GradPlanes(*(torch.zeros(n, c, device=dev) for c in (4, 4, 4, 48)))
    ctx = B.Context(0, 1, 0)
    try:
        for t in range(1, 4):
            g = {"mean_opac": rnd(n, 4), "quat": rnd(n, 4), "scale": torch.cat([rnd(n, 3), torch.zeros(n, 1, device=dev)], 1),
                 "sh": rnd(n, 48)}
            gs = {k: v[idx.to(dev)].double().cpu().numpy() for k, v in g.items()}
            for k in ("mean_opac", "quat", "scale", "sh"):
                getattr(gp, k).copy_(g[k])
            B.bgs_adam_step(ctx, tp, gp, act, None, B.adam_hparams(**H, step=t))
            torch.cuda.synchronize()
            p, st, a = OP.adam_step(p, st, gs, dict(H, step=t))
        lr_of = {"mean_logit": np.r_[[H["lr_mean"]] * 3, H["lr_opacity"]], "quat_raw": H["lr_quat"],
                 "log_scale": H["lr_scale"], "sh": OP.sh_lr(len(idx), H["lr_sh_dc"], H["lr_sh_rest"])}
        for k in ("mean_logit", "quat_raw", "log_scale", "sh"):
            got = getattr(tp, k)[idx.to(dev)].double().cpu().numpy()
            assert np.all(np.abs(got - p[k]) <= 1e-6 * np.abs(p[k]) + 1e-3 * lr_of[k]), k
        got = act.mean_opac[idx.to(dev)].double().cpu().numpy()
        assert np.allclose(got, a["mean_opac"], rtol=2e-6, atol=1e-7)
    finally:
        ctx.close()
