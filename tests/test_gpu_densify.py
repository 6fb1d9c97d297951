"""NEXT-3 density control through the C ABI vs oracle/densify.py.

Statistic: the CUDA view's phi-weighted |dL/dmean2d| (fp32, from the compositing partials) vs the
oracle's fp64 dL/dmean2d of the same view: within 1e-3 relative + 1e-5 of the largest (the
gradient tolerance of north_star), counts exact, at world 1 and 2, with and without phi.
Apply: decisions, counts, output order, levels, copied rows and moments bit-exact; split
children's means within 1e-6 |mu| + 1e-5 s (fp32 rotation of an fp64 normal), their log-scales
within 1e-6; activated planes within 2e-6 relative.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
import synthetic as S  # noqa: E402
from gpu_helpers import GpuStep  # noqa: E402
from oracle import densify as DC  # noqa: E402
from oracle import optim as OP  # noqa: E402

pytestmark = pytest.mark.gpu
TAU, EXT, MINO, DIV, SEED = 2e-4, 0.05, 0.005, 1.6, 77


@pytest.mark.parametrize("M,use_phi", [(1, False), (1, True), (2, True)])
def test_statistic_parity(tiny_scene, M, use_phi):
    cam = tiny_scene.cameras[0]
    dl = S.grad_image(cam["H"], cam["W"])
    phi = np.random.default_rng(3).random(tiny_scene.n) if use_phi else None
    gs = GpuStep(tiny_scene, cam, M=M, dLdC=dl, densify=True, phi=phi)
    st = O.OracleStep(tiny_scene, cam, M=1, dLdC=dl)
    try:
        vis = np.flatnonzero(gs.radius > 0)
        g2d = st.get("g2d").reshape(-1, 9)
        ref, cnt = DC.accumulate(np.zeros(tiny_scene.n), np.zeros(tiny_scene.n), vis, g2d[vis, :2], cam["W"],
                                 cam["H"], phi)
        assert np.array_equal(gs.dc_count, cnt)
        tol = 1e-3 * np.abs(ref) + 1e-5 * np.abs(ref).max()
        assert np.all(np.abs(gs.dc_stat - ref) <= tol), float(np.max(np.abs(gs.dc_stat - ref) - tol))
        assert ref.max() > 0
    finally:
        gs.close()


def _shard(n, seed):
    rng = np.random.default_rng(seed)
    f = np.float32
    logit = rng.normal(0, 3, n)
    logit[rng.random(n) < 0.1] = -8.0                     # some below opacity 0.005 (logit -5.29)
    ls = np.log(np.where(rng.random((n, 1)) < 0.5, rng.uniform(0.005, 0.04, (n, 3)), rng.uniform(0.06, 0.5, (n, 3))))
    params = {"mean_logit": np.c_[rng.uniform(-10, 10, (n, 3)), logit].astype(f),
              "quat_raw": rng.standard_normal((n, 4)).astype(f),
              "log_scale": np.c_[ls, np.zeros(n)].astype(f), "sh": rng.standard_normal((n, 48)).astype(f)}
    state = {m: {k: rng.standard_normal(v.shape).astype(f) for k, v in params.items()} for m in ("m", "v")}
    lod = rng.integers(0, 6, n).astype(np.uint8)
    count = rng.integers(0, 6, n).astype(np.int32)
    stat = (rng.exponential(TAU, n) * np.maximum(count, 1)).astype(f)
    return params, state, lod, stat, count


@pytest.mark.parametrize("world,rank", [(1, 0), (2, 1)])
def test_apply_parity(world, rank):
    import paper_2605_13794_b200.bgs as B
    n = 5003
    params, state, lod, stat, count = _shard(n, 11 + rank)
    dev = "cuda"
    keys = ("mean_logit", "quat_raw", "log_scale", "sh")
    tin = B.TrainParams(*(torch.from_numpy(params[k]).to(dev) for k in keys))
    for j, k in enumerate(keys):
        tin.m[j].copy_(torch.from_numpy(state["m"][k]))
        tin.v[j].copy_(torch.from_numpy(state["v"][k]))
    cap = 3 * n
    tout = B.TrainParams(*(torch.full((cap, c), np.nan, device=dev) for c in (4, 4, 4, 48)))
    lod_out = torch.full((cap,), 255, dtype=torch.uint8, device=dev)
    act = B.GaussianPlanes(torch.zeros(cap, 4, device=dev), torch.zeros(cap, 4, device=dev),
                           torch.zeros(cap, 4, device=dev), tout.sh, lod_out)
    ctxs = B.Context.local_group(world, 0) if world > 1 else [B.Context(0, 1, 0)]
    try:
        nn = B.bgs_densify_apply(ctxs[rank], tin, torch.from_numpy(lod).to(dev), torch.from_numpy(stat).to(dev),
                                 torch.from_numpy(count).to(dev), B.densify_params(TAU, EXT, MINO, DIV, SEED, k_levels=6),
                                 tout, lod_out, act)
        torch.cuda.synchronize()
        ref, rst, rlod, cnt = DC.apply(params, state, lod, stat, count, TAU, EXT, MINO, DIV, SEED, rank, world,
                                       k_levels=6)
        assert cnt["kept"] > 0 and cnt["clones"] > 0 and cnt["splits"] > 0
        # heritage rule at the ceiling: a split of a level-(K-1) parent stays at K-1
        assert rlod.max() == 5 and (rlod[cnt["kept"] + cnt["clones"]:] == 5).any()
        assert nn == len(rlod)
        assert np.array_equal(lod_out.cpu().numpy()[:nn], rlod)
        K, Cn = cnt["kept"], cnt["clones"]
        copied = slice(0, K + Cn)
        kids = slice(K + Cn, nn)
        for j, k in enumerate(keys):
            got = getattr(tout, k).cpu().numpy()[:nn]
            assert np.array_equal(got[copied], ref[k][copied].astype(np.float32)), k
            for mom, arr in (("m", tout.m[j]), ("v", tout.v[j])):
                gm = arr.cpu().numpy()[:nn]
                assert np.array_equal(gm, rst[mom][k].astype(np.float32)), (k, mom)
            g, r = got[kids].astype(np.float64), ref[k][kids]
            if k == "mean_logit":
                s = np.exp(params["log_scale"][:, :3].astype(np.float64)).max()
                assert np.all(np.abs(g[:, :3] - r[:, :3]) <= 1e-6 * np.abs(r[:, :3]) + 1e-5 * s)
                assert np.array_equal(g[:, 3], r[:, 3].astype(np.float32))
            elif k == "log_scale":
                assert np.all(np.abs(g - r) <= 1e-6)
            else:
                assert np.array_equal(g, r.astype(np.float32)), k
        mo, qa, sc = OP.activate(ref["mean_logit"], ref["quat_raw"], ref["log_scale"])
        for got, want in ((act.mean_opac, mo), (act.quat, qa), (act.scale, sc)):
            g = got.cpu().numpy()[:nn].astype(np.float64)
            assert np.allclose(g, want, rtol=2e-6, atol=1e-6)
    finally:
        for c in ctxs:
            c.close()


def test_apply_capacity_and_empty():
    import paper_2605_13794_b200.bgs as B
    n = 300
    params, state, lod, stat, count = _shard(n, 5)
    stat[:] = 1.0  # everything densifies
    dev = "cuda"
    keys = ("mean_logit", "quat_raw", "log_scale", "sh")
    tin = B.TrainParams(*(torch.from_numpy(params[k]).to(dev) for k in keys))
    tout = B.TrainParams(*(torch.zeros(n, c, device=dev) for c in (4, 4, 4, 48)))  # too small
    ctx = B.Context(0, 1, 0)
    try:
        with pytest.raises(B.BgsError) as e:
            B.bgs_densify_apply(ctx, tin, torch.from_numpy(lod).to(dev), torch.from_numpy(stat).to(dev),
                                torch.from_numpy(count).to(dev), B.densify_params(TAU, EXT, MINO, DIV, SEED), tout,
                                torch.zeros(n, dtype=torch.uint8, device=dev), None)
        assert "CAPACITY" in str(e.value)
        assert math.isfinite(float(tout.mean_logit.sum().item()))
    finally:
        ctx.close()


def test_apply_full_size_sampled():
    """A 2M-row shard: category totals exact (oracle decisions over every row), and 3000 sampled
    kept originals / clones / children at their oracle positions (kept: rank among kept; clones:
    K + rank among clones; children: K + C + c S + rank among split parents)."""
    import paper_2605_13794_b200.bgs as B
    n = 2_000_003
    params, state, lod, stat, count = _shard(n, 99)
    dev = "cuda"
    keys = ("mean_logit", "quat_raw", "log_scale", "sh")
    tin = B.TrainParams(*(torch.from_numpy(params[k]).to(dev) for k in keys))
    for j, k in enumerate(keys):
        tin.m[j].copy_(torch.from_numpy(state["m"][k]))
        tin.v[j].copy_(torch.from_numpy(state["v"][k]))
    cap = 2 * n + 1
    tout = B.TrainParams(*(torch.empty(cap, c, device=dev) for c in (4, 4, 4, 48)))
    lod_out = torch.empty(cap, dtype=torch.uint8, device=dev)
    ctx = B.Context(0, 1, 0)
    try:
        nn = B.bgs_densify_apply(ctx, tin, torch.from_numpy(lod).to(dev), torch.from_numpy(stat).to(dev),
                                 torch.from_numpy(count).to(dev), B.densify_params(TAU, EXT, MINO, DIV, SEED), tout,
                                 lod_out, None)
        torch.cuda.synchronize()
        keep, clone, split = DC.decide(params, stat, count, TAU, EXT, MINO)
        K, Cn, Sn = int(keep.sum()), int(clone.sum()), int(split.sum())
        assert nn == K + Cn + 2 * Sn and Cn > 0 and Sn > 0
        rng = np.random.default_rng(4)
        ck = np.cumsum(keep) - 1
        cc = np.cumsum(clone) - 1
        cs = np.cumsum(split) - 1
        ml_out = tout.mean_logit
        for cat, mask, pos in (("keep", keep, lambda i: ck[i]), ("clone", clone, lambda i: K + cc[i])):
            for i in rng.choice(np.flatnonzero(mask), 1000, replace=False):
                got = ml_out[int(pos(i))].cpu().numpy()
                assert np.array_equal(got, params["mean_logit"][i]), (cat, i)
                assert int(lod_out[int(pos(i))].item()) == int(lod[i]), (cat, i)
        for i in rng.choice(np.flatnonzero(split), 500, replace=False):
            for c in range(2):
                q = K + Cn + c * Sn + int(cs[i])
                got = ml_out[q].double().cpu().numpy()
                # child c of parent gid i: mu + R(q) (s z) with the oracle's sampler
                qr = params["quat_raw"][i].astype(np.float64)
                R = DC.rotation(qr / np.linalg.norm(qr))
                s = np.exp(params["log_scale"][i, :3].astype(np.float64))
                z = np.array([DC.normal01(SEED, int(i), c, a) for a in range(3)])
                want = params["mean_logit"][i, :3].astype(np.float64) + R @ (s * z)
                assert np.all(np.abs(got[:3] - want) <= 1e-6 * np.abs(want) + 1e-5 * s.max()), (i, c)
                assert int(lod_out[q].item()) == min(255, int(lod[i]) + 1)
    finally:
        ctx.close()
