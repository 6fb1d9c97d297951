"""Pins of the NEXT-3 density-control oracle (oracle/densify.py) against SPEC's worked examples
(S:424-441), the 3DGS rules and the statistics the split sampler must have."""
import math

import numpy as np
from scipy import stats

from oracle import densify as DC

TAU, EXT, MINO, DIV = 2e-4, 0.05, 0.005, 1.6


def _shard(n, seed=0):
    rng = np.random.default_rng(seed)
    params = {"mean_logit": np.c_[rng.standard_normal((n, 3)), np.full(n, 2.0)],
              "quat_raw": rng.standard_normal((n, 4)),
              "log_scale": np.c_[np.log(np.full((n, 3), 0.01)), np.zeros(n)],
              "sh": rng.standard_normal((n, 48))}
    state = {m: {k: rng.standard_normal(v.shape) for k, v in params.items()} for m in ("m", "v")}
    return params, state, np.arange(n) % 3


def test_accumulate_spec_examples():
    lid = np.array([0, 0, 1])
    d = np.array([[0.1 / 500, 0.0], [0.3 / 500, 0.0], [0.2 / 500, 0.0]])  # W = 1000 -> NDC norms .1 .3 .2
    st, c = DC.accumulate(np.zeros(2), np.zeros(2), lid, d, 1000, 10)
    assert np.allclose(st, [0.4, 0.2]) and list(c) == [2, 1]           # phi = 1 -> sum, count 2
    st0, c0 = DC.accumulate(np.zeros(2), np.zeros(2), lid, d, 1000, 10, phi=np.array([0.0, 1.0]))
    assert st0[0] == 0.0 and c0[0] == 2                                 # phi = 0 never grows
    sth, _ = DC.accumulate(np.zeros(2), np.zeros(2), lid, d, 1000, 10, phi=np.array([0.5, 0.25]))
    assert np.allclose(sth, [0.5 * 0.4, 0.25 * 0.2])                    # scaled per Gaussian


def test_no_trigger_leaves_scene_unchanged():
    p, s, lod = _shard(20)
    out, st, ol, cnt = DC.apply(p, s, lod, np.zeros(20), np.ones(20), TAU, EXT, MINO, DIV, 1)
    assert cnt == dict(kept=20, clones=0, splits=0)
    for k in p:
        assert np.array_equal(out[k], p[k]) and np.array_equal(st["m"][k], s["m"][k])
    assert np.array_equal(ol, lod)


def test_clone_one_small_gaussian():
    p, s, lod = _shard(10)
    stat = np.zeros(10)
    stat[4] = 3 * TAU * 2
    count = np.full(10, 2)
    out, st, ol, cnt = DC.apply(p, s, lod, stat, count, TAU, EXT, MINO, DIV, 1)
    assert len(ol) == 11 and cnt["clones"] == 1                       # N + 1
    assert ol[10] == lod[4]                                           # heritage: clone keeps the level
    for k in p:
        assert np.array_equal(out[k][10], p[k][4]) and not st["m"][k][10].any()
        assert np.array_equal(out[k][:10], p[k])


def test_split_one_large_gaussian():
    p, s, lod = _shard(10)
    p["log_scale"][6, :3] = np.log([0.2, 0.1, 0.07])
    stat = np.zeros(10)
    stat[6] = 1.0
    out, st, ol, cnt = DC.apply(p, s, lod, stat, np.ones(10), TAU, EXT, MINO, DIV, 7)
    assert len(ol) == 11 and cnt["splits"] == 1                       # parent removed, 2 children
    assert list(ol[9:]) == [lod[6] + 1] * 2                           # heritage: split increments
    assert np.allclose(out["log_scale"][9:, :3], p["log_scale"][6, :3] - math.log(1.6))
    assert not np.array_equal(out["mean_logit"][9], out["mean_logit"][10])
    keep = [i for i in range(10) if i != 6]
    assert np.array_equal(out["sh"][:9], p["sh"][keep])


def test_split_heritage_clamped_at_finest_level():
    """SPEC apply_heritage examples: clone keeps l, split gives min(l + 1, K - 1), so
    (K - 1, split) -> K - 1 and every level stays in [0, K - 1]."""
    K = 6
    p, s, lod = _shard(4)
    lod[:] = [0, K - 1, K - 2, K - 1]
    p["log_scale"][[1, 2], :3] = np.log(0.5)                          # 1, 2 split; 3 clones
    stat = np.zeros(4)
    stat[1:] = 1.0
    out, _, ol, cnt = DC.apply(p, s, lod, stat, np.ones(4), TAU, EXT, MINO, DIV, 3, k_levels=K)
    assert cnt == dict(kept=2, clones=1, splits=2)
    # kept originals (0, 3), the clone of 3, first children (1, 2), second children (1, 2)
    assert list(ol) == [0, K - 1, K - 1, K - 1, K - 1, K - 1, K - 1]
    assert ol.max() <= K - 1


def test_prune_low_opacity_including_children():
    p, s, lod = _shard(6)
    p["mean_logit"][[1, 3], 3] = math.log(0.004 / 0.996)              # opacity 0.004 < 0.005
    p["log_scale"][3, :3] = np.log(0.5)
    stat = np.zeros(6)
    stat[3] = 1.0
    out, _, ol, cnt = DC.apply(p, s, lod, stat, np.ones(6), TAU, EXT, MINO, DIV, 1)
    assert len(ol) == 4 and cnt == dict(kept=4, clones=0, splits=0)


def test_normal_sampler_is_standard_normal():
    z = np.array([DC.normal01(3, g, c, a) for g in range(4000) for c in range(2) for a in range(3)])
    assert abs(z.mean()) < 0.02 and abs(z.var() - 1) < 0.03
    assert stats.kstest(z, "norm").pvalue > 1e-3


def test_split_children_follow_the_parent_covariance():
    """Children offsets mu_c - mu over many seeds have covariance R diag(s^2) R^T (the parent's
    Sigma): catches a transposed R, a wrong scale axis or a missing rotation."""
    p, s, lod = _shard(1, 4)
    p["log_scale"][0, :3] = np.log([0.3, 0.1, 0.05])
    q = p["quat_raw"][0] / np.linalg.norm(p["quat_raw"][0])
    R = DC.rotation(q)
    sig = R @ np.diag(np.array([0.3, 0.1, 0.05]) ** 2) @ R.T
    offs = []
    for seed in range(3000):
        out, _, _, _ = DC.apply(p, s, lod, np.ones(1), np.ones(1), TAU, EXT, MINO, DIV, seed)
        offs.append(out["mean_logit"][:, :3] - p["mean_logit"][0, :3])
    o = np.concatenate(offs)
    cov = o.T @ o / len(o)
    assert np.allclose(cov, sig, atol=0.06 * sig.max()), (cov, sig)
    assert np.allclose(R @ R.T, np.eye(3), atol=1e-12)
