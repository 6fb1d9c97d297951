"""NEXT-3 density-control oracle: the phi-reweighted statistic and clone / split / prune with the
LOD heritage rule, plain numpy (TEST INFRASTRUCTURE ONLY; shares no code with csrc/densify.cu).

Definitions followed (readings R37, R39, R40):
  statistic: stat_i += phi_i * |(dL/dmx * W/2, dL/dmy * H/2)|, count_i += 1 for
    every Gaussian the view projected (radius > 0); phi = 1 without a report.
  apply (3DGS adaptive density control; heritage P:194): avg = stat / max(1, count) (fp32);
    densify avg >= tau; split when max_j s_ij > dense_extent, else clone; prune opacity <
    min_opacity (parents and children: children copy the opacity).  Decisions in fp32 on
    l < logit(m) and max log s > log(e) (thresholds rounded once from double).
  order: kept originals (input order), clones (parent order), first children, second children.
  clone = copy (level kept); split child = mu + R(q) (s * z), log s - log(split_div), level + 1,
    z ~ N(0, I) by Box-Muller on the (seed, key) uniforms of oracle/simplify.py (R30 generator),
    key = 2k and 2k + 1, k = 8 gid + 3 child + axis.  Adam moments kept for originals, zero for
    new rows.
Pins: tests/test_oracle_densify.py.
"""
from __future__ import annotations

import math

import numpy as np

from oracle.simplify import uniform01


def normal01(seed: int, gid: int, child: int, axis: int) -> float:
    """Box-Muller standard normal of (seed, gid, child, axis)."""
    k = gid * 8 + 3 * child + axis
    u1 = uniform01(seed, 2 * k)
    u2 = uniform01(seed, 2 * k + 1)
    return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)


def accumulate(stat, count, lidx, dmean2d, W: int, H: int, phi=None):
    """stat (f64 copy) += phi * |dL/dmean2d in NDC| and count += 1 over the view's records."""
    stat = np.asarray(stat, np.float64).copy()
    count = np.asarray(count, np.int64).copy()
    d = np.asarray(dmean2d, np.float64)
    norm = np.sqrt((d[:, 0] * (W / 2.0)) ** 2 + (d[:, 1] * (H / 2.0)) ** 2)
    w = np.ones(len(lidx)) if phi is None else np.asarray(phi, np.float64)[lidx]
    np.add.at(stat, lidx, w * norm)
    np.add.at(count, lidx, 1)
    return stat, count


def rotation(q):
    """R(q) of a unit quaternion (w, x, y, z)."""
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def decide(params: dict, stat, count, tau: float, dense_extent: float, min_opacity: float):
    """Per row (keep, clone, split) booleans, decisions in fp32 (R39)."""
    f = np.float32
    logit = np.asarray(params["mean_logit"], np.float32)[:, 3]
    ls = np.asarray(params["log_scale"], np.float32)[:, :3]
    logit_min = f(math.log(min_opacity / (1.0 - min_opacity)))
    log_ext = f(math.log(dense_extent))
    alive = ~(logit < logit_min)
    c = np.maximum(np.asarray(count, np.int64), 1).astype(np.float32)
    avg = (np.asarray(stat, np.float32) / c).astype(np.float32)
    dens = avg >= f(tau)
    big = ls.max(axis=1) > log_ext
    return alive & ~(dens & big), alive & dens & ~big, alive & dens & big


def apply(params: dict, state: dict, lod, stat, count, tau, dense_extent, min_opacity, split_div, seed,
          rank: int = 0, world: int = 1, k_levels: int = 256):
    """New (params, state, lod) of the shard; params / state keyed like oracle/optim.py.
    Heritage rule (SPEC apply_heritage): a clone keeps the parent's level, a split
    child gets min(l + 1, K - 1) so every level stays in [0, K - 1]."""
    keep, clone, split = decide(params, stat, count, tau, dense_extent, min_opacity)
    keys = ("mean_logit", "quat_raw", "log_scale", "sh")
    P = {k: np.asarray(params[k], np.float64) for k in keys}
    Sm = {k: np.asarray(state["m"][k], np.float64) for k in keys}
    Sv = {k: np.asarray(state["v"][k], np.float64) for k in keys}
    lod = np.asarray(lod, np.int64)
    out = {k: [] for k in keys}
    om = {k: [] for k in keys}
    ov = {k: [] for k in keys}
    olod = []

    def emit(i, fresh, **over):
        for k in keys:
            out[k].append(over.get(k, P[k][i]))
            om[k].append(np.zeros_like(P[k][i]) if fresh else Sm[k][i])
            ov[k].append(np.zeros_like(P[k][i]) if fresh else Sv[k][i])
        olod.append(min(k_levels - 1, lod[i] + over.get("dlod", 0)))

    for i in np.flatnonzero(keep):
        emit(i, False)
    for i in np.flatnonzero(clone):
        emit(i, True)
    sp = np.flatnonzero(split)
    for c in range(2):
        for i in sp:
            q = P["quat_raw"][i]
            R = rotation(q / np.linalg.norm(q))
            s = np.exp(P["log_scale"][i, :3])
            gid = int(i) * world + rank
            z = np.array([normal01(seed, gid, c, a) for a in range(3)])
            ml = P["mean_logit"][i].copy()
            ml[:3] = ml[:3] + R @ (s * z)
            ls = P["log_scale"][i].copy()
            ls[:3] = ls[:3] - math.log(split_div)
            emit(i, True, mean_logit=ml, log_scale=ls, dlod=1)
    n = len(olod)
    res = {k: (np.array(out[k]) if n else np.zeros((0,) + P[k].shape[1:])) for k in keys}
    st = {"m": {k: (np.array(om[k]) if n else np.zeros((0,) + P[k].shape[1:])) for k in keys},
          "v": {k: (np.array(ov[k]) if n else np.zeros((0,) + P[k].shape[1:])) for k in keys}}
    return res, st, np.array(olod, np.int64), dict(kept=int(keep.sum()), clones=int(clone.sum()),
                                                   splits=int(split.sum()))
