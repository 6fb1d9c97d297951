"""CPU oracle of the scheduled simplification: the scoring report's phi,
the two pruning passes and the index-parity redistribution of the survivors.

TEST INFRASTRUCTURE ONLY (like oracle/__init__.py): imported by tests/ and nothing in the
product package.  Plain numpy, written from the paper's text; every decision that floating
point takes is taken here in the same IEEE fp64 operations the kernels use (R30-R33),
and every integer / index decision is exact.

  phi_i = c_vis_i / (c_rad_i + eps), eps = 1e-8             PAPER.md P:187; SPEC S:281 (R17)
  pass 1: "stochastic importance-weighted sampling without replacement: it draws a fixed
          fraction of the current set with sample probability proportional to s_i"
          -> exponential race: keep the top-k by log(u_i)/s_i                        S:303 (R30)
  pass 2: "a deterministic cumulative-mass cut that retains the smallest prefix of Gaussians
          whose summed score reaches a target fraction (we use 99%) of the total"
  "Each pass is followed by an index-parity redistribution that rebalances the survivors
   across shards"
"""
from __future__ import annotations

import numpy as np

EPS = 1e-8
SCORE_QUANTUM_BITS = 24  # R31: the mass cut decides on floor(s * 2^24), like w (D5)
_M64 = (1 << 64) - 1


def phi(c_rad: np.ndarray, c_vis: np.ndarray) -> np.ndarray:
    """phi_i = c^vis_i / (c^rad_i + eps) (fp64)."""
    return c_vis.astype(np.float64) / (c_rad.astype(np.float64) + EPS)


# ---- counter-based uniform generator (R30): u_i depends only on (seed, global id) -----------

def splitmix64(x: int) -> int:
    """One splitmix64 output for state x (Steele, Lea, Flood 2014), written out."""
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def uniform01(seed: int, gid: int) -> float:
    """u in (0, 1): the top 53 bits of splitmix64(seed ^ splitmix64(gid)), plus half a quantum."""
    x = splitmix64((seed ^ splitmix64(gid)) & _M64)
    return ((x >> 11) + 0.5) * (2.0 ** -53)


# ---- pinned natural logarithm (R30): IEEE fp64 operations in a fixed order ------------------

_LN2 = 0.6931471805599453
_SQRT2 = 1.4142135623730951
_SERIES = 12  # terms f^(2k+1)/(2k+1), k < 12: |f| <= 0.1716, f^24/25 < 1e-19


def ln_pinned(u: float) -> float:
    """ln(u) for u > 0 finite: u = m 2^e with m in [sqrt(2)/2, sqrt(2)) (exact split),
    ln(m) = 2 atanh(f), f = (m - 1)/(m + 1), by the odd series in Horner form; every step is
    one correctly rounded IEEE op, so the kernels reproduce it bit for bit."""
    m, e = np.frexp(np.float64(u))  # u = m 2^e, m in [0.5, 1): exact
    m = np.float64(m) * 2.0
    e = int(e) - 1
    if m > _SQRT2:
        m = m * 0.5  # exact
        e += 1
    f = (m - 1.0) / (m + 1.0)
    f2 = f * f
    p = np.float64(1.0) / np.float64(2 * (_SERIES - 1) + 1)
    for k in range(_SERIES - 2, -1, -1):
        p = p * f2 + np.float64(1.0) / np.float64(2 * k + 1)
    lm = (f + f) * p
    return float(np.float64(e) * _LN2 + lm)


def race_key(s: float, seed: int, gid: int) -> float:
    """key = log(u)/s for s > 0; -inf for s = 0 (drawn only after every positive score)."""
    if not s > 0.0:
        return float("-inf")
    return float(np.float64(ln_pinned(uniform01(seed, gid))) / np.float64(s))


def prune_stochastic(s: np.ndarray, gid: np.ndarray, keep_count: int, seed: int) -> np.ndarray:
    """Pass 1: keep the keep_count Gaussians with the largest race keys, ties
    by global id ascending (R30).  Returns a keep mask aligned with s."""
    n = len(s)
    keep = np.zeros(n, bool)
    k = max(0, min(int(keep_count), n))
    if k == 0:
        return keep
    keys = np.array([race_key(float(s[i]), seed, int(gid[i])) for i in range(n)], np.float64)
    order = np.lexsort((gid, -keys))  # key descending, then gid ascending
    keep[order[:k]] = True
    return keep


def score_quanta(s: np.ndarray) -> np.ndarray:
    """R31: q_i = floor(s_i 2^24) (exact in fp64 for s < 2^29), u64."""
    q = np.floor(np.where(s > 0, s, 0.0) * float(1 << SCORE_QUANTUM_BITS))
    return q.astype(np.uint64)


def prune_mass_cut(s: np.ndarray, gid: np.ndarray, num: int, den: int):
    """Pass 2: order by q desc, gid asc; keep the smallest prefix with
    den * sum(prefix q) >= num * sum(q) (exact integers).  num == den keeps every s > 0.
    All-zero scores keep only the first element (smallest gid) and report the warning.
    Returns (keep mask, all_zero)."""
    n = len(s)
    keep = np.zeros(n, bool)
    if n == 0:
        return keep, False
    if num == den:
        keep[:] = s > 0
        if keep.any():
            return keep, False
    q = score_quanta(s)
    total = int(sum(int(x) for x in q))
    order = np.lexsort((gid, -q.astype(np.float64)))  # q < 2^53: exact as float for the sort
    if total == 0:
        keep[order[0]] = True
        return keep, True
    target = num * total
    run = 0
    for j, i in enumerate(order):
        run += int(q[i])
        keep[i] = True
        if den * run >= target:
            break
    return keep, False


def redistribute(keep_by_gid: np.ndarray, M: int):
    """P:185 / P:170: survivors renumbered densely in global-id order (new gid = rank among the
    kept), then sharded by index parity: new rank = new gid mod M, new local = new gid // M.
    Returns new_gid (-1 for pruned) indexed by old gid."""
    new_gid = np.full(len(keep_by_gid), -1, np.int64)
    kept = np.nonzero(keep_by_gid)[0]
    new_gid[kept] = np.arange(len(kept))
    return new_gid
