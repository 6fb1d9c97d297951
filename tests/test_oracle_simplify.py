"""Pins of oracle/simplify.py (NEXT-1: phi, pass-1 stochastic prune, pass-2 mass cut,
index-parity redistribution) against what the paper / SPEC fix and against mathematics,
independent of the oracle's own arithmetic.  CPU only."""
from __future__ import annotations

import math

import numpy as np

from oracle import simplify as SO


# ---- phi --------------------------------------------------------

def test_phi_examples():
    # single view, single splat visible and contributing: phi = 1/(1+eps)  [SPEC S:296]
    assert SO.phi(np.array([1]), np.array([1]))[0] == 1.0 / (1.0 + 1e-8)
    # visible in no view: phi = 0  [SPEC S:295]
    assert SO.phi(np.array([0]), np.array([0]))[0] == 0.0
    # c_vis <= c_rad -> phi in [0, 1)
    rng = np.random.default_rng(0)
    cr = rng.integers(0, 64, 1000)
    cv = (cr * rng.random(1000)).astype(np.int64)
    p = SO.phi(cr, cv)
    assert np.all(p >= 0) and np.all(p < 1.0)


# ---- the generator and the pinned logarithm (R30) ----------------------------------------------

def test_splitmix64_reference_value():
    # first output of splitmix64 from state 0 (published test vector of the algorithm)
    assert SO.splitmix64(0) == 0xE220A8397B1DCDAF


def test_uniform01_is_uniform_and_open():
    u = np.array([SO.uniform01(123, g) for g in range(40000)])
    assert u.min() > 0.0 and u.max() < 1.0
    assert abs(u.mean() - 0.5) < 0.005
    counts, _ = np.histogram(u, bins=20, range=(0, 1))
    chi2 = float(((counts - 2000.0) ** 2 / 2000.0).sum())
    assert chi2 < 45.0  # 19 dof: p ~ 1e-3
    # different seeds give different streams
    assert SO.uniform01(1, 7) != SO.uniform01(2, 7)


def test_ln_pinned_against_library_and_closed_forms():
    rng = np.random.default_rng(1)
    us = list(rng.random(20000)) + [2.0 ** -k for k in range(1, 60)] + [1.0 - 2.0 ** -k for k in range(1, 53)]
    us += [math.sqrt(2) / 2, math.sqrt(2) / 2 * (1 + 2 ** -52), 0.5 * (1 + 1e-9), 2.0 ** -53 * 0.5]
    for u in us:
        if u <= 0:
            continue
        got, ref = SO.ln_pinned(u), math.log(u)
        assert abs(got - ref) <= 2e-15 * abs(ref) + 1e-300, (u, got, ref)  # ~10 ulp
    assert SO.ln_pinned(1.0) == 0.0
    for k in range(1, 40):  # ln(2^-k) = -k ln 2: f = 0, only the exponent term
        assert SO.ln_pinned(2.0 ** -k) == -k * SO._LN2


# ---- pass 1: stochastic prune -------------------------------------------

def test_prune_stochastic_spec_examples():
    s = np.array([0.3, 1.2, 0.0, 4.0])
    gid = np.arange(4)
    assert SO.prune_stochastic(s, gid, 4, seed=5).all()  # keep_fraction = 1: identity  [S:303]
    for seed in range(50):  # scores (1, 0, 0), keep 1: the score-1 Gaussian always survives [S:304]
        assert SO.prune_stochastic(np.array([1.0, 0.0, 0.0]), np.arange(3), 1, seed).tolist() == [True, False, False]


def test_prune_stochastic_sampling_law():
    # scores (10, 1), keep 1 over 10,000 seeded trials: first survives with frequency 10/11 +- 0.02 [S:305]
    s = np.array([10.0, 1.0])
    hits = sum(SO.prune_stochastic(s, np.arange(2), 1, seed)[0] for seed in range(10000))
    assert abs(hits / 10000 - 10 / 11) < 0.02
    # single draw from 4: inclusion probability proportional to s (without-replacement law, k = 1)
    s = np.array([1.0, 2.0, 3.0, 4.0])
    cnt = np.zeros(4)
    for seed in range(20000):
        cnt += SO.prune_stochastic(s, np.arange(4), 1, seed)
    assert np.all(np.abs(cnt / 20000 - s / s.sum()) < 0.015)
    # k = 2 of (1, 1, 2): P(item 2 kept) = 1 - P(it is drawn neither first nor second)
    #   = 1 - (1/4)(1/3)*2 = 5/6 under successive sampling proportional to s
    s = np.array([1.0, 1.0, 2.0])
    kept2 = sum(SO.prune_stochastic(s, np.arange(3), 2, seed)[2] for seed in range(12000))
    assert abs(kept2 / 12000 - 5 / 6) < 0.015


def test_prune_stochastic_zero_scores_only_after_positives():
    rng = np.random.default_rng(3)
    s = np.where(rng.random(500) < 0.3, 0.0, rng.random(500))
    npos = int((s > 0).sum())
    keep = SO.prune_stochastic(s, np.arange(500), npos + 7, seed=9)
    assert keep[s > 0].all()
    zeros = np.nonzero(s == 0)[0]
    assert keep[zeros].sum() == 7 and keep[zeros[:7]].all()  # ties at -inf by global id


# ---- pass 2: mass cut ----------------------------------------------------

def test_mass_cut_spec_examples():
    gid = np.arange(4)
    # target 1.0 retains all Gaussians with s > 0  [S:311]
    keep, warn = SO.prune_mass_cut(np.array([0.2, 0.0, 0.5, 1e-12]), gid, 1, 1)
    assert keep.tolist() == [True, False, True, True] and not warn
    # scores (0.5, 0.3, 0.15, 0.05), target 0.99: first three hold 0.95 < 0.99 -> all four  [S:312]
    keep, _ = SO.prune_mass_cut(np.array([0.5, 0.3, 0.15, 0.05]), gid, 99, 100)
    assert keep.all()
    # a first element whose mass alone reaches the target is the whole prefix  [S:317]
    keep, _ = SO.prune_mass_cut(np.array([0.995, 0.002, 0.002, 0.001]), gid, 99, 100)
    assert keep.tolist() == [True, False, False, False]
    # all-zero scores: only the forced first element, with the warning  [S:310]
    keep, warn = SO.prune_mass_cut(np.zeros(5), np.arange(5), 99, 100)
    assert keep.tolist() == [True, False, False, False, False] and warn


def test_mass_cut_minimal_sufficient_prefix():
    rng = np.random.default_rng(11)
    for trial in range(20):
        n = int(rng.integers(1, 3000))
        s = rng.pareto(1.5, n) * (rng.random(n) < 0.9)
        if trial % 4 == 0:
            s = np.round(s, 1)  # many equal scores: ties by gid
        gid = rng.permutation(n)
        keep, warn = SO.prune_mass_cut(s, gid, 99, 100)
        q = SO.score_quanta(s).astype(object)
        tot = sum(q)
        if tot == 0:
            assert warn and keep.sum() == 1
            continue
        kept = sum(q[keep])
        assert 100 * kept >= 99 * tot  # sufficient
        # minimal: the kept set is a prefix of (q desc, gid asc), and dropping its last
        # (smallest q, then largest gid) member falls below the target
        idx = np.nonzero(keep)[0]
        last = max(idx, key=lambda i: (-q[i], gid[i]))
        assert 100 * (kept - q[last]) < 99 * tot
        for i in np.nonzero(~keep)[0]:
            assert (q[i], -gid[i]) < (q[last], -gid[last])


# ---- redistribution ----------------------------------------------------------------

def test_redistribute_bijection_and_balance():
    rng = np.random.default_rng(2)
    keep = rng.random(1001) < 0.37
    ng = SO.redistribute(keep, 4)
    kept = np.nonzero(keep)[0]
    assert np.array_equal(np.sort(ng[kept]), np.arange(len(kept)))  # bijection onto [0, N')
    assert np.all(np.diff(ng[kept]) > 0)  # global-id order preserved
    assert np.all(ng[~keep] == -1)
    sizes = np.bincount(ng[kept] % 4, minlength=4)
    assert sizes.max() - sizes.min() <= 1  # index parity balances the shards
    # the renumbering does not depend on M; only the split does
    assert np.array_equal(SO.redistribute(keep, 1), ng)
