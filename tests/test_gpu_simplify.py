"""GPU parity of NEXT-1 (phi, pass-1 stochastic prune, pass-2 mass cut, index-parity
redistribution) through the C ABI against oracle/simplify.py: bit-exact keep sets and exact
parameter copies, at M = 1 and through the in-process group at M = 2, 3 (the selection is global
over ranks: gathered per-rank results must equal the oracle's global answer)."""
from __future__ import annotations

import threading

import numpy as np
import pytest
import torch

from oracle import simplify as SO

pytestmark = pytest.mark.gpu


def _per_rank(M, fn):
    """Run fn(rank, ctx, stream) on M contexts (one thread each for M > 1); returns the results."""
    import paper_2605_13794_b200.bgs as B
    ctxs = B.Context.local_group(M, 0) if M > 1 else [B.Context(0, 1, 0)]
    out, errs = [None] * M, []

    def run(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream(0)
            with torch.cuda.stream(st):
                out[r] = fn(r, ctxs[r], st)
                st.synchronize()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    if M == 1:
        run(0)
    else:
        th = [threading.Thread(target=run, args=(r,)) for r in range(M)]
        for t in th:
            t.start()
        for t in th:
            t.join()
    for c in ctxs:
        c.close()
    if errs:
        raise errs[0]
    return out


def _scores(rng, n, kind):
    if kind == "heavy":
        s = rng.pareto(1.2, n) * (rng.random(n) < 0.85)
    elif kind == "ties":
        s = rng.integers(0, 5, n).astype(np.float64) * 0.25
    elif kind == "zeros":
        s = np.zeros(n)
    else:
        s = rng.random(n)
    return s.astype(np.float64)


def test_phi_bit_exact():
    import paper_2605_13794_b200.bgs as B
    rng = np.random.default_rng(0)
    n = 50_000
    cr = rng.integers(0, 70, n).astype(np.uint32)
    cv = (cr * rng.random(n)).astype(np.uint32)
    ctx = B.Context()
    phi = torch.zeros(n, dtype=torch.float64, device="cuda")
    B.bgs_score_phi(ctx, n, torch.from_numpy(cr.view(np.int32)).cuda(), torch.from_numpy(cv.view(np.int32)).cuda(),
                    phi)
    torch.cuda.synchronize()
    assert np.array_equal(phi.cpu().numpy().view(np.uint64), SO.phi(cr, cv).view(np.uint64))
    ctx.close()


@pytest.mark.parametrize("M", [1, 2, 3])
def test_prune_stochastic_bit_exact(M):
    import paper_2605_13794_b200.bgs as B
    rng = np.random.default_rng(10 + M)
    for trial, (n, kind) in enumerate([(1, "uniform"), (7, "heavy"), (3000, "heavy"), (20000, "ties"),
                                       (12000, "uniform"), (500, "zeros")]):
        s = _scores(rng, n, kind)
        for frac in (0.0, 0.37, 0.6, 1.0, 1.2):
            k = int(round(frac * n))
            seed = int(rng.integers(0, 2**63))
            ref = SO.prune_stochastic(s, np.arange(n), k, seed)

            def fn(r, ctx, st, s=s, k=k, seed=seed):
                sl = np.ascontiguousarray(s[r::M])
                keep = torch.full((max(len(sl), 1),), 7, dtype=torch.uint8, device="cuda")
                B.bgs_prune_stochastic(ctx, len(sl), torch.from_numpy(sl).cuda(), k, seed, keep, st)
                return keep[:len(sl)].cpu().numpy()

            got = np.zeros(n, bool)
            for r, kr in enumerate(_per_rank(M, fn)):
                got[r::M] = kr.astype(bool)
            assert np.array_equal(got, ref), (trial, frac, int(got.sum()), int(ref.sum()))


@pytest.mark.parametrize("M", [1, 2, 3])
def test_prune_mass_cut_bit_exact(M):
    import paper_2605_13794_b200.bgs as B
    rng = np.random.default_rng(20 + M)
    cases = [(n, kind) for n, kind in [(1, "uniform"), (9, "heavy"), (5000, "heavy"), (30000, "ties"),
                                        (20000, "uniform"), (300, "zeros")]]
    cases.append((4, "spec"))
    for n, kind in cases:
        s = np.array([0.5, 0.3, 0.15, 0.05]) if kind == "spec" else _scores(rng, n, kind)
        for num, den in ((99, 100), (1, 2), (1, 1), (999, 1000)):
            ref, ref_warn = SO.prune_mass_cut(s, np.arange(n), num, den)

            def fn(r, ctx, st, s=s, num=num, den=den):
                sl = np.ascontiguousarray(s[r::M])
                keep = torch.full((max(len(sl), 1),), 7, dtype=torch.uint8, device="cuda")
                warn = B.bgs_prune_mass_cut(ctx, len(sl), torch.from_numpy(sl).cuda(), num, den, keep, st)
                return keep[:len(sl)].cpu().numpy(), warn

            res = _per_rank(M, fn)
            got = np.zeros(n, bool)
            for r, (kr, warn) in enumerate(res):
                got[r::M] = kr.astype(bool)
                assert warn == ref_warn
            assert np.array_equal(got, ref), (n, kind, num, den, int(got.sum()), int(ref.sum()))


@pytest.mark.parametrize("M", [1, 2, 3])
def test_redistribute_exact_copies(M):
    import paper_2605_13794_b200.bgs as B
    rng = np.random.default_rng(30 + M)
    for n, p in ((1, 1.0), (10, 0.0), (4001, 0.37), (25000, 0.8)):
        mo = rng.standard_normal((n, 4)).astype(np.float32)
        q = rng.standard_normal((n, 4)).astype(np.float32)
        sc = rng.random((n, 4)).astype(np.float32)
        sh = rng.standard_normal((n, 48)).astype(np.float32)
        lod = rng.integers(0, 6, n).astype(np.uint8)
        keep = rng.random(n) < p
        new_gid = SO.redistribute(keep, M)
        nk = int(keep.sum())

        def fn(r, ctx, st):
            t = lambda a: torch.from_numpy(np.ascontiguousarray(a[r::M])).cuda()
            g = B.GaussianPlanes(t(mo), t(q), t(sc), t(sh), t(lod))
            cap = max(1, (nk + M - 1) // M)
            out = B.GaussianPlanes(torch.full((cap, 4), np.nan, device="cuda"), torch.zeros(cap, 4, device="cuda"),
                                   torch.zeros(cap, 4, device="cuda"), torch.zeros(cap, 48, device="cuda"),
                                   torch.zeros(cap, dtype=torch.uint8, device="cuda"))
            kk = torch.from_numpy(np.ascontiguousarray(keep[r::M]).astype(np.uint8)).cuda()
            m = B.bgs_redistribute(ctx, g, kk, out, st)
            return m, [x[:m].cpu().numpy() for x in (out.mean_opac, out.quat, out.scale, out.sh, out.lod)]

        res = _per_rank(M, fn)
        kept = np.nonzero(keep)[0]
        for r, (m, arrs) in enumerate(res):
            mine = kept[new_gid[kept] % M == r]  # old gids landing on rank r, in new-local order
            assert m == len(mine)
            for got, src in zip(arrs, (mo, q, sc, sh, lod)):
                assert np.array_equal(got.view(np.uint8), src[mine].view(np.uint8)), (n, p, r)


@pytest.mark.parametrize("M", [1, 2, 3])
def test_redistribute_unequal_shards(M):
    """After density control the shards differ in size; bgs_shard_sizes reports them and
    bgs_redistribute rebalances in the index-parity order gid = j M + m over slices padded to the
    largest shard (absent rows not kept), exact copies ((100, 200) -> (150, 150))."""
    import paper_2605_13794_b200.bgs as B
    rng = np.random.default_rng(77 + M)
    sizes = [int(x) for x in rng.integers(300, 1400, M)]
    if M == 2:
        sizes = [100, 200]
    n_max = max(sizes)
    rows = {}
    for r in range(M):
        n = sizes[r]
        rows[r] = (rng.standard_normal((n, 4)).astype(np.float32), rng.standard_normal((n, 4)).astype(np.float32),
                   rng.random((n, 4)).astype(np.float32), rng.standard_normal((n, 48)).astype(np.float32),
                   rng.integers(0, 6, n).astype(np.uint8))
    keep_by_gid = np.zeros(n_max * M, bool)
    for r in range(M):
        keep_by_gid[np.arange(sizes[r]) * M + r] = True  # rebalance: every present row survives
    new_gid = SO.redistribute(keep_by_gid, M)
    nk = int(keep_by_gid.sum())

    def fn(r, ctx, st):
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        g = B.GaussianPlanes(*(t(a) for a in rows[r]))
        sz = B.bgs_shard_sizes(ctx, sizes[r])
        cap = max(1, (nk + M - 1) // M)
        out = B.GaussianPlanes(torch.full((cap, 4), np.nan, device="cuda"), torch.zeros(cap, 4, device="cuda"),
                               torch.zeros(cap, 4, device="cuda"), torch.zeros(cap, 48, device="cuda"),
                               torch.zeros(cap, dtype=torch.uint8, device="cuda"))
        kk = torch.ones(max(sizes[r], 1), dtype=torch.uint8, device="cuda")
        m = B.bgs_redistribute(ctx, g, kk, out, st)
        return sz, m, [x[:m].cpu().numpy() for x in (out.mean_opac, out.quat, out.scale, out.sh, out.lod)]

    res = _per_rank(M, fn)
    kept = np.nonzero(keep_by_gid)[0]
    for r, (sz, m, arrs) in enumerate(res):
        assert sz == sizes
        mine = kept[new_gid[kept] % M == r]  # old gids landing on rank r, in new-local order
        assert m == len(mine) == (nk - r + M - 1) // M
        for k, got in enumerate(arrs):
            src = np.stack([rows[g % M][k][g // M] for g in mine]) if len(mine) else got
            assert np.array_equal(got.view(np.uint8), np.asarray(src).view(np.uint8)), (M, r, k)
    if M == 2:
        assert [m for _, m, _ in res] == [150, 150]
