"""CUDA path (through the C ABI) vs the CPU oracle on the same seeded inputs.

Bit-exact: radius, rect, tile ids, per-tile pair counts, sort order, ranges, routing, gate and
cull decisions, record floats (pinned arithmetic), a and n_contrib (except attributed early-stop
flips), c_rad, and c_vis / Cull given identical w_fixed.  Pixels |d| <= 1e-4.  Gradients
|d| <= 1e-3 |g| + 1e-5 max|g| per parameter group.  w_fixed within one fixed-point unit per
contributing pixel + 1e-5 relative.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
import synthetic as S  # noqa: E402
from gpu_helpers import GpuStep, rec_view  # noqa: E402

pytestmark = pytest.mark.gpu
ET_MARGIN = 1e-4  # relative distance of T(1-alpha) to 1e-4 below which an early-stop flip is excused


def _f32(x):
    return np.asarray(x, np.float64).astype(np.float32)


def _flip_info(st, gs, cam, sample=None):
    """Pixels whose early-stop decision actually differs between the oracle and the GPU (exp
    rounding), and the gids whose a / w / gradients those flips can affect (every
    splat of that pixel's list up to the deeper of the two stops).  Candidates (oracle test value
    T(1-alpha) within ET_MARGIN relative of 1e-4) are reported, but only actual flips excuse
    anything.  `sample`: restrict to a boolean pixel mask (tile-sampled oracle runs)."""
    H, W = cam["H"], cam["W"]
    margin = st.get("et_margin").reshape(H, W)
    nc_o = st.get("n_contrib").reshape(H, W)
    cand = margin < ET_MARGIN
    flips = (nc_o != gs.nc) & cand
    if sample is not None:
        cand, flips = cand & sample, flips & sample
    affected = set()
    TX = (W + 15) // 16
    for y, x in zip(*np.nonzero(flips)):
        t = (y // 16) * TX + x // 16
        for r in range(st.M):
            b, e = st.get("tile_range", r)
            if b <= t < e:
                break
        gids = st.get("pair_gid", r)
        lo, hi = st.get("range_lo", r), st.get("range_hi", r)
        upto = max(nc_o[y, x], gs.nc[y, x]) + 1
        lt = t - b
        affected.update(gids[lo[lt]:min(hi[lt], lo[lt] + upto)].tolist())
    return cand, flips, affected


def _excused_ok(st, gs, affected):
    """The excusal stays small: under 1% of the splats that contribute to the view."""
    contributing = int((st.get("a") > 0).sum())
    assert len(affected) <= 0.01 * max(contributing, 1), (len(affected), contributing)


def _check_grads(sc_n, st, gs, keep, group_tol=1e-3, what=""):
    """Parameter gradients vs the oracle: |d| <= 1e-3 |g| + 1e-5 max|g| per group."""
    for name, width in (("d_mean", 3), ("d_quat", 4), ("d_scale", 3), ("d_opac", 1), ("d_sh", 48)):
        ref = st.get(name).reshape(sc_n, width)[keep]
        got = gs.grads[name].reshape(sc_n, width)[keep]
        tol = group_tol * np.abs(ref) + 1e-5 * np.abs(ref).max(initial=0)
        bad = np.abs(got - ref) > tol
        assert not bad.any(), (what, name, int(bad.sum()),
                               float(np.max(np.abs(got - ref) / (np.abs(ref) + 1e-30), initial=0)))


def _check_g2d(st, gs, keep, what=""):
    """The 9 owner-summed compositing partials dL/d(mx, my, A, B, C, o, r, g, b) per splat."""
    g_ref = st.get("g2d").reshape(-1, 9)
    for k in range(9):
        ref, got = g_ref[keep, k], gs.g2d[keep, k]
        tol = 1e-3 * np.abs(ref) + 1e-5 * np.abs(ref).max(initial=0)
        bad = np.abs(got - ref) > tol
        assert not bad.any(), (what, k, int(bad.sum()))


@pytest.fixture(scope="module")
def tiny_run(tiny_scene):
    cam = tiny_scene.cameras[0]
    dl = S.grad_image(cam["H"], cam["W"])
    st = O.OracleStep(tiny_scene, cam, M=1, dLdC=dl)
    gs = GpuStep(tiny_scene, cam, M=1, dLdC=dl)
    yield tiny_scene, cam, dl, st, gs
    gs.close()


def test_project_bit_exact(tiny_run):
    sc, cam, dl, st, gs = tiny_run
    assert np.array_equal(gs.radius, st.get("radius"))
    rec = gs.rank[0]["records"]
    order = np.argsort(rec["gid"])
    gid = rec["gid"][order]
    valid = np.nonzero(st.get("radius") > 0)[0]
    assert np.array_equal(gid, valid)
    m2 = st.get("mean2d").reshape(-1, 2)[valid]
    con = st.get("conic").reshape(-1, 3)[valid]
    for name, ref in (("mx", m2[:, 0]), ("my", m2[:, 1]), ("A", con[:, 0]), ("B", con[:, 1]), ("C", con[:, 2]),
                      ("depth", st.get("depth")[valid])):
        assert np.array_equal(rec[name][order].view(np.uint32), _f32(ref).view(np.uint32)), name
    assert np.array_equal(rec["rgb"][order].view(np.uint32), _f32(st.get("rgb").reshape(-1, 3)[valid]).view(np.uint32))
    assert np.array_equal(rec["rect"][order], st.get("rect").reshape(-1, 4)[valid])
    q = gs.rank[0]["q_project"]
    assert q["F"] == len(valid) and q["P_all"] == st.get("n_pairs_total")[0]


def test_sort_and_ranges_bit_exact(tiny_run):
    sc, cam, dl, st, gs = tiny_run
    o = gs.rank[0]
    vals = o["vals"]
    tiles = o["key_tile"]
    dbits = o["recv"]["depth"][vals].view(np.uint32)
    gid = o["recv"]["gid"][vals]
    assert np.array_equal(tiles, st.get("pair_tile", 0))
    assert np.array_equal(gid, st.get("pair_gid", 0))
    assert np.array_equal(dbits, _f32(st.get("depth")[gid]).view(np.uint32))
    assert np.array_equal(o["ranges"][:, 0], st.get("range_lo", 0))
    assert np.array_equal(o["ranges"][:, 1], st.get("range_hi", 0))
    # sorted keys non-decreasing in every tile
    keys = o["keys"]
    same_tile = tiles[1:] == tiles[:-1]
    assert np.all(keys[1:][same_tile] >= keys[:-1][same_tile])


@pytest.mark.parametrize("M", [1, 3])
def test_bucket_sort_path_matches(tiny_scene, tiny_run, monkeypatch, M):
    """BGS_SORT=bucket (per-tile bucket sort, bucket.cu) gives the oracle's pair order and ranges
    and the same image at world 1 and at M = 3 (in-process group); its keys are f32 bits(depth) - lo
    (C_DLO holds 0xffffffff - lo), non-decreasing in every tile."""
    sc, cam, dl, st1, gs = tiny_run
    st = st1 if M == 1 else O.OracleStep(sc, cam, M=M, dLdC=dl)
    monkeypatch.setenv("BGS_SORT", "bucket")
    g2 = GpuStep(sc, cam, M=M, dLdC=dl)
    try:
        for r in range(M):
            o2 = g2.rank[r]
            b, _ = st.get("tile_range", r)
            assert np.array_equal(o2["recv"]["gid"][o2["vals"]], st.get("pair_gid", r))
            assert np.array_equal(o2["key_tile"] + b, st.get("pair_tile", r))
            assert np.array_equal(o2["ranges"][:, 0], st.get("range_lo", r))
            assert np.array_equal(o2["ranges"][:, 1], st.get("range_hi", r))
            dbits = o2["recv"]["depth"][o2["vals"]].view(np.uint32)
            lo = np.uint32(0xFFFFFFFF - int(o2["counters"][6] & np.uint64(0xFFFFFFFF)))
            assert np.array_equal(o2["keys"], dbits - lo)
        assert np.array_equal(g2.img, gs.img) and np.array_equal(g2.nc, gs.nc)
    finally:
        g2.close()


def test_raster_fwd_parity(tiny_run):
    sc, cam, dl, st, gs = tiny_run
    H, W = cam["H"], cam["W"]
    cand, flips, affected = _flip_info(st, gs, cam)
    img = st.get("img").reshape(3, H, W)
    T = st.get("t_final").reshape(H, W)
    ok = ~flips
    assert np.abs(gs.img - img)[:, ok].max() <= 1e-4
    assert np.abs(gs.T - T)[ok].max() <= 1e-5
    assert np.array_equal(gs.nc[ok], st.get("n_contrib").reshape(H, W)[ok])
    a_o, w_o = st.get("a"), st.get("w_fixed")
    mism = np.nonzero(gs.a != a_o)[0]
    assert set(mism.tolist()) <= affected, (len(mism), flips.sum())
    keep = np.ones(sc.n, bool)
    keep[list(affected)] = False
    dw = np.abs(gs.w.astype(np.float64) - w_o.astype(np.float64))
    assert np.all(dw[keep] <= a_o[keep] + 1e-5 * w_o[keep].astype(np.float64))
    _excused_ok(st, gs, affected)
    print(f"flip candidates {cand.sum()}, flips {flips.sum()}, affected splats {len(affected)}")


def test_backward_parity(tiny_run):
    """All 9 compositing partials and every parameter gradient of every splat except those whose
    list holds an actual early-stop flip (<= 1% of the contributing splats; 0 on this scene)."""
    sc, cam, dl, st, gs = tiny_run
    _, flips, affected = _flip_info(st, gs, cam)
    _excused_ok(st, gs, affected)
    keep = np.ones(sc.n, bool)
    keep[list(affected)] = False
    contributing = st.get("a") > 0
    assert (keep & contributing).sum() >= 0.99 * contributing.sum()
    _check_g2d(st, gs, keep, "tiny")
    _check_grads(sc.n, st, gs, keep, what="tiny")


def test_importance_parity(tiny_run):
    sc, cam, dl, st, gs = tiny_run
    # same w_fixed -> bit-exact selection; s is the same fp64 expression
    ref = O.importance(gs.radius, gs.w, gs.a)
    assert np.array_equal(gs.c_rad, ref["c_rad"])
    assert np.array_equal(gs.c_vis, ref["c_vis"])
    assert np.array_equal(gs.cull_bits, S.unpack_bits(ref["cull"], sc.n))
    np.testing.assert_allclose(gs.s, ref["s"], rtol=1e-12, atol=0)
    # against the oracle's own w: s within the fixed-point bound
    ref2 = O.importance(st.get("radius"), st.get("w_fixed"), st.get("a"))
    _, _, affected = _flip_info(st, gs, cam)
    keep = np.ones(sc.n, bool)
    keep[list(affected)] = False
    np.testing.assert_allclose(gs.s[keep], ref2["s"][keep], rtol=2e-5, atol=1e-9)


@pytest.fixture(params=["coarse", "coop"])
def imp_mode(request, monkeypatch):
    """a12 at world 1: the coarse-histogram path (default) and the cooperative one (BGS_IMP=coop)."""
    if request.param == "coop":
        monkeypatch.setenv("BGS_IMP", "coop")
    return request.param


def test_importance_dense_path_bit_exact(imp_mode):
    """bgs_importance with caller-supplied dense w_fixed equals the oracle selection on the same
    values, including heavy ties (count-only gid select) and an empty view."""
    import paper_2605_13794_b200.bgs as B
    ctx = B.Context()
    rng = np.random.default_rng(5)
    for trial in range(10):
        n = int(rng.integers(1, 200_000))
        if trial == 0:
            w = np.zeros(n, np.uint64)
        elif trial < 3:
            w = (rng.integers(0, 4, n) * (1 << 20)).astype(np.uint64)  # massive ties
        elif trial < 6:
            w = rng.integers(0, 1 << 40, n).astype(np.uint64) * rng.integers(0, 2, n).astype(np.uint64)
        elif trial == 6:
            # one dominant item: the crossing bin of the first round holds only it (early exit)
            w = rng.integers(1, 1 << 20, n).astype(np.uint64)
            w[rng.integers(0, n)] = np.uint64(1 << 45)
        elif trial == 7:
            # heavy-tailed (log-uniform) weights, as the rasterizer produces: crossing bins thin out
            # after a few rounds
            w = np.exp(rng.uniform(np.log(1e3), np.log(1e12), n)).astype(np.uint64)
        elif trial == 8:
            # a unique item straddling the 99% cut with equal high bits to many others
            w = np.full(n, np.uint64(1 << 30)) + rng.integers(0, 1 << 8, n).astype(np.uint64)
        else:
            # two items only; either may be the threshold
            n = 2
            w = np.array([(1 << 33) + 5, (1 << 33) + 3], np.uint64)
        a = np.where(w > 0, rng.integers(1, 300, n), 0).astype(np.uint32)
        rad = np.where(a > 0, 4, rng.integers(0, 2, n) * 4).astype(np.int32)
        ref = O.importance(rad, w, a)
        dev = "cuda"
        s = torch.zeros(n, dtype=torch.float64, device=dev)
        crad = torch.zeros(n, dtype=torch.int32, device=dev)
        cvis = torch.zeros(n, dtype=torch.int32, device=dev)
        cull = torch.zeros((n + 31) // 32, dtype=torch.int32, device=dev)
        B.bgs_importance(ctx, n, torch.from_numpy(rad).to(dev), torch.from_numpy(w.view(np.int64)).to(dev),
                         torch.from_numpy(a.view(np.int32)).to(dev), s, crad, cvis, cull)
        torch.cuda.synchronize()
        assert np.array_equal(cvis.cpu().numpy().view(np.uint32), ref["c_vis"]), trial
        assert np.array_equal(cull.cpu().numpy().view(np.uint32), ref["cull"]), trial
        assert np.array_equal(crad.cpu().numpy().view(np.uint32), ref["c_rad"]), trial
        np.testing.assert_allclose(s.cpu().numpy(), ref["s"], rtol=1e-12)
    ctx.close()


@pytest.mark.parametrize("mode", ["coarse", "rounds"])
def test_importance_selection_world3(mode, monkeypatch):
    """a12 at world > 1 on identical w_fixed (dense path, index-parity shards over an in-process group
    of 3): the two-collective path (coarse histogram all-reduce + crossing-bin all-gather, default) and
    the radix-round path (BGS_IMP=rounds) both select bit-exactly the oracle's global top-99% set,
    including heavy ties (gid order), one dominant item, heavy tails and an empty view."""
    import threading
    import paper_2605_13794_b200.bgs as B
    if mode == "rounds":
        monkeypatch.setenv("BGS_IMP", "rounds")
    M = 3
    rng = np.random.default_rng(11)
    for trial in range(7):
        n = int(rng.integers(2, 120_000))
        if trial == 0:
            w = np.zeros(n, np.uint64)
        elif trial == 1:
            w = (rng.integers(0, 4, n) * (1 << 20)).astype(np.uint64)  # massive ties
        elif trial == 2:
            w = rng.integers(1, 1 << 20, n).astype(np.uint64)
            w[rng.integers(0, n)] = np.uint64(1 << 45)  # one dominant item
        elif trial == 3:
            w = np.exp(rng.uniform(np.log(1e3), np.log(1e12), n)).astype(np.uint64)
        elif trial == 4:
            w = np.full(n, np.uint64(1 << 30)) + rng.integers(0, 1 << 8, n).astype(np.uint64)
        elif trial == 5:
            w = np.full(n, np.uint64(12345))  # every item in one coarse bin, all tied
        else:
            w = rng.integers(0, 1 << 40, n).astype(np.uint64) * rng.integers(0, 2, n).astype(np.uint64)
        a = np.where(w > 0, rng.integers(1, 300, n), 0).astype(np.uint32)
        rad = np.where(a > 0, 4, 0).astype(np.int32)
        ref = O.importance(rad, w, a)
        ctxs = B.Context.local_group(M, 0)
        res = [None] * M
        errs = []

        def run(r):
            try:
                torch.cuda.set_device(0)
                st = torch.cuda.Stream()
                with torch.cuda.stream(st):
                    dev = "cuda"
                    ids = np.arange(r, n, M)
                    m = len(ids)
                    s_ = torch.zeros(max(m, 1), dtype=torch.float64, device=dev)
                    cr = torch.zeros(max(m, 1), dtype=torch.int32, device=dev)
                    cv = torch.zeros(max(m, 1), dtype=torch.int32, device=dev)
                    cu = torch.zeros(max(1, (m + 31) // 32), dtype=torch.int32, device=dev)
                    B.bgs_importance(ctxs[r], m, torch.from_numpy(rad[ids]).to(dev),
                                     torch.from_numpy(w[ids].view(np.int64)).to(dev),
                                     torch.from_numpy(a[ids].view(np.int32)).to(dev), s_, cr, cv, cu, stream=st)
                    st.synchronize()
                    res[r] = (cv.cpu().numpy()[:m].view(np.uint32), S.unpack_bits(cu.cpu().numpy(), m),
                              ctxs[r].batch_stats()["collectives"])
            except Exception as e:  # pragma: no cover
                errs.append(e)

        th = [threading.Thread(target=run, args=(r,)) for r in range(M)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for c in ctxs:
            c.close()
        if errs:
            raise errs[0]
        cvis = np.zeros(n, np.uint32)
        cull = np.zeros(n, bool)
        for r in range(M):
            cvis[r::M], cull[r::M] = res[r][0], res[r][1]
        assert np.array_equal(cvis, ref["c_vis"]), (mode, trial)
        assert np.array_equal(cull, S.unpack_bits(ref["cull"], n)), (mode, trial)
        if mode == "coarse":
            assert all(res[r][2] <= 2 for r in range(M)), [res[r][2] for r in range(M)]


@pytest.mark.parametrize("M", [2, 3, 4])
def test_multirank_local_group_parity(tiny_scene, tiny_run, M):
    """The M > 1 kernels (tile costs, owner map, dest masks, pack, exchange, reverse gather-sum,
    distributed radix select) on one GPU through the in-process transport: owner map and routing
    bit-exact vs the oracle at the same M; pixels / n_contrib / w / a bitwise equal to the GPU
    M = 1 run ("identical to what a single-GPU renderer would produce")."""
    sc, cam, dl, st1, gs1 = tiny_run
    st = O.OracleStep(sc, cam, M=M, dLdC=dl)
    gs = GpuStep(sc, cam, M=M, dLdC=dl)
    try:
        owner = st.get("owner")
        for r in range(M):
            assert np.array_equal(gs.rank[r]["owner"], owner)
            q = gs.rank[r]["q"]
            b, e = st.get("tile_range", r)
            assert (q["tile_begin"], q["tile_end"]) == (b, e)
            assert q["P"] == len(st.get("pair_tile", r))
            assert q["R"] == len(st.get("recv", r))
            # received set and sorted pair sequence per owner
            tiles = gs.rank[r]["key_tile"] + b
            gids = gs.rank[r]["recv"]["gid"][gs.rank[r]["vals"]]
            assert np.array_equal(tiles, st.get("pair_tile", r))
            assert np.array_equal(gids, st.get("pair_gid", r))
        counts = st.get("counts").reshape(M, M)
        for r in range(M):
            assert gs.rank[r]["q"]["D"] == counts[r].sum()
        assert np.array_equal(gs.img, gs1.img) and np.array_equal(gs.T, gs1.T) and np.array_equal(gs.nc, gs1.nc)
        assert np.array_equal(gs.a, gs1.a) and np.array_equal(gs.w, gs1.w)
        assert np.array_equal(gs.c_vis, gs1.c_vis) and np.array_equal(gs.cull_bits, gs1.cull_bits)
        # against the oracle at the same M (owner partials summed in dest-rank order, O10): pixels,
        # counts, a, w and every gradient, excusing only actual early-stop flips
        H, W = cam["H"], cam["W"]
        cand, flips, affected = _flip_info(st, gs, cam)
        _excused_ok(st, gs, affected)
        ok = ~flips
        assert np.abs(gs.img - st.get("img").reshape(3, H, W))[:, ok].max() <= 1e-4
        assert np.array_equal(gs.nc[ok], st.get("n_contrib").reshape(H, W)[ok])
        keep = np.ones(sc.n, bool)
        keep[list(affected)] = False
        assert np.array_equal(gs.a[keep], st.get("a")[keep])
        w_o = st.get("w_fixed").astype(np.float64)
        assert np.all(np.abs(gs.w.astype(np.float64) - w_o)[keep] <= st.get("a")[keep] + 1e-5 * w_o[keep])
        _check_g2d(st, gs, keep, f"M={M}")
        _check_grads(sc.n, st, gs, keep, what=f"M={M}")
    finally:
        gs.close()


@pytest.mark.parametrize("M", [2, 3])
def test_importance_only_reverse(tiny_scene, tiny_run, M):
    """BGS_IMPORTANCE_ONLY: the scoring pass's reverse exchange carries only (w, a),
    12 B per record; w, a, s, c_rad, c_vis and the Cull column are bit-identical to the full 48-B
    reverse and to world 1."""
    sc, cam, dl, st1, gs1 = tiny_run
    full = GpuStep(sc, cam, M=M, flags=1)  # NO_COLOR, forward only: the scoring pass
    imp = GpuStep(sc, cam, M=M, flags=1, imp_only=True)
    try:
        for f in ("a", "w", "c_rad", "c_vis", "cull_bits"):
            assert np.array_equal(getattr(imp, f), getattr(full, f)), f
            assert np.array_equal(getattr(imp, f), getattr(gs1, f)), f
        np.testing.assert_allclose(imp.s, full.s, rtol=1e-15, atol=0)
        assert not imp.g2d.any()  # no gradients travel in this mode
    finally:
        full.close()
        imp.close()


def test_route_given_owner_map(tiny_scene, tiny_run):
    """bgs_route's tile_owner_in: the oracle's owner map passed in reproduces the
    a3 split's routing; a map that is not contiguous runs is refused on every rank."""
    import paper_2605_13794_b200.bgs as B
    sc, cam, dl, st1, gs1 = tiny_run
    M = 3
    st = O.OracleStep(sc, cam, M=M, dLdC=dl)
    gs = GpuStep(sc, cam, M=M, dLdC=dl, owner_in=st.get("owner"))
    try:
        for r in range(M):
            assert np.array_equal(gs.rank[r]["owner"], st.get("owner"))
            assert gs.rank[r]["R_route"] == len(st.get("recv", r))
        assert np.array_equal(gs.img, gs1.img) and np.array_equal(gs.nc, gs1.nc)
    finally:
        gs.close()
    bad = st.get("owner").copy()
    bad[0], bad[-1] = bad[-1], bad[0]
    with pytest.raises(B.BgsError, match="tile_owner_in"):
        GpuStep(sc, cam, M=M, dLdC=dl, owner_in=bad)


@pytest.mark.gpu
def test_project_bwd_needs_colour_projection(tiny_scene):
    """a11 reads the colour Jacobian a2 leaves in the arena (include/bgs.h): after a BGS_NO_COLOR
    projection of the view, bgs_project_bwd is refused with a contract error instead of reading a
    stale Jacobian."""
    import torch
    import paper_2605_13794_b200.bgs as B
    cam = tiny_scene.cameras[0]
    H, W = cam["H"], cam["W"]
    ctx = B.Context(0, 1, 0)
    g = B.GaussianPlanes.from_scene(tiny_scene, "cuda")
    grads = g.zeros_grads()
    n = tiny_scene.n
    radius = torch.zeros(n, dtype=torch.int32, device="cuda")
    rgb, T = torch.zeros(3, H, W, device="cuda"), torch.zeros(H, W, device="cuda")
    nc = torch.zeros(H, W, dtype=torch.int32, device="cuda")
    dl = torch.from_numpy(S.grad_image(H, W)).cuda()
    c = B.camera(cam)
    B.bgs_project(ctx, g, c, None, None, B.BGS_NO_COLOR, radius)
    B.bgs_route(ctx)
    B.bgs_sort_tiles(ctx)
    B.bgs_raster_fwd(ctx, 0, rgb, T, nc)
    B.bgs_raster_bwd(ctx, dl, T, nc)
    B.bgs_route_reverse(ctx)
    with pytest.raises(B.BgsError, match="NO_COLOR"):
        B.bgs_project_bwd(ctx, g, c, grads)
    # the same view with colour goes through
    B.bgs_project(ctx, g, c, None, None, 0, radius)
    B.bgs_route(ctx)
    B.bgs_sort_tiles(ctx)
    B.bgs_raster_fwd(ctx, 0, rgb, T, nc)
    B.bgs_raster_bwd(ctx, dl, T, nc)
    B.bgs_route_reverse(ctx)
    B.bgs_project_bwd(ctx, g, c, grads)
    torch.cuda.synchronize()
    assert torch.isfinite(grads.mean_opac).all() and grads.mean_opac.abs().sum() > 0


def test_gate_and_cull_bit_exact():
    sc = S.gen_city("rubble", n=200_000, W=576, H=432, V=4)
    cam = sc.cameras[2]
    gate = dict(enabled=1, l_max=3, d0=sc.d0 * 4)
    cull = S.random_cull_column(sc.n, 0.8, seed=2)
    for M in (1, 2):
        st = O.OracleStep(sc, cam, gate=gate, cull_global=cull, M=M)
        gs = GpuStep(sc, cam, M=M, gate=gate, cull_global=cull)
        try:
            assert np.array_equal(gs.radius, st.get("radius"))
            for r in range(M):
                assert gs.rank[r]["q"]["n_lod"] == st.get("n_lod")[r]
                assert gs.rank[r]["q"]["n_active"] == st.get("n_keep")[r]
                assert gs.rank[r]["q"]["fallback"] == st.get("fallback")[r]
            img = st.get("img").reshape(3, cam["H"], cam["W"])
            cand = st.get("et_margin").reshape(cam["H"], cam["W"]) < ET_MARGIN
            assert np.abs(gs.img - img)[:, ~cand].max() <= 1e-4
        finally:
            gs.close()


def test_building_full_size_gated_sampled():
    """BASELINE configs[2] at full size (Building-shaped, 8M Gaussians, 1152x864) with the LOD gate
    (d0 = 4 x median camera distance, the bench's setting) and a seeded Cull column: gate / cull
    counts, the fallback decision, radius and every record bit-exact; pixels and n_contrib on a 1/16
    tile sample (the oracle composites only those tiles)."""
    sc = S.gen_city("building")
    cam = sc.cameras[3]
    gate = dict(enabled=1, l_max=sc.k_levels - 1, d0=sc.d0 * 4)
    cull = S.random_cull_column(sc.n, 0.9, seed=5)
    st = O.OracleStep(sc, cam, gate=gate, cull_global=cull, M=1, tile_frac=1.0 / 16, threads=16)
    gs = GpuStep(sc, cam, M=1, gate=gate, cull_global=cull, importance=False)
    try:
        assert np.array_equal(gs.radius, st.get("radius"))
        q = gs.rank[0]["q"]
        assert q["n_lod"] == st.get("n_lod")[0] and q["n_active"] == st.get("n_keep")[0]
        assert q["fallback"] == st.get("fallback")[0]
        rec = gs.rank[0]["records"]
        order = np.argsort(rec["gid"])
        valid = np.nonzero(st.get("radius") > 0)[0]
        assert np.array_equal(rec["gid"][order], valid)
        m2 = st.get("mean2d").reshape(-1, 2)[valid]
        assert np.array_equal(rec["mx"][order].view(np.uint32), _f32(m2[:, 0]).view(np.uint32))
        assert np.array_equal(rec["rgb"][order].view(np.uint32),
                              _f32(st.get("rgb").reshape(-1, 3)[valid]).view(np.uint32))
        H, W = cam["H"], cam["W"]
        sample = _tile_sample(H, W)
        _, flips, _ = _flip_info(st, gs, cam, sample)
        ok = sample & ~flips
        assert np.abs(gs.img - st.get("img").reshape(3, H, W))[:, ok].max(initial=0) <= 1e-4
        assert np.array_equal(gs.nc[ok], st.get("n_contrib").reshape(H, W)[ok])
    finally:
        gs.close()


def test_spatial_order_layout():
    """bgs_spatial_order: a permutation whose Morton codes (recomputed here in float64 from the
    same bounding box) never decrease except at quantisation-boundary ties; a step on the
    reordered shard matches the oracle on the same relabelled scene."""
    import paper_2605_13794_b200.bgs as B
    sc = S.gen_city("rubble", n=300_000, W=576, H=432, V=4)
    ctx = B.Context()
    g = B.GaussianPlanes.from_scene(sc, "cuda")
    perm = B.spatial_order(ctx, g).cpu().numpy()
    ctx.close()
    assert np.array_equal(np.sort(perm), np.arange(sc.n))
    mu = sc.means.astype(np.float64)
    lo, hi = mu.min(0), mu.max(0)
    q = np.clip(np.floor((mu - lo) * (65535.0 / (hi - lo))), 0, 65535).astype(np.uint64)

    def spread(v):
        out = np.zeros_like(v)
        for b in range(16):
            out |= ((v >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b)
        return out

    code = spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1)) | (spread(q[:, 2]) << np.uint64(2))
    c = code[perm]
    assert (np.diff(c.astype(np.float64)) < 0).mean() < 1e-3
    sc2 = sc.subset(perm)
    cam = sc2.cameras[1]
    st = O.OracleStep(sc2, cam, M=1)
    gs = GpuStep(sc2, cam, M=1, importance=False)
    try:
        assert np.array_equal(gs.radius, st.get("radius"))
        o = gs.rank[0]
        assert np.array_equal(o["recv"]["gid"][o["vals"]], st.get("pair_gid", 0))
    finally:
        gs.close()


def _tile_sample(H, W, stride=16):
    """Pixels of the tiles t = 0, stride, 2 stride, ... (the oracle's tile_frac sample)."""
    TX = (W + 15) // 16
    sample = np.zeros((H, W), bool)
    for t in range(0, TX * ((H + 15) // 16), stride):
        ty, tx = divmod(t, TX)
        sample[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16] = True
    return sample


@pytest.fixture(scope="module")
def rubble_full():
    """BASELINE configs[1] at full size (6M Gaussians, 1152x864), view 7, in the bench's launch
    configuration.  dL/dC is the seeded noise image zeroed outside a 1/16 tile sample, so the
    oracle's tile-sampled compositing backward (tile_frac = 1/16) sees the same upstream gradient
    as the GPU's full-image backward: every parameter gradient is then comparable."""
    sc = S.gen_city("rubble")
    cam = sc.cameras[7]
    H, W = cam["H"], cam["W"]
    sample = _tile_sample(H, W)
    dl = S.grad_image(H, W) * sample[None]
    st = O.OracleStep(sc, cam, M=1, tile_frac=1.0 / 16, dLdC=dl)
    gs = GpuStep(sc, cam, M=1, dLdC=dl)
    yield sc, cam, sample, st, gs
    gs.close()


def test_block_bounds_cull_is_exact():
    """Hierarchical culling (bgs_shard_bounds + bgs_gaussians.bounds) on the Z-ordered full Rubble
    shard: for several views, radius, the records, F, P_all and |A| are bit-identical to the
    per-Gaussian path (a culled block's Gaussians all have empty rects)."""
    import paper_2605_13794_b200.bgs as B
    sc = S.gen_city("rubble")
    ctx = B.Context(0, 1, 0)
    g = B.GaussianPlanes.from_scene(sc, "cuda")
    perm = B.spatial_order(ctx, g)
    g = B.GaussianPlanes(g.mean_opac[perm].contiguous(), g.quat[perm].contiguous(), g.scale[perm].contiguous(),
                         g.sh[perm].contiguous(), g.lod[perm].contiguous())
    gb = B.GaussianPlanes(g.mean_opac, g.quat, g.scale, g.sh, g.lod)
    bounds = B.bgs_shard_bounds(ctx, gb)
    torch.cuda.synchronize()
    # the boxes hold their blocks (spot check against torch on a few blocks)
    b = bounds.cpu().numpy()
    mo, scl = g.mean_opac.cpu().numpy(), g.scale.cpu().numpy()
    for blk in (0, 17, len(b) - 1):
        rows = slice(blk * 1024, min(sc.n, blk * 1024 + 1024))
        assert np.array_equal(b[blk, :3], mo[rows, :3].min(0)) and np.array_equal(b[blk, 4:7], mo[rows, :3].max(0))
        assert b[blk, 3] == scl[rows, :3].max()
    for v in (0, 7, 31, 50):
        cam = B.camera(sc.cameras[v])
        out = []
        for gg in (g, gb):
            radius = torch.full((sc.n,), -1, dtype=torch.int32, device="cuda")
            B.bgs_project(ctx, gg, cam, None, None, 0, radius)
            q = ctx.query()
            rec = rec_view(ctx.debug_buffer("records"))
            order = np.argsort(rec["gid"])
            out.append((radius.cpu().numpy(), q, {k: v_[order] for k, v_ in rec.items()}))
        (r0, q0, c0), (r1, q1, c1) = out
        assert np.array_equal(r0, r1), v
        assert (q0["F"], q0["P_all"], q0["n_active"]) == (q1["F"], q1["P_all"], q1["n_active"]), v
        for k in c0:
            assert np.array_equal(c0[k], c1[k]), (v, k)
    ctx.close()


def test_full_size_sampled(rubble_full):
    """Projection, records, the complete sorted pair sequence and ranges bit-exact at full size;
    pixels and n_contrib on the 1/16 tile sample (the ones the oracle composites)."""
    sc, cam, sample, st, gs = rubble_full
    assert np.array_equal(gs.radius, st.get("radius"))
    rec = gs.rank[0]["records"]
    order = np.argsort(rec["gid"])
    valid = np.nonzero(st.get("radius") > 0)[0]
    assert np.array_equal(rec["gid"][order], valid)
    m2 = st.get("mean2d").reshape(-1, 2)[valid]
    assert np.array_equal(rec["mx"][order].view(np.uint32), _f32(m2[:, 0]).view(np.uint32))
    assert np.array_equal(rec["rgb"][order].view(np.uint32),
                          _f32(st.get("rgb").reshape(-1, 3)[valid]).view(np.uint32))
    o = gs.rank[0]
    assert np.array_equal(o["key_tile"], st.get("pair_tile", 0))
    assert np.array_equal(o["recv"]["gid"][o["vals"]], st.get("pair_gid", 0))
    assert np.array_equal(o["ranges"][:, 0], st.get("range_lo", 0))
    assert np.array_equal(o["ranges"][:, 1], st.get("range_hi", 0))
    H, W = cam["H"], cam["W"]
    cand, flips, affected = _flip_info(st, gs, cam, sample)
    ok = sample & ~flips
    assert ok.sum() > 0.05 * H * W
    img = st.get("img").reshape(3, H, W)
    assert np.abs(gs.img - img)[:, ok].max() <= 1e-4
    assert np.array_equal(gs.nc[ok], st.get("n_contrib").reshape(H, W)[ok])
    print(f"full size: flip candidates {cand.sum()}, flips {flips.sum()}, affected {len(affected)}")


def test_full_size_sampled_gradients(rubble_full):
    """All 9 compositing partials and all parameter gradients of the 6M-Gaussian view (upstream
    gradient on the 1/16 tile sample) against the fp64 oracle, excusing only actual flips."""
    sc, cam, sample, st, gs = rubble_full
    _, flips, affected = _flip_info(st, gs, cam, sample)
    _excused_ok(st, gs, affected)
    keep = np.ones(sc.n, bool)
    keep[list(affected)] = False
    touched = np.abs(st.get("g2d").reshape(-1, 9)).sum(1) > 0
    assert touched.sum() > 10_000
    _check_g2d(st, gs, keep, "rubble")
    _check_grads(sc.n, st, gs, keep, what="rubble")


def test_full_size_importance(rubble_full):
    """a12 on the full 6M shard: c_rad, c_vis and the Cull column bit-exact against the oracle's
    selection (std::sort and scan, O12) on the GPU's own w_fixed and a; s the same fp64 sum."""
    sc, cam, sample, st, gs = rubble_full
    assert (gs.w > 0).sum() > 100_000
    ref = O.importance(gs.radius, gs.w, gs.a)
    assert np.array_equal(gs.c_rad, ref["c_rad"])
    assert np.array_equal(gs.c_vis, ref["c_vis"])
    assert np.array_equal(gs.cull_bits, S.unpack_bits(ref["cull"], sc.n))
    np.testing.assert_allclose(gs.s, ref["s"], rtol=1e-12, atol=0)
    # w and a on the sampled tiles: the oracle composites only those, so a splat lying wholly
    # inside them has comparable totals
    H, W = cam["H"], cam["W"]
    TX = (W + 15) // 16
    rect = st.get("rect").reshape(-1, 4)
    in_sample = np.zeros(sc.n, bool)
    vis = np.nonzero(st.get("radius") > 0)[0]
    r = rect[vis]
    single = (r[:, 2] - r[:, 0] == 1) & (r[:, 3] - r[:, 1] == 1)
    t = r[:, 1] * TX + r[:, 0]
    in_sample[vis[single & (t % 16 == 0)]] = True
    _, _, affected = _flip_info(st, gs, cam, sample)
    in_sample[list(affected)] = False
    assert in_sample.sum() > 1000
    assert np.array_equal(gs.a[in_sample], st.get("a")[in_sample])
    w_o = st.get("w_fixed").astype(np.float64)[in_sample]
    assert np.all(np.abs(gs.w[in_sample].astype(np.float64) - w_o) <= st.get("a")[in_sample] + 1e-5 * w_o)


@pytest.mark.parametrize("city,view", [("residence", 5), ("matrixcity", 2)])
def test_full_size_ragged_configs(city, view):
    """BASELINE configs[3] (Residence-shaped, 8M Gaussians, 1368x912: the last tile column is 8
    pixels wide) and configs[4] (MatrixCity-shaped, 20M Gaussians, 1920x1080: the last tile row is 8
    pixels high) at full size: radius, records, the complete pair sequence and ranges bit-exact;
    pixels, n_contrib, the 9 compositing partials and every parameter gradient on a 1/16 tile sample
    that includes ragged tiles (dL/dC zeroed outside it); c_rad / c_vis / Cull bit-exact on the
    GPU's own w and a."""
    sc = S.gen_city(city)
    cam = sc.cameras[view]
    H, W = cam["H"], cam["W"]
    TX, TY = (W + 15) // 16, (H + 15) // 16
    assert W % 16 == 8 or H % 16 == 8
    sample = _tile_sample(H, W)
    # the sample reaches the ragged column / row (tiles t = 0 mod 16)
    ragged = [t for t in range(0, TX * TY, 16) if t % TX == TX - 1 or t // TX == TY - 1]
    assert ragged
    dl = S.grad_image(H, W) * sample[None]
    st = O.OracleStep(sc, cam, M=1, tile_frac=1.0 / 16, dLdC=dl, threads=16)
    gs = GpuStep(sc, cam, M=1, dLdC=dl)
    try:
        assert np.array_equal(gs.radius, st.get("radius"))
        rec = gs.rank[0]["records"]
        order = np.argsort(rec["gid"])
        valid = np.nonzero(st.get("radius") > 0)[0]
        assert np.array_equal(rec["gid"][order], valid)
        m2 = st.get("mean2d").reshape(-1, 2)[valid]
        assert np.array_equal(rec["mx"][order].view(np.uint32), _f32(m2[:, 0]).view(np.uint32))
        o = gs.rank[0]
        assert np.array_equal(o["key_tile"], st.get("pair_tile", 0))
        assert np.array_equal(o["recv"]["gid"][o["vals"]], st.get("pair_gid", 0))
        assert np.array_equal(o["ranges"][:, 0], st.get("range_lo", 0))
        assert np.array_equal(o["ranges"][:, 1], st.get("range_hi", 0))
        _, flips, affected = _flip_info(st, gs, cam, sample)
        ok = sample & ~flips
        assert ok.sum() > 0.05 * H * W
        img = st.get("img").reshape(3, H, W)
        assert np.abs(gs.img - img)[:, ok].max() <= 1e-4
        assert np.array_equal(gs.nc[ok], st.get("n_contrib").reshape(H, W)[ok])
        # the sampled ragged tiles composited something (their partial blocks are compared above)
        assert sum(int(gs.nc[(t // TX) * 16:(t // TX + 1) * 16, (t % TX) * 16:(t % TX + 1) * 16].sum())
                   for t in ragged) > 0
        _excused_ok(st, gs, affected)
        keep = np.ones(sc.n, bool)
        keep[list(affected)] = False
        _check_g2d(st, gs, keep, city)
        _check_grads(sc.n, st, gs, keep, what=city)
        ref = O.importance(gs.radius, gs.w, gs.a)
        assert np.array_equal(gs.c_rad, ref["c_rad"])
        assert np.array_equal(gs.c_vis, ref["c_vis"])
        assert np.array_equal(gs.cull_bits, S.unpack_bits(ref["cull"], sc.n))
    finally:
        gs.close()


@pytest.mark.parametrize("split", ["default", "0"])
@pytest.mark.parametrize("case", ["empty", "single", "ragged", "behind_and_offscreen", "dense_tile", "faint"])
def test_edge_cases(case, split, monkeypatch):
    if split == "0":  # every tile on the two-pixels-per-lane work unit
        monkeypatch.setenv("BGS_SPLIT_TILES", "0")
    if case == "empty":
        sc = S.gen_small(1, 5, 40, 24)
        sc.means[:, 2] = -3.0  # everything behind the camera
    elif case == "single":
        sc = S.gen_small(2, 1, 33, 33, spread=0.01)
    elif case == "ragged":
        sc = S.gen_tiny(n=3000, W=250, H=181, seed=4)
        sc.cameras = [S.make_camera(250, 181, np.eye(3), np.zeros(3))]
    elif case == "behind_and_offscreen":
        sc = S.gen_small(3, 400, 64, 48, spread=4.0)
    elif case == "faint":
        # the tile footprint (R5): a third of the splats below the alpha cut everywhere (o < 1/255:
        # radius > 0, a record, but no tile), a third faint (footprint far inside the 3DGS rect), the
        # rest strongly anisotropic (footprint a thin band of the rect)
        sc = S.gen_tiny(n=3000, W=128, H=96, seed=6)
        sc.cameras = [S.make_camera(128, 96, np.eye(3), np.zeros(3))]
        k = np.arange(sc.n) % 3
        sc.opac[k == 0] = 0.003
        sc.opac[k == 1] = 0.01
        sc.scales[k == 2] *= np.array([3.0, 0.15, 0.15], np.float32)
    else:
        # thousands of pairs in single tiles (long onesweep runs of one digit, many partitions)
        sc = S.gen_small(4, 9000, 64, 64, spread=0.08, sigma_range=(0.002, 0.01))
    cam = sc.cameras[0]
    dl = S.grad_image(cam["H"], cam["W"], seed=3)
    st = O.OracleStep(sc, cam, dLdC=dl)
    gs = GpuStep(sc, cam, dLdC=dl)
    try:
        assert np.array_equal(gs.radius, st.get("radius"))
        H, W = cam["H"], cam["W"]
        _, flips, _ = _flip_info(st, gs, cam)
        assert np.abs(gs.img - st.get("img").reshape(3, H, W))[:, ~flips].max(initial=0) <= 1e-4
        assert np.array_equal(gs.nc[~flips], st.get("n_contrib").reshape(H, W)[~flips])
        o = gs.rank[0]
        tiles = o["key_tile"]
        assert np.array_equal(tiles, st.get("pair_tile", 0))
        assert np.array_equal(o["recv"]["gid"][o["vals"]], st.get("pair_gid", 0))
        _, flips, affected = _flip_info(st, gs, cam)
        keep = np.ones(sc.n, bool)
        keep[list(affected)] = False
        assert np.array_equal(gs.a[keep], st.get("a")[keep])
        _check_g2d(st, gs, keep, case)
        _check_grads(sc.n, st, gs, keep, what=case)
        if case == "faint":
            rect, rect3 = st.get("rect").reshape(-1, 4), st.get("rect3").reshape(-1, 4)
            vis = gs.radius > 0
            below = vis & (sc.opac.ravel() < 1 / 255)
            assert below.sum() > 100 and np.all(rect[below, 2] == rect[below, 0])  # no tile
            assert np.all(gs.a[below] == 0) and all(np.all(v.reshape(sc.n, -1)[below] == 0) for v in gs.grads.values())
            area = lambda r: (r[:, 2] - r[:, 0]) * (r[:, 3] - r[:, 1])
            assert area(rect[vis]).sum() < 0.7 * area(rect3[vis]).sum()
        if case == "empty":
            assert np.all(gs.img == 0) and np.all(gs.T == 1) and np.all(gs.nc == 0)
            assert gs.rank[0]["q"]["F"] == 0 and gs.rank[0]["q"]["P"] == 0
            assert all(np.all(v == 0) for v in gs.grads.values())
    finally:
        gs.close()


def test_views_in_flight_match_sequential(tiny_scene):
    """Two views on two contexts / streams at once (the bench's views in flight) give the same
    images, counts and cull columns as running them one after the other, and the same gradients
    and scores up to the order of the float reductions."""
    import paper_2605_13794_b200.bgs as B
    sc = tiny_scene
    cams = [sc.cameras[0], S.make_camera(256, 256, np.eye(3), np.array([0.3, -0.2, 0.5]))]
    dev = "cuda"
    n = sc.n
    g = B.GaussianPlanes.from_scene(sc, dev)
    H, W = 256, 256
    dl = torch.from_numpy(S.grad_image(H, W)).to(dev)

    def run(concurrent):
        ctxs = [B.Context(), B.Context()]
        grads = g.zeros_grads()
        s = torch.zeros(n, dtype=torch.float64, device=dev)
        cr = torch.zeros(n, dtype=torch.int32, device=dev)
        cv = torch.zeros(n, dtype=torch.int32, device=dev)
        outs = []
        streams = [torch.cuda.Stream(), torch.cuda.Stream()]
        for k, cam in enumerate(cams):
            o = dict(radius=torch.zeros(n, dtype=torch.int32, device=dev), rgb=torch.zeros(3, H, W, device=dev),
                     T=torch.zeros(H, W, device=dev), nc=torch.zeros(H, W, dtype=torch.int32, device=dev),
                     cull=torch.zeros((n + 31) // 32, dtype=torch.int32, device=dev))
            ctx = ctxs[k] if concurrent else ctxs[0]
            st = streams[k] if concurrent else streams[0]
            B.bgs_view_step(ctx, g, B.camera(cam), None, None, 0, o["radius"], o["rgb"], o["T"], o["nc"], dl, grads,
                            B.importance_out(s, cr, cv, o["cull"]), st)
            outs.append(o)
        torch.cuda.synchronize()
        for c in ctxs:
            c.close()
        return outs, grads, s, cr, cv

    seq = run(False)
    par = run(True)
    for a, b in zip(seq[0], par[0]):
        for k in a:
            assert torch.equal(a[k], b[k]), k
    for name in ("mean_opac", "quat", "scale", "sh"):
        # float atomics make even two sequential runs differ in summation order: the gradient
        # tolerance of the oracle parity tests
        x, y = getattr(seq[1], name), getattr(par[1], name)
        assert torch.all((x - y).abs() <= 1e-3 * x.abs() + 1e-5 * float(x.abs().max())), name
    assert torch.equal(seq[3], par[3]) and torch.equal(seq[4], par[4])
    assert torch.allclose(seq[2], par[2], rtol=1e-12, atol=0)


@pytest.mark.parametrize("split", ["0", "all"])
def test_raster_work_units_parity(tiny_scene, monkeypatch, split):
    """Both compositing work units against the oracle: every tile as one CTA with two pixels per
    lane and the row-half skip (split 0: the path most Rubble tiles take) and every tile as two
    half-tile CTAs with one pixel per lane (the heavy-tile path)."""
    monkeypatch.setenv("BGS_SPLIT_TILES", "0" if split == "0" else "100000")
    sc = tiny_scene
    cam = sc.cameras[0]
    dl = S.grad_image(cam["H"], cam["W"])
    st = O.OracleStep(sc, cam, M=1, dLdC=dl)
    gs = GpuStep(sc, cam, M=1, dLdC=dl)
    try:
        H, W = cam["H"], cam["W"]
        cand, flips, affected = _flip_info(st, gs, cam)
        ok = ~flips
        assert np.abs(gs.img - st.get("img").reshape(3, H, W))[:, ok].max() <= 1e-4
        assert np.array_equal(gs.nc[ok], st.get("n_contrib").reshape(H, W)[ok])
        _excused_ok(st, gs, affected)
        keep = np.ones(sc.n, bool)
        keep[list(affected)] = False
        assert np.array_equal(gs.a[keep], st.get("a")[keep])
        _check_g2d(st, gs, keep, f"split {split}")
        _check_grads(sc.n, st, gs, keep, what=f"split {split}")
    finally:
        gs.close()
