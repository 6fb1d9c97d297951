"""Pins of the CPU oracle against things other than itself.

Each test names the pin and the PAPER.md / SPEC.md passage it follows.  None of the expected
values comes from the CUDA path.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import synthetic as S

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _one_scene(means, quats=None, scales=None, opac=None, sh=None, lod=None, W=33, H=33, R=None, t=None, fx=None):
    n = len(means)
    means = np.asarray(means, np.float32).reshape(n, 3)
    quats = np.tile(np.array([1, 0, 0, 0], np.float32), (n, 1)) if quats is None else np.asarray(quats, np.float32)
    scales = np.full((n, 3), 0.05, np.float32) if scales is None else np.asarray(scales, np.float32).reshape(n, 3)
    opac = np.full(n, 0.5, np.float32) if opac is None else np.asarray(opac, np.float32)
    if sh is None:
        sh = np.zeros((n, 16, 3), np.float32)
    lod = np.zeros(n, np.uint8) if lod is None else np.asarray(lod, np.uint8)
    cam = S.make_camera(W, H, np.eye(3) if R is None else R, np.zeros(3) if t is None else t, fx=fx, fy=fx)
    return S.Scene(means, quats, scales, opac, sh, lod, [cam], d0=1.0), cam


def _albedo_sh(rgb):
    sh = np.zeros((16, 3), np.float32)
    sh[0] = (np.asarray(rgb, np.float64) - 0.5) / S.SH_C0
    return sh


# ------------------------------------------------------------------------------------------
# P2: compositing worked example (Eq.2)
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("M", [1, 3])
def test_P2_two_half_alpha_splats(M):
    ex = GOLDEN["compositing_two_half_alpha"]
    sh = np.stack([_albedo_sh([0.9, 0.2, 0.4]), _albedo_sh([0.1, 0.7, 0.3])])
    sc, cam = _one_scene([[0, 0, 4.0], [0, 0, 5.0]], opac=ex["alpha"], sh=sh)
    st = O.OracleStep(sc, cam, M=M)
    rgb = st.get("rgb").reshape(2, 3)
    img = st.get("img").reshape(3, 33, 33)
    T = st.get("t_final").reshape(33, 33)
    c = 16  # (W-1)/2 is an integer pixel centre: G = 1 there, so alpha = o exactly
    w1, w2 = ex["weights"]
    expect = np.float32(rgb[0] * w1) + np.float32(rgb[1] * w2)
    np.testing.assert_allclose(img[:, c, c], expect, rtol=0, atol=1e-7)
    assert T[c, c] == np.float32(ex["t_final"])
    assert st.get("n_contrib").reshape(33, 33)[c, c] == 2


def test_P2_empty_scene_is_black():
    ex = GOLDEN["compositing_empty"]
    sc, cam = _one_scene([[0, 0, -5.0]])  # behind the camera -> culled -> empty
    st = O.OracleStep(sc, cam)
    assert np.all(st.get("img") == 0.0) and ex["pixel"] == [0.0, 0.0, 0.0]
    assert np.all(st.get("t_final") == np.float32(ex["t_final"]))
    assert np.all(st.get("radius") == 0)
    assert st.get("n_pairs_total")[0] == 0


# ------------------------------------------------------------------------------------------
# P3: closed form for one isotropic Gaussian on the optical axis (EWA; R3, R4)
# ------------------------------------------------------------------------------------------
def _iso_axis(ratio, o=0.8, W=257):
    f = np.float32(0.9 * W)
    z = np.float32(10.0)
    sigma = np.float32(ratio * float(z) / float(f))
    sc, cam = _one_scene([[0, 0, float(z)]], scales=[[sigma] * 3], opac=[o], W=W, H=W)
    return sc, cam, float(f) * float(sigma) / float(z)


def test_P3_isotropic_closed_form_radius_and_conic():
    sc, cam, r = _iso_axis(5.0)
    st = O.OracleStep(sc, cam)
    v = r * r + 0.3
    c = (257 - 1) / 2
    assert tuple(st.get("mean2d")) == (c, c)
    A, B, Cc = st.get("conic")
    assert B == 0.0
    np.testing.assert_allclose([A, Cc], [1 / v, 1 / v], rtol=2e-6)
    # radius = ceil(3 sqrt(v + sqrt(0.1))) = ceil(15.18) = 16 (vanilla 3DGS eigenvalue guard)
    assert st.get("radius")[0] == 16


def test_P3_eigenvalue_guard_changes_radius():
    # f sigma / z = sqrt(15.5): v = 15.8; with the 0.1 guard radius 13, without it 12
    sc, cam, r = _iso_axis(math.sqrt(15.5))
    st = O.OracleStep(sc, cam)
    v = r * r + 0.3
    assert math.ceil(3 * math.sqrt(v)) == 12
    assert st.get("radius")[0] == 13


def test_P3_footprint_lattice_count_and_weight():
    o = 0.8
    sc, cam, r = _iso_axis(5.0, o=o)
    st = O.OracleStep(sc, cam)
    v = r * r + 0.3
    c = 128
    # rect of a radius-16 splat centred on pixel 128: tiles [floor((c-16)/16), floor((c+16+15)/16)) = [7, 9)
    xs = np.arange(7 * 16, 9 * 16)
    dx, dy = np.meshgrid(xs - c, xs - c)
    r2 = (dx * dx + dy * dy).astype(np.float64)
    qual = r2 <= 2 * v * math.log(255 * o)  # alpha = o e^{-r^2/2v} >= 1/255
    a_expect = int(qual.sum())
    w_expect = float(np.sum(np.minimum(0.99, o * np.exp(-r2[qual] / (2 * v)))))
    assert st.get("a")[0] == a_expect
    np.testing.assert_allclose(st.get("w")[0], w_expect, rtol=2e-6)
    # continuum: integral of o e^{-r^2/2v} over the disc = 2 pi v o (1 - 1/(255 o))
    assert abs(w_expect - 2 * math.pi * v * o * (1 - 1 / (255 * o))) / w_expect < 2e-3
    img = st.get("img").reshape(3, 257, 257)
    rgb = st.get("rgb")
    np.testing.assert_allclose(img[:, c, c], min(0.99, o) * rgb, rtol=1e-6)


# ------------------------------------------------------------------------------------------
# P4: covariance Sigma = R(q) S^2 R(q)^T observed through the projection
# ------------------------------------------------------------------------------------------
def _sigma_from_projection(q, s):
    """Recover Sigma from three axis-aligned cameras, each with the Gaussian on its axis."""
    from scipy.spatial.transform import Rotation
    out = {}
    rots = {"z": np.eye(3), "y": Rotation.from_euler("x", 90, degrees=True).as_matrix(),
            "x": Rotation.from_euler("y", -90, degrees=True).as_matrix()}
    for name, Rc in rots.items():
        Rc = Rc.astype(np.float32)
        z = 10.0
        mu = Rc.T.astype(np.float64) @ np.array([0, 0, z])  # world point on this camera's axis
        sc, cam = _one_scene([mu], quats=[q], scales=[s], W=257, H=257, R=Rc)
        st = O.OracleStep(sc, cam)
        A, B, Cc = st.get("conic")
        cov = np.linalg.inv(np.array([[A, B], [B, Cc]])) - 0.3 * np.eye(2)
        f = cam["fx"]
        out[name] = (cov / (f / z) ** 2, Rc.astype(np.float64))
    return out


@pytest.mark.parametrize("case", ["identity", "axis", "random"])
def test_P4_covariance(case):
    from scipy.spatial.transform import Rotation
    rng = np.random.default_rng(3)
    if case == "identity":
        q, s = np.array([1, 0, 0, 0.0]), np.array([1.0, 1.0, 1.0]) * 0.05
    elif case == "axis":
        q, s = np.array([1, 0, 0, 0.0]), np.array([2.0, 1.0, 1.0]) * 0.05
    else:
        q = rng.standard_normal(4)
        q /= np.linalg.norm(q)
        s = rng.uniform(0.02, 0.08, 3)
    q = q.astype(np.float32)
    s = s.astype(np.float32)
    Rq = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()  # scipy is scalar-last
    Sigma = Rq @ np.diag(s.astype(np.float64) ** 2) @ Rq.T
    if case == "identity":
        np.testing.assert_allclose(Sigma, np.eye(3) * 0.05 ** 2, atol=1e-12)
    obs = _sigma_from_projection(q, s)
    for name, (blk, Rc) in obs.items():
        Sc = Rc @ Sigma @ Rc.T  # camera-frame covariance; its xy block is what projects
        np.testing.assert_allclose(blk, Sc[:2, :2], rtol=2e-4, atol=2e-9)
    ev = np.sort(np.linalg.eigvalsh(Sigma))
    np.testing.assert_allclose(ev, np.sort(s.astype(np.float64) ** 2), rtol=1e-6)


# ------------------------------------------------------------------------------------------
# P5: mean2d = direct pinhole projection; cov2d = J_fd Sigma_cam J_fd^T + 0.3 I (EWA, textbook)
# ------------------------------------------------------------------------------------------
def test_P5_projection_matches_pinhole_and_fd_jacobian():
    from scipy.spatial.transform import Rotation
    rng = np.random.default_rng(5)
    n = 200
    Rc = Rotation.from_euler("xyz", [12, -7, 25], degrees=True).as_matrix().astype(np.float32)
    t = np.array([0.3, -0.2, 1.0], np.float32)
    W = H = 128
    pc = np.stack([rng.uniform(-1.2, 1.2, n), rng.uniform(-1.2, 1.2, n), rng.uniform(4, 8, n)], 1)
    mu = ((pc - t) @ Rc.astype(np.float64))  # world = R^T (pc - t)
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    s = rng.uniform(0.03, 0.2, (n, 3))
    sc, cam = _one_scene(mu, quats=q, scales=s, opac=np.full(n, 0.9), W=W, H=H, R=Rc, t=t)
    st = O.OracleStep(sc, cam)
    valid = st.get("radius") > 0
    assert valid.sum() > 150
    fx, fy, cx, cy = cam["fx"], cam["fy"], cam["cx"], cam["cy"]
    R64 = Rc.astype(np.float64)
    mu32 = sc.means.astype(np.float64)
    p = mu32 @ R64.T + t.astype(np.float64)
    m2 = np.stack([fx * p[:, 0] / p[:, 2] + cx, fy * p[:, 1] / p[:, 2] + cy], 1)
    np.testing.assert_allclose(st.get("mean2d").reshape(n, 2)[valid], m2[valid], atol=2e-4)

    def pi(x):
        return np.array([fx * x[0] / x[2] + cx, fy * x[1] / x[2] + cy])

    conic = st.get("conic").reshape(n, 3)
    q32 = sc.quats.astype(np.float64)
    for i in np.nonzero(valid)[0][:60]:
        h = 1e-5
        J = np.stack([(pi(p[i] + h * e) - pi(p[i] - h * e)) / (2 * h) for e in np.eye(3)], 1)
        Rq = Rotation.from_quat([q32[i, 1], q32[i, 2], q32[i, 3], q32[i, 0]]).as_matrix()
        Sig = Rq @ np.diag(sc.scales[i].astype(np.float64) ** 2) @ Rq.T
        cov = J @ (R64 @ Sig @ R64.T) @ J.T + 0.3 * np.eye(2)
        A, B, C_ = conic[i]
        np.testing.assert_allclose(np.linalg.inv(np.array([[A, B], [B, C_]])), cov, rtol=1e-4, atol=1e-5)


# ------------------------------------------------------------------------------------------
# P6: SH basis = real spherical harmonics up to 3DGS's fixed per-function sign
# ------------------------------------------------------------------------------------------
def test_P6_sh_basis_is_real_sph_harm():
    from scipy.special import sph_harm_y
    rng = np.random.default_rng(6)
    dirs = rng.standard_normal((64, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    Yo = np.stack([O.sh_basis(d) for d in dirs])
    theta = np.arccos(np.clip(dirs[:, 2], -1, 1))
    phi = np.arctan2(dirs[:, 1], dirs[:, 0])
    for l in range(4):
        for m in range(-l, l + 1):
            k = l * l + l + m
            Y = sph_harm_y(l, abs(m), theta, phi)
            if m > 0:
                yr = math.sqrt(2) * (-1) ** m * Y.real
            elif m < 0:
                yr = math.sqrt(2) * (-1) ** m * Y.imag
            else:
                yr = Y.real
            np.testing.assert_allclose(np.abs(Yo[:, k]), np.abs(yr), rtol=1e-9, atol=1e-12)
            big = np.abs(yr) > 1e-3
            sg = np.sign(Yo[big, k] * yr[big])
            assert np.all(sg == sg[0]), (l, m)


# ------------------------------------------------------------------------------------------
# P1: tiled oracle == per-pixel brute force over all splats (Eq.2), any M
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("M", [1, 2, 5])
def test_P1_tiled_equals_bruteforce(tiny_scene, M):
    st = O.OracleStep(tiny_scene, tiny_scene.cameras[0], M=M)
    img, T, _ = st.bruteforce()
    assert np.array_equal(img.ravel(), st.get("img"))
    assert np.array_equal(T.ravel(), st.get("t_final"))


# ------------------------------------------------------------------------------------------
# P7: compositing invariants (R10)
# ------------------------------------------------------------------------------------------
def test_P7_transmittance_and_weights(tiny_scene):
    st = O.OracleStep(tiny_scene, tiny_scene.cameras[0])
    T = st.get("t_final")
    assert T.min() >= np.float32(1e-4)  # early stop excludes the splat that would cross 1e-4
    assert (T < 1e-3).mean() > 0.1  # the scene does exercise early termination
    w, wf, a = st.get("w"), st.get("w_fixed"), st.get("a")
    assert np.all(w >= 0)
    assert np.array_equal(w > 0, a > 0) and np.array_equal(wf > 0, a > 0)
    # total visibility mass = total absorbed transmittance (telescoping sum of Eq.2 weights)
    np.testing.assert_allclose(w.sum(), np.sum(1.0 - T.astype(np.float64)), rtol=1e-5)
    # fixed-point w within 2^-25 per contributing pixel term
    assert np.all(np.abs(wf / 2.0 ** 24 - w) <= a * 2.0 ** -25 + 1e-12)


def test_P7_conservation_per_pixel():
    sc = S.gen_tiny(n=3000, seed=9)
    sc.sh[:] = 0
    sc.sh[:, 0, :] = np.float32(0.5 / S.SH_C0)  # every colour ~= 1
    st = O.OracleStep(sc, sc.cameras[0])
    rgb = st.get("rgb").reshape(-1, 3)
    cval = rgb[st.get("radius") > 0][0, 0]
    img = st.get("img").reshape(3, -1).astype(np.float64)
    T = st.get("t_final").astype(np.float64)
    np.testing.assert_allclose(img[0] / cval + T, 1.0, atol=2e-5)


def test_P7_deletion_never_decreases_other_weights(tiny_scene):
    # Removing a splat can only raise the transmittance seen by the splats behind it.  (SPEC
    # S:167 states the inequality the other way round; reading R28.)
    st = O.OracleStep(tiny_scene, tiny_scene.cameras[0])
    w = st.get("w")
    g = int(np.argmax(w))
    keep = np.ones(tiny_scene.n, bool)
    keep[g] = False
    st2 = O.OracleStep(tiny_scene.subset(np.nonzero(keep)[0]), tiny_scene.cameras[0])
    w2 = st2.get("w")
    w1 = w[keep]
    assert np.all(w2 >= w1 * (1 - 1e-5) - 1e-9)
    assert np.any(w2 > w1 * (1 + 1e-3))


# ------------------------------------------------------------------------------------------
# P8: LOD gate (Eq.4-6)
# ------------------------------------------------------------------------------------------
def _level_log_form(d, d0, lmax):
    x = math.log2(d0 / d)
    return max(0, min(lmax, math.floor(x + 0.5)))  # round half up (R18)


def test_P8_level_examples():
    ex = GOLDEN["level_at"]
    d0 = 100.0
    for ratio, level in ex["cases"]:
        d = ratio * d0
        assert _level_log_form(d, d0, 5) == level
        for l in range(0, 4):
            thr_keep = l == 0 or d * d <= O.d2_threshold(d0, l)
            assert thr_keep == (l <= level)


def test_P8_threshold_form_equals_log_form():
    rng = np.random.default_rng(8)
    d0 = 437.5
    n_checked = 0
    for _ in range(200_000):
        d = float(np.float32(d0 * 2.0 ** rng.uniform(-6, 3)))
        l = int(rng.integers(0, 6))
        lmax = int(rng.integers(0, 6))
        x = math.log2(d0 / d)
        if abs((x + 0.5) - round(x + 0.5)) < 1e-6:
            continue  # measure-zero boundary
        d2 = np.float32(np.float32(d) * np.float32(d))
        keep_thr = l <= lmax and (l == 0 or d2 <= np.float32(O.d2_threshold(d0, l)))
        keep_log = l <= _level_log_form(d, d0, lmax)
        assert keep_thr == keep_log
        n_checked += 1
    assert n_checked > 199_000


def test_P8_gate_cull_fallback_sets():
    sc = S.gen_city("rubble", n=20_000, W=320, H=240, V=4)
    cam = sc.cameras[1]
    gate = dict(enabled=1, l_max=3, d0=sc.d0 * 4)
    cull = S.random_cull_column(sc.n, 0.7, seed=4)
    st = O.OracleStep(sc, cam, gate=gate, cull_global=cull, M=2)
    # Eq.5 predicate in fp64 log form, per Gaussian
    d = np.linalg.norm(sc.means.astype(np.float64) - cam["campos"].astype(np.float64), axis=1)
    x = np.log2(gate["d0"] / d)
    Lv = np.clip(np.floor(x + 0.5), 0, gate["l_max"])
    lod_ok = sc.lod <= Lv
    frac = np.abs((x + 0.5) - np.round(x + 0.5))
    ok = frac > 1e-5
    assert np.array_equal(st.get("lod_ok").astype(bool)[ok], lod_ok[ok])
    culled = S.unpack_bits(cull, sc.n)
    n_lod, n_keep, fb = st.get("n_lod"), st.get("n_keep"), st.get("fallback")
    assert not fb.any()
    keep = st.get("keep").astype(bool)
    assert np.array_equal(keep, st.get("lod_ok").astype(bool) & ~culled)  # Eq.6: A = L \ Cull
    sizes = np.array([len(range(m, sc.n, 2)) for m in range(2)])
    assert np.all(n_keep <= n_lod) and np.all(n_lod <= sizes)
    ex = GOLDEN["active_set"]
    assert sorted(set(ex["gate_pass"]) - set(ex["cull"])) == ex["active"]
    # all-level-0 shard: the gate keeps everything -> ratio 1 > 0.95 -> fallback
    sc0 = sc.subset(np.arange(sc.n))
    sc0.lod = np.zeros(sc.n, np.uint8)
    st0 = O.OracleStep(sc0, cam, gate=gate, M=2)
    assert st0.get("fallback").all()


# ------------------------------------------------------------------------------------------
# P9: sort / ranges / routing completeness (Eq.2 order P:156; R12)
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("M", [1, 4])
def test_P9_pairs_complete_sorted_and_routed(tiny_scene, M):
    st = O.OracleStep(tiny_scene, tiny_scene.cameras[0], M=M)
    rect = st.get("rect").reshape(-1, 4)
    radius = st.get("radius")
    depth = st.get("depth")
    TX = 16
    expected = set()
    for i in np.nonzero(radius > 0)[0]:
        x0, y0, x1, y1 = rect[i]
        for y in range(y0, y1):
            for x in range(x0, x1):
                expected.add((y * TX + x, int(i)))
    got = []
    owner = st.get("owner")
    for r in range(M):
        tiles, gids = st.get("pair_tile", r), st.get("pair_gid", r)
        b, e = st.get("tile_range", r)
        assert np.all((tiles >= b) & (tiles < e)) and np.all(owner[b:e] == r)
        for q in range(1, len(tiles)):  # (tile, depth, gid) strictly increasing
            k0 = (tiles[q - 1], depth[gids[q - 1]], gids[q - 1])
            k1 = (tiles[q], depth[gids[q]], gids[q])
            assert k0 < k1
        lo, hi = st.get("range_lo", r), st.get("range_hi", r)
        for lt in range(e - b):
            sel = np.nonzero(tiles == b + lt)[0]
            if len(sel):
                assert lo[lt] == sel[0] and hi[lt] == sel[-1] + 1 and len(sel) == hi[lt] - lo[lt]
            else:
                assert lo[lt] == hi[lt] == 0
        got += list(zip(tiles.tolist(), gids.tolist()))
    assert len(got) == len(expected) and set(got) == expected
    F = int((radius > 0).sum())
    mask = st.get("dest_mask")
    counts = st.get("counts").reshape(M, M)
    D = int(sum(bin(int(v)).count("1") for v in mask))
    assert counts.sum() == D <= M * F
    recv_total = sum(len(st.get("recv", r)) for r in range(M))
    assert recv_total == D
    # a splat is routed to r iff one of its tiles is owned by r
    for i in np.nonzero(radius > 0)[0][:500]:
        x0, y0, x1, y1 = rect[i]
        owners = {int(owner[y * TX + x]) for y in range(y0, y1) for x in range(x0, x1)}
        assert owners == {r for r in range(M) if mask[i] >> r & 1}


def test_P9_shard_map_golden():
    ex = GOLDEN["shard_map"]
    sc = S.gen_small(0, ex["n"], 16, 16)
    assert np.array_equal(np.arange(ex["n"])[ex["rank"]::ex["M"]], ex["owned"])
    sh = sc.shard(ex["rank"], ex["M"])
    np.testing.assert_array_equal(sh.means, sc.means[ex["owned"]])


# ------------------------------------------------------------------------------------------
# P10: distributed invariance "identical to what a single-GPU renderer would produce"
# ------------------------------------------------------------------------------------------
def test_P10_M_invariance(tiny_scene):
    dl = S.grad_image(256, 256)
    ref = O.OracleStep(tiny_scene, tiny_scene.cameras[0], M=1, dLdC=dl)
    for M in (2, 3, 4, 8):
        st = O.OracleStep(tiny_scene, tiny_scene.cameras[0], M=M, dLdC=dl)
        for f in ("img", "t_final", "n_contrib", "w_fixed", "a", "radius"):
            assert np.array_equal(st.get(f), ref.get(f)), (M, f)
        np.testing.assert_allclose(st.get("d_mean"), ref.get("d_mean"), rtol=1e-9, atol=1e-15)


def test_threaded_oracle_is_bit_identical(tiny_scene):
    """The multi-core baseline (bench.py cpu_baseline) runs the same oracle with host threads:
    every output, including the fp64 sums, must be bit-identical to the sequential run."""
    dl = S.grad_image(256, 256)
    for M in (1, 3):
        ref = O.OracleStep(tiny_scene, tiny_scene.cameras[0], M=M, dLdC=dl, threads=1)
        st = O.OracleStep(tiny_scene, tiny_scene.cameras[0], M=M, dLdC=dl, threads=4)
        for f in ("img", "t_final", "n_contrib", "et_margin", "w", "w_fixed", "a", "radius", "g2d", "d_mean",
                  "d_quat", "d_scale", "d_opac", "d_sh", "margins"):
            assert np.array_equal(st.get(f), ref.get(f)), (M, f)


def test_tile_partition_invariants(tiny_scene):
    """Reading R24 (P:170 cites Scaling-3DGS without an algorithm): parity unpinned beyond these."""
    for M in (1, 2, 3, 4, 8):
        st = O.OracleStep(tiny_scene, tiny_scene.cameras[0], M=M)
        owner = st.get("owner")
        c = st.get("tile_pairs").astype(np.int64) + 1
        assert owner[0] == 0 and np.all(np.diff(owner) >= 0) and owner.max() <= M - 1
        run = np.bincount(owner, weights=c, minlength=M)
        assert run.max() <= c.sum() / M + c.max() + 1e-9


# ------------------------------------------------------------------------------------------
# P12: importance (Eq.3; c_rad / c_vis / Cull P:132; R15-R17)
# ------------------------------------------------------------------------------------------
def test_P12_golden_single_and_uncovered():
    ex = GOLDEN["importance_single"]
    r = O.importance([5, 0], [int(ex["w"] * 2 ** 24), 0], [ex["a"], 0])
    np.testing.assert_allclose(r["s"][0], ex["s"], rtol=1e-8)
    assert r["c_rad"][0] == ex["c_rad"] and r["c_vis"][0] == ex["c_vis"]
    ex0 = GOLDEN["importance_uncovered"]
    assert r["s"][1] == ex0["s"] and (r["cull"][0] >> 1 & 1) == ex0["cull"]


def test_P12_mass_cut_golden():
    ex = GOLDEN["mass_cut_prefix"]
    w = [int(v * 2 ** 30) for v in ex["scores"]]
    r = O.importance([1] * 4, w, [1] * 4, mass_num=ex["target_num"], mass_den=ex["target_den"])
    assert r["in_set"].sum() == ex["retained"]


def test_P12_selection_vs_sort_and_scan():
    rng = np.random.default_rng(12)
    for trial in range(20):
        n = int(rng.integers(1, 3000))
        w = rng.integers(0, 50, n).astype(np.uint64) * rng.integers(0, 2, n).astype(np.uint64)
        if trial % 3 == 0:
            w = (w * np.uint64(1 << 30)).astype(np.uint64)
        a = np.where(w > 0, rng.integers(1, 100, n), 0).astype(np.uint32)
        rad = np.where(a > 0, 3, rng.integers(0, 2, n) * 3).astype(np.int32)
        r = O.importance(rad, w, a)
        # independent sort-and-scan in Python integers
        pop = sorted((int(v), i) for i, v in enumerate(w) if v > 0)
        pop.sort(key=lambda t: (-t[0], t[1]))
        total = sum(v for v, _ in pop)
        chosen, pref = set(), 0
        for v, i in pop:
            if total == 0 or 100 * pref >= 99 * total:
                break
            chosen.add(i)
            pref += v
        assert set(np.nonzero(r["in_set"])[0].tolist()) == chosen
        assert np.all(r["c_vis"] <= r["c_rad"])
        culled = S.unpack_bits(r["cull"], n)
        assert np.array_equal(culled, ~r["in_set"])
        if total:
            assert 100 * int(w[~r["in_set"]].sum()) <= total  # culled mass <= 1%
        s_expect = np.where(a > 0, (w.astype(np.float64) / 2 ** 24) / (a + 1e-8), 0.0)
        np.testing.assert_allclose(r["s"], s_expect, rtol=1e-12)


# ------------------------------------------------------------------------------------------
# P17: the alpha-cut threshold thr = -ln(255 o) (SPEC S:137 alpha_min = 1/255; D3) is computed
# with a fixed-sequence fp64 ln (reading R30) so that both sides round the same value; pinned
# here against libm's correctly rounded log, not against itself.
# ------------------------------------------------------------------------------------------
def test_P17_fixed_ln_matches_libm():
    rng = np.random.default_rng(17)
    u = np.concatenate([np.exp(rng.uniform(np.log(1e-6), np.log(1e6), 20000)),
                        255.0 * rng.uniform(0.0, 1.0, 20000).astype(np.float32).astype(np.float64),
                        [1.0, 2.0, 0.5, 255.0, math.sqrt(2.0), math.nextafter(math.sqrt(2.0), 2.0)]])
    u = u[u > 0]
    for x in u:
        got, ref = O.ln_fixed(float(x)), math.log(float(x))
        # within 2 ulp of the correctly rounded value (the series truncation is < 1e-19 relative)
        assert abs(got - ref) <= 2 * math.ulp(ref) + 1e-300, (x, got, ref)
    assert O.ln_fixed(1.0) == 0.0
    for k in range(-20, 21):
        assert abs(O.ln_fixed(2.0 ** k) - k * math.log(2.0)) <= math.ulp(k * math.log(2.0)) + 1e-300


def test_P17_threshold_bits():
    """thr(o) is float32(-ln(255 o)): equal to the rounding of libm's value except where that
    double lies within an ulp of a float rounding boundary (then one float ulp apart at most);
    and alpha >= 1/255 <=> power >= thr on a dense grid of powers."""
    rng = np.random.default_rng(3)
    o = np.concatenate([rng.uniform(0.004, 1.0, 20000), [1.0 / 255 + 1e-7, 0.5, 0.99, 1.0 - 1e-7]]).astype(np.float32)
    same = 0
    for v in o:
        t = O.thr(float(v))
        ref = np.float32(-math.log(255.0 * float(v)))
        assert abs(np.float64(t) - np.float64(ref)) <= np.spacing(np.float32(abs(ref)) + np.float32(1e-30)), v
        same += t == ref
    assert same >= len(o) - 2
    for v in (0.05, 0.3, 0.8):
        t = O.thr(v)
        p = np.float64(np.float32(t))
        # a power just above thr keeps alpha above 1/255 (up to the float rounding of thr)
        assert np.float32(v) * math.exp(p + 1e-6) >= 1.0 / 255 * (1 - 1e-6)
        assert np.float32(v) * math.exp(p - 1e-3) < 1.0 / 255


# ------------------------------------------------------------------------------------------
# P6b: the SH colour is evaluated along the viewing ray, camera -> Gaussian (3DGS convention,
# d = (mu - c_v)/|mu - c_v|).  A splat whose only view-dependent term is the band-1 x
# function is brighter seen from the side where the ray runs along +x; a reversed direction
# (c_v - mu) swaps the two colours.
# ------------------------------------------------------------------------------------------
def test_P6b_view_direction_sign():
    mu = np.array([[0.3, -0.2, 0.1]], np.float32)
    k_x = None
    Yx = O.sh_basis([1.0, 0.0, 0.0])
    for k in (1, 2, 3):  # the band-1 function that varies along x (P6: real SH up to sign)
        if abs(Yx[k]) > 0.4:
            k_x = k
    assert k_x is not None and abs(O.sh_basis([0, 1.0, 0])[k_x]) < 1e-12
    sh = np.zeros((1, 16, 3), np.float32)
    sh[0, k_x, 0] = 0.2 / Yx[k_x]  # red = 0.5 + 0.2 x_dir
    out = {}
    for side, f in (("minus_x", 1.0), ("plus_x", -1.0)):
        pos = mu[0].astype(np.float64) - 5.0 * f * np.array([1.0, 0, 0])
        R = np.array([[0, 1, 0], [0, 0, f], [f, 0, 0]], np.float64)  # rows right, down, forward = f e_x
        assert np.isclose(np.linalg.det(R), 1.0)
        sc, _ = _one_scene(mu, sh=sh, W=33, H=33)
        cam = S.make_camera(33, 33, R, -R @ pos)
        sc.cameras = [cam]
        st = O.OracleStep(sc, cam)
        assert st.get("radius")[0] > 0
        out[side] = st.get("rgb").reshape(-1, 3)[0, 0]
    # camera on the -x side: the ray camera -> Gaussian runs along +x
    assert abs(out["minus_x"] - 0.7) < 1e-6 and abs(out["plus_x"] - 0.3) < 1e-6, out


# ------------------------------------------------------------------------------------------
# P18: the tile footprint (reading R5) = the 3DGS rect cut to the box of the alpha >= 1/255
# ellipse.  Pinned against the alpha test written out in fp64 numpy (Eq.2's N(p) membership,
# R9: alpha = o exp(power) >= 1/255), not against the oracle's own box: every pixel centre of the
# 3DGS rect where a splat passes the cut must lie in one of its footprint tiles.  P1 (tiled ==
# brute force over the 3DGS rects, any M) pins the same property through the rendered image.
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("seed", [1, 2])
def test_P18_footprint_holds_every_passing_pixel(seed):
    sc = S.gen_tiny(seed=seed, n=3000)
    cam = sc.cameras[0]
    st = O.OracleStep(sc, cam)
    TX = (cam["W"] + 15) // 16
    rad = st.get("radius")
    fp = st.get("rect").reshape(-1, 4)
    r3 = st.get("rect3").reshape(-1, 4)
    m2 = st.get("mean2d").reshape(-1, 2)
    con = st.get("conic").reshape(-1, 3)
    opac = sc.opac.astype(np.float64).ravel()
    valid = np.nonzero(rad > 0)[0]
    assert np.all(fp[valid, 0] >= r3[valid, 0]) and np.all(fp[valid, 1] >= r3[valid, 1])
    assert np.all(fp[valid, 2] <= r3[valid, 2]) and np.all(fp[valid, 3] <= r3[valid, 3])
    area = lambda r: np.maximum(r[:, 2] - r[:, 0], 0) * np.maximum(r[:, 3] - r[:, 1], 0)
    a_fp, a_r3 = area(fp[valid]).sum(), area(r3[valid]).sum()
    assert a_fp < 0.95 * a_r3  # the cut does remove tiles on this (anisotropic, low-opacity) scene
    checked = 0
    for i in valid:
        x0, y0, x1, y1 = r3[i]
        if (x1 - x0) * (y1 - y0) > 9:
            continue
        xs = np.arange(x0 * 16, min(x1 * 16, cam["W"]))
        ys = np.arange(y0 * 16, min(y1 * 16, cam["H"]))
        dx = m2[i, 0] - xs[None, :]
        dy = m2[i, 1] - ys[:, None]
        A, B, C = con[i]
        power = -0.5 * (A * dx * dx + C * dy * dy) - B * dx * dy
        passing = (power <= 0) & (opac[i] * np.exp(power) >= 1.0 / 255.0 * (1 + 1e-6))
        py, px = np.nonzero(passing)
        tx, ty = xs[px] // 16, ys[py] // 16
        inside = (tx >= fp[i, 0]) & (tx < fp[i, 2]) & (ty >= fp[i, 1]) & (ty < fp[i, 3])
        assert inside.all(), (i, fp[i], r3[i])
        checked += 1
    assert checked > 1000
