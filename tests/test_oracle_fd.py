"""P11: the oracle's analytic backward (O9-O11) against fp64 central finite differences.

PAPER.md P:161 "Training optimizes these primitive attributes", "gradients propagate
through both the rasterizer and the screen-space routing"; SPEC S:151 / S:585 (FD check on a
10-Gaussian 32x32 scene, h = 1e-4 relative).  The forward here is the pure-fp64
instantiation of the oracle (flag F64), so the FD quotient is exact to ~1e-9.  Scenes are
chosen away from every discontinuity (alpha cut, 0.99 clamp, early stop, integer radius and
rect): the test asserts the margins before differencing.
"""
import numpy as np

import oracle as O
import synthetic as S

GROUPS = ("means", "quats", "scales", "opac", "sh")
GRAD_NAME = {"means": "d_mean", "quats": "d_quat", "scales": "d_scale", "opac": "d_opac", "sh": "d_sh"}


def _loss(scene, cam, dl, M=1):
    st = O.OracleStep(scene, cam, M=M, flags=O.F64, dLdC=dl)
    return float(np.dot(st.get("img64"), dl.ravel().astype(np.float64))), st


def _safe(st, h_scale):
    thr, clamp, integ = st.get("margins")
    T = st.get("t_final")
    return thr > 50 * h_scale and clamp > 50 * h_scale and integ > 1e-3 and T.min() > 0.05


def _scene(seed, n=10, W=32, rot=False, clamp_case=False):
    sc = S.gen_small(seed, n, W, W, spread=1.0, depth=6.0, sigma_range=(0.08, 0.35), opac_range=(0.25, 0.6))
    if rot:
        from scipy.spatial.transform import Rotation
        Rc = Rotation.from_euler("xyz", [10, -15, 20], degrees=True).as_matrix()
        t = np.array([0.2, -0.1, 0.5])
        pc = sc.means.astype(np.float64)
        sc.means = ((pc - t) @ Rc).astype(np.float32)  # so that R mu + t = pc
        sc.cameras = [S.make_camera(W, W, Rc, t)]
    if clamp_case:
        # centre beyond the +-1.3 tan(fov/2) clamp, large enough to still cover the image
        sc.means[0] = np.array([5.5, 0.3, 6.0], np.float32)
        sc.scales[0] = np.array([1.6, 1.2, 1.4], np.float32)
        sc.opac[0] = np.float32(0.3)
    return sc


def _find_safe_scene(**kw):
    for seed in range(200):
        sc = _scene(seed, **kw)
        dl = S.grad_image(sc.cameras[0]["H"], sc.cameras[0]["W"], seed=seed + 1, sigma=1.0)
        L0, st = _loss(sc, sc.cameras[0], dl)
        rad = st.get("radius")
        if kw.get("clamp_case") and rad[0] == 0:
            continue
        if (rad > 0).sum() >= 0.8 * sc.n and _safe(st, 1e-5) and st.get("rgb").reshape(-1, 3)[rad > 0].min() > 0.02:
            return sc, dl, st
    raise AssertionError("no discontinuity-free scene found")


def _fd_check(sc, dl, st, rel_h=1e-6, rtol=1e-4):
    cam = sc.cameras[0]
    worst = {}
    for g in GROUPS:
        arr = getattr(sc, g)
        ana = st.get(GRAD_NAME[g]).reshape(arr.shape[0], -1)
        flat = arr.reshape(arr.shape[0], -1)
        gmax = np.abs(ana).max()
        assert gmax > 0, g
        errs = []
        for i in range(arr.shape[0]):
            if st.get("radius")[i] == 0:
                assert np.all(ana[i] == 0)
                continue
            for j in range(flat.shape[1]):
                x0 = flat[i, j]
                h = np.float32(max(abs(float(x0)), 0.05) * rel_h)
                xp, xm = np.float32(x0 + h), np.float32(x0 - h)
                flat[i, j] = xp
                Lp, _ = _loss(sc, cam, dl)
                flat[i, j] = xm
                Lm, _ = _loss(sc, cam, dl)
                flat[i, j] = x0
                fd = (Lp - Lm) / (float(xp) - float(xm))
                err = abs(fd - ana[i, j])
                assert err <= rtol * abs(ana[i, j]) + 1e-6 * gmax, (g, i, j, fd, ana[i, j])
                errs.append(err / (rtol * abs(ana[i, j]) + 1e-6 * gmax))
        worst[g] = max(errs) if errs else 0.0
    return worst


def test_P11_fd_identity_camera():
    sc, dl, st = _find_safe_scene(n=8)
    w = _fd_check(sc, dl, st)
    assert all(v <= 1.0 for v in w.values()), w
    assert w["means"] < 1e-2 and w["quats"] < 1e-2  # geometry grads: FD agreement far inside the bar


def test_P11_fd_rotated_camera():
    sc, dl, st = _find_safe_scene(n=6, rot=True)
    _fd_check(sc, dl, st)


def test_P11_fd_jacobian_clamp_true_derivative():
    sc, dl, st = _find_safe_scene(n=4, clamp_case=True)
    # the first Gaussian is clamped in x: check its position gradient (true clamp derivative, R8)
    fx, cx = sc.cameras[0]["fx"], sc.cameras[0]["cx"]
    lim = (32 - cx) / fx + 0.3 * (0.5 * 32 / fx)
    assert sc.means[0, 0] / sc.means[0, 2] > lim
    _fd_check(sc, dl, st)


def test_P11_zero_upstream_gives_zero_grads():
    sc = _scene(3)
    dl = np.zeros((3, 32, 32), np.float32)
    st = O.OracleStep(sc, sc.cameras[0], flags=O.F64, dLdC=dl)
    for g in GROUPS:
        assert np.all(st.get(GRAD_NAME[g]) == 0)


def test_P11_fp32_backward_matches_fp64_backward():
    """The parity reference (fp32 forward decisions, fp64 backward) agrees with the pure-fp64
    path on a smooth scene: the fp32 forward only perturbs the Jacobians at ~1e-7."""
    sc, dl, st64 = _find_safe_scene(n=10)
    st32 = O.OracleStep(sc, sc.cameras[0], dLdC=dl)
    for g in GROUPS:
        a, b = st32.get(GRAD_NAME[g]), st64.get(GRAD_NAME[g])
        np.testing.assert_allclose(a, b, rtol=1e-4, atol=1e-5 * np.abs(b).max())
