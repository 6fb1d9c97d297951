"""Seeded synthetic inputs for the BlitzGS per-view splatting step.

This module is the ONLY thing shared between the CUDA path (``paper_2605_13794_b200``)
and the CPU oracle (``oracle/``).  It produces *inputs* only: Gaussian parameters
(already activated: unit quaternions, positive scales, opacities in (0,1)), SH
coefficients, LOD labels, cameras and the upstream image gradient dL/dC.  It holds
none of the method's arithmetic (no projection, no compositing, no gate).

Recipes follow SURVEY.md §8(d) ("Synthetic aerial-city generator"); the paper
publishes no per-view statistics (§4, P:336 names only the datasets), so
every distribution below is a stated choice, repeated in DESIGN.md §3.

Array conventions (numpy, C-contiguous):
  means  float32 [N,3]   world position (z up for the city scenes)
  quats  float32 [N,4]   unit quaternion (w, x, y, z)
  scales float32 [N,3]   per-axis standard deviation (> 0)
  opac   float32 [N]     opacity in (0, 1)
  sh     float32 [N,16,3] SH degree-3 coefficients, coefficient-major, RGB inner
  lod    uint8   [N]     LOD label in [0, K-1]
Camera (dict): fx, fy, cx, cy (float), W, H (int), R float32[3,3] world->camera
(row-major; camera looks along +z, x right, y down), t float32[3],
campos float32[3] (= -R^T t, the camera centre c_v of Eq. 5), near (float).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SH_C0 = 0.28209479177387814  # only used to *encode* an albedo into the DC coefficient


@dataclass
class Scene:
    means: np.ndarray
    quats: np.ndarray
    scales: np.ndarray
    opac: np.ndarray
    sh: np.ndarray
    lod: np.ndarray
    cameras: list = field(default_factory=list)
    d0: float = 1.0
    k_levels: int = 1
    name: str = "scene"

    @property
    def n(self) -> int:
        return int(self.means.shape[0])

    def subset(self, idx: np.ndarray) -> "Scene":
        return Scene(self.means[idx], self.quats[idx], self.scales[idx], self.opac[idx],
                     self.sh[idx], self.lod[idx], self.cameras, self.d0, self.k_levels, self.name)

    def shard(self, rank: int, world: int) -> "Scene":
        """Index-parity shard G^(m) = {g_i : i mod M = m} (§3.2)."""
        return self.subset(np.arange(rank, self.n, world))


# ----------------------------------------------------------------------------------------
# rotations (input construction only)
# ----------------------------------------------------------------------------------------

def matrix_to_quat(Rm: np.ndarray) -> np.ndarray:
    """Rotation matrices [N,3,3] (columns = local axes in world) -> unit quats (w,x,y,z)."""
    Rm = np.asarray(Rm, dtype=np.float64)
    n = Rm.shape[0]
    q = np.empty((n, 4), dtype=np.float64)
    tr = Rm[:, 0, 0] + Rm[:, 1, 1] + Rm[:, 2, 2]
    m0 = tr > 0
    s = np.sqrt(np.maximum(tr[m0] + 1.0, 1e-30)) * 2
    q[m0, 0] = 0.25 * s
    q[m0, 1] = (Rm[m0, 2, 1] - Rm[m0, 1, 2]) / s
    q[m0, 2] = (Rm[m0, 0, 2] - Rm[m0, 2, 0]) / s
    q[m0, 3] = (Rm[m0, 1, 0] - Rm[m0, 0, 1]) / s
    rest = ~m0
    i0 = rest & (Rm[:, 0, 0] > Rm[:, 1, 1]) & (Rm[:, 0, 0] > Rm[:, 2, 2])
    s = np.sqrt(np.maximum(1.0 + Rm[i0, 0, 0] - Rm[i0, 1, 1] - Rm[i0, 2, 2], 1e-30)) * 2
    q[i0, 0] = (Rm[i0, 2, 1] - Rm[i0, 1, 2]) / s
    q[i0, 1] = 0.25 * s
    q[i0, 2] = (Rm[i0, 0, 1] + Rm[i0, 1, 0]) / s
    q[i0, 3] = (Rm[i0, 0, 2] + Rm[i0, 2, 0]) / s
    i1 = rest & ~i0 & (Rm[:, 1, 1] > Rm[:, 2, 2])
    s = np.sqrt(np.maximum(1.0 + Rm[i1, 1, 1] - Rm[i1, 0, 0] - Rm[i1, 2, 2], 1e-30)) * 2
    q[i1, 0] = (Rm[i1, 0, 2] - Rm[i1, 2, 0]) / s
    q[i1, 1] = (Rm[i1, 0, 1] + Rm[i1, 1, 0]) / s
    q[i1, 2] = 0.25 * s
    q[i1, 3] = (Rm[i1, 1, 2] + Rm[i1, 2, 1]) / s
    i2 = rest & ~i0 & ~i1
    s = np.sqrt(np.maximum(1.0 + Rm[i2, 2, 2] - Rm[i2, 0, 0] - Rm[i2, 1, 1], 1e-30)) * 2
    q[i2, 0] = (Rm[i2, 1, 0] - Rm[i2, 0, 1]) / s
    q[i2, 1] = (Rm[i2, 0, 2] + Rm[i2, 2, 0]) / s
    q[i2, 2] = (Rm[i2, 1, 2] + Rm[i2, 2, 1]) / s
    q[i2, 3] = 0.25 * s
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return q


def random_quats(rng: np.random.Generator, n: int) -> np.ndarray:
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return q


def _normalize_f32_quats(q: np.ndarray) -> np.ndarray:
    q = np.asarray(q, dtype=np.float64)
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    return q.astype(np.float32)


# ----------------------------------------------------------------------------------------
# cameras
# ----------------------------------------------------------------------------------------

def make_camera(W: int, H: int, R: np.ndarray, t: np.ndarray, fx: float | None = None,
                fy: float | None = None, cx: float | None = None, cy: float | None = None,
                near: float = 0.01) -> dict:
    fx = 0.9 * W if fx is None else fx
    fy = 0.9 * W if fy is None else fy
    cx = (W - 1) / 2.0 if cx is None else cx
    cy = (H - 1) / 2.0 if cy is None else cy
    R = np.asarray(R, dtype=np.float32).reshape(3, 3)
    t = np.asarray(t, dtype=np.float32).reshape(3)
    campos = (-(R.astype(np.float64).T @ t.astype(np.float64))).astype(np.float32)
    return dict(fx=float(np.float32(fx)), fy=float(np.float32(fy)), cx=float(np.float32(cx)),
                cy=float(np.float32(cy)), W=int(W), H=int(H), R=R, t=t, campos=campos,
                near=float(np.float32(near)))


def look_camera(W: int, H: int, pos: np.ndarray, yaw: float, pitch: float, **kw) -> dict:
    """Camera at `pos` (world, z up) heading `yaw`, pitched `pitch` (negative = down)."""
    f = np.array([math.cos(pitch) * math.cos(yaw), math.cos(pitch) * math.sin(yaw), math.sin(pitch)])
    r = np.array([math.sin(yaw), -math.cos(yaw), 0.0])
    d = np.cross(f, r)
    R = np.stack([r, d, f])  # rows: camera x (right), y (down), z (forward)
    t = -R @ np.asarray(pos, dtype=np.float64)
    return make_camera(W, H, R, t, **kw)


def grad_image(H: int, W: int, seed: int = 7, sigma: float = 1e-3) -> np.ndarray:
    """Upstream dL/dC: seeded Gaussian noise [3,H,W] float32."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return (rng.standard_normal((3, H, W), dtype=np.float32) * np.float32(sigma)).astype(np.float32)


def target_image(H: int, W: int, seed: int = 9) -> np.ndarray:
    """Ground-truth image I_b of Eq.7 for the supervision tests and bench: seeded smooth colour
    field (a few random plane waves per channel) plus pixel noise, clipped to [0, 1], float32
    [3,H,W].  No method arithmetic."""
    rng = np.random.Generator(np.random.PCG64(seed))
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    img = np.empty((3, H, W), np.float64)
    for c in range(3):
        f = 0.45 + np.zeros((H, W))
        for _ in range(4):
            kx, ky = rng.uniform(-0.08, 0.08, 2)
            f += rng.uniform(0.05, 0.15) * np.sin(kx * xx + ky * yy + rng.uniform(0, 2 * np.pi))
        img[c] = f + 0.05 * rng.standard_normal((H, W))
    return np.clip(img, 0.0, 1.0).astype(np.float32)


# ----------------------------------------------------------------------------------------
# tiny scene (configs[0])
# ----------------------------------------------------------------------------------------

def _sh_from_albedo(rng, albedo: np.ndarray, noise: float = 0.05) -> np.ndarray:
    n = albedo.shape[0]
    sh = np.zeros((n, 16, 3), dtype=np.float32)
    sh[:, 0, :] = ((albedo + rng.normal(0, noise, (n, 3)) - 0.5) / SH_C0).astype(np.float32)
    for l in (1, 2, 3):
        lo, hi = l * l, (l + 1) * (l + 1)
        sh[:, lo:hi, :] = rng.normal(0, 0.05 * 2.0 ** (-l), (n, hi - lo, 3)).astype(np.float32)
    return sh


def _opacity(rng, n: int) -> np.ndarray:
    """Mixture 0.6*Beta(4,1.5) + 0.4*U(0.02,0.5) (SURVEY.md §8(d) 'Opacity')."""
    pick = rng.random(n) < 0.6
    o = np.where(pick, rng.beta(4.0, 1.5, n), rng.uniform(0.02, 0.5, n))
    return np.clip(o, 0.005, 0.995).astype(np.float32)


def gen_tiny(seed: int = 1, n: int = 10_000, W: int = 256, H: int = 256, k_levels: int = 4) -> Scene:
    """configs[0]: 10k Gaussians in a 4x4x4 box centred 6 units in front of one 256x256
    camera (fx=fy=0.9W), radii ~3-40 px, dense centre so early termination triggers."""
    rng = np.random.Generator(np.random.PCG64(seed))
    # dense centre: half from a narrow normal, half uniform in the box
    m1 = rng.normal(0.0, 0.6, (n // 2, 3))
    m2 = rng.uniform(-2.0, 2.0, (n - n // 2, 3))
    means = np.concatenate([m1, m2])
    means = np.clip(means, -2.0, 2.0)
    means[:, 2] += 6.0
    rng.shuffle(means)
    # world sigma for a ~3..40 px radius at z~6, f=230: f*s/z in [0.5, 13]
    base = np.exp(rng.uniform(math.log(0.012), math.log(0.33), n))
    aniso = np.exp(rng.normal(0.0, 0.35, (n, 3)))
    scales = (base[:, None] * aniso).astype(np.float32)
    quats = _normalize_f32_quats(random_quats(rng, n))
    opac = _opacity(rng, n)
    sh = _sh_from_albedo(rng, rng.uniform(0.05, 0.95, (n, 3)))
    lod = rng.integers(0, k_levels, n).astype(np.uint8)
    cam = make_camera(W, H, np.eye(3), np.zeros(3))
    return Scene(means.astype(np.float32), quats, scales, opac, sh, lod, [cam], d0=6.0,
                 k_levels=k_levels, name="tiny")


def gen_small(seed: int, n: int, W: int, H: int, spread: float = 1.0, depth: float = 6.0,
              sigma_range=(0.05, 0.3), opac_range=(0.3, 0.9)) -> Scene:
    """Small hand-sized scenes for finite-difference and edge-case tests."""
    rng = np.random.Generator(np.random.PCG64(seed))
    means = rng.uniform(-spread, spread, (n, 3))
    means[:, 2] = depth + rng.uniform(-spread, spread, n)
    scales = rng.uniform(sigma_range[0], sigma_range[1], (n, 3)).astype(np.float32)
    quats = _normalize_f32_quats(random_quats(rng, n))
    opac = rng.uniform(opac_range[0], opac_range[1], n).astype(np.float32)
    sh = _sh_from_albedo(rng, rng.uniform(0.2, 0.8, (n, 3)))
    sh[:, 1:, :] *= 4.0
    lod = np.zeros(n, dtype=np.uint8)
    cam = make_camera(W, H, np.eye(3), np.zeros(3), fx=0.9 * W, fy=0.9 * W)
    return Scene(means.astype(np.float32), quats, scales, opac, sh, lod, [cam], d0=depth,
                 k_levels=1, name=f"small{n}")


# ----------------------------------------------------------------------------------------
# aerial city (configs[1..4])
# ----------------------------------------------------------------------------------------

CITY_CONFIGS = {
    # name: (N, W, H, grid G, occupancy p_b, scene seed)
    "rubble": (6_000_000, 1152, 864, 24, 0.25, 11),
    "building": (8_000_000, 1152, 864, 32, 0.5, 12),
    "residence": (8_000_000, 1368, 912, 40, 0.6, 13),
    "matrixcity": (20_000_000, 1920, 1080, 64, 0.7, 14),
}


def _heightfield(rng, L):
    k = rng.uniform(0.5, 4.0, (8, 2)) * (2 * math.pi / L)
    ph = rng.uniform(0, 2 * math.pi, 8)
    amp = 0.01 * L / 8.0

    def h(x, y):
        z = np.zeros_like(x)
        for i in range(8):
            z += amp * np.sin(k[i, 0] * x + k[i, 1] * y + ph[i])
        return z

    def grad(x, y):
        gx = np.zeros_like(x)
        gy = np.zeros_like(x)
        for i in range(8):
            c = amp * np.cos(k[i, 0] * x + k[i, 1] * y + ph[i])
            gx += c * k[i, 0]
            gy += c * k[i, 1]
        return gx, gy

    return h, grad


def _frames_from_normals(nrm: np.ndarray, rng) -> np.ndarray:
    """Orthonormal frames [N,3,3] with columns (t1, t2, n), random in-plane angle."""
    n = nrm / np.linalg.norm(nrm, axis=1, keepdims=True)
    a = np.where(np.abs(n[:, 2:3]) < 0.9, np.array([[0, 0, 1.0]]), np.array([[1.0, 0, 0]]))
    t1 = np.cross(a, n)
    t1 /= np.linalg.norm(t1, axis=1, keepdims=True)
    t2 = np.cross(n, t1)
    th = rng.uniform(0, 2 * math.pi, n.shape[0])[:, None]
    u1 = np.cos(th) * t1 + np.sin(th) * t2
    u2 = np.cross(n, u1)
    return np.stack([u1, u2, n], axis=2)


def gen_city(name: str = "rubble", n: int | None = None, W: int | None = None, H: int | None = None,
             V: int = 64, K: int = 6, seed: int | None = None, L: float = 1000.0) -> Scene:
    """Seeded aerial-city scene: ground heightfield + G x G building grid,
    Gaussians on surfaces by area (ground .45, roofs .20, facades .30, vegetation .05),
    K LOD levels with P(l) ~ 2^l and tangent sigma s0*2^-l*LogNormal(0,.25), normal sigma
    0.15*tangent, V cameras on a lawnmower path (altitude U(.25L,.4L), pitch U(-90,-40) deg,
    fx=fy=0.9W).  d0 = median camera->centroid distance (reading R19)."""
    N0, W0, H0, G, pb, seed0 = CITY_CONFIGS[name]
    n = N0 if n is None else n
    W = W0 if W is None else W
    H = H0 if H is None else H
    seed = seed0 if seed is None else seed
    rng = np.random.Generator(np.random.PCG64(seed))
    hfun, hgrad = _heightfield(rng, L)

    # --- buildings
    cell = L / G
    occ = rng.random((G, G)) < pb
    bi, bj = np.nonzero(occ)
    nb = bi.size
    fw = rng.uniform(0.4, 0.8, nb) * cell
    fd = rng.uniform(0.4, 0.8, nb) * cell
    cxb = (bi + 0.5) * cell + rng.uniform(-0.1, 0.1, nb) * cell
    cyb = (bj + 0.5) * cell + rng.uniform(-0.1, 0.1, nb) * cell
    hb = np.exp(rng.normal(math.log(0.03 * L), 0.6, nb))
    base = hfun(cxb, cyb)
    albedo_b = rng.uniform(0.15, 0.9, (nb, 3))

    # --- cameras (lawnmower)
    cams = []
    rows = max(1, int(round(math.sqrt(V / 2))))
    per_row = int(math.ceil(V / rows))
    crng = np.random.Generator(np.random.PCG64(seed + 1000))
    for v in range(V):
        r = v // per_row
        c = v % per_row
        frac = (c + 0.5) / per_row
        if r % 2 == 1:
            frac = 1 - frac
        x = 0.1 * L + 0.8 * L * frac
        y = 0.1 * L + 0.8 * L * (r + 0.5) / rows
        z = crng.uniform(0.25 * L, 0.4 * L)
        yaw = 0.0 if r % 2 == 0 else math.pi
        yaw += crng.uniform(-0.3, 0.3)
        pitch = math.radians(crng.uniform(-90.0, -40.0))
        cams.append(look_camera(W, H, np.array([x, y, z]), yaw, pitch))
    centroid = np.array([L / 2, L / 2, 0.0])
    d0 = float(np.median([np.linalg.norm(c["campos"] - centroid) for c in cams]))
    f = 0.9 * W
    s0 = 4.0 * d0 / f  # level-0 splats ~12 px radius at d0: 3*f*s0/d0 = 12

    # --- category counts
    n_ground = int(0.45 * n)
    n_roof = int(0.20 * n) if nb else 0
    n_fac = int(0.30 * n) if nb else 0
    n_veg = n - n_ground - n_roof - n_fac

    means = np.empty((n, 3), dtype=np.float64)
    normals = np.empty((n, 3), dtype=np.float64)
    albedo = np.empty((n, 3), dtype=np.float64)
    o = 0
    # ground
    gx = rng.uniform(0, L, n_ground)
    gy = rng.uniform(0, L, n_ground)
    means[o:o + n_ground] = np.stack([gx, gy, hfun(gx, gy)], 1)
    dx, dy = hgrad(gx, gy)
    normals[o:o + n_ground] = np.stack([-dx, -dy, np.ones_like(dx)], 1)
    albedo[o:o + n_ground] = np.array([0.35, 0.38, 0.3]) + rng.normal(0, 0.08, (n_ground, 3))
    o += n_ground
    if nb:
        # roofs by area
        area = fw * fd
        b = rng.choice(nb, n_roof, p=area / area.sum())
        u = rng.uniform(-0.5, 0.5, (n_roof, 2))
        means[o:o + n_roof] = np.stack([cxb[b] + u[:, 0] * fw[b], cyb[b] + u[:, 1] * fd[b], base[b] + hb[b]], 1)
        normals[o:o + n_roof] = np.array([0, 0, 1.0])
        albedo[o:o + n_roof] = albedo_b[b] * 0.8
        o += n_roof
        # facades by area (4 walls per building)
        wall_len = np.stack([fw, fd, fw, fd], 1)
        wall_area = (wall_len * hb[:, None]).ravel()
        wsel = rng.choice(nb * 4, n_fac, p=wall_area / wall_area.sum())
        b = wsel // 4
        side = wsel % 4
        u = rng.uniform(-0.5, 0.5, n_fac)
        hz = rng.uniform(0, 1, n_fac) * hb[b] + base[b]
        px = np.where(side == 0, cxb[b] + u * fw[b], np.where(side == 2, cxb[b] + u * fw[b],
                      np.where(side == 1, cxb[b] + 0.5 * fw[b], cxb[b] - 0.5 * fw[b])))
        py = np.where(side == 0, cyb[b] - 0.5 * fd[b], np.where(side == 2, cyb[b] + 0.5 * fd[b],
                      cyb[b] + u * fd[b]))
        means[o:o + n_fac] = np.stack([px, py, hz], 1)
        nx = np.where(side == 1, 1.0, np.where(side == 3, -1.0, 0.0))
        ny = np.where(side == 0, -1.0, np.where(side == 2, 1.0, 0.0))
        normals[o:o + n_fac] = np.stack([nx, ny, np.zeros_like(nx)], 1)
        albedo[o:o + n_fac] = albedo_b[b]
        o += n_fac
    # vegetation blobs near the ground
    vx = rng.uniform(0, L, n_veg)
    vy = rng.uniform(0, L, n_veg)
    means[o:o + n_veg] = np.stack([vx, vy, hfun(vx, vy) + rng.uniform(0.5, 8.0, n_veg)], 1)
    normals[o:o + n_veg] = rng.standard_normal((n_veg, 3)) + 1e-6
    albedo[o:o + n_veg] = np.array([0.2, 0.45, 0.15]) + rng.normal(0, 0.06, (n_veg, 3))
    o += n_veg
    assert o == n

    # --- LOD levels P(l) ~ 2^l and scales
    pl = 2.0 ** np.arange(K)
    lod = rng.choice(K, n, p=pl / pl.sum()).astype(np.uint8)
    sig_t = s0 * 2.0 ** (-lod.astype(np.float64)) * np.exp(rng.normal(0, 0.25, n))
    aniso = np.exp(rng.normal(0, 0.2, (n, 2)))
    scales = np.stack([sig_t * aniso[:, 0], sig_t * aniso[:, 1], 0.15 * sig_t], 1).astype(np.float32)
    frames = _frames_from_normals(normals, rng)
    quats = matrix_to_quat(frames)
    veg = np.zeros(n, dtype=bool)
    veg[n - n_veg:] = True
    quats[veg] = random_quats(rng, int(veg.sum()))
    quats = _normalize_f32_quats(quats)

    perm = rng.permutation(n)  # global ids carry no spatial order (index parity is not spatial)
    means = means[perm].astype(np.float32)
    quats = quats[perm]
    scales = scales[perm]
    lod = lod[perm]
    albedo = np.clip(albedo[perm], 0.02, 0.98)
    opac = _opacity(rng, n)
    sh = np.empty((n, 16, 3), dtype=np.float32)
    CH = 1 << 20
    for s in range(0, n, CH):
        e = min(n, s + CH)
        sh[s:e] = _sh_from_albedo(rng, albedo[s:e])
    return Scene(means, quats, scales, opac, sh, lod, cams, d0=d0, k_levels=K, name=name)


def random_cull_column(n: int, keep_frac: float, seed: int) -> np.ndarray:
    """A seeded Cull column (1 = culled) packed into uint32 words, bit j of word j//32."""
    rng = np.random.Generator(np.random.PCG64(seed))
    bits = rng.random(n) >= keep_frac
    return pack_bits(bits)


def pack_bits(bits: np.ndarray) -> np.ndarray:
    bits = np.asarray(bits, dtype=bool)
    nw = (bits.size + 31) // 32
    padded = np.zeros(nw * 32, dtype=bool)
    padded[:bits.size] = bits
    b = padded.reshape(nw, 32).astype(np.uint64)
    words = (b << np.arange(32, dtype=np.uint64)).sum(axis=1).astype(np.uint32)
    return words


def unpack_bits(words: np.ndarray, n: int) -> np.ndarray:
    words = np.asarray(words, dtype=np.uint32)
    b = (words[:, None] >> np.arange(32, dtype=np.uint32)) & 1
    return b.ravel()[:n].astype(bool)
