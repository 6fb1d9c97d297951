"""ctypes wrapper of the CPU oracle (oracle/bgs_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package never imports this module.
Parity status of every function is listed in DESIGN.md §5 ("Oracle pins").
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bgs_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

CXXFLAGS = ["-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["g++", *CXXFLAGS, "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


class _Scene(C.Structure):
    _fields_ = [("n", C.c_int64), ("mean", C.c_void_p), ("quat", C.c_void_p), ("scale", C.c_void_p),
                ("opac", C.c_void_p), ("sh", C.c_void_p), ("lod", C.c_void_p)]


class _Camera(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("W", C.c_int32), ("H", C.c_int32), ("R", C.c_float * 9), ("t", C.c_float * 3),
                ("campos", C.c_float * 3), ("near_clip", C.c_float)]


class _Gate(C.Structure):
    _fields_ = [("enabled", C.c_int32), ("l_max", C.c_int32), ("d0", C.c_double),
                ("fb_num", C.c_int32), ("fb_den", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.or_step.restype = C.c_void_p
        _lib.or_step.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                C.c_int32]
        _lib.or_free.argtypes = [C.c_void_p]
        _lib.or_set_threads.restype = C.c_int32
        _lib.or_set_threads.argtypes = [C.c_int32]
        _lib.or_get.restype = C.c_int64
        _lib.or_get.argtypes = [C.c_void_p, C.c_char_p, C.c_int32, C.c_void_p]
        _lib.or_d2_threshold.restype = C.c_float
        _lib.or_d2_threshold.argtypes = [C.c_double, C.c_int32]
        _lib.or_thr.restype = C.c_float
        _lib.or_thr.argtypes = [C.c_float]
        _lib.or_ln.restype = C.c_double
        _lib.or_ln.argtypes = [C.c_double]
        _lib.or_sh_basis.argtypes = [C.c_double, C.c_double, C.c_double, C.c_void_p]
        _lib.or_bruteforce.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.or_importance.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    return _lib


def set_threads(n: int) -> int:
    """Host threads of the oracle's per-Gaussian and per-tile loops (1 = sequential).  Results are
    bit-identical for every count (bgs_oracle.cpp: tile increments replayed in tile order).
    Returns the count in effect."""
    return int(lib().or_set_threads(int(n)))


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _camera(cam: dict) -> _Camera:
    c = _Camera()
    c.fx, c.fy, c.cx, c.cy = cam["fx"], cam["fy"], cam["cx"], cam["cy"]
    c.W, c.H = cam["W"], cam["H"]
    c.R[:] = [float(v) for v in np.asarray(cam["R"], np.float32).ravel()]
    c.t[:] = [float(v) for v in np.asarray(cam["t"], np.float32).ravel()]
    c.campos[:] = [float(v) for v in np.asarray(cam["campos"], np.float32).ravel()]
    c.near_clip = cam["near"]
    return c


_FIELD_DTYPES = {
    "lod_ok": np.uint8, "keep": np.uint8, "n_lod": np.int64, "n_keep": np.int64, "fallback": np.int64,
    "radius": np.int32, "tile_pairs": np.int32, "owner": np.int32, "dest_mask": np.uint8, "counts": np.int64,
    "img": np.float32, "t_final": np.float32, "n_contrib": np.int32, "et_margin": np.float32, "w": np.float64,
    "w_fixed": np.uint64, "a": np.uint32, "g2d": np.float64, "d_mean": np.float64, "d_quat": np.float64,
    "d_scale": np.float64, "d_opac": np.float64, "d_sh": np.float64, "n_pairs_total": np.int64,
    "mean2d": np.float64, "conic": np.float64, "depth": np.float64, "rgb": np.float64, "thr": np.float64,
    "rect": np.int32, "rect3": np.int32, "phase_seconds": np.float64, "img64": np.float64, "margins": np.float64, "tile_range": np.int32, "recv": np.int64, "pair_tile": np.int32, "pair_gid": np.int64,
    "range_lo": np.int64, "range_hi": np.int64,
}

NO_COLOR = 1
F64 = 2


class OracleStep:
    """One simulated view step at M ranks (O1..O11 of DESIGN.md §5)."""

    def __init__(self, scene, cam: dict, gate: dict | None = None, cull_global: np.ndarray | None = None,
                 M: int = 1, flags: int = 0, dLdC: np.ndarray | None = None, tile_frac: float = 1.0,
                 threads: int = 1):
        L = lib()
        self._keep = []
        n = scene.n
        arrs = [np.ascontiguousarray(scene.means, np.float32), np.ascontiguousarray(scene.quats, np.float32),
                np.ascontiguousarray(scene.scales, np.float32), np.ascontiguousarray(scene.opac, np.float32),
                np.ascontiguousarray(scene.sh, np.float32).reshape(n, 48), np.ascontiguousarray(scene.lod, np.uint8)]
        self._keep += arrs
        sc = _Scene(n, *[_ptr(a) for a in arrs])
        cm = _camera(cam)
        g = gate or {}
        gt = _Gate(int(g.get("enabled", 0)), int(g.get("l_max", 31)), float(g.get("d0", 1.0)),
                   int(g.get("fb_num", 19)), int(g.get("fb_den", 20)))
        cull = None if cull_global is None else np.ascontiguousarray(cull_global, np.uint32)
        dl = None if dLdC is None else np.ascontiguousarray(dLdC, np.float32)
        self._keep += [cull, dl]
        self.M = M
        self.n = n
        self.cam = cam
        self.threads = set_threads(threads)
        t0 = time.perf_counter()
        stride = max(1, int(round(1.0 / tile_frac)))
        try:
            self._h = L.or_step(C.byref(sc), C.byref(cm), C.byref(gt), _ptr(cull), M, flags, _ptr(dl), stride)
        finally:
            set_threads(1)
        self.seconds = time.perf_counter() - t0

    def get(self, name: str, rank: int = 0) -> np.ndarray:
        L = lib()
        cnt = L.or_get(self._h, name.encode(), rank, None)
        if cnt < 0:
            raise KeyError(name)
        out = np.empty(cnt, dtype=_FIELD_DTYPES[name])
        L.or_get(self._h, name.encode(), rank, _ptr(out))
        return out

    def seconds_by_phase(self) -> dict:
        v = self.get("phase_seconds")
        return dict(project=float(v[0]), route_sort=float(v[1]), composite=float(v[2]), project_bwd=float(v[3]))

    def bruteforce(self):
        H, W = self.cam["H"], self.cam["W"]
        img = np.zeros((3, H, W), np.float32)
        T = np.zeros((H, W), np.float32)
        cnt = np.zeros((H, W), np.int32)
        lib().or_bruteforce(self._h, _ptr(img), _ptr(T), _ptr(cnt))
        return img, T, cnt

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().or_free(self._h)
                self._h = None
        except Exception:
            pass


def d2_threshold(d0: float, l: int) -> float:
    return float(lib().or_d2_threshold(d0, l))


def thr(o: float) -> float:
    """O3 alpha-cut threshold thr = (float)(-ln(255 o)) with the oracle's fixed-sequence ln."""
    return float(lib().or_thr(float(o)))


def ln_fixed(u: float) -> float:
    return float(lib().or_ln(float(u)))


def sh_basis(d) -> np.ndarray:
    Y = np.zeros(16, np.float64)
    lib().or_sh_basis(float(d[0]), float(d[1]), float(d[2]), _ptr(Y))
    return Y


def importance(radius, w_fixed, a, s=None, c_rad=None, c_vis=None, mass_num=99, mass_den=100):
    """O12 (Eq.3, c_rad/c_vis/Cull).  Global arrays in gid order.  Returns dict."""
    n = len(radius)
    radius = np.ascontiguousarray(radius, np.int32)
    w_fixed = np.ascontiguousarray(w_fixed, np.uint64)
    a = np.ascontiguousarray(a, np.uint32)
    s = np.zeros(n, np.float64) if s is None else np.array(s, np.float64)
    c_rad = np.zeros(n, np.uint32) if c_rad is None else np.array(c_rad, np.uint32)
    c_vis = np.zeros(n, np.uint32) if c_vis is None else np.array(c_vis, np.uint32)
    cull = np.zeros((n + 31) // 32, np.uint32)
    in_set = np.zeros(n, np.uint8)
    lib().or_importance(n, _ptr(radius), _ptr(w_fixed), _ptr(a), mass_num, mass_den, _ptr(s), _ptr(c_rad),
                        _ptr(c_vis), _ptr(cull), _ptr(in_set))
    return dict(s=s, c_rad=c_rad, c_vis=c_vis, cull=cull, in_set=in_set.astype(bool))
