"""Thin ctypes binding of libbgs (include/bgs.h): argument marshalling only.

Every step of the per-view path runs in the sm_100a kernels of libbgs.so.  PyTorch supplies
device memory (tensors), streams and, for world > 1, the process group used to broadcast the
NCCL unique id.  There is no CPU fallback: if libbgs.so is missing, importing this module
raises; if no CUDA device is present, every call returns BGS_ERR_CUDA and raises BgsError.
Function names follow the C ABI (bgs_project, bgs_route, ...).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# BGS_LIB selects an in-tree A/B variant (libbgs_<name>.so, build.py --name); default libbgs.so
LIB_PATH = os.path.join(_HERE, os.path.basename(os.environ.get("BGS_LIB", "libbgs.so")))

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libbgs.so not built ({LIB_PATH}); run `python -m paper_2605_13794_b200.build` "
                      "(or __graft_entry__.build()) — there is no CPU fallback")
_lib = C.CDLL(LIB_PATH)

BGS_NO_COLOR = 1
BGS_IMPORTANCE = 2
BGS_GRAPH = 4
BGS_IMPORTANCE_ONLY = 8
BGS_Q_COUNT = 14
Q_NAMES = ("n_local", "n_lod", "n_active", "F", "D", "R", "P", "tile_begin", "tile_end", "fallback",
           "sort_passes", "P_all", "width", "height")
STATUS = {0: "BGS_OK", 1: "BGS_ERR_INVALID_ARGUMENT", 2: "BGS_ERR_CAPACITY", 3: "BGS_ERR_CUDA",
          4: "BGS_ERR_NCCL", 5: "BGS_ERR_CONTRACT", 6: "BGS_ERR_INTERNAL"}
DEBUG = {"records": 0, "rec_lidx": 1, "recv": 2, "keys": 3, "vals": 4, "ranges": 5, "acc": 6, "acc_local": 7,
         "owner": 8, "dest_mask": 9, "tile_pairs": 10, "counters": 11}


class BgsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class bgs_camera(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("width", C.c_int32), ("height", C.c_int32), ("R", C.c_float * 9), ("t", C.c_float * 3),
                ("campos", C.c_float * 3), ("near_clip", C.c_float)]


class bgs_batch_view(C.Structure):
    _fields_ = [("cam", bgs_camera), ("cull_column", C.c_void_p), ("radius_out", C.c_void_p), ("rgb", C.c_void_p),
                ("t_final", C.c_void_p), ("n_contrib", C.c_void_p), ("dL_drgb", C.c_void_p),
                ("cull_out", C.c_void_p), ("sup", C.c_void_p), ("dL_scratch", C.c_void_p)]


class bgs_gaussians(C.Structure):
    _fields_ = [("n_local", C.c_int64), ("mean_opac", C.c_void_p), ("quat", C.c_void_p), ("scale", C.c_void_p),
                ("sh", C.c_void_p), ("lod", C.c_void_p), ("bounds", C.c_void_p)]


class bgs_gaussian_grads(C.Structure):
    _fields_ = [("mean_opac", C.c_void_p), ("quat", C.c_void_p), ("scale", C.c_void_p), ("sh", C.c_void_p)]


class bgs_lod_gate(C.Structure):
    _fields_ = [("enabled", C.c_int32), ("l_max", C.c_int32), ("d0", C.c_double), ("fallback_num", C.c_int32),
                ("fallback_den", C.c_int32)]


class bgs_importance_out(C.Structure):
    _fields_ = [("s", C.c_void_p), ("c_rad", C.c_void_p), ("c_vis", C.c_void_p), ("cull_out", C.c_void_p),
                ("mass_num", C.c_int32), ("mass_den", C.c_int32)]


class bgs_gaussians_out(C.Structure):
    _fields_ = [("capacity", C.c_int64), ("mean_opac", C.c_void_p), ("quat", C.c_void_p), ("scale", C.c_void_p),
                ("sh", C.c_void_p), ("lod", C.c_void_p)]


_vp = C.c_void_p
_SIGS = {
    "bgs_get_unique_id": [_vp],
    "bgs_ctx_create": [C.c_int32, C.c_int32, _vp, C.c_int32, _vp],
    "bgs_ctx_create_local_group": [C.c_int32, C.c_int32, _vp],
    "bgs_ctx_destroy": [_vp],
    "bgs_query": [_vp, _vp],
    "bgs_debug_buffer": [_vp, C.c_int32, _vp, _vp],
    "bgs_project": [_vp, _vp, _vp, _vp, _vp, C.c_uint32, _vp, _vp],
    "bgs_route": [_vp, _vp, _vp, _vp, _vp],
    "bgs_sort_tiles": [_vp, _vp],
    "bgs_raster_fwd": [_vp, C.c_uint32, _vp, _vp, _vp, _vp],
    "bgs_raster_bwd": [_vp, _vp, _vp, _vp, _vp],
    "bgs_route_reverse": [_vp, C.c_uint32, _vp],
    "bgs_project_bwd": [_vp, _vp, _vp, _vp, _vp],
    "bgs_importance": [_vp, C.c_int64, _vp, _vp, _vp, C.c_int32, C.c_int32, _vp, _vp, _vp, _vp, _vp],
    "bgs_view_step": [_vp, _vp, _vp, _vp, _vp, C.c_uint32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "bgs_view_step_host": [_vp, _vp, _vp, _vp, _vp, C.c_uint32, _vp, _vp, _vp, _vp, _vp, _vp],
    "bgs_view_step_host_async": [_vp, _vp, _vp, _vp, _vp, C.c_uint32, _vp, _vp, _vp, _vp, _vp, _vp],
    "bgs_spatial_order": [_vp, _vp, C.c_int64, _vp, _vp],
    "bgs_set_stage_timing": [_vp, C.c_int32],
    "bgs_stage_times": [_vp, _vp],
    "bgs_score_phi": [_vp, C.c_int64, _vp, _vp, _vp, _vp],
    "bgs_prune_stochastic": [_vp, C.c_int64, _vp, C.c_int64, C.c_uint64, _vp, _vp],
    "bgs_prune_mass_cut": [_vp, C.c_int64, _vp, C.c_int32, C.c_int32, _vp, _vp, _vp],
    "bgs_redistribute": [_vp, _vp, _vp, _vp, _vp, _vp],
    "bgs_shard_sizes": [_vp, C.c_int64, _vp],
    "bgs_loss_photo": [_vp, _vp, _vp, C.c_float, C.c_float, _vp, _vp, _vp],
    "bgs_loss_scale": [_vp, _vp, C.c_float, _vp, _vp, _vp],
    "bgs_train_view_step": [_vp, _vp, _vp, _vp, _vp, C.c_uint32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "bgs_adam_step": [_vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "bgs_densify_accumulate": [_vp, C.c_int64, _vp, _vp, _vp, _vp],
    "bgs_visibility_mask": [_vp, C.c_int64, _vp, _vp, _vp],
    "bgs_shard_bounds": [_vp, _vp, _vp, _vp],
    "bgs_batch_step": [_vp, C.c_int32, _vp, _vp, C.c_uint32, _vp, _vp, _vp, _vp],
    "bgs_batch_view_ctx": [_vp, C.c_int32, _vp],
    "bgs_batch_stats": [_vp, _vp],
    "bgs_densify_apply": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "bgs_train_view_step_host_async": [_vp, _vp, _vp, _vp, _vp, C.c_uint32, _vp, _vp, C.c_float, C.c_float, C.c_float,
                                       _vp, _vp, _vp, _vp],
}
for _name, _args in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = C.c_int
_lib.bgs_last_error.argtypes = [_vp]
_lib.bgs_last_error.restype = C.c_char_p
_lib.bgs_launch_count.argtypes = [_vp]
_lib.bgs_launch_count.restype = C.c_int64
_lib.bgs_host_sync_count.argtypes = [_vp]
_lib.bgs_host_sync_count.restype = C.c_int64

EXPORTS = tuple(_SIGS) + ("bgs_last_error", "bgs_launch_count", "bgs_host_sync_count")


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return C.c_void_p(t.data_ptr())
    if isinstance(t, np.ndarray):
        return t.ctypes.data_as(C.c_void_p)
    return t


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    if isinstance(stream, torch.cuda.Stream):
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(int(stream))


# ------------------------------------------------------------------------------------------
# context
# ------------------------------------------------------------------------------------------
class Context:
    """One rank's bgs_ctx.  world > 1: pass the 128-byte NCCL unique id (see unique_id())."""

    def __init__(self, rank: int = 0, world: int = 1, device: int = 0, nccl_uid: bytes | None = None, _handle=None):
        self.rank, self.world, self.device = rank, world, device
        if _handle is not None:
            self._h = _handle
            return
        h = C.c_void_p()
        uid = None if nccl_uid is None else C.create_string_buffer(bytes(nccl_uid), 128)
        st = _lib.bgs_ctx_create(rank, world, uid, device, C.byref(h))
        if st != 0:
            raise BgsError(st, "bgs_ctx_create")
        self._h = h

    @staticmethod
    def local_group(world: int, device: int = 0) -> list["Context"]:
        arr = (C.c_void_p * world)()
        st = _lib.bgs_ctx_create_local_group(world, device, arr)
        if st != 0:
            raise BgsError(st, "bgs_ctx_create_local_group")
        return [Context(r, world, device, _handle=C.c_void_p(arr[r])) for r in range(world)]

    @property
    def handle(self):
        return self._h

    def check(self, st: int, what: str):
        if st != 0:
            raise BgsError(st, f"{what}: {_lib.bgs_last_error(self._h).decode(errors='replace')}")

    def host_syncs(self) -> int:
        return int(_lib.bgs_host_sync_count(self._h))

    def launches(self) -> int:
        return int(_lib.bgs_launch_count(self._h))

    def query(self) -> dict:
        out = (C.c_int64 * BGS_Q_COUNT)()
        self.check(_lib.bgs_query(self._h, out), "bgs_query")
        return dict(zip(Q_NAMES, list(out)))

    def debug_buffer(self, name: str, dtype=torch.uint8) -> torch.Tensor:
        """Copy of an arena intermediate (parity tests only)."""
        p = C.c_void_p()
        nbytes = C.c_int64()
        self.check(_lib.bgs_debug_buffer(self._h, DEBUG[name], C.byref(p), C.byref(nbytes)), "bgs_debug_buffer")
        n = int(nbytes.value)
        out = torch.empty(n, dtype=torch.uint8, device=f"cuda:{self.device}")
        if n and p.value:
            torch.cuda.synchronize(self.device)
            st = _cudart().cudaMemcpy(C.c_void_p(out.data_ptr()), p, C.c_size_t(n), 3)  # device to device
            if int(st) != 0:
                raise RuntimeError(f"cudaMemcpy failed: {st}")
            # a device-to-device cudaMemcpy does not block the host, and it runs on the legacy
            # stream, which torch's non-blocking streams do not wait for: finish it before `out` is used
            torch.cuda.synchronize(self.device)
        return out.view(dtype) if n else out

    def close(self):
        if getattr(self, "_h", None) and not getattr(self, "_borrowed", False):
            _lib.bgs_ctx_destroy(self._h)
        self._h = None

    def batch_view(self, b: int) -> "Context":
        """Borrowed Context of view slot b of the last bgs_batch_step (query / debug_buffer only)."""
        h = C.c_void_p()
        self.check(_lib.bgs_batch_view_ctx(self._h, int(b), C.byref(h)), "bgs_batch_view_ctx")
        c = Context(self.rank, self.world, self.device, _handle=h)
        c._borrowed = True
        return c

    def batch_stats(self) -> dict:
        out = (C.c_int64 * 6)()
        self.check(_lib.bgs_batch_stats(self._h, out), "bgs_batch_stats")
        return dict(zip(("host_syncs", "collectives", "batches", "graph_launches", "graph_instantiations",
                         "graph_fallbacks"), list(out)))


_CUDART = None


def _cudart():
    """The CUDA runtime torch already loaded (for raw device-to-device copies of debug views)."""
    global _CUDART
    if _CUDART is None:
        import glob
        cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                                       "libcudart.so*")) + ["libcudart.so.12", "libcudart.so"]
        for c in cands:
            try:
                _CUDART = C.CDLL(c)
                break
            except OSError:
                continue
        if _CUDART is None:
            raise RuntimeError("libcudart not found")
        _CUDART.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
        _CUDART.cudaMemcpy.restype = C.c_int
    return _CUDART


def unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = _lib.bgs_get_unique_id(buf)
    if st != 0:
        raise BgsError(st, "bgs_get_unique_id")
    return buf.raw


# ------------------------------------------------------------------------------------------
# structs
# ------------------------------------------------------------------------------------------
def camera(cam: dict) -> bgs_camera:
    c = bgs_camera()
    c.fx, c.fy, c.cx, c.cy = cam["fx"], cam["fy"], cam["cx"], cam["cy"]
    c.width, c.height = int(cam["W"]), int(cam["H"])
    c.R[:] = [float(v) for v in np.asarray(cam["R"], np.float32).ravel()]
    c.t[:] = [float(v) for v in np.asarray(cam["t"], np.float32).ravel()]
    c.campos[:] = [float(v) for v in np.asarray(cam["campos"], np.float32).ravel()]
    c.near_clip = float(cam["near"])
    return c


def lod_gate(enabled: bool = False, l_max: int = 31, d0: float = 1.0, num: int = 19, den: int = 20) -> bgs_lod_gate:
    return bgs_lod_gate(int(enabled), int(l_max), float(d0), int(num), int(den))


class GaussianPlanes:
    """Activated parameters of one shard in the ABI layout (float4 rows, SH [n][48])."""

    def __init__(self, mean_opac, quat, scale, sh, lod, bounds=None):
        self.mean_opac, self.quat, self.scale, self.sh, self.lod = mean_opac, quat, scale, sh, lod
        self.bounds = bounds  # optional block bounds (bgs_shard_bounds) for hierarchical culling
        self.n = int(mean_opac.shape[0])

    @staticmethod
    def from_arrays(means, opac, quats, scales, sh, lod, device="cuda") -> "GaussianPlanes":
        n = int(np.asarray(means).shape[0])
        mo = np.empty((n, 4), np.float32)
        mo[:, :3] = means
        mo[:, 3] = opac
        sc = np.zeros((n, 4), np.float32)
        sc[:, :3] = scales
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)
        return GaussianPlanes(t(mo), t(np.asarray(quats, np.float32)), t(sc),
                              t(np.asarray(sh, np.float32).reshape(n, 48)), t(np.asarray(lod, np.uint8)))

    @staticmethod
    def from_scene(scene, device="cuda") -> "GaussianPlanes":
        return GaussianPlanes.from_arrays(scene.means, scene.opac, scene.quats, scene.scales, scene.sh, scene.lod,
                                          device)

    def struct(self) -> bgs_gaussians:
        return bgs_gaussians(self.n, self.mean_opac.data_ptr(), self.quat.data_ptr(), self.scale.data_ptr(),
                             self.sh.data_ptr(), self.lod.data_ptr(),
                             self.bounds.data_ptr() if self.bounds is not None else None)

    def zeros_grads(self) -> "GradPlanes":
        z = lambda t: torch.zeros_like(t, dtype=torch.float32)
        return GradPlanes(z(self.mean_opac), z(self.quat), z(self.scale), z(self.sh))


class GradPlanes:
    def __init__(self, mean_opac, quat, scale, sh):
        self.mean_opac, self.quat, self.scale, self.sh = mean_opac, quat, scale, sh

    def struct(self) -> bgs_gaussian_grads:
        return bgs_gaussian_grads(self.mean_opac.data_ptr(), self.quat.data_ptr(), self.scale.data_ptr(),
                                  self.sh.data_ptr())

    def zero_(self):
        for t in (self.mean_opac, self.quat, self.scale, self.sh):
            t.zero_()


# ------------------------------------------------------------------------------------------
# the ABI calls (same names as include/bgs.h)
# ------------------------------------------------------------------------------------------
def bgs_project(ctx: Context, g: GaussianPlanes, cam: bgs_camera, gate: bgs_lod_gate | None, cull_column,
                flags: int, radius_out: torch.Tensor, stream=None):
    gs = g.struct()
    ctx.check(_lib.bgs_project(ctx.handle, C.byref(gs), C.byref(cam), C.byref(gate) if gate is not None else None,
                               _ptr(cull_column), flags, _ptr(radius_out), _stream(stream)), "bgs_project")


def bgs_route(ctx: Context, tile_owner_out=None, stream=None, tile_owner_in=None) -> int:
    """a3 + a4; returns R (records received by this rank)."""
    r = C.c_int64(0)
    ctx.check(_lib.bgs_route(ctx.handle, _ptr(tile_owner_in), _ptr(tile_owner_out), C.byref(r), _stream(stream)),
              "bgs_route")
    return int(r.value)


def bgs_sort_tiles(ctx: Context, stream=None):
    ctx.check(_lib.bgs_sort_tiles(ctx.handle, _stream(stream)), "bgs_sort_tiles")


def bgs_raster_fwd(ctx: Context, flags: int, rgb, t_final, n_contrib, stream=None):
    ctx.check(_lib.bgs_raster_fwd(ctx.handle, flags, _ptr(rgb), _ptr(t_final), _ptr(n_contrib), _stream(stream)),
              "bgs_raster_fwd")


def bgs_raster_bwd(ctx: Context, dL_drgb, t_final, n_contrib, stream=None):
    ctx.check(_lib.bgs_raster_bwd(ctx.handle, _ptr(dL_drgb), _ptr(t_final), _ptr(n_contrib), _stream(stream)),
              "bgs_raster_bwd")


def bgs_route_reverse(ctx: Context, stream=None, flags: int = 0):
    """a10; flags BGS_IMPORTANCE_ONLY: (w, a) only, 12 B per record (scoring sweeps)."""
    ctx.check(_lib.bgs_route_reverse(ctx.handle, int(flags), _stream(stream)), "bgs_route_reverse")


def bgs_project_bwd(ctx: Context, g: GaussianPlanes, cam: bgs_camera, grads: GradPlanes, stream=None):
    gs, gr = g.struct(), grads.struct()
    ctx.check(_lib.bgs_project_bwd(ctx.handle, C.byref(gs), C.byref(cam), C.byref(gr), _stream(stream)),
              "bgs_project_bwd")


def bgs_importance(ctx: Context, n_local: int, radius, w_fixed, a, s, c_rad, c_vis, cull_out, mass_num=99,
                   mass_den=100, stream=None):
    ctx.check(_lib.bgs_importance(ctx.handle, int(n_local), _ptr(radius), _ptr(w_fixed), _ptr(a), mass_num, mass_den,
                                  _ptr(s), _ptr(c_rad), _ptr(c_vis), _ptr(cull_out), _stream(stream)),
              "bgs_importance")


def bgs_shard_sizes(ctx: Context, n_local: int) -> list:
    """Every rank's shard size (host list), for a skew-triggered redistribution policy."""
    out = (C.c_int64 * ctx.world)()
    ctx.check(_lib.bgs_shard_sizes(ctx.handle, int(n_local), out), "bgs_shard_sizes")
    return [int(v) for v in out]


def bgs_loss_photo(ctx: Context, rgb, target, lam: float, batch_inv: float, dL_drgb, out, stream=None):
    """NEXT-4, Eq.7: out (device f64[3]) = {l_v, L1, SSIM}; dL_drgb overwritten on owned tiles."""
    ctx.check(_lib.bgs_loss_photo(ctx.handle, _ptr(rgb), _ptr(target), float(lam), float(batch_inv), _ptr(dL_drgb),
                                  _ptr(out), _stream(stream)), "bgs_loss_photo")


def bgs_loss_scale(ctx: Context, g: GaussianPlanes, beta: float, grads: GradPlanes, out, stream=None):
    """NEXT-4, Eq.8: out (device f64[2]) = {L_scale, |V|}; grads.scale += beta/|V| on argmin axes."""
    gs = g.struct()
    gr = grads.struct()
    ctx.check(_lib.bgs_loss_scale(ctx.handle, C.byref(gs), float(beta), C.byref(gr), _ptr(out),
                                  _stream(stream)), "bgs_loss_scale")


class bgs_train_params(C.Structure):
    _fields_ = [("n_local", C.c_int64), ("mean_logit", C.c_void_p), ("quat_raw", C.c_void_p),
                ("log_scale", C.c_void_p), ("sh", C.c_void_p), ("m", C.c_void_p * 4), ("v", C.c_void_p * 4)]


class bgs_adam_hparams(C.Structure):
    _fields_ = [("lr_mean", C.c_float), ("lr_opacity", C.c_float), ("lr_quat", C.c_float), ("lr_scale", C.c_float),
                ("lr_sh_dc", C.c_float), ("lr_sh_rest", C.c_float), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("step", C.c_int32)]


class TrainParams:
    """Raw parameters of a shard + Adam moments (bgs_train_params), torch device tensors."""

    def __init__(self, mean_logit, quat_raw, log_scale, sh):
        self.mean_logit, self.quat_raw, self.log_scale, self.sh = mean_logit, quat_raw, log_scale, sh
        self.m = [torch.zeros_like(t) for t in (mean_logit, quat_raw, log_scale, sh)]
        self.v = [torch.zeros_like(t) for t in (mean_logit, quat_raw, log_scale, sh)]

    @property
    def n(self) -> int:
        return int(self.mean_logit.shape[0])

    def struct(self) -> bgs_train_params:
        s = bgs_train_params()
        s.n_local = self.n
        s.mean_logit, s.quat_raw = self.mean_logit.data_ptr(), self.quat_raw.data_ptr()
        s.log_scale, s.sh = self.log_scale.data_ptr(), self.sh.data_ptr()
        for k in range(4):
            s.m[k] = self.m[k].data_ptr()
            s.v[k] = self.v[k].data_ptr()
        return s


def adam_hparams(lr_mean=1.6e-4, lr_opacity=0.05, lr_quat=1e-3, lr_scale=5e-3, lr_sh_dc=2.5e-3,
                 lr_sh_rest=2.5e-3 / 20, beta1=0.9, beta2=0.999, eps=1e-15, step=1) -> bgs_adam_hparams:
    """Defaults: the 3DGS parameter groups (reading R38)."""
    return bgs_adam_hparams(lr_mean, lr_opacity, lr_quat, lr_scale, lr_sh_dc, lr_sh_rest, beta1, beta2, eps, step)


def bgs_adam_step(ctx: Context, p: TrainParams, grads: GradPlanes, act: GaussianPlanes, visible,
                  h: bgs_adam_hparams, stream=None):
    """NEXT-3: fused activation chain rule + Adam; writes act (activated planes), zeroes grads."""
    ps = p.struct()
    gr = grads.struct()
    ao = bgs_gaussians_out(act.mean_opac.shape[0], act.mean_opac.data_ptr(), act.quat.data_ptr(),
                           act.scale.data_ptr(), act.sh.data_ptr(), act.lod.data_ptr())
    ctx.check(_lib.bgs_adam_step(ctx.handle, C.byref(ps), C.byref(gr), C.byref(ao), _ptr(visible), C.byref(h),
                                 _stream(stream)), "bgs_adam_step")


class bgs_densify_params(C.Structure):
    _fields_ = [("grad_threshold", C.c_float), ("dense_extent", C.c_float), ("min_opacity", C.c_float),
                ("split_div", C.c_float), ("seed", C.c_uint64), ("k_levels", C.c_int32)]


def densify_params(grad_threshold=2e-4, dense_extent=0.01, min_opacity=0.005, split_div=1.6,
                   seed=0, k_levels=256) -> bgs_densify_params:
    """3DGS defaults (tau 2e-4, opacity 0.005, split / 1.6); dense_extent = percent_dense * extent;
    k_levels = K (split children's level is min(l + 1, K - 1))."""
    return bgs_densify_params(grad_threshold, dense_extent, min_opacity, split_div, seed, k_levels)


def bgs_visibility_mask(ctx: Context, n_local: int, radius, mask, stream=None):
    """mask (int32 [ceil(n/32)], caller-zeroed per batch) |= bits of radius > 0."""
    ctx.check(_lib.bgs_visibility_mask(ctx.handle, int(n_local), _ptr(radius), _ptr(mask), _stream(stream)),
              "bgs_visibility_mask")


def bgs_densify_accumulate(ctx: Context, n_local: int, phi, stat, count, stream=None):
    ctx.check(_lib.bgs_densify_accumulate(ctx.handle, int(n_local), _ptr(phi), _ptr(stat), _ptr(count),
                                          _stream(stream)), "bgs_densify_accumulate")


def bgs_densify_apply(ctx: Context, p_in: TrainParams, lod_in, stat, count, dp: bgs_densify_params,
                      p_out: TrainParams, lod_out, act_out: GaussianPlanes | None, stream=None) -> int:
    """NEXT-3 clone / split / prune; p_out rows = capacity; returns the new row count."""
    si, so = p_in.struct(), p_out.struct()
    ao = None
    if act_out is not None:
        ao = bgs_gaussians_out(act_out.mean_opac.shape[0], act_out.mean_opac.data_ptr(), act_out.quat.data_ptr(),
                               act_out.scale.data_ptr(), act_out.sh.data_ptr(), act_out.lod.data_ptr())
    n = C.c_int64(0)
    ctx.check(_lib.bgs_densify_apply(ctx.handle, C.byref(si), _ptr(lod_in), _ptr(stat), _ptr(count), C.byref(dp),
                                     C.byref(so), _ptr(lod_out), C.byref(ao) if ao is not None else None,
                                     C.byref(n), _stream(stream)), "bgs_densify_apply")
    return int(n.value)


class bgs_supervision(C.Structure):
    _fields_ = [("target", C.c_void_p), ("lam", C.c_float), ("batch_inv", C.c_float), ("beta", C.c_float),
                ("loss_out", C.c_void_p)]


def supervision(target, lam: float, batch_inv: float, beta: float, loss_out) -> bgs_supervision:
    return bgs_supervision(_ptr(target), float(lam), float(batch_inv), float(beta), _ptr(loss_out))


def bgs_train_view_step(ctx: Context, g: GaussianPlanes, cam: bgs_camera, gate, cull_column, flags, radius_out,
                        sup: bgs_supervision, rgb, t_final, n_contrib, dL_scratch, grads: GradPlanes | None,
                        importance: bgs_importance_out | None, stream=None):
    gs = g.struct()
    gr = grads.struct() if grads is not None else None
    ctx.check(_lib.bgs_train_view_step(ctx.handle, C.byref(gs), C.byref(cam),
                                       C.byref(gate) if gate is not None else None, _ptr(cull_column), flags,
                                       _ptr(radius_out), C.byref(sup), _ptr(rgb), _ptr(t_final), _ptr(n_contrib),
                                       _ptr(dL_scratch), C.byref(gr) if gr is not None else None,
                                       C.byref(importance) if importance is not None else None, _stream(stream)),
              "bgs_train_view_step")


def bgs_train_view_step_host_async(ctx: Context, g: GaussianPlanes, cam: bgs_camera, gate, cull_column, flags,
                                   radius_out, target_host, lam: float, batch_inv: float, beta: float, loss_host,
                                   grads: GradPlanes | None, importance: bgs_importance_out | None, stream=None):
    gs = g.struct()
    gr = grads.struct() if grads is not None else None
    ctx.check(_lib.bgs_train_view_step_host_async(ctx.handle, C.byref(gs), C.byref(cam),
                                                  C.byref(gate) if gate is not None else None, _ptr(cull_column),
                                                  flags, _ptr(radius_out), _ptr(target_host), float(lam),
                                                  float(batch_inv), float(beta), _ptr(loss_host),
                                                  C.byref(gr) if gr is not None else None,
                                                  C.byref(importance) if importance is not None else None,
                                                  _stream(stream)),
              "bgs_train_view_step_host_async")


def batch_view(cam: bgs_camera, radius_out, rgb, t_final, n_contrib, dL_drgb=None, cull_column=None,
               cull_out=None, sup: "bgs_supervision | None" = None, dL_scratch=None) -> bgs_batch_view:
    """One view of bgs_batch_step.  sup (a bgs_supervision, kept alive by the returned struct)
    makes the view supervised: Eq.7-8 write its dL/dC into dL_scratch."""
    v = bgs_batch_view(cam, _ptr(cull_column), _ptr(radius_out), _ptr(rgb), _ptr(t_final), _ptr(n_contrib),
                       _ptr(dL_drgb), _ptr(cull_out), C.cast(C.pointer(sup), C.c_void_p) if sup is not None else None,
                       _ptr(dL_scratch))
    v._sup = sup
    return v


def bgs_batch_step(ctx: Context, g: GaussianPlanes, views, gate=None, flags: int = 0, grads: GradPlanes | None = None,
                   importance: bgs_importance_out | None = None, stream=None):
    """NEXT-2: a1..a11 (+a12) of len(views) views in one call (one host read, one exchange per batch).
    views: a list of bgs_batch_view or a prebuilt ctypes array of them."""
    arr = views if isinstance(views, C.Array) else (bgs_batch_view * len(views))(*views)
    gs = g.struct()
    gr = grads.struct() if grads is not None else None
    ctx.check(_lib.bgs_batch_step(ctx.handle, len(views), C.byref(gs), C.byref(gate) if gate is not None else None,
                                  int(flags), arr, C.byref(gr) if gr is not None else None,
                                  C.byref(importance) if importance is not None else None, _stream(stream)),
              "bgs_batch_step")


def bgs_view_step(ctx: Context, g: GaussianPlanes, cam: bgs_camera, gate, cull_column, flags, radius_out, rgb, t_final,
                  n_contrib, dL_drgb, grads: GradPlanes | None, importance: bgs_importance_out | None, stream=None):
    gs = g.struct()
    gr = grads.struct() if grads is not None else None
    ctx.check(_lib.bgs_view_step(ctx.handle, C.byref(gs), C.byref(cam), C.byref(gate) if gate is not None else None,
                                 _ptr(cull_column), flags, _ptr(radius_out), _ptr(rgb), _ptr(t_final),
                                 _ptr(n_contrib), _ptr(dL_drgb), C.byref(gr) if gr is not None else None,
                                 C.byref(importance) if importance is not None else None, _stream(stream)),
              "bgs_view_step")


def bgs_view_step_host(ctx: Context, g: GaussianPlanes, cam: bgs_camera, gate, cull_column, flags, radius_out,
                       dL_host: torch.Tensor, rgb_host: torch.Tensor, grads: GradPlanes | None,
                       importance: bgs_importance_out | None, stream=None):
    gs = g.struct()
    gr = grads.struct() if grads is not None else None
    ctx.check(_lib.bgs_view_step_host(ctx.handle, C.byref(gs), C.byref(cam),
                                      C.byref(gate) if gate is not None else None, _ptr(cull_column), flags,
                                      _ptr(radius_out), _ptr(dL_host), _ptr(rgb_host),
                                      C.byref(gr) if gr is not None else None,
                                      C.byref(importance) if importance is not None else None, _stream(stream)),
              "bgs_view_step_host")


BOUNDS_BLOCK = 1024


def bgs_shard_bounds(ctx: Context, g: "GaussianPlanes", bounds=None, stream=None):
    """Block bounds of the shard for hierarchical culling (a1); returns the f32 [blocks][8] tensor and
    attaches it to g (g.bounds), so subsequent steps with g skip off-screen blocks."""
    nb = max(1, (g.n + BOUNDS_BLOCK - 1) // BOUNDS_BLOCK)
    if bounds is None:
        bounds = torch.empty(nb, 8, dtype=torch.float32, device=g.mean_opac.device)
    gs = g.struct()
    ctx.check(_lib.bgs_shard_bounds(ctx.handle, C.byref(gs), _ptr(bounds), _stream(stream)), "bgs_shard_bounds")
    g.bounds = bounds
    return bounds


def bgs_spatial_order(ctx: Context, mean_opac: torch.Tensor, perm_out: torch.Tensor, stream=None):
    ctx.check(_lib.bgs_spatial_order(ctx.handle, _ptr(mean_opac), int(mean_opac.shape[0]), _ptr(perm_out),
                                     _stream(stream)), "bgs_spatial_order")


def spatial_order(ctx: Context, g: GaussianPlanes) -> torch.Tensor:
    """Z-order permutation of a shard (perm[new] = old local index), computed by libbgs."""
    perm = torch.empty(max(g.n, 1), dtype=torch.int32, device=g.mean_opac.device)
    bgs_spatial_order(ctx, g.mean_opac, perm)
    return perm[:g.n].long()


def importance_out(s, c_rad, c_vis, cull_out, num=99, den=100) -> bgs_importance_out:
    return bgs_importance_out(s.data_ptr(), c_rad.data_ptr(), c_vis.data_ptr(), cull_out.data_ptr(), num, den)


# ------------------------------------------------------------------------------------------
# NEXT-1: scoring report phi, scheduled simplification, index-parity redistribution
# ------------------------------------------------------------------------------------------
def bgs_score_phi(ctx: Context, n_local: int, c_rad, c_vis, phi, stream=None):
    ctx.check(_lib.bgs_score_phi(ctx.handle, int(n_local), _ptr(c_rad), _ptr(c_vis), _ptr(phi), _stream(stream)),
              "bgs_score_phi")


def bgs_prune_stochastic(ctx: Context, n_local: int, s, keep_count: int, seed: int, keep_out, stream=None):
    ctx.check(_lib.bgs_prune_stochastic(ctx.handle, int(n_local), _ptr(s), int(keep_count), int(seed) & (2**64 - 1),
                                        _ptr(keep_out), _stream(stream)), "bgs_prune_stochastic")


def bgs_prune_mass_cut(ctx: Context, n_local: int, s, num: int, den: int, keep_out, stream=None) -> bool:
    """Returns the all-zero warning flag."""
    flag = C.c_int32(0)
    ctx.check(_lib.bgs_prune_mass_cut(ctx.handle, int(n_local), _ptr(s), int(num), int(den), _ptr(keep_out),
                                      C.byref(flag), _stream(stream)), "bgs_prune_mass_cut")
    return bool(flag.value)


def bgs_redistribute(ctx: Context, g: GaussianPlanes, keep, out: GaussianPlanes, stream=None) -> int:
    """Survivors of `g` (keep != 0) renumbered and re-sharded into `out` (capacity = out.n rows);
    returns this rank's new shard size."""
    gs = g.struct()
    o = bgs_gaussians_out(out.n, out.mean_opac.data_ptr(), out.quat.data_ptr(), out.scale.data_ptr(),
                          out.sh.data_ptr(), out.lod.data_ptr() if out.lod is not None else None)
    n_out = C.c_int64(0)
    ctx.check(_lib.bgs_redistribute(ctx.handle, C.byref(gs), _ptr(keep), C.byref(o), C.byref(n_out),
                                    _stream(stream)), "bgs_redistribute")
    return int(n_out.value)


def bgs_set_stage_timing(ctx: Context, enable: bool):
    ctx.check(_lib.bgs_set_stage_timing(ctx.handle, int(bool(enable))), "bgs_set_stage_timing")


STAGES = ("project", "route", "sort", "raster_fwd", "loss", "raster_bwd", "route_reverse", "project_bwd",
          "importance")


def bgs_stage_times(ctx: Context) -> dict:
    """Device ms per stage of the most recent bgs_view_step (stage timing enabled)."""
    out = (C.c_float * len(STAGES))()
    ctx.check(_lib.bgs_stage_times(ctx.handle, out), "bgs_stage_times")
    return dict(zip(STAGES, [float(x) for x in out]))


def bgs_view_step_host_async(ctx: Context, g: GaussianPlanes, cam: bgs_camera, gate, cull_column, flags, radius_out,
                             dL_host: torch.Tensor, rgb_host: torch.Tensor, grads: GradPlanes | None,
                             importance: bgs_importance_out | None, stream=None):
    """Non-blocking host-buffer step: rgb_host is valid after `stream` is synchronised."""
    gs = g.struct()
    gr = grads.struct() if grads is not None else None
    ctx.check(_lib.bgs_view_step_host_async(ctx.handle, C.byref(gs), C.byref(cam),
                                            C.byref(gate) if gate is not None else None, _ptr(cull_column), flags,
                                            _ptr(radius_out), _ptr(dL_host), _ptr(rgb_host),
                                            C.byref(gr) if gr is not None else None,
                                            C.byref(importance) if importance is not None else None,
                                            _stream(stream)), "bgs_view_step_host_async")
