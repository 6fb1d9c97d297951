"""Algorithmic bytes / operations per stage of one view.

These are what the METHOD must move or compute, not what a kernel happens to do:
  a1+a2 project      16 N (mu,o) + 1 N (lod) + N/8 (cull column, if any) + 32 A (q, s of active)
                     + 192 F (SH of in-frustum) + 52 F (record + index) + 48 F (colour Jacobian
                     along the view direction + clamp bits, for a11) + 4 N (radius)           [bytes]
  a5-a7 sort         16 R (rect, depth of received) + 8 P (u32 key + u32 value written) + 16 P
                     per executed 8-bit radix pass (read + write) + 4 P (ranges pass)     [bytes]
  a8 raster fwd      SURVEY §8(d): ~17 FP32 lane-ops per CONTRIBUTING (pixel, splat) pair (dx,dy 2,
                     power 3 (one FMUL + 2 FFMA in the pinned order), cut 2, exp 1 MUFU, alpha 2,
                     test T(1-alpha) 2, w = alpha T 1, colour 3, T update 1).  The contributing pairs are
                     A = sum over splats of a_{i,v} (measured per view by the instrumented forward):
                     every exact kernel must evaluate them in full, whatever it culls.  [ALU]
  a9 raster bwd      SURVEY §8(d): ~45 FP32 lane-ops per contributing pair (recompute dx, dy, power,
                     exp, alpha 9, T recovery 3, colour grads 6, dL/dalpha 8, clamp + G dL/dalpha 3,
                     dL/do 1, mean2d / conic partials 12, accumulation 3).                   [ALU]
                     Diagnostic beside it (`frac_E_min`): the DESIGN.md recount (19 fwd / 33 bwd) per
                     E_min entry (every list entry up to a pixel's last contributor, sum of n_contrib);
                     exact box culling skips most of those, so that fraction can exceed 1.
  a10 reverse (M>1)  48 D (send back) + 48 D (gather)                                     [bytes]
  a11 project bwd    48 F (mu, o, q, s) + 48 F (colour Jacobian + clamp bits) + 52 F (partials +
                     index) + 2 x 236 F (grads RMW; the SH row itself is read once, by a2)  [bytes]
  a12 importance     52 F (w, a, index) + 2 x 16 F (s, c_rad, c_vis RMW) + N/8 (Cull)    [bytes]
  NEXT-4 loss        213 FP32 ops per image element (3 H W): window statistics 3 products +
                     5 maps x 2 separable 11-tap passes = 113, SSIM and its partials 25,
                     3 partial maps x 2 passes = 66, dS, L1 sign, sums 9 (the 5 px halo a
                     32x32 tile recomputes is not counted)                                [ALU]
Peaks: HBM = MEASURED_PEAKS.json hbm_gbs (copy bandwidth); ALU = 148 SMs x 128 FP32 lanes x
sm_max clock = 37.2 T lane-op/s (one FP32 instruction per lane per clock; an FFMA is ONE lane-op,
so this is an instruction rate, not a FLOP rate).
"""
from __future__ import annotations

FWD_OPS = 17.0       # per contributing pair
BWD_OPS = 45.0
FWD_OPS_EMIN = 19.0  # per E_min entry (DESIGN.md recount; diagnostic)
BWD_OPS_EMIN = 33.0
LOSS_OPS = 213.0
KERNEL = {"project": "k_cull+k_project+k_color", "sort": "k_emit+k_onesweep+k_ranges_fixup",
          "raster_fwd": "k_raster_fwd", "raster_bwd": "k_raster_bwd", "project_bwd": "k_project_bwd+k_project_bwd_shg",
          "importance": "k_imp_coop", "loss": "k_loss_photo"}
ALU_UNIT = "T lane-op/s"


def _avg(qs, k):
    return sum(q[k] for q in qs) / max(1, len(qs))


def stage_rooflines(stage_ms, qs, n_local, W, H, world, peaks, sm_mhz=None, E=None, cull=False, traffic=None,
                    A=None, names=None, with_loss=False):
    """traffic: optional {stage: DRAM bytes per view} from a committed ncu capture (profiles/)."""
    traffic = traffic or {}
    N = float(n_local)
    A_contrib = A  # contributing (pixel, splat) pairs
    A, F, R, D, P = (_avg(qs, k) for k in ("n_active", "F", "R", "D", "P"))
    passes = _avg(qs, "sort_passes")
    hbm = float(peaks["hbm_gbs"])
    alu = 148 * 128 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12  # T ops/s
    names = names or ("project", "route", "sort", "raster_fwd", "loss", "raster_bwd", "route_reverse", "project_bwd",
                      "importance")
    bytes_ = {
        "project": 16 * N + N + (N / 8 if cull else 0) + 32 * A + 192 * F + 52 * F + 48 * F + 4 * N,
        "route": (48 * D + 48 * R) if world > 1 else 0.0,
        "sort": 16 * R + 8 * P + 16 * P * passes + 4 * P,
        "route_reverse": (96 * D) if world > 1 else 0.0,
        "project_bwd": 48 * F + 48 * F + 52 * F + 2 * 236 * F,
        "importance": 52 * F + 32 * F + N / 8,
    }
    E = float(E) if E is not None else 0.0
    Ac = float(A_contrib) if A_contrib is not None else 0.0
    ops = {"raster_fwd": FWD_OPS * Ac, "raster_bwd": BWD_OPS * Ac}
    ops_e = {"raster_fwd": FWD_OPS_EMIN * E, "raster_bwd": BWD_OPS_EMIN * E}
    out = []
    for name, ms in zip(names, stage_ms):
        ms = float(ms)
        if name == "loss":
            if with_loss:
                out.append(loss_roofline(ms, W, H, peaks, traffic.get(name)))
            continue
        if name in ops:
            ach = ops[name] / (ms * 1e-3) / 1e12 if ms > 0 else 0.0
            ach_e = ops_e[name] / (ms * 1e-3) / 1e12 if ms > 0 else 0.0
            k = FWD_OPS if name == "raster_fwd" else BWD_OPS
            out.append(dict(stage=name, kernel=KERNEL[name], ms=round(ms, 4), bound="alu", achieved=round(ach, 3),
                            peak=round(alu, 2), unit=ALU_UNIT, frac=round(ach / alu, 4), traffic=traffic.get(name),
                            work=f"{ops[name]:.3e} lane-ops per view ({k:.0f} x {Ac:.4g} contributing pairs)",
                            frac_E_min=round(ach_e / alu, 4),
                            work_E_min=f"{ops_e[name]:.3e} ({FWD_OPS_EMIN if k == FWD_OPS else BWD_OPS_EMIN:.0f}"
                                       f" x E_min {E:.4g})"))
        else:
            b = bytes_.get(name, 0.0)
            ach = b / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
            out.append(dict(stage=name, kernel=KERNEL.get(name, name), ms=round(ms, 4), bound="hbm",
                            achieved=round(ach, 1), peak=hbm, unit="GB/s", frac=round(ach / hbm, 4),
                            traffic=traffic.get(name), work=f"{b:.3e} bytes per view"))
    return out


def loss_roofline(ms, W, H, peaks, traffic=None):
    alu = 148 * 128 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
    o = LOSS_OPS * 3.0 * W * H
    ach = o / (ms * 1e-3) / 1e12 if ms > 0 else 0.0
    return dict(stage="loss", kernel=KERNEL["loss"], ms=round(ms, 4), bound="alu", achieved=round(ach, 3),
                peak=round(alu, 2), unit=ALU_UNIT, frac=round(ach / alu, 4), traffic=traffic,
                work=f"{o:.3e} lane-ops ({LOSS_OPS:.0f} x 3 H W)")


def load_traffic(path):
    """{stage: dram bytes per view} from profiles/ncu_traffic.json (profiles/make_traffic.py)."""
    import json
    import os
    if not os.path.exists(path):
        return {}
    d = json.load(open(path))
    return {k: v["dram_bytes_per_view"] for k, v in d.get("stages", {}).items()}
