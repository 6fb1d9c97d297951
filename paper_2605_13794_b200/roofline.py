"""Algorithmic bytes / operations per stage of one view.

These are what the METHOD must move or compute, not what a kernel happens to do:
  a1+a2 project      16 N (mu,o) + 1 N (lod) + N/8 (cull column, if any) + 32 A (q, s of active)
                     + 192 F (SH of in-frustum) + 52 F (record + index) + 4 N (radius)      [bytes]
  a5-a7 sort         16 R (rect, depth of received) + 8 P (u32 key + u32 value written) + 16 P
                     per executed 8-bit radix pass (read + write) + 4 P (ranges pass)     [bytes]
  a8 raster fwd      19 FP32 ops per (pixel, list entry) up to the pixel's last contributor
                     (SURVEY §8(d)'s E_min = sum of n_contrib): dx,dy 2, power 5, alpha cut 1,
                     exp 1, alpha = min(.99, oG) 2, w = alpha T and T -= w 2, early stop 1,
                     colour 3, w and a sums 2                                              [ALU]
  a9 raster bwd      33 FP32 ops per E_min entry: recompute dx,dy,power,cut,exp,alpha 11,
                     T_k = T_{k+1}/(1-alpha) 3, w 1, colour grads 3, dL/dalpha (c.dL,
                     T c.dL - s/(1-alpha), s update) 6, G dL/dalpha 1, dL/do 1, mean2d/conic
                     moments 7                                                            [ALU]
                     (MUFU and FFMA count as one op.)  Exact culling skips most E_min entries
                     (a splat whose alpha >= 1/255 ellipse misses a warp's 8x8 block cannot
                     contribute there), so this fraction can exceed 1 on scenes with large
                     splats.  `frac_contributing` is the strict bound beside it: the same ops per
                     CONTRIBUTING (pixel, splat) pair (A = sum over splats of a_{i,v}), which every
                     exact kernel must evaluate in full; on Rubble A is ~6% of E_min, i.e. most
                     evaluations a block-culled kernel issues do not contribute.
  a10 reverse (M>1)  48 D (send back) + 48 D (gather)                                     [bytes]
  a11 project bwd    240 F (params) + 52 F (partials + index) + 2 x 236 F (grads RMW)     [bytes]
  a12 importance     52 F (w, a, index) + 2 x 16 F (s, c_rad, c_vis RMW) + N/8 (Cull)    [bytes]
  NEXT-4 loss        213 FP32 ops per image element (3 H W): window statistics 3 products +
                     5 maps x 2 separable 11-tap passes = 113, SSIM and its partials 25,
                     3 partial maps x 2 passes = 66, dS, L1 sign, sums 9 (the 5 px halo a
                     32x32 tile recomputes is not counted)                                [ALU]
Peaks: HBM = MEASURED_PEAKS.json hbm_gbs (copy bandwidth); ALU = 148 SMs x 128 FP32 lanes x
sm_max clock (one FP32 instruction per lane per clock; FFMA counted as one op).
"""
from __future__ import annotations

FWD_OPS = 19.0
BWD_OPS = 33.0
LOSS_OPS = 213.0


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
        "project": 16 * N + N + (N / 8 if cull else 0) + 32 * A + 192 * F + 52 * F + 4 * N,
        "route": (48 * D + 48 * R) if world > 1 else 0.0,
        "sort": 16 * R + 8 * P + 16 * P * passes + 4 * P,
        "route_reverse": (96 * D) if world > 1 else 0.0,
        "project_bwd": 240 * F + 52 * F + 2 * 236 * F,
        "importance": 52 * F + 32 * F + N / 8,
    }
    E = float(E) if E is not None else 0.0
    Ac = float(A_contrib) if A_contrib is not None else E
    ops = {"raster_fwd": FWD_OPS * E, "raster_bwd": BWD_OPS * E}
    ops_a = {"raster_fwd": FWD_OPS * Ac, "raster_bwd": BWD_OPS * Ac}
    out = []
    for name, ms in zip(names, stage_ms):
        ms = float(ms)
        if name == "loss":
            if not with_loss:
                continue  # no supervision in this step (the stage events bracket nothing)
            o = LOSS_OPS * 3.0 * W * H
            ach = o / (ms * 1e-3) / 1e12
            out.append(dict(stage=name, ms=round(ms, 4), bound="alu", achieved=round(ach, 3), peak=round(alu, 2),
                            unit="TFLOP/s", frac=round(ach / alu, 4), traffic=traffic.get(name),
                            work=f"{o:.3e} ops ({LOSS_OPS:.0f} x 3 H W)"))
        elif name in ops:
            ach = ops[name] / (ms * 1e-3) / 1e12 if ms > 0 else 0.0
            ach_a = ops_a[name] / (ms * 1e-3) / 1e12 if ms > 0 else 0.0
            k = FWD_OPS if name == "raster_fwd" else BWD_OPS
            out.append(dict(stage=name, ms=round(ms, 4), bound="alu", achieved=round(ach, 3), peak=round(alu, 2),
                            unit="TFLOP/s", frac=round(ach / alu, 4), traffic=traffic.get(name),
                            work=f"{ops[name]:.3e} ops ({k:.0f} x E_min)",
                            frac_contributing=round(ach_a / alu, 4)))
        else:
            b = bytes_.get(name, 0.0)
            ach = b / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
            out.append(dict(stage=name, ms=round(ms, 4), bound="hbm", achieved=round(ach, 1), peak=hbm,
                            unit="GB/s", frac=round(ach / hbm, 4), traffic=traffic.get(name), work=f"{b:.3e} bytes"))
    return out


def load_traffic(path):
    """{stage: dram bytes per view} from profiles/ncu_traffic.json (profiles/make_traffic.py)."""
    import json
    import os
    if not os.path.exists(path):
        return {}
    d = json.load(open(path))
    return {k: v["dram_bytes_per_view"] for k, v in d.get("stages", {}).items()}
