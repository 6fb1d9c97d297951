"""Host logic of the measurement: the per-stage algorithmic work and the
roofline fractions bench.py reports, checked against the formulas written out by hand."""
import math

from paper_2605_13794_b200 import roofline as R

PEAKS = {"hbm_gbs": 6463.0, "sm_max_mhz": 1965.0}
Q = [dict(n_active=6e6, F=8e5, R=8e5, D=8e5, P=1.6e6, sort_passes=4)]


def _by_stage(out):
    return {d["stage"]: d for d in out}


def test_alu_peak_is_lane_instruction_rate():
    # 148 SMs x 128 FP32 lanes x 1965 MHz = 37.2 T lane-op/s (an FFMA counts once)
    out = _by_stage(R.stage_rooflines([0.2], Q, 6e6, 1152, 864, 1, PEAKS, A=2e7, names=("raster_bwd",)))
    assert math.isclose(out["raster_bwd"]["peak"], round(148 * 128 * 1965e6 / 1e12, 2))
    assert out["raster_bwd"]["unit"] == "T lane-op/s" and out["raster_bwd"]["bound"] == "alu"


def test_raster_fraction_on_contributing_pairs():
    A = 1.957e7
    ms = 0.2187
    out = _by_stage(R.stage_rooflines([ms], Q, 6e6, 1152, 864, 1, PEAKS, A=A, E=3.2e8, names=("raster_bwd",)))
    ach = 45 * A / (ms * 1e-3) / 1e12
    assert math.isclose(out["raster_bwd"]["achieved"], round(ach, 3))
    assert math.isclose(out["raster_bwd"]["frac"], round(ach / (148 * 128 * 1965e6 / 1e12), 4))
    assert 0 < out["raster_bwd"]["frac"] < 1
    fwd = _by_stage(R.stage_rooflines([0.16], Q, 6e6, 1152, 864, 1, PEAKS, A=A, E=3.2e8, names=("raster_fwd",)))
    assert math.isclose(fwd["raster_fwd"]["achieved"], round(17 * A / 0.16e-3 / 1e12, 3))


def test_hbm_stage_bytes():
    N, F, P, A = 6e6, 8e5, 1.6e6, 6e6
    names = ("project", "sort", "project_bwd", "importance")
    out = _by_stage(R.stage_rooflines([0.1] * 4, Q, N, 1152, 864, 1, PEAKS, names=names))
    want = {
        # mu, o + lod + q, s of active + SH of in-frustum + record + index + colour Jacobian + radius
        "project": 16 * N + N + 32 * A + 192 * F + 52 * F + 48 * F + 4 * N,
        # received rects / depths + pair write + 4 executed passes (read + write) + ranges
        "sort": 16 * F + 8 * P + 16 * P * 4 + 4 * P,
        # mu, o, q, s + colour Jacobian + partials + index + gradient rows read and written
        "project_bwd": 48 * F + 48 * F + 52 * F + 2 * 236 * F,
        "importance": 52 * F + 32 * F + N / 8,
    }
    for k, b in want.items():
        assert out[k]["work"] == f"{b:.3e} bytes per view", k
        assert math.isclose(out[k]["achieved"], round(b / 0.1e-3 / 1e9, 1)), k
        assert math.isclose(out[k]["frac"], round(b / 0.1e-3 / 1e9 / 6463.0, 4)), k


def test_world1_has_no_exchange_bytes():
    out = _by_stage(R.stage_rooflines([0.003, 0.003], Q, 6e6, 1152, 864, 1, PEAKS, names=("route", "route_reverse")))
    assert out["route"]["achieved"] == 0 and out["route_reverse"]["achieved"] == 0
    out2 = _by_stage(R.stage_rooflines([0.003], Q, 6e6, 1152, 864, 2, PEAKS, names=("route_reverse",)))
    assert out2["route_reverse"]["work"] == f"{96 * 8e5:.3e} bytes per view"


def test_loss_roofline():
    d = R.loss_roofline(0.1115, 1152, 864, PEAKS)
    assert math.isclose(d["achieved"], round(213 * 3 * 1152 * 864 / 0.1115e-3 / 1e12, 3))
