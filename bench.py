#!/usr/bin/env python
"""Benchmark of the BlitzGS per-view distributed splatting step (fwd+bwd views/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config rubble] [--impl reference]

N > 1: launched by torch.distributed.run (one rank per GPU, NCCL).  A STEP is one training batch of
B = 4 views (the paper's mini-batch; `--batch`), every view through the unit of work of
SURVEY §8(d): a1 gate + a2 projection -> a3/a4 ownership + all-to-all -> a5-a7 pair emission /
onesweep sort / ranges -> a8 compositing -> a9 backward -> a10 reverse exchange -> a11 projection
backward.  a12 (importance) is timed separately (`with_importance`, `scoring`).  The per-view image
gradient dL/dC is a fixed seeded tensor (the Eq.7 loss is outside the unit; the `train` block adds
it).  Rank 0 prints ONE JSON line.  See DESIGN.md §7 for every number's definition.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd+bwd views/s"
CONFIG_SHAPES = {
    # name: (label, gate on?) -- shapes in synthetic.CITY_CONFIGS
    "rubble": ("Mill-19 Rubble-shaped synthetic aerial scene (6M Gaussians, 1152x864)", False),
    "building": ("Mill-19 Building-shaped synthetic scene (8M Gaussians, 1152x864), LOD gate + importance mask",
                 True),
    "residence": ("UrbanScene3D Residence-shaped synthetic scene (8M Gaussians, 1368x912)", False),
    "matrixcity": ("MatrixCity aerial-shaped synthetic city (20M Gaussians, 1920x1080)", False),
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50, help="timed steps (batches of --batch views)")
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--batch", type=int, default=4, help="views per step (B = 4, P:342), all in flight")
    p.add_argument("--config", default="rubble", choices=sorted(CONFIG_SHAPES))
    p.add_argument("--impl", default="native", choices=["native", "reference"])
    p.add_argument("--n", type=int, default=None, help="override Gaussian count (debug only)")
    p.add_argument("--views", type=int, default=64)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--gate", choices=["config", "on", "off"], default="config",
                   help="LOD gate + importance mask: the config's default, or forced (Table-2-style toggles)")
    p.add_argument("--mask", choices=["config", "on", "off"], default="config",
                   help="importance Cull mask: the config's default, or forced (independent of the gate)")
    p.add_argument("--layout", default="morton", choices=["morton", "input"],
                   help="shard storage order: Z-order (bgs_spatial_order) or the generator's random ids")
    p.add_argument("--host-threads", type=int, default=0,
                   help="1: one host thread per in-flight context (the ABI's one-ctx-per-host-thread model)")
    p.add_argument("--quick", action="store_true", help="headline, e2e and stages only (no train/scoring/simplify)")
    p.add_argument("--no-bounds", action="store_true", help="no block bounds (per-Gaussian culling only)")
    return p.parse_args()


def submit_views(fn, inflight: int, ids, threaded: bool, device: int):
    """Enqueue view ids[j] on in-flight context j % inflight via fn(k, v).  threaded: one host thread
    per context (ctypes releases the GIL inside the ABI calls)."""
    if not threaded or inflight == 1:
        for j, v in enumerate(ids):
            fn(j % inflight, v)
        return
    import torch
    errs = []

    def worker(k):
        try:
            torch.cuda.set_device(device)
            for j, v in enumerate(ids):
                if j % inflight == k:
                    fn(k, v)
        except Exception as e:  # surfaced after the join
            errs.append(e)

    th = [threading.Thread(target=worker, args=(k,)) for k in range(inflight)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]


# ------------------------------------------------------------------------------------------
# clocks sampling (NVML / nvidia-smi during the timed region)
# ------------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clock-event reason bits (nvml.h): sw power cap 0x4, hw slowdown 0x8, sw thermal 0x20, hw thermal 0x40
    REASON_BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.t = None
        self.nvml = None
        self.samples = []
        self.stop_flag = False

    def _nvml_sample(self):
        import pynvml
        sm = pynvml.nvmlDeviceGetClockInfo(self.nvml, pynvml.NVML_CLOCK_SM)
        rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(self.nvml)
        self.samples.append((sm, rs))

    def _nvml_loop(self):
        while not self.stop_flag:
            try:
                self._nvml_sample()
            except Exception:
                return
            time.sleep(0.001)

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.device]) if vis else self.device
            self.nvml = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.nvml, pynvml.NVML_CLOCK_SM)
            self._nvml_sample()
            self.t = threading.Thread(target=self._nvml_loop, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.nvml is not None:
            self.stop_flag = True
            if self.t:
                self.t.join(timeout=2)
            try:
                self._nvml_sample()
            except Exception:
                pass
            sm = [s for s, _ in self.samples]
            reasons = sorted(n for n, bit in self.REASON_BITS.items() if any(r & bit for _, r in self.samples))
            return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": float(self.max_mhz),
                    "reasons": reasons, "samples": len(sm), "source": "nvml"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def clocks_ok(clk: dict) -> bool:
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    if bad & set(clk.get("reasons") or []):
        return False
    sm, mx = clk.get("sm_mhz"), clk.get("sm_max_mhz")
    return not (sm and mx and sm < 0.7 * mx and "sw_power_cap" not in (clk.get("reasons") or []))


def config_dict(args, label, gate_on, mask_on, N_all, W, H, world, batch):
    return {"workload": label, "config": args.config, "gaussians": int(N_all), "width": W, "height": H,
            "views": args.views, "lod_gate": gate_on, "importance_mask": mask_on,
            "parallelism": f"index-parity shards x {world}, tile-owner all-to-all",
            "unit_of_work": "a1-a11 per view (SURVEY 8(d)); a12 importance timed separately"}


# ------------------------------------------------------------------------------------------
# the native arm
# ------------------------------------------------------------------------------------------
def run_native(args):
    import torch
    import torch.distributed as dist

    import paper_2605_13794_b200.bgs as B
    import synthetic as S

    from paper_2605_13794_b200 import dist as D

    rank, world, local = D.env_rank_world()
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    tdev = torch.device(dev)
    batch = max(1, args.batch)
    if world > 1:
        D.init("nccl", tdev)
        ctxs = []
        for _ in range(batch):  # one communicator per in-flight ctx
            uid = D.broadcast_bytes(B.unique_id() if rank == 0 else None, 128, tdev)
            ctxs.append(B.Context(rank, world, local, uid))
    else:
        ctxs = [B.Context(0, 1, local) for _ in range(batch)]
    ctx = ctxs[0]

    label, gate_default = CONFIG_SHAPES[args.config]
    gate_on = gate_default if args.gate == "config" else args.gate == "on"
    mask_on = gate_default if args.mask == "config" else args.mask == "on"  # independent toggles (Table 2)
    t0 = time.perf_counter()
    scene = S.gen_city(args.config, n=args.n, V=args.views)
    gen_s = time.perf_counter() - t0
    shard = scene.shard(rank, world)
    g = B.GaussianPlanes.from_scene(shard, dev)
    n_local = shard.n
    if args.layout == "morton":
        # framework layout: each shard stored in Z-order (bgs_spatial_order), ids relabelled
        perm = B.spatial_order(ctx, g)
        g = B.GaussianPlanes(g.mean_opac[perm].contiguous(), g.quat[perm].contiguous(), g.scale[perm].contiguous(),
                             g.sh[perm].contiguous(), g.lod[perm].contiguous())
        if world == 1:
            scene = scene.subset(perm.cpu().numpy())  # the oracle baseline sees the same labelling
        torch.cuda.synchronize()
    if not args.no_bounds:
        # block bounds of the (Z-ordered) shard: a1 skips the blocks that cannot reach the image
        B.bgs_shard_bounds(ctx, g)
        torch.cuda.synchronize()
    W, H = scene.cameras[0]["W"], scene.cameras[0]["H"]
    cams = [B.camera(c) for c in scene.cameras]
    # d0: 4x the median camera distance (R19) so the gate is selective, not degenerate
    gate = B.lod_gate(True, scene.k_levels - 1, scene.d0 * 4) if gate_on else None
    grads = g.zeros_grads()
    nw = (max(n_local, 1) + 31) // 32
    s_imp = torch.zeros(max(n_local, 1), dtype=torch.float64, device=dev)
    c_rad = torch.zeros(max(n_local, 1), dtype=torch.int32, device=dev)
    c_vis = torch.zeros(max(n_local, 1), dtype=torch.int32, device=dev)
    dl = torch.from_numpy(S.grad_image(H, W)).to(dev)
    l2_flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    per = []
    for k in range(batch):
        per.append(dict(stream=torch.cuda.Stream(dev), radius=torch.zeros(max(n_local, 1), dtype=torch.int32,
                                                                          device=dev),
                        rgb=torch.zeros(3, H, W, device=dev), Tf=torch.zeros(H, W, device=dev),
                        nc=torch.zeros(H, W, dtype=torch.int32, device=dev),
                        cull=torch.zeros(nw, dtype=torch.int32, device=dev)))
    stream = per[0]["stream"]

    cull_cols = None
    if mask_on:
        # per-view Cull columns from one untimed importance sweep (Building config)
        cull_cols = []
        p = per[0]
        with torch.cuda.stream(stream):
            for v, cam in enumerate(cams):
                cc = torch.zeros(nw, dtype=torch.int32, device=dev)
                B.bgs_view_step(ctx, g, cam, None, None, B.BGS_NO_COLOR, p["radius"], p["rgb"], p["Tf"], p["nc"],
                                None, None, B.importance_out(s_imp, c_rad, c_vis, cc), stream)
                cull_cols.append(cc)
        stream.synchronize()

    def cull_of(v):
        return cull_cols[v % len(cams)] if cull_cols is not None else None

    def imp_of(k):
        return B.importance_out(s_imp, c_rad, c_vis, per[k]["cull"], 99, 100)

    def view_on(k, v, with_imp=False):
        p = per[k]
        B.bgs_view_step(ctxs[k], g, cams[v % len(cams)], gate, cull_of(v), 0, p["radius"], p["rgb"], p["Tf"],
                        p["nc"], dl, grads, imp_of(k) if with_imp else None, p["stream"])

    def barrier():
        if world > 1:
            dist.barrier()

    # the ctx arenas are grow-only and sized by the largest view seen: one untimed pass over the
    # camera set per ctx brings them to steady state (as after the first epoch of training)
    for k in range(batch):
        for v in range(len(cams)):
            view_on(k, v, with_imp=True)
    torch.cuda.synchronize()
    barrier()

    # ---- per-stage breakdown: one view at a time, L2 flushed before each (a1-a11; then a1-a12
    # for the importance stage), library-side stage events
    def stage_loop(n_views, with_imp):
        stage_ms = np.zeros(len(B.STAGES))
        qs, tot, E_sum, A_sum = [], 0.0, 0.0, 0.0
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        p = per[0]
        B.bgs_set_stage_timing(ctx, True)
        with torch.cuda.stream(stream):
            for k in range(n_views):
                v = args.warmup + k
                l2_flush.zero_()
                stream.synchronize()
                ev[0].record(stream)
                B.bgs_view_step(ctx, g, cams[v % len(cams)], gate, cull_of(v), 0, p["radius"], p["rgb"], p["Tf"],
                                p["nc"], dl, grads, imp_of(0) if with_imp else None, stream)
                ev[1].record(stream)
                stream.synchronize()
                st = B.bgs_stage_times(ctx)
                stage_ms += np.array([st[n] for n in B.STAGES])
                tot += ev[0].elapsed_time(ev[1])
                qs.append(ctx.query())
                E_sum += float(p["nc"].sum(dtype=torch.int64).item())
                if with_imp:  # contributing (pixel, splat) pairs = sum of a over the received splats
                    acc = ctx.debug_buffer("acc")
                    if acc.numel():
                        A_sum += float(acc.view(torch.int32).view(-1, 12)[:, 9].sum(dtype=torch.int64).item())
        B.bgs_set_stage_timing(ctx, False)
        return stage_ms / n_views, qs, tot / n_views, E_sum / n_views, A_sum / n_views

    n_stage = min(max(args.steps, 8), 64)
    stage_avg, qs, single_ms, E_avg, _ = stage_loop(n_stage, False)
    imp_avg, qs_imp, single_imp_ms, _, A_avg = stage_loop(n_stage, True)
    stage_avg = stage_avg.copy()
    stage_avg[list(B.STAGES).index("importance")] = imp_avg[list(B.STAGES).index("importance")]
    torch.cuda.synchronize()
    barrier()
    single_ms = D.max_over_ranks(single_ms, tdev)
    single_imp_ms = D.max_over_ranks(single_imp_ms, tdev)

    # ---- the headline: K steps, each a batch of B views in flight (one ctx + stream per view),
    # sharing the shard and the gradient buffers (accumulated with reductions); no L2 flush between
    # views (they overlap; every view reads the 1.45 GB shard, > the 126 MB L2)
    def timed_batches(fn, n_steps, warm):
        submit_views(fn, batch, [k for k in range(warm * batch)], bool(args.host_threads), local)
        torch.cuda.synchronize()
        barrier()
        ev_start = torch.cuda.Event(enable_timing=True)
        ev_end = [torch.cuda.Event(enable_timing=True) for _ in range(batch)]
        clocks = ClockSampler(local)
        clocks.start()
        l0 = sum(c.launches() for c in ctxs)
        h0 = sum(c.host_syncs() for c in ctxs)
        ev_start.record(per[0]["stream"])
        for k in range(1, batch):
            per[k]["stream"].wait_event(ev_start)
        submit_views(fn, batch, [warm * batch + j for j in range(n_steps * batch)], bool(args.host_threads), local)
        for k in range(batch):
            ev_end[k].record(per[k]["stream"])
        torch.cuda.synchronize()
        launches = sum(c.launches() for c in ctxs) - l0
        hsyncs = sum(c.host_syncs() for c in ctxs) - h0
        clk = clocks.stop()
        ms = max(ev_start.elapsed_time(e) for e in ev_end)
        barrier()
        return D.max_over_ranks(ms, tdev), launches, hsyncs, clk

    head_ms, launches, hsyncs, clk = timed_batches(lambda k, v: view_on(k, v), args.steps, args.warmup)
    if not clocks_ok(clk):  # rejected clocks: re-measure once
        head_ms, launches, hsyncs, clk = timed_batches(lambda k, v: view_on(k, v), args.steps, args.warmup)
        clk["remeasured"] = True
    n_views = args.steps * batch
    ms_per_step = head_ms / args.steps
    views_per_s = 1000.0 * n_views / head_ms

    imp_ms, imp_launches, _, _ = timed_batches(lambda k, v: view_on(k, v, True), args.steps, 1)

    # ---- NEXT-2: the same steps through bgs_batch_step (one call per batch of B views: one host
    # read and, at world > 1, one exchange per batch), eagerly and as a CUDA graph (BGS_GRAPH)
    batch_api = batch_step_timing(args, B, g, cams, gate, cull_of, per, dl, grads, batch, barrier, D, tdev, world,
                                  rank, local)
    with_importance = {"metric": "fwd+bwd views/s with a12 (importance, Cull column) per view",
                       "value": round(1000.0 * n_views / imp_ms, 3), "unit": "views/s",
                       "ms_per_step": round(imp_ms / args.steps, 4), "gpu_launches": int(imp_launches)}

    # ---- per-view workload statistics (summed over ranks)
    def avg(key, qq):
        return float(np.mean([q[key] for q in qq]))

    P_rank = avg("P", qs)
    stats = D.sum_over_ranks([P_rank, avg("F", qs), avg("R", qs), avg("D", qs), avg("n_active", qs), float(n_local),
                              float(A_avg)], tdev)
    P_all, F_all, R_all, D_all, A_all, N_all, Acontrib_all = [float(x) for x in stats]
    P_max = D.max_over_ranks(P_rank, tdev)
    pairs_per_s = P_all * views_per_s

    # ---- e2e: the same steps through the host-buffer ABI call (pinned dL/dC H2D and the rendered
    # image D2H inside the timed region, per view), wall clock, max over ranks
    dl_host = torch.from_numpy(S.grad_image(H, W)).pin_memory()
    rgb_hosts = [torch.empty(3, H, W).pin_memory() for _ in range(batch)]

    def host_view(k, v):
        p = per[k]
        B.bgs_view_step_host_async(ctxs[k], g, cams[v % len(cams)], gate, cull_of(v), 0, p["radius"], dl_host,
                                   rgb_hosts[k], grads, None, p["stream"])

    submit_views(host_view, batch, list(range(batch)), False, local)
    torch.cuda.synchronize()
    barrier()
    t1 = time.perf_counter()
    submit_views(host_view, batch, [args.warmup * batch + j for j in range(n_views)], bool(args.host_threads), local)
    torch.cuda.synchronize()
    e2e_s = D.max_over_ranks(time.perf_counter() - t1, tdev)
    e2e_views = n_views / e2e_s

    result = {
        "metric": METRIC, "value": round(views_per_s, 3), "unit": "views/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": dict(config_dict(args, label, gate_on, mask_on, N_all, W, H, world, batch),
                       shard_layout=args.layout, host_threads=bool(args.host_threads),
                       block_bounds=not args.no_bounds,
                       l2=("inputs exceed L2 (every view reads the 1.45 GB shard); the B views of a step overlap "
                           "and are not flushed between; stages_ms / single_view_ms: one view at a time, L2 "
                           "flushed (256 MB write) before each"),
                       arena="pre-grown by one untimed pass over the cameras per ctx before the warm-up steps"),
        "views_per_step": batch,
        "single_view_ms": round(single_ms, 4),
        "single_view_with_importance_ms": round(single_imp_ms, 4),
        "splat_pairs_per_s": round(pairs_per_s, 1),
        "with_importance": with_importance,
        "batch_step": batch_api,
        "per_view": {"pairs_P": P_all, "records_F": F_all, "received_R": R_all, "sent_D": D_all,
                     "active_A": A_all, "duplication_D_over_F": (D_all / F_all if F_all else None),
                     "nvlink_bytes": 48.0 * (D_all - F_all) * 2 if world > 1 else 0.0,
                     "E_min_pixel_entries": round(E_avg, 1),
                     "contributing_pairs": round(Acontrib_all, 1),
                     "gate_keep": (avg("n_lod", qs) / n_local) if gate_on and n_local else None,
                     "owned_pairs_max_over_mean": (P_max * world / P_all) if P_all else None},
        "gpu_launches": int(launches),
        "gpu_launches_per_view": round(launches / n_views, 2),
        "host_syncs_per_view": round(hsyncs / n_views, 3),
        "clocks": clk,
        "scene_gen_s": round(gen_s, 2),
    }

    extra = {}
    if not args.quick:
        extra["scoring"] = scoring(args, B, ctxs, per, g, cams, gate, cull_of, s_imp, c_rad, c_vis, l2_flush,
                                   batch, barrier, D, tdev, n_local, local)
        extra["train"] = train_iterations(args, B, S, ctxs, per, g, cams, gate, cull_of, imp_of, stream, l2_flush,
                                          batch, barrier, D, tdev, H, W, n_local, local)
        extra["simplify"] = simplify(args, B, ctx, g, s_imp, c_rad, c_vis, stream, barrier, D, tdev, n_local, N_all)

    # ---- rooflines: the dominant kernel on the contributing-pair basis
    from paper_2605_13794_b200.roofline import load_traffic, stage_rooflines
    peaks = load_peaks()
    traffic = (load_traffic(os.path.join(ROOT, "profiles", "ncu_traffic.json"))
               if args.config == "rubble" and world == 1 else None)
    roof = stage_rooflines(stage_avg, qs_imp, n_local=n_local, W=W, H=H, world=world, peaks=peaks, E=E_avg,
                           A=A_avg, cull=cull_cols is not None, traffic=traffic, names=B.STAGES)
    dominant = max((r for r in roof if r["stage"] != "importance"), key=lambda r: r["ms"])
    result["stages_ms"] = {n: round(float(v), 4) for n, v in zip(B.STAGES, stage_avg) if n != "loss"}
    result["roofline"] = {k: dominant[k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic")}
    result["roofline"]["kernel"] = dominant.get("kernel", dominant["stage"])
    result["roofline"]["basis"] = dominant["work"]
    result["roofline_stages"] = roof
    result.update(extra)
    if "train" in extra and extra["train"].get("loss_stage_ms"):
        from paper_2605_13794_b200.roofline import loss_roofline
        extra["train"]["loss_roofline"] = loss_roofline(extra["train"]["loss_stage_ms"], W, H, peaks)
    result["e2e"] = {"value": round(e2e_views, 3), "unit": "views/s", "h2d_bytes_per_step": int(batch * 3 * H * W * 4),
                     "d2h_bytes_per_step": int(batch * 3 * H * W * 4),
                     "path": "bgs_view_step_host_async (pinned host dL/dC in, rendered image out, per view)"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(scene, args, cams_idx=args.warmup)
    if rank == 0:
        print(json.dumps(result), flush=True)
    for c in ctxs:
        c.close()
    if world > 1:
        dist.destroy_process_group()


def batch_step_timing(args, B, g, cams, gate, cull_of, per, dl, grads, batch, barrier, D, tdev, world, rank, local):
    """K steps through bgs_batch_step (NEXT-2), device-timed like the headline; per batch: launches,
    host syncs and collectives (the library's counters)."""
    import torch
    import torch.distributed as dist
    if world > 1:
        uid = D.broadcast_bytes(B.unique_id() if rank == 0 else None, 128, tdev)
        bctx = B.Context(rank, world, local, uid)
    else:
        bctx = B.Context(0, 1, local)
    stream = per[0]["stream"]
    V = len(cams)
    n_arr = V // batch if V % batch == 0 else V
    arrs = []
    for i in range(n_arr):
        vs = []
        for k in range(batch):
            v = (i * batch + k) % V
            p = per[k]
            vs.append(B.batch_view(cams[v], p["radius"], p["rgb"], p["Tf"], p["nc"], dl, cull_column=cull_of(v)))
        arrs.append((B.bgs_batch_view * batch)(*vs))
    out = {}
    for name, flags in (("eager", 0), ("graph", B.BGS_GRAPH)):
        with torch.cuda.stream(stream):
            # every batch of the camera cycle once (grows the slot arenas to steady state, as the
            # per-view contexts' warm-up pass does), then the warm-up steps
            for i in range(n_arr + args.warmup + 1):
                B.bgs_batch_step(bctx, g, arrs[i % n_arr], gate, flags, grads, None, stream)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            s0 = bctx.batch_stats()
            l0, h0 = bctx.launches(), bctx.host_syncs()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for i in range(args.steps):
                B.bgs_batch_step(bctx, g, arrs[(args.warmup + 1 + i) % n_arr], gate, flags, grads, None, stream)
            e1.record(stream)
            torch.cuda.synchronize()
        ms = D.max_over_ranks(e0.elapsed_time(e1), tdev)
        s1 = bctx.batch_stats()
        nv = args.steps * batch
        out[name] = {"value": round(1000.0 * nv / ms, 3), "unit": "views/s", "ms_per_step": round(ms / args.steps, 4),
                     "gpu_launches_per_view": round((bctx.launches() - l0) / nv, 2),
                     "host_syncs_per_view": round((bctx.host_syncs() - h0) / nv, 3),
                     "collectives_per_step": round((s1["collectives"] - s0["collectives"]) / args.steps, 2),
                     "graph_launches": s1["graph_launches"] - s0["graph_launches"],
                     "graph_instantiations": s1["graph_instantiations"] - s0["graph_instantiations"],
                     "graph_fallbacks": s1["graph_fallbacks"] - s0["graph_fallbacks"]}
        if world > 1:
            dist.barrier()
    bctx.close()
    out["note"] = ("bgs_batch_step: B views per call on internal view slots, one host read per batch, at world > 1 "
                   "one tile-cost all-reduce + one count exchange + one record all-to-all + one reverse per batch; "
                   "graph = everything after the host read recorded as one CUDA graph (updated in place)")
    return out


def scoring(args, B, ctxs, per, g, cams, gate, cull_of, s_imp, c_rad, c_vis, l2_flush, batch, barrier, D, tdev,
            n_local, local):
    """scoring views/s: the a12 sweep step = NO_COLOR projection, routing, sort,
    instrumented forward, reverse exchange of (w, a), importance; no backward.  One view at a time
    (L2 flushed) and with the sweep's views in flight."""
    import torch

    def score_on(k, v):
        p = per[k]
        st_k = p["stream"]
        cam = cams[v % len(cams)]
        B.bgs_project(ctxs[k], g, cam, gate, cull_of(v), B.BGS_NO_COLOR, p["radius"], st_k)
        B.bgs_route(ctxs[k], None, st_k)
        B.bgs_sort_tiles(ctxs[k], st_k)
        B.bgs_raster_fwd(ctxs[k], B.BGS_IMPORTANCE, p["rgb"], p["Tf"], p["nc"], st_k)
        B.bgs_route_reverse(ctxs[k], st_k, B.BGS_IMPORTANCE_ONLY)
        B.bgs_importance(ctxs[k], n_local, p["radius"], None, None, s_imp, c_rad, c_vis, p["cull"], 99, 100, st_k)

    stream = per[0]["stream"]
    sev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    score_ms = 0.0
    n1 = min(max(args.steps, 8), 64)
    with torch.cuda.stream(stream):
        for k in range(args.warmup + n1):
            if k >= args.warmup:
                l2_flush.zero_()
                stream.synchronize()
                sev[0].record(stream)
            score_on(0, k)
            if k >= args.warmup:
                sev[1].record(stream)
                stream.synchronize()
                score_ms += sev[0].elapsed_time(sev[1])
    score_ms = D.max_over_ranks(score_ms, tdev) / n1
    torch.cuda.synchronize()
    barrier()
    n_views = args.steps * batch
    sev_start = torch.cuda.Event(enable_timing=True)
    sev_end = [torch.cuda.Event(enable_timing=True) for _ in range(batch)]
    sev_start.record(per[0]["stream"])
    for k in range(1, batch):
        per[k]["stream"].wait_event(sev_start)
    submit_views(score_on, batch, list(range(n_views)), bool(args.host_threads), local)
    for k in range(batch):
        sev_end[k].record(per[k]["stream"])
    torch.cuda.synchronize()
    inflight_ms = D.max_over_ranks(max(sev_start.elapsed_time(e) for e in sev_end), tdev) / n_views
    return {"metric": "scoring views/s (a1-a8 NO_COLOR + a10 + a12, no backward)",
            "value": round(1000.0 / score_ms, 3) if score_ms > 0 else None, "unit": "views/s",
            "ms_per_view": round(score_ms, 4),
            "note": "value: one view at a time, L2 flushed before each; in_flight: the sweep's views overlapped "
                    "like the training batch (one ctx + stream each)",
            "in_flight": {"value": round(1000.0 / inflight_ms, 3), "unit": "views/s",
                          "ms_per_view": round(inflight_ms, 4), "views_in_flight": batch}}


def train_iterations(args, B, S, ctxs, per, g0, cams, gate, cull_of, imp_of, stream, l2_flush, batch, barrier, D,
                     tdev, H, W, n_local, local):
    """NEXT-4 + NEXT-3: MEASURED training iterations on a copy of the shard.  One iteration = B
    supervised views in flight (bgs_train_view_step: a1-a11 with Eq.7 L1+SSIM on the owned tiles
    writing dL/dC, Eq.8 scale regulariser; + the density statistic of each view, + the batch's
    visibility mask) -> one fused selective Adam step (bgs_adam_step) writing the activated planes
    the next iteration renders.  Device-timed (events), max over ranks; e2e through the
    host-buffer supervised call (target H2D, loss D2H)."""
    import torch
    dev = f"cuda:{local}"
    lam, binv, beta = 0.2, 1.0 / batch, 0.01 / batch
    tgts = [torch.from_numpy(S.target_image(H, W, seed=9 + k)).to(dev) for k in range(4)]
    mo = g0.mean_opac
    o = mo[:, 3].clamp(1e-6, 1 - 1e-6)
    tp = B.TrainParams(torch.cat([mo[:, :3], torch.log(o / (1 - o))[:, None]], 1).contiguous(), g0.quat.clone(),
                       torch.log(g0.scale.clamp_min(1e-30)).contiguous(), g0.sh.clone())
    tp.log_scale[:, 3] = 0
    g = B.GaussianPlanes(mo.clone(), g0.quat.clone(), g0.scale.clone(), tp.sh, g0.lod)  # rendered + written
    if g0.bounds is not None:
        B.bgs_shard_bounds(ctxs[0], g, stream=stream)  # refreshed after every optimizer step below
    grads = g.zeros_grads()
    nw = (max(n_local, 1) + 31) // 32
    vis = torch.zeros(nw, dtype=torch.int32, device=dev)
    dc_stat = torch.zeros(max(n_local, 1), dtype=torch.float32, device=dev)
    dc_count = torch.zeros(max(n_local, 1), dtype=torch.int32, device=dev)
    for p in per:
        p["dl"] = torch.zeros(3, H, W, device=dev)
        p["loss"] = torch.zeros(5, dtype=torch.float64, device=dev)
    ev_fork = torch.cuda.Event()
    ev_join = [torch.cuda.Event() for _ in range(batch)]
    state = {"step": 0}

    def iteration(it, stages=False):
        # fork: every view waits for the previous iteration's Adam step (stream 0)
        ev_fork.record(stream)
        for k in range(batch):
            p = per[k]
            if k:
                p["stream"].wait_event(ev_fork)
            v = it * batch + k
            B.bgs_train_view_step(ctxs[k], g, cams[v % len(cams)], gate, cull_of(v), 0, p["radius"],
                                  B.supervision(tgts[v % 4], lam, binv, beta, p["loss"]), p["rgb"], p["Tf"],
                                  p["nc"], p["dl"], grads, None, p["stream"])
            B.bgs_densify_accumulate(ctxs[k], n_local, None, dc_stat, dc_count, p["stream"])
            B.bgs_visibility_mask(ctxs[k], n_local, p["radius"], vis, p["stream"])
            ev_join[k].record(p["stream"])
        for k in range(1, batch):
            stream.wait_event(ev_join[k])
        state["step"] += 1
        with torch.cuda.stream(stream):
            B.bgs_adam_step(ctxs[0], tp, grads, g, vis, B.adam_hparams(step=state["step"]), stream)
            if g.bounds is not None:
                B.bgs_shard_bounds(ctxs[0], g, g.bounds, stream)
            vis.zero_()

    for it in range(args.warmup):
        iteration(it)
    torch.cuda.synchronize()
    barrier()
    # stage breakdown of the supervised view (one at a time, L2 flushed): the loss stage
    st_loss = 0.0
    B.bgs_set_stage_timing(ctxs[0], True)
    nst = min(max(args.steps, 8), 32)
    with torch.cuda.stream(stream):
        for k in range(nst):
            l2_flush.zero_()
            stream.synchronize()
            p = per[0]
            B.bgs_train_view_step(ctxs[0], g, cams[k % len(cams)], gate, cull_of(k), 0, p["radius"],
                                  B.supervision(tgts[k % 4], lam, binv, beta, p["loss"]), p["rgb"], p["Tf"], p["nc"],
                                  p["dl"], grads, None, stream)
            stream.synchronize()
            st_loss += B.bgs_stage_times(ctxs[0])["loss"]
    B.bgs_set_stage_timing(ctxs[0], False)
    grads.zero_()
    torch.cuda.synchronize()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    losses = []
    ev0.record(stream)
    for it in range(args.steps):
        iteration(args.warmup + it)
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = D.max_over_ranks(ev0.elapsed_time(ev1), tdev) / args.steps
    losses = [float(p["loss"][0].item()) for p in per]
    barrier()
    # end to end: each view's target uploaded from pinned memory, its loss read back
    tgt_h = [torch.from_numpy(S.target_image(H, W, seed=9 + k)).pin_memory() for k in range(batch)]
    loss_h = [torch.zeros(5, dtype=torch.float64).pin_memory() for _ in range(batch)]

    def host_iteration(it):
        ev_fork.record(stream)
        for k in range(batch):
            p = per[k]
            if k:
                p["stream"].wait_event(ev_fork)
            v = it * batch + k
            B.bgs_train_view_step_host_async(ctxs[k], g, cams[v % len(cams)], gate, cull_of(v), 0, p["radius"],
                                             tgt_h[k], lam, binv, beta, loss_h[k], grads, None, p["stream"])
            B.bgs_visibility_mask(ctxs[k], n_local, p["radius"], vis, p["stream"])
            ev_join[k].record(p["stream"])
        for k in range(1, batch):
            stream.wait_event(ev_join[k])
        state["step"] += 1
        with torch.cuda.stream(stream):
            B.bgs_adam_step(ctxs[0], tp, grads, g, vis, B.adam_hparams(step=state["step"]), stream)
            if g.bounds is not None:
                B.bgs_shard_bounds(ctxs[0], g, g.bounds, stream)
            vis.zero_()

    host_iteration(0)
    torch.cuda.synchronize()
    barrier()
    t1 = time.perf_counter()
    for it in range(args.steps):
        host_iteration(1 + it)
    torch.cuda.synchronize()
    e2e_it = args.steps / D.max_over_ranks(time.perf_counter() - t1, tdev)
    adam = adam_step_timing(B, g, grads, tp, ctxs[0], stream, n_local, l2_flush, per, args, D, tdev, batch)
    dens = densify_timing(B, ctxs[0], tp, g, dc_stat, dc_count, stream, n_local, D, tdev)
    out = {"metric": "training iterations/s (B views: a1-a11 + Eq.7 L1+SSIM + Eq.8 + density statistic, then one "
                     "selective Adam step; NEXT-4 + NEXT-3)",
           "value": round(1000.0 / ms, 3), "unit": "it/s", "ms_per_iteration": round(ms, 4),
           "views_per_s": round(1000.0 * batch / ms, 3), "views_per_iteration": batch,
           "lambda": lam, "batch_inv": binv, "beta": beta, "loss_last_batch": losses,
           "loss_stage_ms": round(st_loss / nst, 4),
           "e2e": {"value": round(e2e_it, 3), "unit": "it/s", "h2d_bytes_per_step": int(batch * 3 * H * W * 4),
                   "d2h_bytes_per_step": int(batch * 40)},
           "adam": adam, "densify": dens}
    del tp, g, grads
    return out


def adam_step_timing(B, g, grads, tp, ctx, stream, n_local, l2_flush, per, args, D, tdev, batch):
    """bgs_adam_step on the shard, device-timed (L2 flushed before each), dense and with the
    visibility mask of a batch of views."""
    import torch
    dev = g.mean_opac.device
    nw = (max(n_local, 1) + 31) // 32
    mask = torch.zeros(nw, dtype=torch.int32, device=dev)
    for p in per[:batch]:
        B.bgs_visibility_mask(ctx, n_local, p["radius"], mask, stream)
    torch.cuda.synchronize()
    rows = float(sum(bin(int(x) & 0xffffffff).count("1") for x in mask.cpu().numpy().tolist()))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    out = {}
    with torch.cuda.stream(stream):
        for name, m in (("dense", None), ("selective", mask)):
            tot = 0.0
            for k in range(args.warmup + args.steps):
                l2_flush.zero_()
                stream.synchronize()
                ev[0].record(stream)
                B.bgs_adam_step(ctx, tp, grads, g, m, B.adam_hparams(step=k + 1), stream)
                ev[1].record(stream)
                stream.synchronize()
                if k >= args.warmup:
                    tot += ev[0].elapsed_time(ev[1])
            out[f"{name}_ms"] = round(D.max_over_ranks(tot / args.steps, tdev), 4)
    # algorithmic bytes per updated row: read raw 240 + grads 240 + m 240 + v 240; write raw 240 +
    # m 240 + v 240 + activated 48 (SH aliases the raw plane) + zeroed grads 240
    per_row = 4 * 240 + 4 * 240 + 48
    peaks = load_peaks()
    for name, nrows in (("dense", float(n_local)), ("selective", rows)):
        ach = per_row * nrows / (out[f"{name}_ms"] * 1e-3) / 1e9 if out[f"{name}_ms"] > 0 else 0.0
        out[f"{name}_roofline"] = {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"],
                                   "unit": "GB/s", "frac": round(ach / peaks["hbm_gbs"], 4), "rows": int(nrows),
                                   "work": f"{per_row} B x rows"}
    out["note"] = ("one optimizer step per batch of B views (P:342); selective = rows projected by any view of the "
                   "batch (bgs_visibility_mask), dense = every row of the shard")
    return out


def densify_timing(B, ctx, tp, g, dc_stat, dc_count, stream, n_local, D, tdev):
    """NEXT-3 density control on the shard with the statistic of the timed training views (tau =
    the 99th percentile of the per-Gaussian average so that ~1% densify; 3DGS's 2e-4 is scale-
    dependent), extent 10 units (1% of the 1000-unit scene): wall time of the HOST-SYNC call."""
    import torch
    dev = g.mean_opac.device
    with torch.cuda.stream(stream):
        avg = (dc_stat[:n_local] / dc_count[:n_local].clamp_min(1).float())
        tau = float(torch.quantile(avg[avg > 0][:1 << 24].float(), 0.99).item()) if bool((avg > 0).any()) else 1.0
        cap = 2 * n_local + 1
        tout = B.TrainParams(*(torch.empty(cap, c, device=dev) for c in (4, 4, 4, 48)))
        lod_out = torch.empty(cap, dtype=torch.uint8, device=dev)
        act2 = B.GaussianPlanes(torch.empty(cap, 4, device=dev), torch.empty(cap, 4, device=dev),
                                torch.empty(cap, 4, device=dev), tout.sh, lod_out)
        dp = B.densify_params(tau, 10.0, 0.005, 1.6, 1234)
        B.bgs_densify_apply(ctx, tp, g.lod, dc_stat, dc_count, dp, tout, lod_out, act2, stream)  # warm-up
        stream.synchronize()
        t1 = time.perf_counter()
        n_new = B.bgs_densify_apply(ctx, tp, g.lod, dc_stat, dc_count, dp, tout, lod_out, act2, stream)
        stream.synchronize()
        ms = (time.perf_counter() - t1) * 1e3
    # algorithmic bytes: read every input row (raw 240 + m, v 480 + lod 1 + stat, count 8), write
    # every output row (raw + m + v 720 + activated 48 + lod 1)
    byt = n_local * (240 + 480 + 1 + 8) + n_new * (720 + 48 + 1)
    hbm = load_peaks()["hbm_gbs"]
    del tout, act2
    return {"apply_ms": round(D.max_over_ranks(ms, tdev), 4), "rows_in": int(n_local), "rows_out": int(n_new),
            "tau": tau, "dense_extent": 10.0,
            "roofline": {"bound": "hbm", "achieved": round(byt / (ms * 1e-3) / 1e9, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(byt / (ms * 1e-3) / 1e9 / hbm, 4)},
            "note": "statistic accumulated by every timed training view (bgs_densify_accumulate); apply is "
                    "HOST-SYNC, wall time incl. the count round trip"}


def simplify(args, B, ctx, g, s_imp, c_rad, c_vis, stream, barrier, D, tdev, n_local, N_all):
    """NEXT-1 scheduled simplification on the shard with the s / c_rad / c_vis the timed views
    accumulated (one pass each; HOST-SYNC calls, wall time between barriers)."""
    import torch
    out = {}
    dev = g.mean_opac.device
    with torch.cuda.stream(stream):
        phi = torch.empty(max(n_local, 1), dtype=torch.float64, device=dev)
        keep = torch.empty(max(n_local, 1), dtype=torch.uint8, device=dev)
        cap = n_local + 1
        out_g = B.GaussianPlanes(torch.empty(cap, 4, device=dev), torch.empty(cap, 4, device=dev),
                                 torch.empty(cap, 4, device=dev), torch.empty(cap, 48, device=dev),
                                 torch.empty(cap, dtype=torch.uint8, device=dev))
        N_glob = int(N_all)

        def timed(fn):
            fn()  # warm-up: first calls grow the ctx arena (cudaMalloc)
            stream.synchronize()
            barrier()
            t1 = time.perf_counter()
            r = fn()
            stream.synchronize()
            return r, round(D.max_over_ranks((time.perf_counter() - t1) * 1e3, tdev), 3)

        _, out["phi_ms"] = timed(lambda: B.bgs_score_phi(ctx, n_local, c_rad, c_vis, phi, stream))
        _, out["pass1_stochastic_ms"] = timed(
            lambda: B.bgs_prune_stochastic(ctx, n_local, s_imp, int(round(0.6 * N_glob)), 1234, keep, stream))
        n_keep1 = D.sum_over_ranks([float(keep[:n_local].sum().item())], tdev)[0]
        _, out["pass2_mass_cut_ms"] = timed(lambda: B.bgs_prune_mass_cut(ctx, n_local, s_imp, 99, 100, keep, stream))
        n_keep2 = D.sum_over_ranks([float(keep[:n_local].sum().item())], tdev)[0]
        _, out["redistribute_ms"] = timed(lambda: B.bgs_redistribute(ctx, g, keep, out_g, stream))
        out.update({"gaussians": N_glob, "kept_pass1": int(n_keep1), "kept_pass2": int(n_keep2),
                    "note": "keep_fraction 0.6 (S:318 default), target 99/100; scores from the timed views"})
        del out_g
    return out


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "source": "measured (MEASURED_PEAKS.json)",
                "sm_max_mhz": d.get("sm_max_mhz", 1965.0)}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)", "sm_max_mhz": 1965.0}


# ------------------------------------------------------------------------------------------
# oracle baselines (the one other place bench.py executes oracle/)
# ------------------------------------------------------------------------------------------
def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def oracle_view(scene, v, threads: int, frac_tiles: float = 1.0):
    """One fwd+bwd view of the workload through the oracle (a1-a11: projection, ownership, routing,
    sort, compositing fwd+bwd, projection backward), compositing on a `frac_tiles` sample."""
    import oracle as O
    import synthetic as S
    cam = scene.cameras[v % len(scene.cameras)]
    dl = S.grad_image(cam["H"], cam["W"])
    t0 = time.perf_counter()
    st = O.OracleStep(scene, cam, M=1, dLdC=dl, tile_frac=frac_tiles, threads=threads)
    secs = time.perf_counter() - t0
    return secs, st.seconds_by_phase(), st.threads


def cpu_baseline(scene, args, cams_idx=0):
    """The oracle as it stands, on this host's cores: (i) all cores on one FULL view of the
    workload, (ii) one thread on a 1/8 tile sample of another view, composite scaled x8."""
    import oracle as O
    cores = host_cores()
    secs, phases, used = oracle_view(scene, cams_idx, cores)
    frac = 1.0 / 8
    s1, ph1, _ = oracle_view(scene, cams_idx + 1, 1, frac)
    per_view_1 = ph1["project"] + ph1["route_sort"] + ph1["composite"] / frac + ph1["project_bwd"]
    return {"value": round(1.0 / secs, 5), "unit": "views/s", "cores": used, "kind": "oracle",
            "sample": f"one full view (a1-a11, all {scene.n} Gaussians, every tile) of the same workload on "
                      f"{used} host threads ({secs:.1f} s)",
            "nproc": cores, "cpu_model": cpu_model(),
            "phases_s": {k: round(v, 3) for k, v in phases.items()},
            "single_thread": {"value": round(1.0 / per_view_1, 5), "unit": "views/s", "cores": 1,
                              "sample": f"one view, compositing fwd+bwd of a {frac:.3f} tile sample scaled "
                                        f"x{1 / frac:.0f} ({s1:.1f} s)",
                              "phases_s": {k: round(v, 3) for k, v in ph1.items()}},
            "oracle_lib": os.path.basename(O.build())}


def run_reference(args):
    """The base contract's reference arm for this tier: the CPU oracle, as it stands, on the box's
    host cores, on the native arm's workload.  Each timed step = one batch of B FULL views (a1-a11
    of every view, all tiles); warm-up steps composite a 1/64 tile sample of one view."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import synthetic as S
    label, gate_default = CONFIG_SHAPES[args.config]
    gate_on = gate_default if args.gate == "config" else args.gate == "on"
    mask_on = gate_default if args.mask == "config" else args.mask == "on"
    if gate_on or mask_on:
        print(json.dumps({"impl": "reference", "unavailable": "the oracle reference arm covers the ungated "
                                                              "configs only (rubble, residence, matrixcity)"}))
        return
    batch = 1  # one view per reference step (the CPU has no views in flight)
    t0 = time.perf_counter()
    scene = S.gen_city(args.config, n=args.n, V=args.views)
    gen_s = time.perf_counter() - t0
    cores = host_cores()
    for w in range(args.warmup):
        oracle_view(scene, w, cores, 1.0 / 64)
    tot = 0.0
    phase_tot = {}
    used = cores
    for k in range(args.steps):
        secs, ph, used = oracle_view(scene, args.warmup + k, cores)
        tot += secs
        for kk, v in ph.items():
            phase_tot[kk] = phase_tot.get(kk, 0.0) + v
    v = args.steps * batch / tot
    W, H = scene.cameras[0]["W"], scene.cameras[0]["H"]
    out = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "views/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1000 * tot / args.steps, 2),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": config_dict(args, label, gate_on, mask_on, scene.n, W, H, world, batch),
           "views_per_step": batch,
           "cpu_baseline": {"value": round(v, 6), "unit": "views/s", "cores": used, "kind": "oracle",
                            "nproc": cores, "cpu_model": cpu_model(),
                            "sample": f"each step one FULL view (a1-a11 of all {scene.n} Gaussians, every tile) on "
                                      f"{used} host threads; warm-up steps on 1/64 tile samples",
                            "phases_s_per_view": {kk: round(x / args.steps, 3) for kk, x in phase_tot.items()}},
           "e2e": {"value": round(v, 6), "unit": "views/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "scene_gen_s": round(gen_s, 2)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_native(a)
