#!/usr/bin/env python
"""Benchmark of the BlitzGS per-view distributed splatting step (fwd+bwd views/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config rubble] [--impl reference]

N > 1: launched by torch.distributed.run (one rank per GPU, NCCL).  One step = one view through
every SURVEY §8(a) row: a1 gate + a2 projection -> a3/a4 ownership + all-to-all -> a5-a7 pair
emission / onesweep sort / ranges -> a8 compositing (+ w, a) -> a9 backward -> a10 reverse
exchange -> a11 projection backward -> a12 importance (Eq.3, top-99% mass, Cull column).
The per-view image gradient dL/dC is a fixed seeded tensor (the Eq.7 loss is outside the path).
Rank 0 prints ONE JSON line.  See DESIGN.md §7 for every number's definition.
"""
from __future__ import annotations

import argparse
import json
import os
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
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="rubble", choices=sorted(CONFIG_SHAPES))
    p.add_argument("--impl", default="native", choices=["native", "reference"])
    p.add_argument("--n", type=int, default=None, help="override Gaussian count (debug only)")
    p.add_argument("--views", type=int, default=64)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--stages", action="store_true", help="also print per-stage timings to stderr")
    p.add_argument("--layout", default="morton", choices=["morton", "input"],
                   help="shard storage order: Z-order (bgs_spatial_order) or the generator's random ids")
    p.add_argument("--host-threads", type=int, default=0,
                   help="1: one host thread per in-flight context (the ABI's one-ctx-per-host-thread model), so "
                        "a context's HOST-SYNC calls block only its own thread; 0: one thread submits all views")
    p.add_argument("--inflight", type=int, default=4,
                   help="views in flight per rank (one ctx + stream each); 4 = the paper's batch of B = 4 "
                        "views per step (P:342). Measured on Rubble (second session): 1 -> 1219, 4 -> 1383, "
                        "6 -> 1388, 8 -> 1386 views/s")
    return p.parse_args()


def submit_views(fn, inflight: int, ids, threaded: bool, device: int):
    """Enqueue view ids[j] on in-flight context j % inflight via fn(k, v).  threaded: one host thread
    per context (ctypes releases the GIL inside the ABI calls), so the host round trip of one view's
    HOST-SYNC projection does not hold back the submission of the other contexts' views."""
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
# clocks sampling (nvidia-smi during the timed region)
# ------------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.t = None
        self.nvml = None
        self.samples = []
        self.stop_flag = False

    # NVML clock-event reason bits (nvml.h): sw power cap 0x4, hw slowdown 0x8, sw thermal 0x20,
    # hw thermal 0x40
    REASON_BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

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
        # NVML polling (~1 ms) so that a short timed region still has samples; nvidia-smi otherwise
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
    inflight = max(1, args.inflight)
    if world > 1:
        D.init("nccl", torch.device(dev))
        ctxs = []
        for _ in range(inflight):  # one communicator per in-flight ctx
            uid = D.broadcast_bytes(B.unique_id() if rank == 0 else None, 128, torch.device(dev))
            ctxs.append(B.Context(rank, world, local, uid))
    else:
        ctxs = [B.Context(0, 1, local) for _ in range(inflight)]
    ctx = ctxs[0]

    label, gate_on = CONFIG_SHAPES[args.config]
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
    W, H = scene.cameras[0]["W"], scene.cameras[0]["H"]
    cams = [B.camera(c) for c in scene.cameras]
    # d0: 4x the median camera distance (R19) so the gate is selective, not degenerate
    gate = B.lod_gate(True, scene.k_levels - 1, scene.d0 * 4) if gate_on else None
    stream = torch.cuda.Stream(dev)
    grads = g.zeros_grads()
    radius = torch.zeros(max(n_local, 1), dtype=torch.int32, device=dev)
    rgb = torch.zeros(3, H, W, device=dev)
    Tf = torch.zeros(H, W, device=dev)
    nc = torch.zeros(H, W, dtype=torch.int32, device=dev)
    s_imp = torch.zeros(max(n_local, 1), dtype=torch.float64, device=dev)
    c_rad = torch.zeros(max(n_local, 1), dtype=torch.int32, device=dev)
    c_vis = torch.zeros(max(n_local, 1), dtype=torch.int32, device=dev)
    cull_cols = None
    imp = B.importance_out(s_imp, c_rad, c_vis, torch.zeros((max(n_local, 1) + 31) // 32, dtype=torch.int32,
                                                             device=dev))
    dl = torch.from_numpy(S.grad_image(H, W)).to(dev)
    l2_flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    if gate_on:
        # Building config: per-view Cull columns from one untimed importance sweep
        cull_cols = []
        with torch.cuda.stream(stream):
            for v, cam in enumerate(cams):
                cc = torch.zeros((max(n_local, 1) + 31) // 32, dtype=torch.int32, device=dev)
                B.bgs_view_step(ctx, g, cam, None, None, B.BGS_NO_COLOR, radius, rgb, Tf, nc, None, None,
                                B.importance_out(s_imp, c_rad, c_vis, cc), stream)
                cull_cols.append(cc)
        stream.synchronize()

    stage_names = B.STAGES
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    cull_out = torch.zeros((max(n_local, 1) + 31) // 32, dtype=torch.int32, device=dev)
    imp_view = B.importance_out(s_imp, c_rad, c_vis, cull_out, 99, 100)

    def one_view(v, record):
        # one step = one bgs_view_step call (a1..a12; the library records its stage events)
        cam = cams[v % len(cams)]
        cull = cull_cols[v % len(cams)] if cull_cols is not None else None
        if record:
            ev[0].record(stream)
        B.bgs_view_step(ctx, g, cam, gate, cull, 0, radius, rgb, Tf, nc, dl, grads, imp_view, stream)
        if record:
            ev[1].record(stream)

    def barrier():
        if world > 1:
            dist.barrier()

    with torch.cuda.stream(stream):
        # the ctx arena is grow-only and sized by the largest view seen: one untimed pass over the
        # camera set brings it to its steady state (as after the first epoch of a training run),
        # then the W warm-up views
        for v in range(len(cams)):
            one_view(v, False)
        for w in range(args.warmup):
            one_view(w, False)
        stream.synchronize()
        barrier()
        # one view at a time, L2 flushed before each: the per-stage breakdown and single_view_ms
        stage_ms = np.zeros(len(stage_names))
        qs = []
        total_ms = 0.0
        E_sum = 0.0
        A_sum = 0.0
        B.bgs_set_stage_timing(ctx, True)
        for k in range(args.steps):
            l2_flush.zero_()  # between timed views: evict the L2 (inputs also exceed it)
            stream.synchronize()
            one_view(args.warmup + k, True)
            stream.synchronize()
            st = B.bgs_stage_times(ctx)
            stage_ms += np.array([st[n] for n in stage_names])
            total_ms += ev[0].elapsed_time(ev[1])
            qs.append(ctx.query())
            E_sum += float(nc.sum(dtype=torch.int64).item())  # outside the timed events
            # contributing (pixel, splat) pairs = sum of a over this rank's received splats
            acc = ctx.debug_buffer("acc")
            if acc.numel():
                A_sum += float(acc.view(torch.int32).view(-1, 12)[:, 9].sum(dtype=torch.int64).item())
        B.bgs_set_stage_timing(ctx, False)
    torch.cuda.synchronize()
    barrier()
    single_ms = D.max_over_ranks(total_ms, torch.device(dev)) / args.steps

    # ---- the headline: `inflight` views in flight per rank, one ctx + stream each, sharing the
    # shard, the gradient buffers and the importance outputs (all accumulated with reductions);
    # no L2 flush between views (they overlap; every view's inputs exceed the 126 MB L2 anyway)
    per = [dict(stream=stream, radius=radius, rgb=rgb, Tf=Tf, nc=nc, cull=cull_out)]
    for k in range(1, inflight):
        per.append(dict(stream=torch.cuda.Stream(dev), radius=torch.zeros_like(radius), rgb=torch.zeros_like(rgb),
                        Tf=torch.zeros_like(Tf), nc=torch.zeros_like(nc), cull=torch.zeros_like(cull_out)))

    def view_on(k, v):
        p = per[k]
        cam = cams[v % len(cams)]
        cull = cull_cols[v % len(cams)] if cull_cols is not None else None
        B.bgs_view_step(ctxs[k], g, cam, gate, cull, 0, p["radius"], p["rgb"], p["Tf"], p["nc"], dl, grads,
                        B.importance_out(s_imp, c_rad, c_vis, p["cull"], 99, 100), p["stream"])

    for k in range(1, inflight):  # arena warm-up of the other contexts
        with torch.cuda.stream(per[k]["stream"]):
            for v in range(len(cams)):
                view_on(k, v)
    torch.cuda.synchronize()
    barrier()
    ev_start = torch.cuda.Event(enable_timing=True)
    ev_end = [torch.cuda.Event(enable_timing=True) for _ in range(inflight)]
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = sum(c.launches() for c in ctxs)
    ev_start.record(per[0]["stream"])
    for k in range(1, inflight):
        per[k]["stream"].wait_event(ev_start)
    submit_views(view_on, inflight, [args.warmup + k for k in range(args.steps)], bool(args.host_threads), local)
    for k in range(inflight):
        ev_end[k].record(per[k]["stream"])
    torch.cuda.synchronize()
    launches = sum(c.launches() for c in ctxs) - launches0
    clk = clocks.stop()
    total_ms = max(ev_start.elapsed_time(e) for e in ev_end)
    barrier()
    total_ms_max = D.max_over_ranks(total_ms, torch.device(dev))
    ms_per_view = total_ms_max / args.steps
    views_per_s = 1000.0 / ms_per_view

    # ---- per-view workload statistics (summed over ranks)
    P_rank = float(np.mean([q["P"] for q in qs]))
    stats = D.sum_over_ranks([P_rank, np.mean([q["F"] for q in qs]), np.mean([q["R"] for q in qs]),
                              np.mean([q["D"] for q in qs]), np.mean([q["n_active"] for q in qs]), float(n_local)],
                             torch.device(dev))
    P_all, F_all, R_all, D_all, A_all, N_all = [float(x) for x in stats]
    pairs_per_s = P_all * views_per_s

    # ---- e2e: same metric through the host-buffer ABI call (H2D of dL/dC, D2H of the image)
    # (bgs_view_step_host_async on every in-flight ctx, one pinned output image per ctx; wall clock
    # from the first call to the synchronisation of every stream, each view's dL/dC uploaded and
    # image downloaded inside the region)
    dl_host = torch.from_numpy(S.grad_image(H, W)).pin_memory()
    rgb_hosts = [torch.empty(3, H, W).pin_memory() for _ in range(inflight)]

    def host_view(k, v):
        p = per[k]
        B.bgs_view_step_host_async(ctxs[k], g, cams[v % len(cams)], gate,
                                   cull_cols[v % len(cams)] if cull_cols is not None else None, 0, p["radius"],
                                   dl_host, rgb_hosts[k], grads,
                                   B.importance_out(s_imp, c_rad, c_vis, p["cull"], 99, 100), p["stream"])

    for k in range(inflight):
        host_view(k, k)
    torch.cuda.synchronize()
    barrier()
    t1 = time.perf_counter()
    submit_views(host_view, inflight, [args.warmup + k for k in range(args.steps)], bool(args.host_threads), local)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t1
    e2e_views = args.steps / D.max_over_ranks(e2e_s, torch.device(dev))

    # ---- NEXT-4 supervised training step: bgs_train_view_step = a1..a12 with Eq.7 (L1 + SSIM on
    # the owned tiles, its gradient as this view's dL/dC) and Eq.8 (scale regulariser); lambda 0.2
    # (3DGS), B = 4 views per step (batch_inv 1/4), beta 0.01 / B; one seeded target image
    train = train_step(args, B, S, ctxs, per, g, cams, gate, cull_cols, grads, s_imp, c_rad, c_vis, stream, l2_flush,
                       inflight, barrier, dev, H, W, n_local, world)

    # ---- scoring views/s: the a12 sweep step = NO_COLOR projection, routing,
    # sort, instrumented forward, reverse exchange of (w, a), importance; no backward
    sev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with torch.cuda.stream(stream):
        score_ms = 0.0
        for k in range(args.warmup + args.steps):
            v = args.warmup + k
            cam = cams[v % len(cams)]
            cull = cull_cols[v % len(cams)] if cull_cols is not None else None
            if k >= args.warmup:
                l2_flush.zero_()
                stream.synchronize()
                sev[0].record(stream)
            B.bgs_project(ctx, g, cam, gate, cull, B.BGS_NO_COLOR, radius, stream)
            B.bgs_route(ctx, None, stream)
            B.bgs_sort_tiles(ctx, stream)
            B.bgs_raster_fwd(ctx, B.BGS_IMPORTANCE, rgb, Tf, nc, stream)
            B.bgs_route_reverse(ctx, stream)
            B.bgs_importance(ctx, n_local, radius, None, None, s_imp, c_rad, c_vis, cull_out, 99, 100, stream)
            if k >= args.warmup:
                sev[1].record(stream)
                stream.synchronize()
                score_ms += sev[0].elapsed_time(sev[1])
    score_ms_max = D.max_over_ranks(score_ms, torch.device(dev)) / args.steps

    # the same sweep step with the views in flight (a scoring pass sweeps all V training views, so
    # its views overlap like the training batch's): one ctx + stream per view in flight
    def score_on(k, v):
        p = per[k]
        cam = cams[v % len(cams)]
        cull = cull_cols[v % len(cams)] if cull_cols is not None else None
        st_k = p["stream"]
        B.bgs_project(ctxs[k], g, cam, gate, cull, B.BGS_NO_COLOR, p["radius"], st_k)
        B.bgs_route(ctxs[k], None, st_k)
        B.bgs_sort_tiles(ctxs[k], st_k)
        B.bgs_raster_fwd(ctxs[k], B.BGS_IMPORTANCE, p["rgb"], p["Tf"], p["nc"], st_k)
        B.bgs_route_reverse(ctxs[k], st_k)
        B.bgs_importance(ctxs[k], n_local, p["radius"], None, None, s_imp, c_rad, c_vis, p["cull"], 99, 100, st_k)

    for k in range(inflight):
        score_on(k, args.warmup + k)
    torch.cuda.synchronize()
    barrier()
    sev_start = torch.cuda.Event(enable_timing=True)
    sev_end = [torch.cuda.Event(enable_timing=True) for _ in range(inflight)]
    sev_start.record(per[0]["stream"])
    for k in range(1, inflight):
        per[k]["stream"].wait_event(sev_start)
    submit_views(score_on, inflight, [args.warmup + k for k in range(args.steps)], bool(args.host_threads), local)
    for k in range(inflight):
        sev_end[k].record(per[k]["stream"])
    torch.cuda.synchronize()
    score_inflight_ms = D.max_over_ranks(max(sev_start.elapsed_time(e) for e in sev_end),
                                         torch.device(dev)) / args.steps
    P_max = D.max_over_ranks(P_rank, torch.device(dev))

    # ---- NEXT-1 scheduled simplification on the same shard, with the s / c_rad / c_vis the
    # timed views accumulated (one pass each; HOST-SYNC calls, wall time between barriers)
    simplify = {}
    with torch.cuda.stream(stream):
        phi = torch.empty(max(n_local, 1), dtype=torch.float64, device=dev)
        keep = torch.empty(max(n_local, 1), dtype=torch.uint8, device=dev)
        cap = (n_local + 1)
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
            return r, D.max_over_ranks((time.perf_counter() - t1) * 1e3, torch.device(dev))

        _, simplify["phi_ms"] = timed(lambda: B.bgs_score_phi(ctx, n_local, c_rad, c_vis, phi, stream))
        _, simplify["pass1_stochastic_ms"] = timed(
            lambda: B.bgs_prune_stochastic(ctx, n_local, s_imp, int(round(0.6 * N_glob)), 1234, keep, stream))
        n_keep1 = D.sum_over_ranks([float(keep[:n_local].sum().item())], torch.device(dev))[0]
        _, simplify["pass2_mass_cut_ms"] = timed(lambda: B.bgs_prune_mass_cut(ctx, n_local, s_imp, 99, 100, keep,
                                                                              stream))
        n_keep2 = D.sum_over_ranks([float(keep[:n_local].sum().item())], torch.device(dev))[0]
        n_new, simplify["redistribute_ms"] = timed(lambda: B.bgs_redistribute(ctx, g, keep, out_g, stream))
        simplify.update({"gaussians": N_glob, "kept_pass1": int(n_keep1), "kept_pass2": int(n_keep2),
                         "note": "keep_fraction 0.6 (S:318 default), target 99/100; scores from the timed views"})
        del out_g

    # ---- roofline of every stage, dominant one reported at top level
    from paper_2605_13794_b200.roofline import load_traffic, stage_rooflines
    peaks = load_peaks()
    stage_avg = stage_ms / args.steps
    traffic = (load_traffic(os.path.join(ROOT, "profiles", "ncu_traffic.json"))
               if args.config == "rubble" and world == 1 else None)
    roof = stage_rooflines(stage_avg, qs, n_local=n_local, W=W, H=H, world=world, peaks=peaks,
                           sm_mhz=clk.get("sm_mhz"), E=E_sum / args.steps, A=A_sum / args.steps,
                           cull=cull_cols is not None, traffic=traffic, names=stage_names)
    dominant = max(roof, key=lambda r: r["ms"])
    train_roof = stage_rooflines(train.pop("stages_avg"), qs, n_local=n_local, W=W, H=H, world=world, peaks=peaks,
                                 E=E_sum / args.steps, A=A_sum / args.steps, cull=cull_cols is not None,
                                 traffic=traffic, names=stage_names, with_loss=True)
    train["loss_roofline"] = next((r for r in train_roof if r["stage"] == "loss"), None)

    result = {
        "metric": METRIC, "value": round(views_per_s, 3), "unit": "views/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_view, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": label, "config": args.config, "gaussians": int(N_all), "width": W, "height": H,
                   "views": len(cams), "lod_gate": gate_on, "importance_mask": gate_on,
                   "parallelism": f"index-parity shards x {world}, tile-owner all-to-all",
                   "shard_layout": args.layout,
                   "views_in_flight": inflight,
                   "host_threads": bool(args.host_threads),
                   "l2": ("inputs exceed L2 (shard 1.8 GB per view read); views in flight are not flushed "
                          "between; single_view_ms / stages_ms: one view at a time, L2 flushed (256 MB write) "
                          "before each"),
                   "arena": "pre-grown by one untimed pass over the cameras before the warm-up views"},
        "single_view_ms": round(single_ms, 4),
        "splat_pairs_per_s": round(pairs_per_s, 1),
        "per_view": {"pairs": P_all, "records_F": F_all, "received_R": R_all, "sent_D": D_all,
                     "active": A_all, "duplication_D_over_F": (D_all / F_all if F_all else None),
                     "E_pixel_entries": round(E_sum / args.steps, 1),
                     "contributing_pairs": round(A_sum / args.steps, 1),
                     "gate_keep": (float(np.mean([q["n_lod"] for q in qs])) / n_local) if gate_on and n_local else None,
                     "owned_pairs_max_over_mean": (P_max * world / P_all) if P_all else None},
        "scoring": {"metric": "scoring views/s (a1-a8 NO_COLOR + a10 + a12, no backward)",
                    "value": round(1000.0 / score_ms_max, 3) if score_ms_max > 0 else None, "unit": "views/s",
                    "ms_per_view": round(score_ms_max, 4),
                    "note": "value: one view at a time, L2 flushed before each; in_flight: the sweep's views "
                            "overlapped like the training batch (one ctx + stream each)",
                    "in_flight": {"value": round(1000.0 / score_inflight_ms, 3), "unit": "views/s",
                                  "ms_per_view": round(score_inflight_ms, 4), "views_in_flight": inflight}},
        "simplify": {k: (round(v, 3) if isinstance(v, float) else v) for k, v in simplify.items()},
        "train": train,
        "stages_ms": {n: round(float(v), 4) for n, v in zip(stage_names, stage_avg)},
        "roofline": dict({k: dominant[k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic")},
                         basis=(f"{dominant['work']} per view (SURVEY 8(d) per-unit ops x E_min); exceeds 1 when "
                                "exact box culling skips list entries that cannot contribute; the strict "
                                "contributing-pair basis is frac_contributing in roofline_stages"
                                if dominant["bound"] == "alu" else f"{dominant['work']} per view (SURVEY 8(d))")),
        "roofline_kernel": dominant["stage"],
        "roofline_stages": roof,
        "e2e": {"value": round(e2e_views, 3), "unit": "views/s", "h2d_bytes_per_step": int(3 * H * W * 4),
                "d2h_bytes_per_step": int(3 * H * W * 4)},
        "gpu_launches": int(launches),
        "clocks": clk,
        "scene_gen_s": round(gen_s, 2),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(scene, args)
    if rank == 0:
        print(json.dumps(result), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def train_step(args, B, S, ctxs, per, g, cams, gate, cull_cols, grads, s_imp, c_rad, c_vis, stream, l2_flush,
               inflight, barrier, dev, H, W, n_local, world):
    """NEXT-4: the supervised step (bgs_train_view_step) timed like the headline (views in flight,
    device events, max over ranks), its stage breakdown (one view at a time, L2 flushed), and its
    end-to-end rate through bgs_train_view_step_host_async (target image H2D, loss D2H)."""
    import torch
    from paper_2605_13794_b200 import dist as D
    lam, binv, beta = 0.2, 0.25, 0.01 / 4
    tgt = torch.from_numpy(S.target_image(H, W)).to(dev)
    for p in per:
        p["dl"] = torch.zeros(3, H, W, device=dev)
        p["loss"] = torch.zeros(5, dtype=torch.float64, device=dev)
    # NEXT-3 density statistic, accumulated by every training view (3DGS: every iteration of the
    # densification window), phi from the importance counts the views accumulate
    dc_stat = torch.zeros(max(n_local, 1), dtype=torch.float32, device=dev)
    dc_count = torch.zeros(max(n_local, 1), dtype=torch.int32, device=dev)

    def train_on(k, v):
        p = per[k]
        B.bgs_train_view_step(ctxs[k], g, cams[v % len(cams)], gate,
                              cull_cols[v % len(cams)] if cull_cols is not None else None, 0, p["radius"],
                              B.supervision(tgt, lam, binv, beta, p["loss"]), p["rgb"], p["Tf"], p["nc"], p["dl"],
                              grads, B.importance_out(s_imp, c_rad, c_vis, p["cull"], 99, 100), p["stream"])
        B.bgs_densify_accumulate(ctxs[k], n_local, None, dc_stat, dc_count, p["stream"])

    for k in range(inflight):
        with torch.cuda.stream(per[k]["stream"]):
            for w in range(args.warmup):
                train_on(k, w)
    torch.cuda.synchronize()
    barrier()
    # stage breakdown: one view at a time, L2 flushed before each
    stages = np.zeros(len(B.STAGES))
    with torch.cuda.stream(stream):
        B.bgs_set_stage_timing(ctxs[0], True)
        for k in range(args.steps):
            l2_flush.zero_()
            stream.synchronize()
            train_on(0, args.warmup + k)
            stream.synchronize()
            st = B.bgs_stage_times(ctxs[0])
            stages += np.array([st[n] for n in B.STAGES])
        B.bgs_set_stage_timing(ctxs[0], False)
    torch.cuda.synchronize()
    barrier()
    # headline-style: views in flight
    ev_start = torch.cuda.Event(enable_timing=True)
    ev_end = [torch.cuda.Event(enable_timing=True) for _ in range(inflight)]
    ev_start.record(per[0]["stream"])
    for k in range(1, inflight):
        per[k]["stream"].wait_event(ev_start)
    submit_views(train_on, inflight, [args.warmup + k for k in range(args.steps)], bool(args.host_threads),
                 int(str(dev).split(":")[-1]))
    for k in range(inflight):
        ev_end[k].record(per[k]["stream"])
    torch.cuda.synchronize()
    ms = D.max_over_ranks(max(ev_start.elapsed_time(e) for e in ev_end), torch.device(dev)) / args.steps
    loss = per[0]["loss"].cpu().tolist()
    barrier()
    # end to end: every view's target uploaded from pinned memory, its loss read back
    tgt_h = [torch.from_numpy(S.target_image(H, W, seed=9 + k)).pin_memory() for k in range(inflight)]
    loss_h = [torch.zeros(5, dtype=torch.float64).pin_memory() for _ in range(inflight)]

    def host_on(k, v):
        p = per[k]
        B.bgs_train_view_step_host_async(ctxs[k], g, cams[v % len(cams)], gate,
                                         cull_cols[v % len(cams)] if cull_cols is not None else None, 0,
                                         p["radius"], tgt_h[k], lam, binv, beta, loss_h[k], grads,
                                         B.importance_out(s_imp, c_rad, c_vis, p["cull"], 99, 100), p["stream"])

    for k in range(inflight):
        host_on(k, k)
    torch.cuda.synchronize()
    barrier()
    t1 = time.perf_counter()
    submit_views(host_on, inflight, [args.warmup + k for k in range(args.steps)], bool(args.host_threads),
                 int(str(dev).split(":")[-1]))
    torch.cuda.synchronize()
    e2e = args.steps / D.max_over_ranks(time.perf_counter() - t1, torch.device(dev))
    # NEXT-3: the optimizer step of the batch (bgs_adam_step) on this rank's shard, dense (every row)
    # and selective (rows some view of the batch projected: the union of the records' c_rad bits)
    adam = adam_step_timing(B, S, g, grads, ctxs[0], stream, dev, n_local, l2_flush, cams, gate, cull_cols, per,
                            s_imp, c_rad, c_vis, args, dc_stat, dc_count)
    return {"metric": "supervised training views/s (a1-a12 + Eq.7 L1+SSIM on owned tiles + Eq.8, NEXT-4)",
            "value": round(1000.0 / ms, 3), "unit": "views/s", "ms_per_view": round(ms, 4),
            "lambda": lam, "batch_inv": binv, "beta": beta,
            "stages_ms": {n: round(float(v) / args.steps, 4) for n, v in zip(B.STAGES, stages)},
            "stages_avg": stages / args.steps,
            "loss_last_view": {"l": loss[0], "L1": loss[1], "SSIM": loss[2], "L_scale": loss[3], "V": loss[4]},
            "e2e": {"value": round(e2e, 3), "unit": "views/s", "h2d_bytes_per_step": int(3 * H * W * 4),
                    "d2h_bytes_per_step": 40},
            "adam": adam,
            "batch_of_4_views_per_s": {
                "dense_adam": round(4000.0 / (4 * ms + adam["dense_ms"]), 3),
                "selective_adam": round(4000.0 / (4 * ms + adam["selective_ms"]), 3)}}


def adam_step_timing(B, S, g, grads, ctx, stream, dev, n_local, l2_flush, cams, gate, cull_cols, per, s_imp, c_rad,
                     c_vis, args, dc_stat, dc_count):
    """bgs_adam_step on the shard: raw planes derived from the activated ones, device-timed (L2
    flushed before each), dense and with the visibility mask of a 4-view batch."""
    import torch
    from paper_2605_13794_b200 import dist as D
    mo = g.mean_opac
    o = mo[:, 3].clamp(1e-6, 1 - 1e-6)
    ml = torch.cat([mo[:, :3], torch.log(o / (1 - o))[:, None]], 1).contiguous()
    tp = B.TrainParams(ml, g.quat.clone(), torch.log(g.scale.clamp_min(1e-30)).contiguous(), g.sh.clone())
    tp.log_scale[:, 3] = 0
    act = B.GaussianPlanes(torch.empty_like(mo), torch.empty_like(g.quat), torch.empty_like(g.scale), tp.sh, g.lod)
    # the batch's visible rows: radius > 0 in any of 4 views (from the in-flight contexts' last views)
    vis = torch.zeros(max(n_local, 1), dtype=torch.bool, device=dev)
    for p in per[:4]:
        vis |= p["radius"][:max(n_local, 1)] > 0
    bits = vis.view(-1)
    pad = (-bits.numel()) % 32
    words = torch.nn.functional.pad(bits.to(torch.int64), (0, pad)).view(-1, 32)
    mask = (words << torch.arange(32, device=dev, dtype=torch.int64)).sum(1).to(torch.int64)
    mask = torch.where(mask >= 2 ** 31, mask - 2 ** 32, mask).to(torch.int32).contiguous()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    out = {}
    with torch.cuda.stream(stream):
        for name, m in (("dense", None), ("selective", mask)):
            tot = 0.0
            for k in range(args.warmup + args.steps):
                l2_flush.zero_()
                stream.synchronize()
                ev[0].record(stream)
                B.bgs_adam_step(ctx, tp, grads, act, m, B.adam_hparams(step=k + 1), stream)
                ev[1].record(stream)
                stream.synchronize()
                if k >= args.warmup:
                    tot += ev[0].elapsed_time(ev[1])
            out[f"{name}_ms"] = round(D.max_over_ranks(tot / args.steps, torch.device(dev)), 4)
    rows = float(vis[:n_local].sum().item())
    # algorithmic bytes per updated row: read raw 240 + grads 240 + m 240 + v 240; write raw 240 +
    # m 240 + v 240 + activated 48 (SH aliases the raw plane) + zeroed grads 240
    per_row = 4 * 240 + 4 * 240 + 48
    peaks_gbs = load_peaks()["hbm_gbs"]
    for name, nrows in (("dense", float(n_local)), ("selective", rows)):
        ach = per_row * nrows / (out[f"{name}_ms"] * 1e-3) / 1e9 if out[f"{name}_ms"] > 0 else 0.0
        out[f"{name}_roofline"] = {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks_gbs, "unit": "GB/s",
                                   "frac": round(ach / peaks_gbs, 4), "rows": int(nrows),
                                   "work": f"{per_row} B x rows"}
    out["note"] = ("one optimizer step per batch of B = 4 views (P:342); selective = rows projected by any view "
                   "of the batch (visibility mask), dense = every row of the shard")
    # NEXT-3 density control on the shard with the statistic of the timed training views (tau chosen
    # as the 99th percentile of the per-Gaussian average so that ~1% densify; 3DGS's 2e-4 is scale-
    # dependent), extent 1% of the scene (1000 units): wall time of the HOST-SYNC call
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
        out["densify"] = {"apply_ms": round(D.max_over_ranks(ms, torch.device(dev)), 4), "rows_in": int(n_local),
                          "rows_out": int(n_new), "tau": tau, "dense_extent": 10.0,
                          "roofline": {"bound": "hbm", "achieved": round(byt / (ms * 1e-3) / 1e9, 1),
                                       "peak": peaks_gbs, "unit": "GB/s",
                                       "frac": round(byt / (ms * 1e-3) / 1e9 / peaks_gbs, 4)},
                          "note": "statistic accumulated by every timed training view (bgs_densify_accumulate); "
                                  "apply is HOST-SYNC, wall time incl. the count round trip"}
        del tout, act2
    del tp, act
    return out


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "source": "measured", "sm_max_mhz": d.get("sm_max_mhz", 1965.0)}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)", "sm_max_mhz": 1965.0}


# ------------------------------------------------------------------------------------------
# oracle baselines (the one other place bench.py executes oracle/)
# ------------------------------------------------------------------------------------------
def oracle_sample(scene, views, frac_tiles: float):
    """The oracle's time per view on this workload: full projection + routing + sort of every
    view, compositing fwd+bwd on a `frac_tiles` sample of the tiles, scaled to a whole view."""
    import oracle as O
    import synthetic as S
    cam = scene.cameras[views % len(scene.cameras)]
    dl = S.grad_image(cam["H"], cam["W"])
    st = O.OracleStep(scene, cam, M=1, dLdC=dl, tile_frac=frac_tiles)
    return st.seconds, st.seconds_by_phase()


def cpu_baseline(scene, args):
    import oracle as O
    frac = 1.0 / 8
    secs, phases = oracle_sample(scene, args.warmup, frac)
    comp = phases["composite"] / frac
    per_view = phases["project"] + phases["route_sort"] + comp + phases["project_bwd"]
    return {"value": round(1.0 / per_view, 5), "unit": "views/s", "cores": 1, "kind": "oracle",
            "sample": f"one view of the same workload: oracle projection, ownership, routing and sort of all "
                      f"{scene.n} Gaussians, compositing fwd+bwd of a {frac:.3f} sample of the tiles scaled "
                      f"x{1 / frac:.0f} ({secs:.1f} s of CPU work, 1 thread)",
            "phases_s": {k: round(v, 3) for k, v in phases.items()}, "oracle_lib": os.path.basename(O.build())}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synthetic as S
    label, gate_on = CONFIG_SHAPES[args.config]
    scene = S.gen_city(args.config, n=args.n, V=args.views)
    frac = 1.0 / 16
    for w in range(args.warmup):
        oracle_sample(scene, w, frac)
    tot = 0.0
    phase_tot = {}
    for k in range(args.steps):
        secs, ph = oracle_sample(scene, args.warmup + k, frac)
        per_view = ph["project"] + ph["route_sort"] + ph["composite"] / frac + ph["project_bwd"]
        tot += per_view
        for kk, v in ph.items():
            phase_tot[kk] = phase_tot.get(kk, 0.0) + v
    v = args.steps / tot
    W, H = scene.cameras[0]["W"], scene.cameras[0]["H"]
    out = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "views/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1000 * tot / args.steps, 2),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": label, "config": args.config, "gaussians": scene.n, "width": W, "height": H},
           "cpu_baseline": {"value": round(v, 6), "unit": "views/s", "cores": 1, "kind": "oracle",
                            "sample": f"per step: oracle projection/ownership/sort of all {scene.n} Gaussians of "
                                      f"one view + fwd+bwd compositing of a {frac:.4f} tile sample scaled "
                                      f"x{1 / frac:.0f}"},
           "e2e": {"value": round(v, 6), "unit": "views/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_native(a)
