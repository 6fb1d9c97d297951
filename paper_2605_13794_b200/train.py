"""NEXT-4: the training iteration and its schedule on top of the C ABI.

PAPER.md §4.1: batches of B = 4 views; density control every 500 steps from iteration 2,000 to
20,000; the LOD gate disabled inside that window and engaged afterwards; importance-scoring passes
at T1 = 15,000 (stochastic pruning) and T2 = 40,000 (cumulative-mass pruning), each followed by an
index-parity redistribution; after T1 the density statistic is reweighted by phi.
§3.4: L_max(t) unlocks levels coarse-to-fine on a geometric schedule (reading R21: SPEC
S:398's default, L_max = 0 until step 2,000, then +1 at 2,000 * 2^k up to K - 1).  §3.5 P:213-227:
Eq.7 L1 + SSIM (lambda = 0.2) and Eq.8 (beta = 10) on the owned tiles.

Everything numeric runs in libbgs (bgs_batch_step with supervised views, bgs_visibility_mask,
bgs_densify_accumulate / bgs_densify_apply, bgs_adam_step, the scoring sweep, bgs_prune_*,
bgs_redistribute); this module is the schedule and the host-side bookkeeping of a rank's shard.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Schedule:
    """The paper's iteration schedule (readings R21, R32).  `scaled(f)` shrinks every
    step count by f (short synthetic runs)."""
    dc_start: int = 2000
    dc_end: int = 20000
    dc_every: int = 500
    t1: int = 15000          # first importance-scoring pass: stochastic pruning
    t2: int = 40000          # second pass: cumulative-mass pruning
    unlock_first: int = 2000  # L_max = 0 before, +1 at unlock_first * 2^k
    k_levels: int = 6
    keep_fraction: float = 0.6  # pass-1 keep fraction (S:318 default; reading R32)
    mass_num: int = 99
    mass_den: int = 100

    def scaled(self, f: float) -> "Schedule":
        r = lambda x: max(1, int(round(x * f)))
        return Schedule(r(self.dc_start), r(self.dc_end), r(self.dc_every), r(self.t1), r(self.t2),
                        r(self.unlock_first), self.k_levels, self.keep_fraction, self.mass_num, self.mass_den)

    def l_max(self, t: int) -> int:
        """L_max(t): 0 before unlock_first, then one more level at every doubling of t (integer
        steps unlock_first * 2^k), capped at K - 1; non-decreasing in t."""
        lm, step = 0, self.unlock_first
        while t >= step and lm < self.k_levels - 1:
            lm += 1
            step *= 2
        return lm

    def gate_enabled(self, t: int) -> bool:
        """The LOD gate is disabled inside the density-control window, engaged outside it."""
        return not (self.dc_start <= t <= self.dc_end)

    def densify_due(self, t: int) -> bool:
        return self.dc_start <= t <= self.dc_end and (t - self.dc_start) % self.dc_every == 0

    def accumulate_stats(self, t: int) -> bool:
        return self.dc_start <= t <= self.dc_end

    def phi_active(self, t: int) -> bool:
        """After the first scoring pass the density statistic is reweighted by phi."""
        return t > self.t1

    def scoring_due(self, t: int) -> str | None:
        return "stochastic" if t == self.t1 else ("mass" if t == self.t2 else None)


def epoch_order(n_views: int, seed: int, epoch: int) -> np.ndarray:
    """Training cameras sampled without replacement per epoch (seeded)."""
    return np.random.Generator(np.random.PCG64([seed, epoch])).permutation(n_views)


@dataclass
class StepLog:
    t: int
    loss: float
    l1: float
    ssim: float
    n_gaussians: int
    l_max: int
    gate: bool
    event: str = ""
    extra: dict = field(default_factory=dict)


class Trainer:
    """One rank's training loop (world 1 here; the ABI calls are the same at world > 1 with an NCCL
    ctx per rank).  params: raw parameters (bgs.TrainParams), lod: u8 device tensor, cams: camera
    dicts, targets: device f32 [3][H][W] per camera, d0: the LOD reference distance (R19)."""

    def __init__(self, ctx, params, lod, cams, targets, d0, sched: Schedule, batch: int = 4, lam: float = 0.2,
                 beta: float = 10.0, seed: int = 0, densify=None, device: str = "cuda:0", hp=None,
                 bounds: bool = True):
        import torch

        import paper_2605_13794_b200.bgs as B
        self.B, self.torch = B, torch
        self.ctx, self.p, self.lod = ctx, params, lod
        self.cams = cams
        self.bcams = [B.camera(c) for c in cams]
        self.targets = targets
        self.d0, self.sched, self.batch = float(d0), sched, batch
        self.lam, self.beta, self.seed = lam, beta, seed
        self.dev = device
        self.dp = densify
        self.hp = hp or {}
        self.use_bounds = bounds  # block bounds for hierarchical culling, refreshed after every update
        self.H, self.W = cams[0]["H"], cams[0]["W"]
        self.stream = torch.cuda.Stream(device)
        self.step_count = 0  # Adam step t
        self.cull = None     # per-view Cull columns of the last scoring sweep (N x V bits)
        self.phi = None
        self._order, self._epoch, self._pos = None, -1, 0
        self.per = [dict(rgb=torch.zeros(3, self.H, self.W, device=device),
                         T=torch.zeros(self.H, self.W, device=device),
                         nc=torch.zeros(self.H, self.W, dtype=torch.int32, device=device),
                         dl=torch.zeros(3, self.H, self.W, device=device),
                         loss=torch.zeros(5, dtype=torch.float64, device=device)) for _ in range(batch)]
        self._resize()

    # ---- shard-size dependent buffers
    def _resize(self):
        with self.torch.cuda.stream(self.stream):
            self._resize_on_stream()

    def _resize_on_stream(self):
        torch, B = self.torch, self.B
        n = self.p.n
        self.n = n
        dev = self.dev
        self.act = B.GaussianPlanes(torch.empty(n, 4, device=dev), torch.empty(n, 4, device=dev),
                                    torch.empty(n, 4, device=dev), self.p.sh, self.lod)
        self._activate()
        if self.use_bounds:
            B.bgs_shard_bounds(self.ctx, self.act, stream=self.stream)
        self.grads = self.act.zeros_grads()
        self.stat = torch.zeros(max(n, 1), dtype=torch.float32, device=dev)
        self.count = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        self.vis = torch.zeros((max(n, 1) + 31) // 32, dtype=torch.int32, device=dev)
        for p in self.per:
            p["radius"] = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)

    def _activate(self):
        """Activated planes from the raw ones (R13): the first Adam step rewrites them on device;
        after a resize the planes are formed once here."""
        torch = self.torch
        ml, q, ls = self.p.mean_logit, self.p.quat_raw, self.p.log_scale
        self.act.mean_opac.copy_(torch.cat([ml[:, :3], torch.sigmoid(ml[:, 3:4])], 1))
        self.act.quat.copy_(q / q.norm(dim=1, keepdim=True))
        sc = torch.exp(ls)
        sc[:, 3] = 0
        self.act.scale.copy_(sc)

    def _next_views(self):
        out = []
        for _ in range(self.batch):
            if self._order is None or self._pos >= len(self._order):
                self._epoch += 1
                self._order = epoch_order(len(self.cams), self.seed, self._epoch)
                self._pos = 0
            out.append(int(self._order[self._pos]))
            self._pos += 1
        return out

    # ---- one iteration
    def step(self, t: int) -> StepLog:
        B, torch, sc = self.B, self.torch, self.sched
        gate_on = sc.gate_enabled(t)
        gate = B.lod_gate(True, sc.l_max(t), self.d0) if gate_on else None
        vids = self._next_views()
        sups, views = [], []
        for k, v in enumerate(vids):
            p = self.per[k]
            sup = B.supervision(self.targets[v], self.lam, 1.0 / self.batch, self.beta / self.batch, p["loss"])
            sups.append(sup)
            cull = self.cull[v] if (self.cull is not None and gate_on) else None
            views.append(B.batch_view(self.bcams[v], p["radius"], p["rgb"], p["T"], p["nc"], cull_column=cull,
                                      sup=sup, dL_scratch=p["dl"]))
        st = self.stream
        with torch.cuda.stream(st):
            B.bgs_batch_step(self.ctx, self.act, views, gate, 0, self.grads, None, st)
            for k in range(self.batch):
                if sc.accumulate_stats(t):
                    B.bgs_densify_accumulate(self.ctx.batch_view(k), self.n,
                                             self.phi if sc.phi_active(t) else None, self.stat, self.count, st)
                B.bgs_visibility_mask(self.ctx, self.n, self.per[k]["radius"], self.vis, st)
            self.step_count += 1
            B.bgs_adam_step(self.ctx, self.p, self.grads, self.act, self.vis,
                            B.adam_hparams(step=self.step_count, **self.hp), st)
            if self.use_bounds:
                B.bgs_shard_bounds(self.ctx, self.act, self.act.bounds, st)
            self.vis.zero_()
        event = ""
        if sc.densify_due(t) and self.dp is not None:
            event = self._densify()
        mode = sc.scoring_due(t)
        if mode:
            event += ("; " if event else "") + self._score_and_prune(mode)
        st.synchronize()
        losses = np.stack([p["loss"].cpu().numpy() for p in self.per])
        return StepLog(t, float(losses[:, 0].sum()), float(losses[:, 1].mean()), float(losses[:, 2].mean()), self.n,
                       sc.l_max(t), gate_on, event)

    # ---- density control
    def _densify(self) -> str:
        B, torch = self.B, self.torch
        st = self.stream
        n = self.n
        cap = 2 * n + 1
        dev = self.dev
        out = B.TrainParams(*(torch.empty(cap, c, device=dev) for c in (4, 4, 4, 48)))
        lod_out = torch.empty(cap, dtype=torch.uint8, device=dev)
        with torch.cuda.stream(st):
            n_new = B.bgs_densify_apply(self.ctx, self.p, self.lod, self.stat, self.count, self.dp, out, lod_out, None,
                                        st)
        tp = B.TrainParams(out.mean_logit[:n_new].clone(), out.quat_raw[:n_new].clone(), out.log_scale[:n_new].clone(),
                           out.sh[:n_new].clone())
        tp.m = [m[:n_new].clone() for m in out.m]
        tp.v = [v[:n_new].clone() for v in out.v]
        self.p, self.lod = tp, lod_out[:n_new].clone()
        # the Cull columns index the old rows (pruned originals shift the survivors, new rows are
        # appended): a stale column would mask the wrong Gaussians, so the mask is dropped
        # until the next scoring sweep rebuilds it
        self.cull = None
        if self.phi is not None:  # phi of the new rows is not known until the next sweep: 1
            self.phi = torch.ones(max(n_new, 1), dtype=torch.float64, device=dev)
        self._resize()
        return f"densify {n} -> {n_new}"

    # ---- importance-scoring pass + simplification
    def _score_and_prune(self, mode: str) -> str:
        B, torch = self.B, self.torch
        st = self.stream
        n, dev = self.n, self.dev
        nw = (max(n, 1) + 31) // 32
        s = torch.zeros(max(n, 1), dtype=torch.float64, device=dev)
        c_rad = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        c_vis = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        culls = [torch.zeros(nw, dtype=torch.int32, device=dev) for _ in self.cams]
        p = self.per[0]
        with torch.cuda.stream(st):
            # the sweep renders the full shard (reading R22: gate and cull off), NO_COLOR, instrumented
            for v, cam in enumerate(self.bcams):
                B.bgs_view_step(self.ctx, self.act, cam, None, None, B.BGS_NO_COLOR, p["radius"], p["rgb"], p["T"],
                                p["nc"], None, None, B.importance_out(s, c_rad, c_vis, culls[v], self.sched.mass_num,
                                                                      self.sched.mass_den), st)
            phi = torch.zeros(max(n, 1), dtype=torch.float64, device=dev)
            B.bgs_score_phi(self.ctx, n, c_rad, c_vis, phi, st)
            keep = torch.zeros(max(n, 1), dtype=torch.uint8, device=dev)
            if mode == "stochastic":
                B.bgs_prune_stochastic(self.ctx, n, s, int(round(self.sched.keep_fraction * n)), self.seed + 17, keep, st)
            else:
                B.bgs_prune_mass_cut(self.ctx, n, s, self.sched.mass_num, self.sched.mass_den, keep, st)
            # survivors: parameters, moments, phi and the Cull columns move together (R33, R41)
            n_new = self._compact(keep)
            idx = torch.nonzero(keep[:n].bool()).squeeze(1)
            self.phi = phi[idx].contiguous()
            self.cull = []
            for c in culls:
                bits = ((c.view(-1, 1).to(torch.int64) >> torch.arange(32, device=dev)) & 1).view(-1)[:n][idx]
                pad = (-bits.numel()) % 32
                w = (torch.nn.functional.pad(bits, (0, pad)).view(-1, 32) << torch.arange(32, device=dev)).sum(1)
                self.cull.append(torch.where(w >= 2 ** 31, w - 2 ** 32, w).to(torch.int32).contiguous())
        return f"scoring ({mode}) {n} -> {n_new}"

    def _compact(self, keep) -> int:
        """Index-parity redistribution of the survivors (world 1: order-preserving compaction) of
        the raw planes and both Adam moments (three bgs_redistribute calls with one keep mask)."""
        B, torch = self.B, self.torch
        st = self.stream
        dev = self.dev
        n = self.n
        planes = [(self.p.mean_logit, self.p.quat_raw, self.p.log_scale, self.p.sh)]
        planes += [tuple(self.p.m)] + [tuple(self.p.v)]
        outs = []
        n_new = 0
        for k, (a, b, c, d) in enumerate(planes):
            lod_in = self.lod if k == 0 else torch.zeros(max(n, 1), dtype=torch.uint8, device=dev)
            g = B.GaussianPlanes(a, b, c, d, lod_in)
            o = B.GaussianPlanes(torch.empty(n + 1, 4, device=dev), torch.empty(n + 1, 4, device=dev),
                                 torch.empty(n + 1, 4, device=dev), torch.empty(n + 1, 48, device=dev),
                                 torch.empty(n + 1, dtype=torch.uint8, device=dev))
            n_new = B.bgs_redistribute(self.ctx, g, keep, o, st)
            outs.append(o)
        o = outs[0]
        tp = B.TrainParams(o.mean_opac[:n_new].clone(), o.quat[:n_new].clone(), o.scale[:n_new].clone(),
                           o.sh[:n_new].clone())
        tp.m = [outs[1].mean_opac[:n_new].clone(), outs[1].quat[:n_new].clone(), outs[1].scale[:n_new].clone(),
                outs[1].sh[:n_new].clone()]
        tp.v = [outs[2].mean_opac[:n_new].clone(), outs[2].quat[:n_new].clone(), outs[2].scale[:n_new].clone(),
                outs[2].sh[:n_new].clone()]
        self.p, self.lod = tp, o.lod[:n_new].clone()
        self._resize()
        return n_new


def l_max_table(sched: Schedule, ts) -> list:
    return [sched.l_max(int(t)) for t in ts]


def geometric_unlocks(sched: Schedule) -> list:
    """The iterations at which L_max increments: unlock_first * 2^k, k < K - 1."""
    return [sched.unlock_first * (2 ** k) for k in range(sched.k_levels - 1)]


__all__ = ["Schedule", "Trainer", "StepLog", "epoch_order", "geometric_unlocks", "l_max_table"]
