"""Drive the CUDA path through the C ABI (the binding) and return host numpy views keyed like
the oracle's outputs.  Test infrastructure only."""
from __future__ import annotations

import threading

import numpy as np
import torch

import synthetic as S


def rec_view(raw: torch.Tensor) -> dict:
    """48-B records -> dict of numpy arrays (see include/bgs.h debug buffer 0)."""
    a = raw.cpu().numpy().view(np.float32).reshape(-1, 12)
    u = a.view(np.uint32)
    rect = u[:, 11]
    return dict(mx=a[:, 0], my=a[:, 1], A=a[:, 2], B=a[:, 3], C=a[:, 4], opac=a[:, 5], rgb=a[:, 6:9],
                depth=a[:, 9], gid=u[:, 10].astype(np.int64),
                rect=np.stack([rect & 255, (rect >> 8) & 255, (rect >> 16) & 255, rect >> 24], 1).astype(np.int32))


def acc_view(raw: torch.Tensor) -> dict:
    b = raw.cpu().numpy()
    f = b.view(np.float32).reshape(-1, 12)
    return dict(g=f[:, :9].astype(np.float64), a=f[:, 9].view(np.uint32).copy(),
                w=b.view(np.uint64).reshape(-1, 6)[:, 5].copy())


def decode_key_tiles(keys: np.ndarray, counters: np.ndarray, n_tiles: int) -> np.ndarray:
    """Sorted u32 keys (include/bgs.h debug buffer 3) -> local tile of every pair."""
    lo = 0xFFFFFFFF - int(counters[6] & np.uint64(0xFFFFFFFF))
    hi = int(counters[7] & np.uint64(0xFFFFFFFF))
    nb = max(0, hi - lo).bit_length()
    tbits = max(0, int(n_tiles) - 1).bit_length()
    kd = min(nb, 32 - tbits)
    return (keys.astype(np.uint64) >> np.uint64(kd)).astype(np.int32)


def range_tiles(ranges: np.ndarray, P: int) -> np.ndarray:
    """Local tile of every sorted pair from the per-tile ranges [start, end) (a7; include/bgs.h
    debug buffer 5), which cover [0, P) contiguously in tile order."""
    r = np.asarray(ranges, np.int64).reshape(-1, 2)
    t = np.repeat(np.arange(len(r), dtype=np.int32), np.maximum(r[:, 1] - r[:, 0], 0))
    assert t.size == P, (t.size, P)
    return t


def moments_to_g2d(g: np.ndarray, rec: dict) -> np.ndarray:
    """Accumulator moments (include/bgs.h debug buffer 6) -> dL/d(mx,my,A,B,C,o,r,g,b), with the
    record's own o, A, B, C (bit-identical to the oracle's, test_project_bit_exact)."""
    o, A, B, C = (rec[k].astype(np.float64) for k in ("opac", "A", "B", "C"))
    out = g.copy()
    out[:, 0] = -o * (A * g[:, 0] + B * g[:, 1])
    out[:, 1] = -o * (B * g[:, 0] + C * g[:, 1])
    out[:, 2] = -0.5 * o * g[:, 2]
    out[:, 3] = -o * g[:, 3]
    out[:, 4] = -0.5 * o * g[:, 4]
    return out


class GpuStep:
    """One view through a1..a12 on one ctx (world 1) or an in-process group (world > 1)."""

    def __init__(self, scene, cam, M=1, gate=None, cull_global=None, flags=0, dLdC=None, importance=True,
                 ctxs=None, device=0, target=None, lam=0.2, batch_inv=1.0, beta=None, densify=False, phi=None,
                 owner_in=None, imp_only=False):
        import paper_2605_13794_b200.bgs as B
        self.B = B
        self.M = M
        self.scene, self.cam = scene, cam
        dev = f"cuda:{device}"
        self.ctxs = ctxs or (B.Context.local_group(M, device) if M > 1 else [B.Context(0, 1, device)])
        H, W = cam["H"], cam["W"]
        self.H, self.W = H, W
        self.rank = [dict() for _ in range(M)]
        bcam = B.camera(cam)
        bgate = None if gate is None else B.lod_gate(True, gate.get("l_max", 31), gate["d0"], gate.get("fb_num", 19),
                                                     gate.get("fb_den", 20))
        errors = []

        def run(r):
            try:
                torch.cuda.set_device(device)
                stream = torch.cuda.Stream(device)
                with torch.cuda.stream(stream):
                    sh = scene.shard(r, M)
                    g = B.GaussianPlanes.from_scene(sh, dev)
                    n = sh.n
                    cull = None
                    if cull_global is not None:
                        bits = S.unpack_bits(cull_global, scene.n)[r::M]
                        cull = torch.from_numpy(S.pack_bits(bits).astype(np.int32)).to(dev)
                    radius = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
                    rgb = torch.full((3, H, W), -1.0, device=dev)
                    T = torch.full((H, W), -1.0, device=dev)
                    nc = torch.full((H, W), -1, dtype=torch.int32, device=dev)
                    ctx = self.ctxs[r]
                    owner = torch.zeros(max(1, ((W + 15) // 16) * ((H + 15) // 16)), dtype=torch.int32, device=dev)
                    out = self.rank[r]
                    B.bgs_project(ctx, g, bcam, bgate, cull, flags, radius, stream)
                    out["q_project"] = ctx.query()
                    out["records"] = rec_view(ctx.debug_buffer("records"))
                    out["rec_lidx"] = ctx.debug_buffer("rec_lidx").view(torch.int32).cpu().numpy()
                    oin = None if owner_in is None else torch.from_numpy(np.ascontiguousarray(owner_in, np.int32)).to(dev)
                    out["R_route"] = B.bgs_route(ctx, owner, stream, tile_owner_in=oin)
                    out["owner"] = owner.cpu().numpy()
                    B.bgs_sort_tiles(ctx, stream)
                    out["q"] = ctx.query()
                    out["counters"] = ctx.debug_buffer("counters").view(torch.int64).cpu().numpy().view(np.uint64)
                    out["vals"] = ctx.debug_buffer("vals").view(torch.int32).cpu().numpy()
                    out["ranges"] = ctx.debug_buffer("ranges").view(torch.int32).cpu().numpy().reshape(-1, 2)
                    out["key_tile"] = range_tiles(out["ranges"], out["q"]["P"])
                    # bucket sort (default): keys = f32 bits(depth) - lo, sorted within each tile
                    out["keys"] = ctx.debug_buffer("keys").view(torch.int32).cpu().numpy().view(np.uint32)
                    recv = ctx.debug_buffer("recv") if M > 1 else ctx.debug_buffer("records")
                    out["recv"] = rec_view(recv)
                    out["recv_raw"] = recv
                    B.bgs_raster_fwd(ctx, flags | (B.BGS_IMPORTANCE if importance else 0), rgb, T, nc, stream)
                    if target is not None:  # NEXT-4 Eq.7 on the owned tiles
                        tgt = torch.from_numpy(np.ascontiguousarray(target, np.float32)).to(dev)
                        dlo = torch.full((3, H, W), 7.0, device=dev)  # sentinel: non-owned pixels untouched
                        lo = torch.full((3,), -1.0, dtype=torch.float64, device=dev)
                        B.bgs_loss_photo(ctx, rgb, tgt, lam, batch_inv, dlo, lo, stream)
                        stream.synchronize()
                        out["loss"] = lo.cpu().numpy()
                        out["dl_loss"] = dlo.cpu().numpy()
                    if dLdC is not None:
                        dl = torch.from_numpy(np.ascontiguousarray(dLdC, np.float32)).to(dev)
                        B.bgs_raster_bwd(ctx, dl, T, nc, stream)
                    B.bgs_route_reverse(ctx, stream, B.BGS_IMPORTANCE_ONLY if imp_only else 0)
                    out["acc_local"] = acc_view(ctx.debug_buffer("acc_local"))
                    if densify:  # NEXT-3 statistic of this view
                        stat = torch.zeros(max(n, 1), dtype=torch.float32, device=dev)
                        cnt = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
                        ph = None if phi is None else torch.from_numpy(np.ascontiguousarray(phi[r::M])).to(dev)
                        B.bgs_densify_accumulate(ctx, n, ph, stat, cnt, stream)
                        stream.synchronize()
                        out["dc_stat"] = stat.cpu().numpy()[:n]
                        out["dc_count"] = cnt.cpu().numpy()[:n]
                    grads = g.zeros_grads()
                    if dLdC is not None:
                        B.bgs_project_bwd(ctx, g, bcam, grads, stream)
                    if beta is not None:  # NEXT-4 Eq.8
                        sg = g.zeros_grads()
                        so = torch.full((2,), -1.0, dtype=torch.float64, device=dev)
                        B.bgs_loss_scale(ctx, g, beta, sg, so, stream)
                        stream.synchronize()
                        out["loss_scale"] = so.cpu().numpy()
                        out["g_scale_reg"] = sg.scale.cpu().numpy()
                    if importance:
                        s = torch.zeros(max(n, 1), dtype=torch.float64, device=dev)
                        crad = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
                        cvis = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
                        cullo = torch.zeros(max(1, (n + 31) // 32), dtype=torch.int32, device=dev)
                        B.bgs_importance(ctx, n, radius, None, None, s, crad, cvis, cullo, stream=stream)
                        stream.synchronize()
                        out["s"] = s.cpu().numpy()[:n]
                        out["c_rad"] = crad.cpu().numpy()[:n]
                        out["c_vis"] = cvis.cpu().numpy()[:n]
                        out["cull"] = cullo.cpu().numpy().view(np.uint32)
                    stream.synchronize()
                    out["radius"] = radius.cpu().numpy()[:n]
                    out["rgb"], out["T"], out["nc"] = rgb.cpu().numpy(), T.cpu().numpy(), nc.cpu().numpy()
                    out["grads"] = {k: getattr(grads, k).cpu().numpy() for k in ("mean_opac", "quat", "scale", "sh")}
                    out["launches"] = ctx.launches()
            except Exception as e:  # pragma: no cover - surfaced below
                errors.append((r, e))

        if M == 1:
            run(0)
        else:
            th = [threading.Thread(target=run, args=(r,)) for r in range(M)]
            for t in th:
                t.start()
            for t in th:
                t.join()
        if errors:
            raise errors[0][1]
        self._merge()

    def _merge(self):
        """Assemble global (gid-ordered) arrays and the stitched image."""
        M, n = self.M, self.scene.n
        self.radius = np.zeros(n, np.int32)
        self.img = np.zeros((3, self.H, self.W), np.float32)
        self.T = np.zeros((self.H, self.W), np.float32)
        self.nc = np.zeros((self.H, self.W), np.int32)
        self.a = np.zeros(n, np.uint32)
        self.w = np.zeros(n, np.uint64)
        self.g2d = np.zeros((n, 9))
        self.s = np.zeros(n)
        self.c_rad = np.zeros(n, np.uint32)
        self.c_vis = np.zeros(n, np.uint32)
        self.cull_bits = np.zeros(n, bool)
        self.grads = {k: None for k in ("mean", "opac", "quat", "scale", "sh")}
        gm = np.zeros((n, 4), np.float32)
        gq = np.zeros((n, 4), np.float32)
        gs = np.zeros((n, 4), np.float32)
        gsh = np.zeros((n, 48), np.float32)
        TX = (self.W + 15) // 16
        self.dl_loss = np.full((3, self.H, self.W), np.nan, np.float32) if "dl_loss" in self.rank[0] else None
        self.loss = [self.rank[r].get("loss") for r in range(M)]
        self.loss_scale = [self.rank[r].get("loss_scale") for r in range(M)]
        self.g_scale_reg = np.zeros((n, 4), np.float32) if "g_scale_reg" in self.rank[0] else None
        self.dc_stat = np.zeros(n, np.float32) if "dc_stat" in self.rank[0] else None
        self.dc_count = np.zeros(n, np.int64) if "dc_stat" in self.rank[0] else None
        for r in range(M):
            o = self.rank[r]
            gids = np.arange(r, n, M)
            self.radius[gids] = o["radius"]
            q = o["q"]
            for t in range(q["tile_begin"], q["tile_end"]):
                ty, tx = divmod(t, TX)
                ys, xs = slice(ty * 16, min(self.H, ty * 16 + 16)), slice(tx * 16, min(self.W, tx * 16 + 16))
                self.img[:, ys, xs] = o["rgb"][:, ys, xs]
                self.T[ys, xs] = o["T"][ys, xs]
                self.nc[ys, xs] = o["nc"][ys, xs]
                if self.dl_loss is not None:
                    self.dl_loss[:, ys, xs] = o["dl_loss"][:, ys, xs]
            lid = o["rec_lidx"]
            g = lid.astype(np.int64) * M + r
            acc = o["acc_local"]
            self.a[g] = acc["a"]
            self.w[g] = acc["w"]
            self.g2d[g] = moments_to_g2d(acc["g"], o["records"])
            if "s" in o:
                self.s[gids] = o["s"]
                self.c_rad[gids] = o["c_rad"]
                self.c_vis[gids] = o["c_vis"]
                self.cull_bits[gids] = S.unpack_bits(o["cull"], len(gids))
            if self.dc_stat is not None:
                self.dc_stat[gids] = o["dc_stat"]
                self.dc_count[gids] = o["dc_count"]
            if self.g_scale_reg is not None:
                self.g_scale_reg[gids] = o["g_scale_reg"][:len(gids)]
            gm[gids] = o["grads"]["mean_opac"]
            gq[gids] = o["grads"]["quat"]
            gs[gids] = o["grads"]["scale"]
            gsh[gids] = o["grads"]["sh"].reshape(-1, 48)
        self.grads = dict(d_mean=gm[:, :3].astype(np.float64), d_opac=gm[:, 3].astype(np.float64),
                          d_quat=gq.astype(np.float64), d_scale=gs[:, :3].astype(np.float64),
                          d_sh=gsh.astype(np.float64))

    def close(self):
        for c in self.ctxs:
            c.close()
