"""The NCCL transport at world 2 (one process per GPU, as bench.py --gpus N runs it): ctx creation from a
broadcast unique id, the per-view route / reverse / importance collectives and the batched step's
single exchange, checked against the oracle at M = 2 (owner map, pair order, pixels bitwise equal to
world 1, w / a).  Needs two GPUs (NCCL refuses two ranks on one device); skipped otherwise -- the same
code paths run on one GPU through the in-process transport in test_gpu_parity / test_gpu_batch."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    import paper_2605_13794_b200.bgs as B
    import synthetic as S
    from paper_2605_13794_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(WORLD))
    torch.cuda.set_device(rank)
    dev = torch.device(f"cuda:{rank}")
    dist.init_process_group("nccl", rank=rank, world_size=WORLD, device_id=dev)
    uid = D.broadcast_bytes(B.unique_id() if rank == 0 else None, 128, dev)
    ctx = B.Context(rank, WORLD, rank, uid)
    sc = S.gen_tiny()
    cam = sc.cameras[0]
    sh = sc.shard(rank, WORLD)
    g = B.GaussianPlanes.from_scene(sh, dev)
    grads = g.zeros_grads()
    H, W = cam["H"], cam["W"]
    n = sh.n
    radius = torch.zeros(n, dtype=torch.int32, device=dev)
    rgb = torch.zeros(3, H, W, device=dev)
    T = torch.zeros(H, W, device=dev)
    nc = torch.zeros(H, W, dtype=torch.int32, device=dev)
    dl = torch.from_numpy(S.grad_image(H, W)).to(dev)
    s = torch.zeros(n, dtype=torch.float64, device=dev)
    cr = torch.zeros(n, dtype=torch.int32, device=dev)
    cv = torch.zeros(n, dtype=torch.int32, device=dev)
    cull = torch.zeros((n + 31) // 32, dtype=torch.int32, device=dev)
    owner = torch.zeros(256, dtype=torch.int32, device=dev)
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        B.bgs_project(ctx, g, B.camera(cam), None, None, 0, radius, stream)
        B.bgs_route(ctx, owner, stream)
        B.bgs_sort_tiles(ctx, stream)
        B.bgs_raster_fwd(ctx, B.BGS_IMPORTANCE, rgb, T, nc, stream)
        B.bgs_raster_bwd(ctx, dl, T, nc, stream)
        B.bgs_route_reverse(ctx, stream)
        B.bgs_project_bwd(ctx, g, B.camera(cam), grads, stream)
        B.bgs_importance(ctx, n, radius, None, None, s, cr, cv, cull, stream=stream)
        stream.synchronize()
        q = ctx.query()
        vals = ctx.debug_buffer("vals").view(torch.int32).cpu().numpy()
        recv = ctx.debug_buffer("recv").cpu().numpy().view(np.uint32).reshape(-1, 12)
        # the batched step (one exchange per batch) on the same view twice
        bb = [dict(radius=torch.zeros(n, dtype=torch.int32, device=dev), rgb=torch.zeros(3, H, W, device=dev),
                   T=torch.zeros(H, W, device=dev), nc=torch.zeros(H, W, dtype=torch.int32, device=dev))
              for _ in range(2)]  # each view of a batch has its own outputs (the views run concurrently)
        views = [B.batch_view(B.camera(cam), b["radius"], b["rgb"], b["T"], b["nc"], dl) for b in bb]
        c0 = ctx.batch_stats()["collectives"]
        B.bgs_batch_step(ctx, g, views, None, 0, grads, None, stream)
        stream.synchronize()
        batch_coll = ctx.batch_stats()["collectives"] - c0
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), owner=owner.cpu().numpy(), rgb=rgb.cpu().numpy(),
             nc=nc.cpu().numpy(), tile_begin=q["tile_begin"], tile_end=q["tile_end"],
             pair_gid=recv[vals, 10].astype(np.int64), c_vis=cv.cpu().numpy(), batch_coll=batch_coll,
             rgb_batch=bb[1]["rgb"].cpu().numpy())
    ctx.close()
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < WORLD, reason="NCCL world 2 needs two GPUs")
def test_nccl_world2_matches_oracle(tmp_path):
    import torch.multiprocessing as mp

    import oracle as O
    import synthetic as S
    port = _free_port()
    mp.start_processes(_worker, args=(port, str(tmp_path)), nprocs=WORLD, start_method="spawn")
    sc = S.gen_tiny()
    cam = sc.cameras[0]
    dl = S.grad_image(cam["H"], cam["W"])
    st = O.OracleStep(sc, cam, M=WORLD, dLdC=dl)
    img = np.zeros((3, cam["H"], cam["W"]), np.float32)
    for r in range(WORLD):
        d = np.load(tmp_path / f"rank{r}.npz")
        assert np.array_equal(d["owner"], st.get("owner"))
        b, e = st.get("tile_range", r)
        assert (int(d["tile_begin"]), int(d["tile_end"])) == (b, e)
        assert np.array_equal(d["pair_gid"], st.get("pair_gid", r))
        assert int(d["batch_coll"]) == 4
        assert np.array_equal(d["rgb_batch"], d["rgb"])
        for t in range(b, e):
            ty, tx = divmod(t, 16)
            img[:, ty * 16:ty * 16 + 16, tx * 16:tx * 16 + 16] = d["rgb"][:, ty * 16:ty * 16 + 16, tx * 16:tx * 16 + 16]
    ref = st.get("img").reshape(img.shape)
    assert np.abs(img - ref).max() <= 1e-4
