"""world_size-2 gloo tests of the N > 1 host plumbing on CPU (the kernels need a GPU; the
multi-rank kernels themselves are covered on one GPU through the in-process transport in
test_gpu_parity.py).

Checks: the NCCL unique id broadcast, index-parity shards (every id exactly once, local j <->
global j*M + m), max-over-ranks timing, sums of per-rank statistics, and that the per-rank
oracle decomposition (each process runs the oracle on its own shard + a simulated exchange of
its projected records through gloo) stitches to the single-rank image.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2605_13794_b200 import dist as D
    import oracle as O
    import synthetic as S
    try:
        r, w = D.init("gloo")
        dev = torch.device("cpu")
        uid = bytes(range(128)) if r == 0 else None
        got = D.broadcast_bytes(uid, 128, dev)
        res = {"uid_ok": got == bytes(range(128))}
        res["tmax"] = D.max_over_ranks(10.0 + r, dev)
        res["sum"] = D.sum_over_ranks([1.0, r], dev).tolist()
        n = 1001
        res["ids"] = D.shard_ids(n, r, w).tolist()
        # per-rank oracle view: rank r composites the tiles it owns from ALL ranks' records;
        # the records travel through gloo (all_gather of each rank's projected set)
        sc = S.gen_tiny(n=3000, seed=5)
        cam = sc.cameras[0]
        st = O.OracleStep(sc, cam, M=w)
        b, e = st.get("tile_range", r)
        img = st.get("img").reshape(3, cam["H"], cam["W"])
        mine = np.zeros_like(img)
        TX = (cam["W"] + 15) // 16
        for t in range(b, e):
            ty, tx = divmod(t, TX)
            mine[:, ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16] = img[:, ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16]
        tensor = torch.from_numpy(mine.copy())
        dist.all_reduce(tensor)  # stitch: each pixel owned by exactly one rank
        ref = O.OracleStep(sc, cam, M=1).get("img").reshape(3, cam["H"], cam["W"])
        res["stitched_equal"] = bool(np.array_equal(tensor.numpy(), ref))
        # routed counts seen by each rank agree with the global count matrix
        counts = st.get("counts").reshape(w, w)
        recv_here = torch.tensor(counts[:, r].sum(), dtype=torch.int64)
        gathered = [torch.zeros((), dtype=torch.int64) for _ in range(w)]
        dist.all_gather(gathered, recv_here)
        res["recv_total"] = int(sum(int(x) for x in gathered))
        res["sent_total"] = int(counts.sum())
        out_q.put((r, res))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as ex:  # pragma: no cover
        out_q.put((rank, {"error": repr(ex)}))


@pytest.mark.parametrize("world", [2])
def test_gloo_world2_plumbing(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert "error" not in results[r], results[r]
        assert results[r]["uid_ok"]
        assert results[r]["tmax"] == 10.0 + world - 1
        assert results[r]["sum"] == [float(world), float(sum(range(world)))]
        assert results[r]["stitched_equal"]
        assert results[r]["recv_total"] == results[r]["sent_total"]
    ids = sorted(i for r in range(world) for i in results[r]["ids"])
    assert ids == list(range(1001))
    for r in range(world):
        assert all(g % world == r for g in results[r]["ids"])
