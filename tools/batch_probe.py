"""Host-side timing of bgs_batch_step on the Rubble shard (eager vs graph): host ms per call,
device ms per batch, and the gap between batches (tools only, not a bench number)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_13794_b200.bgs as B  # noqa: E402
import synthetic as S  # noqa: E402

dev = "cuda:0"
torch.cuda.set_device(0)
n = int(os.environ.get("N", "6000000"))
sc = S.gen_city("rubble", n=n)
g = B.GaussianPlanes.from_scene(sc, dev)
ctx = B.Context(0, 1, 0)
perm = B.spatial_order(ctx, g)
g = B.GaussianPlanes(g.mean_opac[perm].contiguous(), g.quat[perm].contiguous(), g.scale[perm].contiguous(),
                     g.sh[perm].contiguous(), g.lod[perm].contiguous())
H, W = 864, 1152
grads = g.zeros_grads()
dl = torch.from_numpy(S.grad_image(H, W)).to(dev)
cams = [B.camera(c) for c in sc.cameras]
per = [dict(radius=torch.zeros(sc.n, dtype=torch.int32, device=dev), rgb=torch.zeros(3, H, W, device=dev),
            T=torch.zeros(H, W, device=dev), nc=torch.zeros(H, W, dtype=torch.int32, device=dev)) for _ in range(4)]
arrs = [(B.bgs_batch_view * 4)(*[B.batch_view(cams[(i * 4 + k) % 64], per[k]["radius"], per[k]["rgb"], per[k]["T"],
                                               per[k]["nc"], dl) for k in range(4)]) for i in range(16)]
stream = torch.cuda.Stream(dev)
for name, flags in (("eager", 0), ("graph", B.BGS_GRAPH)):
    with torch.cuda.stream(stream):
        for i in range(20):
            B.bgs_batch_step(ctx, g, arrs[i % 16], None, flags, grads, None, stream)
        torch.cuda.synchronize()
        hs = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(20):
            t = time.perf_counter()
            B.bgs_batch_step(ctx, g, arrs[i % 16], None, flags, grads, None, stream)
            hs.append((time.perf_counter() - t) * 1e3)
        e1.record(stream)
        torch.cuda.synchronize()
    print(name, "device ms/batch", e0.elapsed_time(e1) / 20, "host ms/call median", np.median(hs), "max", max(hs),
          ctx.batch_stats(), flush=True)
