"""e2e breakdown: host-buffer run_pipeline with / without hit vectors, and the
raw pinned copy bandwidth of this box (H2D 51 MB, D2H 520 MB)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2512_02278_b200 as dvs  # noqa: E402
import torch  # noqa: E402

sys.argv = ["x"]
args = bench.parse()
ctx = dvs.Context(0)
data, queries, index = bench.workload(args, 0, ctx)
ctx.load_index(index)
p = dvs.SearchParams(6, 64, 10, 64, accum="f32")
nq = args.nq
pin = lambda shape, dt: torch.empty(shape, dtype=dt, pin_memory=True)  # noqa: E731
hq = pin((nq, 128), torch.float32)
hq.numpy()[:] = queries
out_t = {"ids": pin((nq, 10), torch.int32), "dists": pin((nq, 10), torch.float32),
         "counts": pin((nq,), torch.int32), "vectors": pin((nq, 10, 128), torch.float32)}
out = {"ids": out_t["ids"].numpy().view(np.uint32), "dists": out_t["dists"].numpy(),
       "counts": out_t["counts"].numpy().view(np.uint32), "vectors": out_t["vectors"].numpy()}
for wv in (True, False):
    for _ in range(2):
        ctx.run_pipeline(hq.numpy(), p, 1, 1, 0, wv, out)
    t0 = time.perf_counter()
    for _ in range(5):
        ctx.run_pipeline(hq.numpy(), p, 1, 1, 0, wv, out)
    print(f"run_pipeline host buffers, vectors={wv}: {(time.perf_counter() - t0) / 5 * 1e3:.2f} ms", flush=True)
d = torch.empty((nq, 10, 128), dtype=torch.float32, device="cuda")
dq = torch.empty((nq, 128), dtype=torch.float32, device="cuda")
for name, dst, src in (("H2D 51MB", dq, hq), ("D2H 512MB", out_t["vectors"], d)):
    for _ in range(2):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(f"{name}: {dt * 1e3:.2f} ms = {src.numel() * 4 / dt / 1e9:.1f} GB/s", flush=True)
