"""K5 assign_top_c time at large C (SURVEY 8f-3 sizing): nq x C x d fp64."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2512_02278_b200 as dvs
    ctx = dvs.Context(0)
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(1)
    for C, d, nq, c in [(64, 128, 100_000, 4), (1024, 128, 100_000, 8), (4096, 128, 100_000, 8), (4096, 96, 1_000_000, 2)]:
        cents = rng.standard_normal((C, d)).astype(np.float32)
        q = torch.from_numpy(rng.standard_normal((nq, d)).astype(np.float32)).to(dev)
        ctx.reset()
        ctx.set_centroids(cents, None, 1)
        out = torch.empty((nq, c), dtype=torch.int32, device=dev)
        for _ in range(2):
            ctx.assign_top_c_device(q.data_ptr(), nq, d, c, out.data_ptr())
        ctx.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            ctx.assign_top_c_device(q.data_ptr(), nq, d, c, out.data_ptr())
        ctx.synchronize()
        ms = (time.perf_counter() - t0) / 3 * 1e3
        print(json.dumps({"clusters": C, "dim": d, "queries": nq, "c": c, "ms": round(ms, 3),
                          "fp64_gflops": round(2.0 * nq * C * d / (ms / 1e3) / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
