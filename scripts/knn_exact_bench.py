"""K6 build_graph on the GPU: byte-like data (fp32 tiles, exact by
construction) vs float data (exact mode: fp32 candidates + fp64 re-rank +
certificate + fp64 fallback).  Host wall clock around the C-ABI call (H2D,
build, D2H), fallback counts from dvsg_last_knn_info."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import paper_2512_02278_b200 as dvs
    from conftest import sift_like
    ctx = dvs.Context(0)
    for n, dim, dg in [(200_000, 128, 32), (1_000_000, 128, 32), (1_000_000, 96, 16)]:
        rng = np.random.default_rng(n + dim)
        for kind in ("bytes", "float"):
            v = sift_like(n, dim, 16, 1) if kind == "bytes" else rng.normal(size=(n, dim)).astype(np.float32)
            ctx.build_graph(v[:2000], dg)  # warm-up
            t0 = time.perf_counter()
            ctx.build_graph(v, dg)
            dt = time.perf_counter() - t0
            mode, fb = ctx.last_knn_info()
            print(json.dumps({"n": n, "dim": dim, "degree": dg, "data": kind, "seconds": round(dt, 3),
                              "exact_mode": mode, "fallback_rows": fb}), flush=True)


if __name__ == "__main__":
    main()
