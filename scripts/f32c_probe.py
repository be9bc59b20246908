"""One cfg4-like K1 launch per accumulation mode (200k x 768 inner product,
k=100, beam 256, 20k queries), for ncu captures of the compensated f32 kernel:

    python scripts/f32c_probe.py --accum f32c [--reps 2]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from scripts.config_shapes import normalised  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--accum", default="f32c")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--nq", type=int, default=20_000)
    ap.add_argument("--metric", default="ip")
    ap.add_argument("--dim", type=int, default=768)
    ap.add_argument("--time", action="store_true")
    a = ap.parse_args()
    import paper_2512_02278_b200 as dvs
    ctx = dvs.Context(0)
    data = normalised(200_000, a.dim, 32, 1)
    queries = normalised(a.nq, a.dim, 32, 2)
    adj = ctx.build_graph(data, 32)
    ctx.load_partition(0, dvs.GraphIndex(data, np.arange(len(data), dtype=np.uint32), 32, adj,
                                         dvs.compute_entry_order(data)))
    p = dvs.SearchParams(6, 256, 100, 256, metric=a.metric, accum=a.accum)
    import time
    for r in range(a.reps):
        t0 = time.perf_counter()
        ids, dists, counts, visited = ctx.beam_search(0, queries, p)
        dt = time.perf_counter() - t0
    print("ok", a.accum, a.metric, a.dim, float(visited.mean()), "qps(host-timed, last rep)=%.0f" % (a.nq / dt) if a.time else "")


if __name__ == "__main__":
    main()
