#!/usr/bin/env python
"""BASELINE configs[4]: batch-size x beam-width sweep on the 100M x 96 config
(the cfg3 index, GPU-built once): QPS / recall@10 / visited per setting at
batches 1k..1M and beams 32..256 (iterations per beam from the calibration),
one JSON line each (device-resident queries, CUDA events, K1 only)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2512_02278_b200 as dvs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--beams", default="16:24,32:14,64:10,128:8,256:6")
    ap.add_argument("--batches", default="1000,10000,100000,1000000")
    ap.add_argument("--accum", default="f32")
    a = ap.parse_args()
    args = bench.parse(["--nq", "1000000", "--recall-sample", "2000"])
    dev = torch.device("cuda", 0)
    ctx = dvs.Context(0)
    w = bench.build_cfg3(args, 0, ctx, dev)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    nq = args.nq
    b = bench.Bufs(torch, nq, 10, args.dim, dev, vectors=False)
    uq = torch.arange(nq, dtype=torch.int32, device=dev)
    up = torch.zeros(nq, dtype=torch.int32, device=dev)
    for spec in a.beams.split(","):
        beam, iters = (int(v) for v in spec.split(":"))
        p = dvs.SearchParams(iters, beam, 10, beam, accum=a.accum)
        for bs in (int(v) for v in a.batches.split(",")):
            def run():
                ctx.search_units_device(w.queries.data_ptr(), bs, args.dim, uq.data_ptr(), up.data_ptr(), bs, p,
                                        b.ids.data_ptr(), b.dists.data_ptr(), b.counts.data_ptr(), b.vis.data_ptr())
            torch.cuda.synchronize()
            run()
            ctx.synchronize()
            reps = max(1, min(20, 200000 // bs))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                run()
            e1.record(stream)
            ctx.synchronize()
            ms = e0.elapsed_time(e1) / reps
            s = min(bs, w.gt.shape[0])
            ids = b.ids[:s].cpu().numpy().view(np.uint32)
            cnt = b.counts[:s].cpu().numpy()
            rec = bench.recall_at_k(ids, cnt, w.gt[:s], 10)
            vis = float(b.vis[:bs].double().mean())
            line = {"n": args.n, "dim": args.dim, "batch": bs, "beam": beam, "iterations": iters,
                    "qps": bs / (ms / 1e3), "ms_per_batch": ms, "recall_at_10": round(rec, 4),
                    "recall_sample": s, "visited_per_query": vis,
                    "alg_gbs": (vis * 4 * args.dim + iters * beam * 128 + 4 * args.dim) * bs / (ms / 1e3) / 1e9}
            print(json.dumps(line), flush=True)
            print(f"[cfg5] bs={bs} w={beam} I={iters}: {line['qps']:,.0f} QPS recall {rec:.4f}", file=sys.stderr,
                  flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
