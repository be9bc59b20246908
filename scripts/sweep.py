"""BASELINE configs[4]-style sweep on the 1M x 128 workload: batch size x beam
width -> QPS (device-resident run_pipeline, CUDA events, L2 flushed) and
recall@10 (exact brute force on the first 1000 queries).  One JSON line per
point.

    python scripts/sweep.py [--out profiles/r01_sweep.jsonl]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--batches", default="1000,10000,100000")
    ap.add_argument("--beams", default="32,64,128,256")
    ap.add_argument("--iterations", type=int, default=6)
    a = ap.parse_args()
    import torch
    import paper_2512_02278_b200 as dvs
    from paper_2512_02278_b200 import synth

    sys.argv = ["x", "--nq", str(max(int(b) for b in a.batches.split(",")))]
    args = bench.parse()
    ctx = dvs.Context(0)
    data, queries, index = bench.workload(args, 0, ctx)
    ctx.load_index(index)
    truth = synth.brute_force_gt(data, queries[:1000], 10)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    out = open(a.out, "w") if a.out else None
    for w in [int(x) for x in a.beams.split(",")]:
        p = dvs.SearchParams(a.iterations, w, 10, w, accum="f32")
        for bs in [int(x) for x in a.batches.split(",")]:
            q = torch.from_numpy(queries[:bs]).to(dev)
            ids = torch.empty((bs, 10), dtype=torch.int32, device=dev)
            dists = torch.empty((bs, 10), dtype=torch.float32, device=dev)
            cnt = torch.empty((bs,), dtype=torch.int32, device=dev)
            vecs = torch.empty((bs, 10, 128), dtype=torch.float32, device=dev)

            def step():
                ctx.run_pipeline_device(q.data_ptr(), bs, 128, p, 1, ids.data_ptr(), dists.data_ptr(),
                                        cnt.data_ptr(), vecs.data_ptr())

            for _ in range(3):
                step()
            ctx.synchronize()
            reps = 5 if bs <= 10000 else 3
            tot = 0.0
            for _ in range(reps):
                flush.fill_(1.0)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                step()
                e1.record(stream)
                stream.synchronize()
                tot += e0.elapsed_time(e1)
            st = ctx.last_search_stats()
            m = min(bs, 1000)
            rec = synth.recall_at_k(ids.cpu().numpy().view(np.uint32)[:m],
                                    cnt.cpu().numpy().view(np.uint32)[:m], truth[:m], 10)
            line = {"beam": w, "iterations": a.iterations, "batch": bs, "qps": bs * reps / (tot / 1e3),
                    "ms_per_batch": tot / reps, "recall_at_10": round(rec, 4),
                    "visited_per_query": st["visited"] / max(st["units"], 1)}
            print(json.dumps(line), flush=True)
            if out:
                out.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
