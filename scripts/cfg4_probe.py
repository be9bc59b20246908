#!/usr/bin/env python
"""BASELINE configs[3] calibration: text-embedding-like 10M x 768 (float,
L2-normalised), inner product, top-100, beam 256; GPU-built graph; sweep of
the iteration count.  One JSON line per setting."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_02278_b200 as dvs  # noqa: E402
from paper_2512_02278_b200 import ivf  # noqa: E402


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--dim", type=int, default=768)
    ap.add_argument("--nq", type=int, default=100_000)
    ap.add_argument("--gt", type=int, default=1000)
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--probe", type=int, default=8)
    ap.add_argument("--keep", type=int, default=12)
    ap.add_argument("--rank", type=int, default=32)
    ap.add_argument("--sweep", default="4x256,6x256,8x256")
    ap.add_argument("--accums", default="f32c,f64")
    args = ap.parse_args()
    dev = "cuda:0"
    ctx = dvs.Context(0)
    t0 = time.time()
    x = ivf.embedding_like_device(args.n, args.dim, rank=args.rank, seed=3, device=dev)
    info = ivf.build_graph_ivf(ctx, x, degree=32, probe=args.probe, dim=args.dim, optimize=True,
                               keep=args.keep, log=log)
    del x
    torch.cuda.empty_cache()
    pv, _, _, _, n = ctx.partition_view_device(0)
    vec = ivf.device_view(pv, (n, args.dim), torch.float32, dev)
    q = ivf.embedding_like_device(args.nq, args.dim, rank=args.rank, seed=4, basis_seed=3, device=dev)
    t1 = time.time()
    gt = ivf.topk_ip_device(vec, q[:args.gt], args.k).cpu().numpy()
    log(f"[cfg4] setup {t1 - t0:.1f}s, ground truth {time.time() - t1:.1f}s")
    nq, k = args.nq, args.k
    ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
    dists = torch.empty((nq, k), dtype=torch.float32, device=dev)
    cnt = torch.empty((nq,), dtype=torch.int32, device=dev)
    vis = torch.empty((nq,), dtype=torch.int64, device=dev)
    uq = torch.arange(nq, dtype=torch.int32, device=dev)
    up = torch.zeros(nq, dtype=torch.int32, device=dev)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    base_ids = None
    for acc in args.accums.split(","):
        for s in args.sweep.split(","):
            it, w = (int(v) for v in s.split("x"))
            p = dvs.SearchParams(it, w, k, w, metric="ip", accum=acc)
            torch.cuda.synchronize()

            def run():
                ctx.search_units_device(q.data_ptr(), nq, args.dim, uq.data_ptr(), up.data_ptr(), nq, p,
                                        ids.data_ptr(), dists.data_ptr(), cnt.data_ptr(), vis.data_ptr())
            run()
            ctx.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run()
            e1.record(stream)
            ctx.synchronize()
            ms = e0.elapsed_time(e1)
            got = ids.cpu().numpy().view(np.uint32).astype(np.int64)
            c = cnt.cpu().numpy()
            r100 = np.mean([len(set(got[i, :c[i]].tolist()) & set(gt[i].tolist())) / k for i in range(args.gt)])
            r10 = np.mean([len(set(got[i, :min(10, c[i])].tolist()) & set(gt[i, :10].tolist())) / 10
                           for i in range(args.gt)])
            v = float(vis.double().mean())
            line = {"n": n, "dim": args.dim, "metric": "ip", "k": k, "iters": it, "beam": w, "accum": acc,
                    "recall@10": round(float(r10), 4), "recall@100": round(float(r100), 4),
                    "qps": nq / (ms / 1e3), "ms": ms, "visited": v,
                    "alg_gbs": (v * 4 * args.dim + it * w * 128 + 4 * args.dim) * nq / (ms / 1e3) / 1e9,
                    "build": {kk: vv for kk, vv in info.items() if kk != "perm"}}
            key = (it, w)
            if acc == "f32c":
                base_ids = base_ids or {}
                base_ids[key] = got.copy()
            elif base_ids and key in base_ids:
                line["ids_identical_to_f32c_frac"] = float(np.mean(np.all(base_ids[key] == got, axis=1)))
            print(json.dumps(line), flush=True)
            log(f"[cfg4] {acc} I={it} w={w}: recall@10 {r10:.4f} @100 {r100:.4f}, {nq / (ms / 1e3):,.0f} QPS, "
                f"visited {v:.0f}, alg {line['alg_gbs']:.0f} GB/s")
    ctx.close()


if __name__ == "__main__":
    main()
