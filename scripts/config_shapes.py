"""K1 at the shapes of BASELINE configs 3 and 4, scaled to one GPU's setup
budget (the exact kNN build of the full 100M / 10M sets is out of reach, see
DESIGN.md): QPS (f32 mode, device-resident queries, CUDA events), recall@k
against exact brute force, and id agreement with the f64 parity mode.

    python scripts/config_shapes.py [--out profiles/r01_config_shapes.jsonl]

cfg3-like: 96-d SIFT-like (rank 16), L2, k=10, beam 64.
cfg4-like: 768-d text-embedding-like (rank 32, L2-normalised rows), inner
product, k=100, beam 256 (cap 3,072; pool kept at I*w = 1,536).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def normalised(n, dim, rank, seed):
    rng = np.random.default_rng(seed)
    a = rng.normal(0.0, 1.0 / np.sqrt(rank), size=(rank, dim)).astype(np.float32)
    z = rng.standard_normal(size=(n, rank), dtype=np.float32)
    x = z @ a + 0.1 * rng.standard_normal(size=(n, dim), dtype=np.float32)
    return (x / np.linalg.norm(x, axis=1, keepdims=True)).astype(np.float32)


def exact_topk(data, queries, k, metric, dev):
    import torch
    x = torch.from_numpy(data).to(dev)
    out = []
    for b in range(0, queries.shape[0], 512):
        q = torch.from_numpy(queries[b:b + 512]).to(dev)
        if metric == "ip":
            d = -(q.double() @ x.double().T)
        else:
            d = (q.double() ** 2).sum(1, keepdim=True) + (x.double() ** 2).sum(1)[None, :] - 2.0 * (q.double() @ x.double().T)
        out.append(torch.topk(d, k, dim=1, largest=False).indices.cpu().numpy())
    return np.concatenate(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--nq", type=int, default=20_000)
    a = ap.parse_args()
    import torch
    import paper_2512_02278_b200 as dvs
    from paper_2512_02278_b200 import synth
    dev = torch.device("cuda", 0)
    ctx = dvs.Context(0)
    shapes = [
        dict(name="cfg3-like 96-d L2", n=2_000_000, dim=96, metric="l2", k=10, beam=64,
             data=lambda n, d: synth.sift_like(n, d, 16, seed=1),
             queries=lambda nq, d: synth.sift_like_queries(nq, d, 16, data_seed=1, seed=2)),
        dict(name="cfg4-like 768-d inner product", n=200_000, dim=768, metric="ip", k=100, beam=256,
             data=lambda n, d: normalised(n, d, 32, 1), queries=lambda nq, d: normalised(nq, d, 32, 2)),
    ]
    out = open(a.out, "w") if a.out else None
    for sh in shapes:
        t0 = time.time()
        data = sh["data"](sh["n"], sh["dim"])
        queries = sh["queries"](a.nq, sh["dim"])
        adj = ctx.build_graph(data, 32)
        g = dvs.GraphIndex(data, np.arange(sh["n"], dtype=np.uint32), 32, adj, dvs.compute_entry_order(data))
        ctx.reset()
        ctx.load_partition(0, g)
        build_s = time.time() - t0
        p = dvs.SearchParams(6, sh["beam"], sh["k"], sh["beam"], metric=sh["metric"], accum="f32")
        d_q = torch.from_numpy(queries).to(dev)
        nq, k = a.nq, sh["k"]
        ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
        dists = torch.empty((nq, k), dtype=torch.float32, device=dev)
        cnt = torch.empty((nq,), dtype=torch.int32, device=dev)
        vis = torch.empty((nq,), dtype=torch.int64, device=dev)
        uq = torch.arange(nq, dtype=torch.int32, device=dev)
        uc = torch.zeros(nq, dtype=torch.int32, device=dev)
        stream = torch.cuda.ExternalStream(ctx.stream, device=dev)

        def run():
            ctx.search_units_device(d_q.data_ptr(), nq, sh["dim"], uq.data_ptr(), uc.data_ptr(), nq, p,
                                    ids.data_ptr(), dists.data_ptr(), cnt.data_ptr(), vis.data_ptr())

        def timed():
            for _ in range(3):
                run()
            ctx.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(3):
                run()
            e1.record(stream)
            stream.synchronize()
            return e0.elapsed_time(e1) / 3

        p_fast = p
        p = dvs.SearchParams(6, sh["beam"], sh["k"], sh["beam"], metric=sh["metric"], accum="f64")
        ms64 = timed()
        p = p_fast
        ms = timed()
        got = ids.cpu().numpy().view(np.uint32)
        counts = cnt.cpu().numpy().view(np.uint32)
        m = 1000
        truth = exact_topk(data, queries[:m], k, sh["metric"], dev)
        rec = synth.recall_at_k(got[:m], counts[:m], truth, k)
        # the f64 parity mode on the same sample: how often the fast mode's ids differ
        p64 = dvs.SearchParams(6, sh["beam"], k, sh["beam"], metric=sh["metric"], accum="f64")
        r64 = ctx.beam_search(0, queries[:m], p64)
        agree = float(np.mean([np.array_equal(got[i, :counts[i]], r64[0][i, :r64[2][i]]) for i in range(m)]))
        st = vis.cpu().numpy().mean()
        # compensated f32 (accum "f32c"): speed and id agreement with f64
        p = dvs.SearchParams(6, sh["beam"], sh["k"], sh["beam"], metric=sh["metric"], accum="f32c")
        ms32c = timed()
        got_c = ids.cpu().numpy().view(np.uint32)
        counts_c = cnt.cpu().numpy().view(np.uint32)
        agree_c = float(np.mean([np.array_equal(got_c[i, :counts_c[i]], r64[0][i, :r64[2][i]]) for i in range(m)]))
        d64 = r64[1]
        dc = dists.cpu().numpy()
        rel = max(float(np.max(np.abs(dc[i, :counts_c[i]] - d64[i, :r64[2][i]]) /
                               np.maximum(np.abs(d64[i, :r64[2][i]]), 1e-30)))
                  for i in range(m) if counts_c[i] > 0 and np.array_equal(got_c[i, :counts_c[i]], r64[0][i, :r64[2][i]]))
        line = {"shape": sh["name"], "n": sh["n"], "dim": sh["dim"], "metric": sh["metric"], "k": k,
                "beam": sh["beam"], "iterations": 6, "queries": nq, "qps": nq / (ms / 1e3), "ms_per_batch": ms,
                "recall_at_k": round(rec, 4), "visited_per_query": float(st),
                "f32_ids_identical_to_f64_mode": agree, "qps_f64_parity_mode": nq / (ms64 / 1e3),
                "qps_f32c_mode": nq / (ms32c / 1e3), "f32c_ids_identical_to_f64_mode": agree_c,
                "f32c_max_rel_dist_diff_vs_f64": rel,
                "setup_s": round(build_s, 1)}
        print(json.dumps(line), flush=True)
        if out:
            out.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
