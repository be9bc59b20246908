"""K1 on fp32 rows vs the byte copy (dvsg_set_vector_storage U8) on the bench
workload (default cfg3), device-resident queries, CUDA events, L2 flushed."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2512_02278_b200 as dvs  # noqa: E402
import torch  # noqa: E402


def main():
    args = bench.parse(sys.argv[1:])
    ctx = dvs.Context(0)
    dev = torch.device("cuda", 0)
    w = bench.build_workload(args, 0, ctx, dev)
    nq = args.nq
    b = bench.Bufs(torch, nq, args.k, args.dim, dev, vectors=False)
    uq = torch.arange(nq, dtype=torch.int32, device=dev)
    up = torch.zeros(nq, dtype=torch.int32, device=dev)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    p = dvs.SearchParams(args.iterations, args.beam, args.k, args.entry, metric=args.metric, accum=args.accum)
    res = {}
    for mode in ("f32", "u8", "f32"):
        ctx.set_vector_storage(mode)

        def run():
            ctx.search_units_device(w.queries.data_ptr(), nq, args.dim, uq.data_ptr(), up.data_ptr(), nq, p,
                                    b.ids.data_ptr(), b.dists.data_ptr(), b.counts.data_ptr(), b.vis.data_ptr())
        run()
        ctx.synchronize()
        ms = []
        for i in range(3):
            flush.fill_(float(i))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run()
            e1.record(stream)
            ctx.synchronize()
            ms.append(e0.elapsed_time(e1))
        ids = b.ids.cpu().numpy().copy()
        res.setdefault(mode, []).append((min(ms), ids))
    same = np.array_equal(res["f32"][0][1], res["u8"][0][1])
    print(json.dumps({"nq": nq, "f32_ms": res["f32"][0][0], "u8_ms": res["u8"][0][0], "f32_again_ms": res["f32"][1][0],
                      "speedup": res["f32"][0][0] / res["u8"][0][0], "ids_identical": bool(same),
                      "lib": os.environ.get("DVSG_LIB", "default")}), flush=True)


if __name__ == "__main__":
    main()
