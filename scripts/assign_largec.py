"""K5 assign_top_c time at large C (SURVEY 8f-3 sizing): the tensor-core path
(TF32 candidates + exact fp64 re-rank + certificate, c <= 24) against the
exact fp64 tile path (forced by c' = 25 > 24; its first c columns are the
reference's top-c, checked equal).  Device-resident queries, CUDA events."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2512_02278_b200 as dvs
    ctx = dvs.Context(0)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    g = torch.Generator(device=dev).manual_seed(1)
    cfgs = [(256, 96, 1_000_000, 8), (1024, 128, 100_000, 8), (4096, 128, 100_000, 8),
            (4096, 96, 1_000_000, 8), (4096, 96, 1_000_000, 1), (16384, 64, 1_000_000, 4)]
    if len(sys.argv) > 1:  # --only C,d,nq,c
        cfgs = [tuple(int(v) for v in sys.argv[2].split(","))]
    for C, d, nq, c in cfgs:
        cents = torch.randn(C, d, device=dev, generator=g).cpu().numpy()
        q = torch.randn(nq, d, device=dev, generator=g)
        ctx.reset()
        ctx.set_centroids(cents, None, 1)
        res = {}
        for tag, cc in (("tc", c), ("fp64_tiles", 25)):
            out = torch.empty((nq, cc), dtype=torch.int32, device=dev)
            ctx.assign_top_c_device(q.data_ptr(), nq, d, cc, out.data_ptr())
            ctx.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 3
            e0.record(stream)
            for _ in range(reps):
                ctx.assign_top_c_device(q.data_ptr(), nq, d, cc, out.data_ptr())
            e1.record(stream)
            ctx.synchronize()
            path, fb = ctx.last_assign_info()
            res[tag] = (e0.elapsed_time(e1) / reps, path, fb, out[:, :c].clone())
        same = bool(torch.equal(res["tc"][3], res["fp64_tiles"][3]))
        print(json.dumps({"clusters": C, "dim": d, "queries": nq, "c": c,
                          "tc_ms": round(res["tc"][0], 3), "tc_path": res["tc"][1], "tc_fallbacks": res["tc"][2],
                          "tiles_ms": round(res["fp64_tiles"][0], 3), "tiles_path": res["fp64_tiles"][1],
                          "speedup": round(res["fp64_tiles"][0] / res["tc"][0], 2),
                          "ids_identical": same,
                          "tc_tf32_tflops": round(2.0 * nq * C * d / (res["tc"][0] / 1e3) / 1e12, 2)}), flush=True)


if __name__ == "__main__":
    main()
