"""Debug (-DDVSG_SHARD_PROFILE build, torchrun): per-unit cycle breakdown of the
node-sharded kernel on real GPUs (origin CTA view)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    import torch
    import torch.distributed as dist
    import paper_2512_02278_b200 as dvs
    from paper_2512_02278_b200._lib import lib
    from paper_2512_02278_b200.dist import prepare_step, setup_sharded
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    os.environ["NCCL_DEBUG"] = "WARN"
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sys.argv = ["x", "--nq", "50000"]
    args = bench.parse()
    ctx = dvs.Context(local)
    data, queries, index = bench.workload(args, rank, ctx)
    g0 = index.graphs[0]
    setup_sharded(ctx, rank, world, data, g0.adjacency, g0.entry_order, g0.global_ids)
    ctx.set_timing(True)
    p = dvs.SearchParams(6, 64, 10, 64, accum="f32")
    dev = torch.device("cuda", local)
    nq = args.nq
    d_q = torch.from_numpy(queries).to(dev)
    ids = torch.empty((nq, 10), dtype=torch.int32, device=dev)
    dd = torch.empty((nq, 10), dtype=torch.float32, device=dev)
    cc = torch.empty((nq,), dtype=torch.int32, device=dev)
    vv = torch.empty((nq,), dtype=torch.int64, device=dev)
    for _ in range(3):
        prepare_step(ctx, dist.barrier)
        ctx.search_sharded_device(d_q.data_ptr(), nq, 128, p, ids.data_ptr(), dd.data_ptr(), cc.data_ptr(), vv.data_ptr())
        ctx.synchronize()
    c = np.zeros(16, np.uint64)
    lib.dvsg_debug_counters(ctx.handle, ctypes.c_void_p(c.ctypes.data))
    units = max(int(c[1]), 1)
    print(f"rank {rank}: K1 ms {ctx.last_timings()['search_ms']:.1f} per unit kcycles: total {c[7]/units/1e3:.1f} "
          f"idle-wait {c[4]/units/1e3:.1f} serve-in-wait {c[5]/units/1e3:.1f} waits/unit {c[6]/units:.2f}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
