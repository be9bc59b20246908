"""Debug (-DDVSG_SHARD_PROFILE build): where an origin CTA's cycles go in the
emulated sharded search: idle waiting, serving while waiting, whole unit."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2512_02278_b200 as dvs  # noqa: E402
from paper_2512_02278_b200._lib import lib  # noqa: E402

sys.argv = ["x", "--nq", "50000"]
args = bench.parse()
ctx = dvs.Context(0)
data, queries, index = bench.workload(args, 0, ctx)
ctx.load_index(index)
ctx.set_timing(True)
p = dvs.SearchParams(args.iterations, args.beam, args.k, args.entry, accum=args.accum)
for R in [1, 2, 4]:
    ctx.beam_search_sharded_emulated(R, queries, p)
    c = np.zeros(16, np.uint64)
    lib.dvsg_debug_counters(ctx.handle, ctypes.c_void_p(c.ctypes.data))
    units = max(int(c[1]), 1)
    print(f"R={R} K1 ms {ctx.last_timings()['search_ms']:.1f}  per unit (kcycles): total {c[7]/units/1e3:.1f}"
          f" idle-wait {c[4]/units/1e3:.1f} serve-in-wait {c[5]/units/1e3:.1f} waits/unit {c[6]/units:.2f}", flush=True)
