"""Debug: survivor-count distribution of K1 (needs a -DDVSG_SORT_STATS build)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2512_02278_b200 as dvs  # noqa: E402
from paper_2512_02278_b200._lib import lib  # noqa: E402

sys.argv = ["x", "--nq", "20000"]
args = bench.parse()
ctx = dvs.Context(0)
data, queries, index = bench.workload(args, 0, ctx)
ctx.load_index(index)
for I, w in [(6, 64)]:
    p = dvs.SearchParams(I, w, 10, w, accum="f32")
    r = ctx.run_pipeline(queries, p, 1, 1, 0, False)
    c = np.zeros(16, np.uint64)
    lib.dvsg_debug_counters(ctx.handle, ctypes.c_void_p(c.ctypes.data))
    nq = queries.shape[0]
    print(dict(units=int(c[1]), visited_per_q=round(c[2] / nq, 1), expanded_per_q=round(c[3] / nq, 1),
               survivors_sorted_per_q=round(c[4] / nq, 1), new_local_per_q=round(c[5] / nq, 1),
               chunks_per_q=round(c[6] / nq, 2), S_entry=round(c[7] / nq, 1),
               S_first_expansion=round(c[8] / nq, 1), S_later_total=round(c[9] / nq, 1)))
