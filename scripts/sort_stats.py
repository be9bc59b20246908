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
    print(dict(units=int(c[1]), visited_per_q=c[2] / nq, expanded_per_q=c[3] / nq,
               S_per_q=c[4] / nq, Sp_per_q=c[5] / nq, chunks_per_q=c[6] / nq,
               S_entry=c[7] / nq, S_iter0=c[8] / nq, S_later=c[9] / nq, M_per_q=c[10] / nq))
