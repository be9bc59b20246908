"""Independent pure-numpy FNSY v1 reader for the tests (index_file.cpp:16-25,
:149-296 layout: magic, u32 version, five length-prefixed LE sections)."""
import os
import struct
from types import SimpleNamespace

import numpy as np

G3_FNSY = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "g3_mixture.fnsy")


def read_fnsy(path):
    raw = open(path, "rb").read()
    assert raw[:4] == b"FNSY" and struct.unpack_from("<I", raw, 4)[0] == 1
    off, secs = 8, {}
    while off < len(raw):
        sid, ln = struct.unpack_from("<IQ", raw, off)
        secs[sid] = memoryview(raw)[off + 12: off + 12 + ln]
        off += 12 + ln
    u32 = lambda mv, o, n=1: np.frombuffer(mv, "<u4", n, o)  # noqa: E731
    c = secs[1]
    C, d = u32(c, 0, 2)
    cents = np.frombuffer(c, "<f4", C * d, 8).reshape(C, d)
    p = secs[2]
    ranks = int(u32(p, 4)[0])
    ctr = u32(p, 8, C).copy()
    g, a, v = secs[3], secs[4], secs[5]
    dg = int(u32(a, 4)[0])
    go, ao, vo = 4, 8, 8
    graphs = []
    for _ in range(C):
        n = int(u32(g, go)[0]); go += 4
        gids = u32(g, go, n).copy(); go += 4 * n
        ao += 4
        adj = u32(a, ao, n * dg).reshape(n, dg).copy(); ao += 4 * n * dg
        vo += 4
        vec = np.frombuffer(v, "<f4", n * d, vo).reshape(n, d).copy(); vo += 4 * n * d
        graphs.append(SimpleNamespace(vectors=vec, global_ids=gids, adjacency=adj,
                                      out_degree=dg, entry_order=None))
    return SimpleNamespace(centroids=cents.copy(), cluster_to_rank=ctr, ranks=ranks,
                           out_degree=dg, graphs=graphs)
