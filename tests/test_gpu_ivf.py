"""GPU tests of the large-index construction path (csrc/ivf_build.cu, ivf.py):
K7 range top-m against numpy, the device compute_entry_order against the
reference's (host restatement pinned in test_oracle.py), the in-place
partition alloc/commit path against the host upload path, the
cluster-restricted graph against the exact build_graph when the probe list
covers every cluster, and the f32-mode upgrade on non-integer data."""
import os

import numpy as np
import pytest

import paper_2512_02278_b200 as dvs
from conftest import sift_like

pytestmark = pytest.mark.gpu
os.environ["DVSG_IVF_CHECK"] = "1"  # host-side bounds checks of every K7 launch

torch = pytest.importorskip("torch")


def _t(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t if dtype is None else t.to(dtype)


def _np_topm(rows, cols, m, exclude_self=False, row_ids=None):
    """(dist, id) top-m with the reference's ordering (exact: integer data)."""
    d = ((rows.astype(np.float64)[:, None, :] - cols.astype(np.float64)[None, :, :]) ** 2).sum(-1)
    out = []
    for i in range(rows.shape[0]):
        key = [(float(np.float32(d[i, j])), j) for j in range(cols.shape[0])
               if not (exclude_self and j == (row_ids[i] if row_ids is not None else i))]
        key.sort()
        out.append([j for _, j in key[:m]])
    return out


@pytest.mark.parametrize("m", [1, 7, 32])
def test_range_topk_matches_numpy(ctx, m):
    from paper_2512_02278_b200 import ivf
    rng = np.random.default_rng(5)
    x = rng.integers(0, 256, size=(700, 40)).astype(np.float32)  # ties on purpose (integers)
    x[:, 36:] = 0
    x[::7, :] = x[3, :]  # exact duplicate rows: (dist, id) tie-break
    xt = _t(x)
    xn = ivf.row_norms(ctx, xt)
    # segments of ragged size, each row against two disjoint column ranges
    off = torch.tensor([0, 5, 200, 333, 700], dtype=torch.int64, device="cuda")
    blocks, _ = ivf.segment_blocks(off)
    ranges = _t(np.array([[0, 150], [400, 700], [10, 20], [30, 699], [0, 700], [700, 700],
                          [100, 400], [500, 600]], np.int32))
    lo = _t(np.array([0, 2, 4, 6, 8], np.int32))
    dists = torch.empty((700, m), dtype=torch.float32, device="cuda")
    ids = ivf.range_topk(ctx, xt, xn, xt, xn, blocks, lo, ranges, m, flags=dvs._lib.RANGE_EXCLUDE_SELF,
                         out_dists=dists).cpu().numpy().view(np.uint32)
    seg_ranges = [[(0, 150), (400, 700)], [(10, 20), (30, 699)], [(0, 700)], [(100, 400), (500, 600)]]
    offs = [0, 5, 200, 333, 700]
    for s in range(4):
        cols = np.concatenate([np.arange(a, b) for a, b in seg_ranges[s]])
        want = _np_topm(x[offs[s]:offs[s + 1]], x[cols], m, True,
                        row_ids=[np.searchsorted(cols, r) if r in set(cols.tolist()) else -1
                                 for r in range(offs[s], offs[s + 1])])
        for i, r in enumerate(range(offs[s], offs[s + 1])):
            w = [int(cols[j]) for j in want[i]]
            assert ids[r, :len(w)].tolist() == w, (s, r)
            if len(w) < m:
                assert (ids[r, len(w):] == 0xFFFFFFFF).all()
            d = ((x[r].astype(np.float64) - x[w].astype(np.float64)) ** 2).sum(1).astype(np.float32)
            assert np.array_equal(dists.cpu().numpy()[r, :len(w)], d)


def test_range_topk_row_map_and_build_pad(ctx):
    from paper_2512_02278_b200 import ivf
    rng = np.random.default_rng(6)
    x = rng.integers(0, 256, size=(300, 16)).astype(np.float32)
    xt = _t(x)
    xn = ivf.row_norms(ctx, xt)
    perm = rng.permutation(300).astype(np.int32)
    off = torch.tensor([0, 300], dtype=torch.int64, device="cuda")
    blocks, _ = ivf.segment_blocks(off)
    lo, rg = ivf._single_list(300, "cuda")
    got = ivf.range_topk(ctx, xt, xn, xt, xn, blocks, lo, rg, 5, flags=dvs._lib.RANGE_EXCLUDE_SELF,
                         row_map=_t(perm)).cpu().numpy().view(np.uint32)
    want = _np_topm(x[perm], x, 5, True, row_ids=perm)
    assert got.tolist() == want
    # build padding: 3-row candidate sets, degree 5 -> cyclic repeat of the 2 others
    lo2 = _t(np.arange(101, dtype=np.int32))
    rg2 = _t(np.stack([np.arange(0, 300, 3), np.arange(3, 303, 3)], 1).astype(np.int32))
    off2 = torch.arange(0, 301, 3, dtype=torch.int64, device="cuda")
    blocks2, _ = ivf.segment_blocks(off2)
    pad = ivf.range_topk(ctx, xt, xn, xt, xn, blocks2, lo2, rg2, 5,
                         flags=dvs._lib.RANGE_EXCLUDE_SELF | dvs._lib.RANGE_BUILD_PAD).cpu().numpy()
    for c in range(100):
        rows = range(3 * c, 3 * c + 3)
        for r in rows:
            others = _np_topm(x[r:r + 1], x[3 * c:3 * c + 3], 3)[0]
            others = [3 * c + j for j in others if 3 * c + j != r]
            assert pad[r].tolist() == [others[j % 2] for j in range(5)]


@pytest.mark.parametrize("kind", ["float", "integer"])
def test_entry_order_device_matches_reference(ctx, oracle, kind):
    rng = np.random.default_rng(7)
    if kind == "float":
        x = rng.normal(size=(5000, 37)).astype(np.float32) * np.float32(3.3)
    else:
        x = sift_like(5000, 96, 16, 3)
    dpad = (x.shape[1] + 3) // 4 * 4
    xp = np.zeros((x.shape[0], dpad), np.float32)
    xp[:, :x.shape[1]] = x
    xt = _t(xp)
    out = torch.empty(x.shape[0], dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    ctx.compute_entry_order_device(xt.data_ptr(), x.shape[0], x.shape[1], dpad, out.data_ptr())
    got = out.cpu().numpy().view(np.uint32)
    assert np.array_equal(got, dvs.compute_entry_order(x))
    assert np.array_equal(got, oracle.compute_entry_order(x))


def _alloc_commit(ctx, x, adj, flags):
    from paper_2512_02278_b200 import ivf
    n, dim = x.shape
    dpad = (dim + 3) // 4 * 4
    pv, pa, pg, pe = ctx.partition_alloc_device(0, n, dim, adj.shape[1])
    v = ivf.device_view(pv, (n, dpad), torch.float32, "cuda")
    v[:, :dim] = _t(x)
    ivf.device_view(pa, adj.shape, torch.int32, "cuda")[:] = _t(adj.view(np.int32))
    torch.cuda.synchronize()
    ctx.partition_commit_device(flags)


def test_partition_commit_equals_host_upload(ctx, oracle):
    x = sift_like(3000, 30, 8, 4)
    adj = oracle.build_graph(x, 16)
    q = sift_like(64, 30, 8, 5)
    p = dvs.SearchParams(6, 32, 10, 32)
    ctx.reset()
    _alloc_commit(ctx, x, adj, dvs._lib.COMMIT_ENTRY_ORDER | dvs._lib.COMMIT_IOTA_IDS)
    assert ctx.index_integral()
    got = ctx.beam_search(0, q, p)
    assert np.array_equal(ctx.entry_order(0), dvs.compute_entry_order(x))
    ctx.reset()
    ctx.load_partition(0, dvs.GraphIndex(x, np.arange(3000, dtype=np.uint32), 16, adj, None))
    want = ctx.beam_search(0, q, p)
    for a, b in zip(got, want):
        assert np.array_equal(a, b)


def test_partition_commit_validates(ctx):
    x = sift_like(100, 8, 4, 4)
    adj = np.zeros((100, 4), np.uint32)
    adj[5, 2] = 100
    ctx.reset()
    with pytest.raises(dvs.FormatError):
        _alloc_commit(ctx, x, adj, dvs._lib.COMMIT_IOTA_IDS)
    ctx.reset()
    xb = x.copy()
    xb[3, 1] = np.nan
    with pytest.raises(dvs.InvalidArgument):
        _alloc_commit(ctx, xb, np.zeros((100, 4), np.uint32), dvs._lib.COMMIT_IOTA_IDS)
    ctx.reset()
    with pytest.raises(dvs.InvalidArgument):
        ctx.partition_commit_device(0)  # nothing allocated
    ctx.reset()


def test_ivf_graph_full_probe_equals_exact_build(ctx, oracle):
    """probe = every cluster: the candidate set is the whole partition, so the
    cluster-restricted graph must be build_graph's exact kNN (in stored order)."""
    from paper_2512_02278_b200 import ivf
    n, dim = 6000, 24
    xt = ivf.sift_like_device(n, dim, rank=8, seed=9, device="cuda")
    xh = xt.cpu().numpy()
    ctx.reset()
    info = ivf.build_graph_ivf(ctx, xt, degree=16, cluster_size=400, probe=1 << 20, n_coarse=4,
                               sample=n, iters=3)
    assert info["probe"] == info["fine_clusters"]  # every cluster probed
    perm = info["perm"].cpu().numpy()
    x = xh[perm]
    adj = ctx_adjacency(ctx, n, 16)
    want = oracle.build_graph(x, 16)
    assert np.array_equal(adj, want)
    assert np.array_equal(ctx.entry_order(0), dvs.compute_entry_order(x))
    ctx.reset()


def ctx_adjacency(ctx, n, dg):
    from paper_2512_02278_b200 import ivf
    pv, pa, pg, pe, rows = ctx.partition_view_device(0)
    assert rows == n
    return ivf.device_view(pa, (n, dg), torch.int32, "cuda").cpu().numpy().view(np.uint32)


def test_ivf_brute_force_matches_library(ctx):
    from paper_2512_02278_b200 import ivf
    x = sift_like(20000, 48, 12, 11)
    q = sift_like(300, 48, 12, 12)
    xt, qt = _t(x), _t(q)
    ids, d = ivf.brute_force_topk(ctx, xt, ivf.row_norms(ctx, xt), qt, 10, splits=7)
    wi, wd = ctx.brute_force_topk(x, q, 10)
    assert np.array_equal(ids.cpu().numpy().astype(np.uint32), wi)
    assert np.array_equal(d.cpu().numpy(), wd)


def test_f32_mode_upgraded_on_float_data(ctx, oracle):
    rng = np.random.default_rng(13)
    x = rng.normal(size=(4000, 64)).astype(np.float32)
    q = rng.normal(size=(200, 64)).astype(np.float32)
    adj = oracle.build_graph(x, 16)
    ctx.reset()
    ctx.load_partition(0, dvs.GraphIndex(x, np.arange(4000, dtype=np.uint32), 16, adj, None))
    assert not ctx.index_integral()
    f32 = ctx.beam_search(0, q, dvs.SearchParams(6, 32, 10, 32, accum="f32"))
    f64 = ctx.beam_search(0, q, dvs.SearchParams(6, 32, 10, 32, accum="f64"))
    for a, b in zip(f32, f64):  # upgraded: the f64 parity mode's results, bit for bit
        assert np.array_equal(a, b)
    ctx.reset()


def _optimize_ref(adj, keep):
    """Restatement of csrc/graph_opt.cu (rank-based detour pruning, reverse
    edges, merge) in plain Python."""
    n, d = adj.shape
    pruned = np.empty_like(adj)
    rev = []
    for v in range(n):
        det = [sum(1 for i in range(j) if (adj[adj[v, i], :j] == adj[v, j]).any()) for j in range(d)]
        order = sorted(range(d), key=lambda j: (det[j], j))
        pruned[v] = adj[v, order]
        rev += [(int(adj[v, order[p]]), order[p], v) for p in range(keep)]
    rev.sort()
    by_u = {}
    for u, _, v in rev:
        by_u.setdefault(u, []).append(v)
    out = np.empty_like(adj)
    for u in range(n):
        cand = list(pruned[u, :keep]) + by_u.get(u, [])[:d - keep] + list(pruned[u, keep:])
        seen, row = set(), []
        for c in cand:
            if c != u and c not in seen:
                seen.add(c)
                row.append(c)
        row = row[:d]
        out[u] = [row[j % len(row)] for j in range(d)] if row else [u] * d
    return out


def test_optimize_graph_matches_restatement(ctx, oracle):
    x = sift_like(1500, 16, 6, 21)
    adj = oracle.build_graph(x, 16)
    want = _optimize_ref(adj.astype(np.int64), 8)
    d_adj = _t(adj.view(np.int32))
    torch.cuda.synchronize()
    ctx.optimize_graph_device(d_adj.data_ptr(), 1500, 16, 8)
    got = d_adj.cpu().numpy().view(np.uint32)
    assert np.array_equal(got, want.astype(np.uint32))


@pytest.mark.parametrize("dim,m,flags", [(40, 7, 1), (96, 32, 1 | 2), (128, 10, 0), (256, 32, 1)])
def test_range_topk_tensor_cores_equal_cuda_cores(ctx, dim, m, flags):
    """K7 on tcgen05 (bf16 operands, fp32 TMEM accumulators) == the CUDA-core
    K7 bit for bit on byte data (every product and partial sum exact)."""
    from paper_2512_02278_b200 import ivf
    rng = np.random.default_rng(dim)
    x = rng.integers(0, 256, size=(1500, dim)).astype(np.float32)
    x[::11] = x[5]  # duplicates: (dist, id) ties
    dpad = (dim + 3) // 4 * 4
    xp = np.zeros((1500, dpad), np.float32)
    xp[:, :dim] = x
    xt = _t(xp)
    xn = ivf.row_norms(ctx, xt)
    xb = ivf.to_bf16(ctx, xt)
    off = torch.tensor([0, 100, 700, 1500], dtype=torch.int64, device="cuda")
    blocks, _ = ivf.segment_blocks(off)
    ranges = _t(np.array([[0, 300], [600, 1500], [20, 21], [900, 1499], [0, 1500]], np.int32))
    lo = _t(np.array([0, 2, 4, 5], np.int32))
    perm = _t(rng.permutation(1500).astype(np.int32))
    for row_map in (None, perm):
        f = flags | (8 if row_map is not None else 0)
        d1 = torch.empty((1500, m), dtype=torch.float32, device="cuda")
        d2 = torch.empty((1500, m), dtype=torch.float32, device="cuda")
        a = ivf.range_topk(ctx, xt, xn, xt, xn, blocks, lo, ranges, m, flags=f, row_map=row_map, out_dists=d1,
                           out_rows=1500)
        b = ivf.range_topk(ctx, xt, xn, xt, xn, blocks, lo, ranges, m, flags=f, row_map=row_map, out_dists=d2,
                           out_rows=1500, rows_bf16=xb, cols_bf16=xb)
        assert torch.equal(a, b)
        assert torch.equal(d1, d2)
    # merge pass over ranges disjoint from each list's first ones
    ranges2 = _t(np.array([[300, 600], [0, 20], [0, 0]], np.int32))
    lo2 = _t(np.array([0, 1, 2, 3], np.int32))
    a2, b2 = a.clone(), b.clone()
    ivf.range_topk(ctx, xt, xn, xt, xn, blocks, lo2, ranges2, m, flags=f | 4, row_map=perm, out_ids=a2, out_dists=d1)
    ivf.range_topk(ctx, xt, xn, xt, xn, blocks, lo2, ranges2, m, flags=f | 4, row_map=perm, out_ids=b2, out_dists=d2,
                   rows_bf16=xb, cols_bf16=xb)
    assert torch.equal(a2, b2) and torch.equal(d1, d2)


def test_ivf_graph_tensor_cores_equal_cuda_cores(ctx):
    from paper_2512_02278_b200 import ivf
    graphs = []
    for tc in (False, True):
        xt = ivf.sift_like_device(40000, 96, rank=12, seed=5, device="cuda")
        ctx.reset()
        ivf.build_graph_ivf(ctx, xt, degree=32, cluster_size=512, probe=6, n_coarse=8, sample=40000, iters=3,
                            optimize=True, keep=12, tensor_cores=tc)
        graphs.append(ctx_adjacency(ctx, 40000, 32).copy())
    assert np.array_equal(graphs[0], graphs[1])
    ctx.reset()


def test_u8_vector_storage_bit_identical(ctx, oracle):
    """dvsg_set_vector_storage(U8): K1 gathers a byte copy of the rows; ids,
    distances, counts and visited equal the f32-storage search (and the
    oracle) in every accumulation mode; float data is refused; the copy is
    dropped when the rows change."""
    from conftest import sift_like
    x = sift_like(6000, 96, 8, 21)
    q = sift_like(300, 96, 8, 22) + 0.25  # float queries: only the rows must be bytes
    adj = oracle.build_graph(x, 16)
    eo = oracle.compute_entry_order(x)
    ctx.reset()
    ctx.load_partition(0, dvs.GraphIndex(x, np.arange(len(x), dtype=np.uint32), 16, adj, eo))
    for accum in ("f32", "f64", "f32c"):
        p = dvs.SearchParams(8, 32, 10, 32, accum=accum)
        ctx.set_vector_storage("f32")
        a = ctx.beam_search(0, q, p)
        ctx.set_vector_storage("u8")
        b = ctx.beam_search(0, q, p)
        for u, v in zip(a, b):
            assert np.array_equal(u, v), accum
    want = oracle.beam_search(x, np.arange(len(x), dtype=np.uint32), adj, eo, q, 8, 32, 10, 32)
    got = ctx.beam_search(0, q, dvs.SearchParams(8, 32, 10, 32, accum="f64"))
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
    ctx.set_vector_storage("f32")
    xf = x + 0.5
    ctx.reset()
    ctx.load_partition(0, dvs.GraphIndex(xf, np.arange(len(x), dtype=np.uint32), 16, adj, eo))
    with pytest.raises(dvs.InvalidArgument):
        ctx.set_vector_storage("u8")
    ctx.reset()
