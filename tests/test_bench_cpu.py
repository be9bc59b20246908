"""Host-side logic of bench.py and the device builder's table helpers (CPU):
workload defaults, the --gpus / WORLD_SIZE contract, recall, the K7 block
tables, and the design-B shard rule used by shard_init_resident."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_workload_defaults():
    a = bench.parse([])
    assert (a.workload, a.n, a.dim, a.nq, a.iterations, a.beam, a.entry, a.k) == \
        ("cfg3", 100_000_000, 96, 1_000_000, 24, 16, 16, 10)
    assert a.metric == "l2" and a.accum == "f32" and a.rank_latent == 16
    c4 = bench.parse(["--workload", "cfg4"])
    assert (c4.n, c4.dim, c4.k, c4.beam, c4.metric, c4.accum, c4.rank_latent) == \
        (10_000_000, 768, 100, 256, "ip", "f64", 32)
    c1 = bench.parse(["--workload", "cfg1", "--nq", "123"])
    assert (c1.n, c1.dim, c1.nq, c1.iterations, c1.beam) == (1_000_000, 128, 123, 6, 64)


def test_gpus_world_size_mismatch_fails_loudly():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"], env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "WORLD_SIZE=2" in (r.stderr + r.stdout)


def test_recall_at_k_matches_definition():
    ids = np.array([[1, 2, 3], [4, 5, 6]], np.uint32)
    cnt = np.array([3, 2], np.uint32)
    truth = np.array([[3, 2, 9], [6, 5, 4]])
    # query 0: {1,2,3} & {3,2,9} = 2; query 1: first 2 ids {4,5} & {6,5,4} = 2
    assert bench.recall_at_k(ids, cnt, truth, 3) == pytest.approx((2 / 3 + 2 / 3) / 2)


def test_segment_blocks_cover_segments_exactly():
    torch = pytest.importorskip("torch")
    from paper_2512_02278_b200 import ivf
    off = torch.tensor([0, 5, 5, 300, 301, 700], dtype=torch.int64)
    b, nb = ivf.segment_blocks(off)
    b = b.numpy()
    assert nb == b.shape[0] == 1 + 0 + 3 + 1 + 4
    assert (b[:, 1] <= 128).all() and (b[:, 1] > 0).all()
    covered = np.zeros(700, int)
    for row0, nrows, lst, out0 in b:
        assert off[lst] <= row0 and row0 + nrows <= off[lst + 1] and out0 == row0
        covered[row0:row0 + nrows] += 1
    assert (covered == 1).all()


def test_shard_rule():
    from paper_2512_02278_b200.dist import owner_of, shard_range
    n, R = 100_000_003, 8
    spans = [shard_range(n, R, r) for r in range(R)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    assert all(spans[i][1] == spans[i + 1][0] for i in range(R - 1))
    for v in (0, 12_500_000, n - 1):
        lo, hi = spans[owner_of(v, n, R)]
        assert lo <= v < hi
