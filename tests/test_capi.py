"""CPU: the C-ABI library loads, exports every symbol include/dvsg.h declares,
and its host-only entry points (entry order, FNSY writer) match the reference.
No device compute here."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "dvsg.h")).read()
    return sorted(set(re.findall(r"\b(dvsg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import paper_2512_02278_b200._lib as L
    declared = _declared_symbols()
    assert len(declared) >= 20
    missing = [s for s in declared if not hasattr(L.lib, s)]
    assert not missing, missing
    assert set(declared) == set(L.EXPORTED), set(declared) ^ set(L.EXPORTED)


def test_library_is_sm100a_only():
    import subprocess
    from paper_2512_02278_b200 import LIB_PATH
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB_PATH],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2512_02278_b200 as dvs
    with pytest.raises(dvs.InternalError, match="CUDA"):
        dvs.Context(0)


def test_status_codes_mirror_reference_exit_codes():
    import paper_2512_02278_b200._lib as L
    assert (L.DVSG_EINVAL, L.DVSG_EFORMAT, L.DVSG_EINTERNAL) == (2, 3, 4)  # commands.cpp:355-361
    assert issubclass(L.InvalidArgument, ValueError)


def test_host_entry_order_matches_oracle(oracle, golden):
    import paper_2512_02278_b200 as dvs
    for name in ("g1_uniform.npz", "g2_siftlike.npz"):
        g = golden(name)
        assert np.array_equal(dvs.compute_entry_order(g["vectors"]), g["entry_order"])
    v = oracle.random_dataset(70000, 8, 3)  # multi-threaded host path
    assert np.array_equal(dvs.compute_entry_order(v), oracle.compute_entry_order(v))


def test_fnsy_writer_roundtrips_reference_file(tmp_path):
    import paper_2512_02278_b200 as dvs
    from fnsy import G3_FNSY, read_fnsy
    idx = read_fnsy(G3_FNSY)
    out = tmp_path / "copy.fnsy"
    built = dvs.BuiltIndex(idx.centroids, idx.cluster_to_rank, idx.ranks, idx.out_degree,
                           [dvs.GraphIndex(g.vectors, g.global_ids, g.out_degree, g.adjacency)
                            for g in idx.graphs])
    dvs.save_index(built, str(out))
    assert open(G3_FNSY, "rb").read() == out.read_bytes()  # bit-exact vs save_index


def test_fnsy_written_file_loads_in_reference(ref, tmp_path):
    import paper_2512_02278_b200 as dvs
    from fnsy import G3_FNSY, read_fnsy
    idx = read_fnsy(G3_FNSY)
    built = dvs.BuiltIndex(idx.centroids, idx.cluster_to_rank, idx.ranks, idx.out_degree,
                           [dvs.GraphIndex(g.vectors, g.global_ids, g.out_degree, g.adjacency)
                            for g in idx.graphs])
    out = tmp_path / "mine.fnsy"
    dvs.save_index(built, str(out))
    r = ref.load_index(str(out)).dump()
    for (v, a, gi, _), g in zip(r["graphs"], idx.graphs):
        assert np.array_equal(v, g.vectors) and np.array_equal(a, g.adjacency)
        assert np.array_equal(gi, g.global_ids)


def test_save_index_rejects_unbuilt():
    import paper_2512_02278_b200 as dvs
    with pytest.raises(dvs.InvalidArgument):
        dvs.save_index(dvs.BuiltIndex(np.zeros((0, 4), np.float32), np.zeros(0, np.uint32), 1, 4), "/tmp/x")


def test_search_params_accum_modes():
    # f64 parity / f32 fast / f32c compensated; anything else is invalid_argument
    import paper_2512_02278_b200 as dvs
    from paper_2512_02278_b200 import _lib
    assert (_lib.ACCUM_F64, _lib.ACCUM_F32, _lib.ACCUM_F32C) == (0, 1, 2)
    for name, code in (("f64", 0), ("f32", 1), ("f32c", 2)):
        assert dvs.SearchParams(6, 64, 10, 64, accum=name).to_c().accum == code
    with pytest.raises(dvs.InvalidArgument):
        dvs.SearchParams(6, 64, 10, 64, accum="f16").to_c()
