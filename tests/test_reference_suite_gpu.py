"""GPU: the reference's OWN unit tests (/root/reference/proj/tests/test_*.cpp,
compiled unchanged by shim/Makefile with shim/doctest.h) run against the
B200 backend: shim/dvs_gpu.cpp replaces src/graph_index.cpp, so every
build_graph / beam_search / visited_count call in them goes through libdvsg.
The binary is built in the build container (it needs the reference sources)
and ships to the GPU box with the snapshot."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "shim", "_build", "ref_tests_gpu")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.isfile(BIN), reason="shim/_build/ref_tests_gpu not built")
def test_reference_unit_tests_pass_on_gpu_backend():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    print(r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert "| 0 failed" in r.stdout
