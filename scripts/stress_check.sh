#!/bin/bash
# Race stress: the GPU parity suite against a build where every block / warp
# barrier is followed by random per-thread sleeps (-DDVSG_STRESS=1, see
# csrc/dvsg_internal.h).  compute-sanitizer is closed on this pool; this is
# the substitute.  Writes gpurun_out/stress/{build.log,pytest.log}.
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/gpurun_out/stress; mkdir -p $OUT
LIB=$ROOT/paper_2512_02278_b200/variants/libdvsg_stress.so
mkdir -p "$(dirname "$LIB")"
if [ ! -f "$LIB" ]; then
  make -s -C $ROOT/paper_2512_02278_b200/csrc -j8 OUT=$LIB OBJ=$ROOT/build/obj_stress EXTRA=-DDVSG_STRESS=1 > $OUT/build.log 2>&1
fi
echo "NANOSLEEP sites in the stress build: $(/usr/local/cuda/bin/cuobjdump -sass $LIB | grep -c NANOSLEEP)" | tee $OUT/pytest.log
# the stress library is the one the test processes load, and it is slower
DVSG_LIB=$LIB python - <<'PY' 2>&1 | tee -a $OUT/pytest.log
import time, numpy as np, os
import paper_2512_02278_b200 as dvs
from paper_2512_02278_b200 import _lib
print("loaded:", _lib.LIB_PATH)
rng = np.random.default_rng(1)
v = rng.integers(0, 255, size=(20000, 64)).astype(np.float32)
ctx = dvs.Context(0)
adj = ctx.build_graph(v, 16)
ctx.load_partition(0, dvs.GraphIndex(v, np.arange(len(v), dtype=np.uint32), 16, adj, None))
q = v[:2000] + 1
ctx.beam_search(0, q, dvs.SearchParams(6, 32, 10, 32, accum="f32"))
t = time.perf_counter(); ctx.beam_search(0, q, dvs.SearchParams(6, 32, 10, 32, accum="f32"))
print("2000-query K1 search: %.1f ms" % ((time.perf_counter() - t) * 1e3))
PY
for rep in 1 2 3; do
  DVSG_LIB=$LIB timeout 1500 python -m pytest $ROOT/tests -q -m gpu -p no:cacheprovider \
    --ignore=$ROOT/tests/test_gpu_fullsize.py 2>&1 | tail -3 | sed "s/^/[rep $rep] /" | tee -a $OUT/pytest.log
done
