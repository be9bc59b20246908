"""HBM random-row gather ceiling on this B200 (north_star's "HBM-gather
roofline"): GB/s of random row reads from a 38.4 GB array (the cfg3 index
size) for row sizes 96 B .. 3 KB, 1-8 rows in flight per warp, grids of
4..16 CTAs/SM.  Compare K1's DRAM GB/s against the best of these rather than
the sequential-copy peak.  One JSON line per setting."""
import ctypes
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "gather", "gather_roofline.cu")
LIB = os.path.join(HERE, "gather", "libgather_roofline.so")


def main():
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                        "-shared", "-Xcompiler", "-fPIC", SRC, "-o", LIB], check=True)
    lib = ctypes.CDLL(LIB)
    lib.gather_run.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64,
                               ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
    dev = torch.device("cuda", 0)
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    total = 100_000_000 * 96  # floats: the cfg3 vector array (38.4 GB)
    base = torch.empty(total, dtype=torch.float32, device=dev)
    base.fill_(1.0)
    g = torch.Generator(device=dev).manual_seed(1)
    for dpad in (24, 96, 128, 768):
        nrows = total // dpad
        nidx = min(20_000_000, 4_000_000_000 // (dpad * 4))
        idx = torch.randint(0, nrows, (nidx,), device=dev, generator=g, dtype=torch.int64).to(torch.int32)
        out = torch.empty(nsm * 16 * 8, dtype=torch.float32, device=dev)
        best = None
        for u in ((1, 2, 4, 8) if dpad <= 128 else (1, 2, 4)):
            for per_sm in (4, 8, 16):
                ms = ctypes.c_float()
                for _ in range(2):
                    rc = lib.gather_run(base.data_ptr(), nrows, dpad, idx.data_ptr(), nidx, out.data_ptr(), u,
                                        nsm * per_sm, ctypes.byref(ms))
                gbs = nidx * dpad * 4 / (ms.value / 1e3) / 1e9
                line = {"row_bytes": dpad * 4, "rows_in_flight_per_warp": u, "ctas_per_sm": per_sm,
                        "gbs": round(gbs, 1), "rc": rc}
                print(json.dumps(line), flush=True)
                if best is None or gbs > best["gbs"]:
                    best = line
        print(json.dumps({"row_bytes": dpad * 4, "best": best}), flush=True)


if __name__ == "__main__":
    main()
