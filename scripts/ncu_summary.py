"""Summarize ncu outputs into profiles/ (run here, on the CPU box).

    python scripts/ncu_summary.py <tag> [gpurun_out]

Reads <dir>/launches.csv (gpu__time_duration launch list of the bench command)
and <dir>/k1_full.ncu-rep (--set full capture of K1), writes
profiles/<tag>_launches.csv (copy), profiles/<tag>_ncu.json and
profiles/k1_traffic.json (DRAM bytes per K1 launch, read by bench.py).
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
]

UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def launch_list(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = {}
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        name = r[hdr["Kernel Name"]]
        unit = r[hdr["Metric Unit"]]
        try:
            v = float(r[hdr["Metric Value"]].replace(",", ""))
        except ValueError:
            continue
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}.get(unit, 1.0)
        short = name.split("(")[0].replace("void ", "")[:90]
        e = out.setdefault(short, {"launches": 0, "ms": 0.0})
        e["launches"] += 1
        e["ms"] += v * scale
    tot = sum(e["ms"] for e in out.values())
    for e in out.values():
        e["share"] = e["ms"] / tot if tot else 0
    return dict(sorted(out.items(), key=lambda kv: -kv[1]["ms"])), tot


def full_capture(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {}
    for i, h in enumerate(hdr):
        if h in METRICS or h == "Kernel Name":
            res[h] = {"value": vals[i], "unit": units[i]}
    return res


def main():
    tag = sys.argv[1]
    d = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    summary = {"tag": tag}
    lpath = os.path.join(d, "launches.csv")
    if os.path.isfile(lpath):
        shutil.copy(lpath, os.path.join(prof, f"{tag}_launches.csv"))
        kernels, tot = launch_list(lpath)
        summary["launch_list"] = {"total_ms": tot, "kernels": kernels,
                                  "note": "ncu --metrics gpu__time_duration.sum --clock-control none "
                                          "of `python bench.py --steps 3 --warmup 3`: cold-cache, "
                                          "serialised; compare shares, not absolutes"}
    fpath = os.path.join(d, "k1_full.ncu-rep")
    if os.path.isfile(fpath):
        m = full_capture(fpath)
        summary["k1_full"] = m
        rd = float(m["dram__bytes_read.sum"]["value"]) * UNIT.get(m["dram__bytes_read.sum"]["unit"], 1)
        wr = float(m["dram__bytes_write.sum"]["value"]) * UNIT.get(m["dram__bytes_write.sum"]["unit"], 1)
        summary["k1_dram_bytes_per_launch"] = rd + wr
        json.dump({"config_key": "n1000000_q100000_w64_I6_f32", "dram_bytes_per_launch": rd + wr,
                   "source": f"profiles/{tag}_ncu.json (ncu --set full, one K1 launch)"},
                  open(os.path.join(prof, "k1_traffic.json"), "w"), indent=1)
    json.dump(summary, open(os.path.join(prof, f"{tag}_ncu.json"), "w"), indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "k1_full"}, indent=1)[:3000])
    if "k1_full" in summary:
        for k, v in summary["k1_full"].items():
            print(f"  {k}: {v['value']} {v['unit']}")


if __name__ == "__main__":
    main()
