"""Sum xg_expand / xg_score times of the last search in a launch list."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/xg/launches.csv")))
hdr = None
out = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            out.append((d["Kernel Name"], float(d["Metric Value"].replace(",", "")) / 1e6))
xs = [o for o in out if "xg_" in o[0]]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
last = xs[-n:]
print("total %.2f ms over the last %d xg launches" % (sum(t for k, t in last), len(last)))
print(" ".join("%.2f" % t for k, t in last))
