"""Per-SASS-region stall samples / instructions of one kernel in an .ncu-rep
(--page source), to find where a kernel spends its time.
    python scripts/ncu_regions.py <rep> [block=100]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 100
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(txt.splitlines()))
h = r[1]
rows = r[2:]
iS = h.index("Warp Stall Sampling (All Samples)")
iI = h.index("Instructions Executed")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_")]
tot = sum(int(x[iS]) for x in rows)
print("samples", tot, "inst %.1fM" % (sum(int(x[iI]) for x in rows) / 1e6))
for b in range(0, len(rows), B):
    blk = rows[b:b + B]
    s = sum(int(x[iS]) for x in blk)
    if s < tot * 0.01:
        continue
    i = sum(int(x[iI]) for x in blk)
    st = {}
    for c in stall_cols:
        v = sum(int(x[c]) if x[c].isdigit() else 0 for x in blk)
        if v:
            st[h[c][6:]] = v
    top = sorted(st.items(), key=lambda kv: -kv[1])[:4]
    ops = set()
    for x in blk:
        t = x[1].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
        if op.split(".")[0] in ("LDG", "STG", "ATOMG", "ATOMS", "SHFL", "BAR", "LDS", "STS", "RED", "ATOM", "MEMBAR", "LD", "ST", "VOTE"):
            ops.add(op.split(".")[0])
    print(f"{b:5d} {100*s/tot:5.1f}% inst {i/1e6:7.1f}M  " + " ".join(f"{k}={100*v/max(s,1):.0f}%" for k, v in top) + "  [" + ",".join(sorted(ops)) + "]")
