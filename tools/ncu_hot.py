# Hottest SASS instructions (warp-stall samples) of one kernel in an
# `ncu --set full --import-source on` report:
#   python tools/ncu_hot.py REPORT.ncu-rep KERNEL_INDEX [TOP]
import csv, io, subprocess, sys

path, kidx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True, check=True).stdout
blocks, cur = [], None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "Kernel Name":
        cur = {"name": row[1], "rows": []}
        blocks.append(cur)
    elif row[0] == "Address":
        cur["hdr"] = row
    elif cur is not None:
        cur["rows"].append(row)
b = blocks[kidx]
h = b["hdr"]
si = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_")]
rows = b["rows"]
tot = sum(int(r[si] or 0) for r in rows)
print(b["name"][:110], "samples", tot, "instructions", len(rows))
agg = {}
for r in rows:
    for i in stall_cols:
        v = int(r[i] or 0)
        if v:
            agg[h[i]] = agg.get(h[i], 0) + v
print("by reason:", ", ".join(f"{k[6:]} {v}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]))
order = sorted(range(len(rows)), key=lambda i: -int(rows[i][si] or 0))[:top]
for i in sorted(order):
    r = rows[i]
    rs = sorted(((int(r[j] or 0), h[j][6:]) for j in stall_cols if int(r[j] or 0)), reverse=True)[:2]
    print(f"{i:5d} {int(r[si] or 0):6d}  {r[1].strip()[:60]:60s} {rs}")
