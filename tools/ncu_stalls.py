"""Top stall locations (source page) of an ncu report."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ci = {n: i for i, n in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


key = "Warp Stall Sampling (All Samples)"
tot = sum(f(r[ci[key]]) for r in data) or 1
stalls = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
agg = {k: sum(f(r[ci[k]]) for r in data) for k in stalls}
print("stall totals:", [(k, round(v / tot * 100, 1)) for v, k in sorted(((v, k) for k, v in agg.items()), reverse=True)[:8]])
data.sort(key=lambda r: -f(r[ci[key]]))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for r in data[:n]:
    top = max(stalls, key=lambda k: f(r[ci[k]]))
    print(f"{f(r[ci[key]]) / tot * 100:5.1f}%  {r[ci['Address']][-6:]}  {r[ci['Source']][:80]:80s} {top}")
