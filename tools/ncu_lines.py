"""Warp-stall samples of an ncu report aggregated per CUDA source line (needs -lineinfo and
--import-source on).  Usage: python tools/ncu_lines.py REPORT [N]"""
import csv
import subprocess
import sys
from collections import defaultdict

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, hdr, cur = None, None, None
samples = defaultdict(float)
reason = defaultdict(lambda: defaultdict(float))
text = {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ci = {n: i for i, n in enumerate(r)}
        stall_cols = [i for i, n in enumerate(r) if n.startswith("stall_") and "Not Issued" not in n]
        continue
    if not hdr or len(r) != len(hdr):
        continue
    if r[0]:  # a source line
        cur = (fname, int(r[0]))
        text[cur] = r[1]
        continue
    if cur is None:
        continue
    try:
        s = float(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    samples[cur] += s
    for i in stall_cols:
        try:
            reason[cur][hdr[i]] += float(r[i] or 0)
        except ValueError:
            pass
tot = sum(samples.values()) or 1.0
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for k, v in sorted(samples.items(), key=lambda kv: -kv[1])[:n]:
    top = max(reason[k].items(), key=lambda kv: kv[1])[0] if reason[k] else ""
    print(f"{v / tot * 100:5.1f}%  {k[0]}:{k[1]:<5d} {top:22s} {text[k].strip()[:80]}")
