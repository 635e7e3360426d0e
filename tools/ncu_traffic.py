"""Average DRAM traffic per launch of one kernel class from an ncu report.

    python tools/ncu_traffic.py REPORT.ncu-rep "conv3x3_tc_kernel<128" "conv3x3_tc<128>" > profiles/dominant_traffic.json

Reads dram__bytes_read.sum + dram__bytes_write.sum and gpu__time_duration.sum of every
launch whose name contains the pattern; bench.py reads the result as roofline.traffic."""
import csv
import json
import subprocess
import sys

rep, pattern, cls = sys.argv[1], sys.argv[2], sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
ci = {n: i for i, n in enumerate(hdr)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0,
         "us": 1e-3, "ns": 1e-6, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
launches = []
for r in rows[2:]:
    if len(r) != len(hdr) or pattern not in r[ci["Kernel Name"]]:
        continue
    val = {m: float(r[ci[m]].replace(",", "")) * scale[units[ci[m]]]
           for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")}
    launches.append(val)
n = len(launches)
rd = sum(v["dram__bytes_read.sum"] for v in launches) / n
wr = sum(v["dram__bytes_write.sum"] for v in launches) / n
ms = sum(v["gpu__time_duration.sum"] for v in launches) / n
print(json.dumps({"kernel_class": cls, "pattern": pattern, "launches": n, "report": rep.split("/")[-1],
                  "dram_bytes_per_launch": rd + wr, "dram_read_per_launch": rd, "dram_write_per_launch": wr,
                  "avg_duration_ms_under_ncu": ms}, indent=1))
