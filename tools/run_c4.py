"""Full multiscale transfer at config C4 (content 6048x8064, style 4226x5319, 4 scales) through
the public API (`multiscale_transfer`), timed per scale.  The paper reports this workload end to
end for the authors' GPU implementation: SPST-fast (600,200,66,30) 13 min, SPST
(600,300,300,300) 74 min (context only -- different hardware and code).

    python tools/run_c4.py [--mode fast|baseline] [--config c4] [--out gpurun_out/c4_fast.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_13459_b200 as spst  # noqa: E402
from paper_2212_13459_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="fast", choices=["fast", "baseline"])
ap.add_argument("--config", default="c4")
ap.add_argument("--scales", type=int, default=4)
ap.add_argument("--out", default=None)
ap.add_argument("--repeat", type=int, default=1, help="runs in one process (later runs are warm)")
a = ap.parse_args()

c = workloads.CONFIGS[a.config]
H, W = c["content"]
u = workloads.synth_content(H, W, 1)
v = workloads.synth_style(*c["style"], 2)
spec = spst.calibrated_vgg19(0)
cfg = spst.RunConfig(n_scales=a.scales, mode=a.mode, extractor=spec)
sched = spst.make_schedule(a.scales, a.mode)
dims = spst.scale_dims((H, W), a.scales)

def run_once():
    marks = {}

    def progress(scale, it, loss, gnorm):
        now = time.perf_counter()
        m = marks.setdefault(scale, {"first": now, "iters": 0, "loss0": loss})
        m["last"], m["iters"], m["loss"], m["gnorm"] = now, it, loss, gnorm

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = spst.multiscale_transfer(u, v, cfg, progress=progress)
    torch.cuda.synchronize()
    total = time.perf_counter() - t0
    rows = []
    prev_end = t0
    for s in sorted(marks):
        m = marks[s]
        # seconds = from the previous scale's last iteration to this scale's last (includes this
        # scale's setup: downsampling, style statistics, content capture, upsampling)
        it_s = (m["last"] - m["first"]) / max(1, m["iters"] - 1)
        rows.append({"scale": s, "dims": list(dims[s - 1]), "iters": m["iters"], "schedule": sched.iters[s - 1],
                     "ms_per_iter": 1e3 * it_s, "seconds": m["last"] - prev_end, "final_loss": m["loss"],
                     "first_loss": m["loss0"]})
        prev_end = m["last"]
    return total, rows, out


runs = []
for r in range(a.repeat):
    total, rows, out = run_once()
    runs.append({"run": r + 1, "kind": "first run of the process" if r == 0 else "warm (same process)",
                 "total_seconds": total, "scales": rows})
    print(f"run {r + 1}: {total:.2f} s " + " ".join(f"s{x['scale']}:{x['ms_per_iter']:.1f}ms/it,{x['seconds']:.2f}s"
                                                 for x in rows), flush=True)
res = {"workload": f"{a.config}: {a.scales}-scale multiscale_transfer, content {H}x{W}, style {c['style']}",
       "mode": a.mode, "schedule": list(sched.iters), "total_seconds": runs[0]["total_seconds"],
       "scales": runs[0]["scales"], "runs": runs,
       "output_finite": bool(np.isfinite(out).all()), "output_range": [float(out.min()), float(out.max())],
       "device": torch.cuda.get_device_name(0)}
print(json.dumps({k: v for k, v in res.items() if k != "runs"}, indent=1))
if a.out:
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
