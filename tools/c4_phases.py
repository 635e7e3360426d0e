"""Where the time between scales goes in the C4 multiscale run: wraps the pipeline's style
statistics, build_problem and minimize (first-iteration evaluations included)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_13459_b200 as spst  # noqa: E402
from paper_2212_13459_b200 import pipeline as P, workloads  # noqa: E402

log = []


def timed(name, fn):
    def w(*a, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        log.append((name, time.perf_counter() - t, r[1].evals if name == "minimize" else None))
        return r
    return w


P._cached_style_stats = timed("style_stats", P._cached_style_stats)
P.build_problem = timed("build_problem", P.build_problem)
P.minimize = timed("minimize", P.minimize)
c = workloads.CONFIGS["c4"]
u = workloads.synth_content(*c["content"], 1)
v = workloads.synth_style(*c["style"], 2)
spec = spst.calibrated_vgg19(0)
for rep in range(2):
    log.clear()
    t0 = time.perf_counter()
    spst.multiscale_transfer(u, v, spst.RunConfig(n_scales=4, mode="fast", extractor=spec))
    print(f"run {rep}: total {time.perf_counter() - t0:.2f} s")
    for name, dt, ev in log:
        print(f"   {name:14s} {dt:6.2f} s" + (f"  evals {ev}" if ev is not None else ""))
