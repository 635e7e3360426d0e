"""Per-kernel device time and GPU idle share of coarse-scale L-BFGS iterations (torch.profiler /
CUPTI).  Diagnostic only -- numbers taken under a profiler are never bench values.

    python tools/coarse_profile.py [--dims 756x1008] [--m 100] [--iters 30]
"""
import argparse
import os
import sys
import time
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_13459_b200 as spst  # noqa: E402
from paper_2212_13459_b200 import workloads  # noqa: E402
from paper_2212_13459_b200.lbfgs import LBFGSConfig, minimize  # noqa: E402
from paper_2212_13459_b200.pipeline import RunConfig, _weights_for_scale, objective_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", default="756x1008")
ap.add_argument("--m", type=int, default=100)
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--stacks", action="store_true", help="attribute device->host copies to Python call sites")
ap.add_argument("--cprofile", action="store_true", help="host-side cProfile of the iterations instead")
a = ap.parse_args()
H, W = (int(t) for t in a.dims.split("x"))
u = workloads.synth_content(H, W, 1)
v = workloads.synth_style(int(H * 0.7), int(W * 0.66), 2)
spec = spst.calibrated_vgg19(0)
p = spst.build_problem(u, v, spec, _weights_for_scale(RunConfig(extractor=spec), spec, (H, W)))
obj = objective_for(p)
x = torch.from_numpy(u).cuda()
x1, _ = minimize(obj, x, LBFGSConfig(history_size=a.m, max_iters=a.m + 5))
torch.cuda.synchronize()
if a.cprofile:
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    minimize(obj, x1, LBFGSConfig(history_size=a.m, max_iters=a.iters))
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
    sys.exit(0)
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU], with_stack=a.stacks) as prof:
    t0 = time.perf_counter()
    x2, tr = minimize(obj, x1, LBFGSConfig(history_size=a.m, max_iters=a.iters))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
its = len(tr.losses) - 1
tot = defaultdict(lambda: [0.0, 0])
spans = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.device_time_total > 0:
        name = e.name.split("(")[0][:60]
        tot[name][0] += e.device_time_total
        tot[name][1] += 1
        spans.append((e.time_range.start, e.time_range.end))
spans.sort()
named = sorted((e.time_range.start, e.time_range.end, e.name.split("(")[0][-40:]) for e in prof.events()
               if e.device_type == torch.autograd.DeviceType.CUDA and e.device_time_total > 0)
gaps = defaultdict(lambda: [0.0, 0])
for (s0, e0, n0), (s1, e1, n1) in zip(named, named[1:]):
    if s1 - e0 > 5:
        gaps[(n0, n1)][0] += s1 - e0
        gaps[(n0, n1)][1] += 1
busy, cur_s, cur_e = 0.0, None, None
for s, e in spans:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
if cur_e is not None:
    busy += cur_e - cur_s
span = (spans[-1][1] - spans[0][0]) if spans else 0
print(f"{a.dims} m={a.m}: {its} iters, wall {1e3 * wall / its:.2f} ms/iter (under profiler); GPU busy "
      f"{busy / 1e3 / its:.2f} ms/iter of {span / 1e3 / its:.2f} ms span ({100 * busy / max(span, 1):.0f} %)")
for name, (us, n) in sorted(tot.items(), key=lambda kv: -kv[1][0])[:30]:
    print(f"  {us / 1e3 / its:8.3f} ms/iter  {n / its:6.1f} launches/iter  {us / n:8.1f} us/launch  {name}")
print("idle gaps > 5 us (after -> before):")
for (n0, n1), (us, n) in sorted(gaps.items(), key=lambda kv: -kv[1][0])[:14]:
    print(f"  {us / 1e3 / its:7.3f} ms/iter  {n / its:5.1f}/iter  {us / n:7.1f} us  {n0} -> {n1}")
if a.stacks:
    sites = defaultdict(int)
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CPU and e.name in ("cudaMemcpyAsync", "cudaMemcpy",
                                                                          "cudaStreamSynchronize"):
            frames = [f for f in (e.stack or []) if "paper_2212_13459_b200" in f or "tools/" in f][:3]
            sites[(e.name, " < ".join(frames))] += 1
    print("runtime copy / sync call sites:")
    for (name, st), n in sorted(sites.items(), key=lambda kv: -kv[1])[:20]:
        print(f"  {n / its:6.1f}/iter  {name}  {st}")
