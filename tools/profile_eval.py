"""One loss+gradient evaluation of config C4 (6048x8064) bracketed by cudaProfilerStart/Stop,
for `ncu --profile-from-start off` launch lists and single-kernel captures."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_13459_b200 as spst  # noqa: E402
from paper_2212_13459_b200 import workloads  # noqa: E402
from paper_2212_13459_b200.pipeline import RunConfig, _weights_for_scale, objective_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--dims", default=None, help="HxW content override (e.g. 756x1008, a coarse C4 scale)")
a = ap.parse_args()
c = workloads.CONFIGS[a.config]
H, W = (int(t) for t in a.dims.split("x")) if a.dims else c["content"]
spec = spst.calibrated_vgg19(0)
u = workloads.synth_content(H, W, 1)
v = workloads.synth_style(*c["style"], 2)
p = spst.build_problem(u, v, spec, _weights_for_scale(RunConfig(extractor=spec), spec, (H, W)))
obj = objective_for(p)
x = torch.from_numpy(u).cuda()
g = torch.empty_like(x)
for _ in range(2):  # warm (scales known, no careful re-runs)
    obj.loss(x)
    obj.grad(g)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(a.reps):
    obj.loss(x)
    obj.grad(g)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
