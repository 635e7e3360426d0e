"""Device time of one loss+gradient evaluation at config C4 (6048x8064), CUDA events, after
warm-up; alternating A/B libraries is done by running this under different SPST_LIB values."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_13459_b200 as spst  # noqa: E402
from paper_2212_13459_b200 import workloads  # noqa: E402
from paper_2212_13459_b200.pipeline import RunConfig, _weights_for_scale, objective_for  # noqa: E402

c = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
H, W = c["content"]
spec = spst.calibrated_vgg19(0)
u = workloads.synth_content(H, W, 1)
p = spst.build_problem(u, workloads.synth_style(*c["style"], 2), spec,
                       _weights_for_scale(RunConfig(extractor=spec), spec, (H, W)))
obj = objective_for(p)
x = torch.from_numpy(u).cuda()
g = torch.empty_like(x)
for _ in range(3):
    obj.loss(x)
    obj.grad(g)
torch.cuda.synchronize()
ts = []
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        obj.loss(x)
        obj.grad(g)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 5)
print(os.environ.get("SPST_LIB", "default"), " ".join(f"{t:.2f}" for t in ts), "ms/eval")
