"""Two L-BFGS iterations of config C4 (after 3 warm-up iterations) inside cudaProfilerStart/Stop,
plus host-side wall-clock for each phase of minimize."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_13459_b200 as spst  # noqa: E402
from paper_2212_13459_b200 import workloads  # noqa: E402
from paper_2212_13459_b200.lbfgs import LBFGSConfig, minimize  # noqa: E402
from paper_2212_13459_b200.pipeline import RunConfig, _weights_for_scale, objective_for  # noqa: E402

c = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
H, W = c["content"]
spec = spst.calibrated_vgg19(0)
u = workloads.synth_content(H, W, 1)
v = workloads.synth_style(*c["style"], 2)
p = spst.build_problem(u, v, spec, _weights_for_scale(RunConfig(extractor=spec), spec, (H, W)))
obj = objective_for(p)
x = torch.from_numpy(u).cuda()
x, _ = minimize(obj, x, LBFGSConfig(history_size=10, max_iters=3))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
t0 = time.time()
x, tr = minimize(obj, x, LBFGSConfig(history_size=10, max_iters=2))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(f"2 iterations {1e3 * (time.time() - t0):.1f} ms, evals {tr.evals}, grads {tr.grads}")
