"""Phase timing of one evaluation at config C4: host wall-clock vs device events per phase."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_13459_b200 as spst  # noqa: E402
from paper_2212_13459_b200 import workloads  # noqa: E402
from paper_2212_13459_b200.pipeline import RunConfig, _weights_for_scale, objective_for  # noqa: E402

c = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
H, W = c["content"]
spec = spst.calibrated_vgg19(0)
u = workloads.synth_content(H, W, 1)
v = workloads.synth_style(*c["style"], 2)
p = spst.build_problem(u, v, spec, _weights_for_scale(RunConfig(extractor=spec), spec, (H, W)))
eng = p.engine
x = torch.from_numpy(u).cuda()
g = torch.empty_like(x)
obj = objective_for(p)
for _ in range(2):
    obj.loss(x)
    obj.grad(g)
torch.cuda.synchronize()


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


for rep in range(3):
    t0 = time.perf_counter()
    e0 = ev()
    eng.forward(x)
    t1 = time.perf_counter()
    e1 = ev()
    counts = [eng.owned_pixels(i) for i in range(len(eng.style_taps))]
    terms, _ = eng.finalize(counts)
    t2 = time.perf_counter()
    e2 = ev()
    cs = float(eng.content_sqdiff().item())
    t3 = time.perf_counter()
    e3 = ev()
    eng.backward(2 * p.weights.lambda_c, g)
    t4 = time.perf_counter()
    e4 = ev()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(f"host ms: fwd {1e3*(t1-t0):.1f} fin {1e3*(t2-t1):.1f} content {1e3*(t3-t2):.1f} bwd {1e3*(t4-t3):.1f} "
          f"tail {1e3*(t5-t4):.1f} | dev ms: fwd {e0.elapsed_time(e1):.1f} fin {e1.elapsed_time(e2):.1f} "
          f"content {e2.elapsed_time(e3):.1f} bwd {e3.elapsed_time(e4):.1f}")
