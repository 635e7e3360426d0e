"""Wall-clock breakdown of L-BFGS iterations at config C4: objective loss / grad vs the rest."""
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
acc = {"loss": 0.0, "grad": 0.0}
loss0, grad0 = obj.loss, obj.grad


def tl(x):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = loss0(x)
    torch.cuda.synchronize()
    acc["loss"] += time.perf_counter() - t
    return r


def tg(o):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = grad0(o)
    torch.cuda.synchronize()
    acc["grad"] += time.perf_counter() - t
    return r


obj.loss, obj.grad = tl, tg
x = torch.from_numpy(u).cuda()
marks = {}


def cb(it, xi, loss, gn):
    torch.cuda.synchronize()
    marks[it] = (time.perf_counter(), dict(acc))


t0 = time.perf_counter()
x, tr = minimize(obj, x, LBFGSConfig(history_size=10, max_iters=8), callback=cb)
for it in range(4, 9):
    (ta, aa), (tb, ab) = marks[it - 1], marks[it]
    print(f"iter {it}: wall {1e3 * (tb - ta):.1f} ms  loss-calls {1e3 * (ab['loss'] - aa['loss']):.1f}  "
          f"grad-calls {1e3 * (ab['grad'] - aa['grad']):.1f}")
print("evals", tr.evals, "grads", tr.grads)
