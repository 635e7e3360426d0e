import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2212_13459_b200 as spst
from paper_2212_13459_b200 import workloads
from paper_2212_13459_b200.pipeline import RunConfig, _weights_for_scale, objective_for
from paper_2212_13459_b200.lbfgs import LBFGSConfig, minimize
H, W = 756, 1008
u = workloads.synth_content(H, W, 1); v = workloads.synth_style(529, 665, 2)
spec = spst.calibrated_vgg19(0)
p = spst.build_problem(u, v, spec, _weights_for_scale(RunConfig(extractor=spec), spec, (H, W)))
obj = objective_for(p)
x = torch.from_numpy(u).cuda()
acc = {"loss": 0.0, "grad": 0.0, "n_loss": 0, "n_grad": 0}
L0, G0 = obj.loss, obj.grad
def tl(xx):
    t = time.perf_counter(); r = L0(xx); acc["loss"] += time.perf_counter() - t; acc["n_loss"] += 1; return r
def tg(o):
    t = time.perf_counter(); r = G0(o); acc["grad"] += time.perf_counter() - t; acc["n_grad"] += 1; return r
for m in (100, 10):
    x1, _ = minimize(obj, x, LBFGSConfig(history_size=m, max_iters=m + 5))  # warm, fill history
    obj.loss, obj.grad = tl, tg
    for k in acc: acc[k] = 0
    torch.cuda.synchronize(); t0 = time.perf_counter()
    x2, tr = minimize(obj, x1, LBFGSConfig(history_size=m, max_iters=m + 40))
    torch.cuda.synchronize(); tot = time.perf_counter() - t0
    its = len(tr.losses) - 1
    obj.loss, obj.grad = L0, G0
    print(f"m={m}: {its} iters, {1e3*tot/its:.2f} ms/iter; loss {1e3*acc['loss']/its:.2f} ms ({acc['n_loss']/its:.2f}/iter), "
          f"grad {1e3*acc['grad']/its:.2f} ms, rest (L-BFGS host+vectors) {1e3*(tot-acc['loss']-acc['grad'])/its:.2f} ms")
