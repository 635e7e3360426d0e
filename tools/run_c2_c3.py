"""Configs C2 and C3 (BASELINE.json configs[1], configs[2]) on one B200 through the public API.

    python tools/run_c2_c3.py [--out gpurun_out/c2_c3.json] [--no-oracle]

C2: single scale, 1512x2016 content, 1024x1024 style, 100 L-BFGS iterations (history 100, as
    the reference's first scale, pipeline.py:32-33).  Before the run, one evaluation at a
    perturbed iterate is checked against the f64 oracle (oracle/spst_oracle.py, whole-image
    restatement of the reference's Algorithm 1 — test infrastructure, run here as the checker
    only): loss within 1e-5, the gradient within the north-star bar max(1e-3, 1.5 x the
    oracle's own f32-vs-f64 difference) and, on our ReLU pattern, within 5e-6 are asserted.
C3: multiscale_transfer with 3 scales, 756x1008 -> 1512x2016 -> 3024x4032 content, style
    2113x2660, fast schedule; per-scale iterations and time.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2212_13459_b200 as spst  # noqa: E402
from paper_2212_13459_b200 import workloads  # noqa: E402
from paper_2212_13459_b200.lbfgs import LBFGSConfig, minimize  # noqa: E402
from paper_2212_13459_b200.pipeline import RunConfig, _weights_for_scale, objective_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/c2_c3.json")
ap.add_argument("--no-oracle", action="store_true")
a = ap.parse_args()
spec = spst.calibrated_vgg19(0)
res = {"device": torch.cuda.get_device_name(0)}

# ---------------------------------------------------------------- C2
c = workloads.CONFIGS["c2"]
H, W = c["content"]
u = workloads.synth_content(H, W, 1)
v = workloads.synth_style(*c["style"], 2)
weights = _weights_for_scale(RunConfig(extractor=spec), spec, (H, W))
p = spst.build_problem(u, v, spec, weights)
rng = np.random.default_rng(3)
xc = np.clip(u + 0.05 * rng.standard_normal(u.shape), 0, 1).astype(np.float32)
loss, g = spst.loss_grad(xc, p)
c2 = {"content": [H, W], "style": list(c["style"]), "loss_at_x": loss}
if not a.no_oracle:
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import spst_oracle as O  # checker only
    t0 = time.time()
    net = O.onet_from_spec(spec)
    po = O.build_problem(u.astype(np.float64), v.astype(np.float64), net,
                         O.default_weights(net, weights.lambda_c), 4096, 160)  # one block: the whole image
    lo, go = O.loss_grad_global(xc.astype(np.float64), po)
    # the f64 network on OUR ReLU pattern isolates arithmetic from sign flips of near-zero
    # pre-activations; the oracle's own f32 path shows the reference's envelope
    _, gm = O.loss_grad_global(xc.astype(np.float64), po, masks=p.engine.relu_masks())
    po32 = O.build_problem(u, v, net, O.default_weights(net, weights.lambda_c), 4096, 160)
    _, g32 = O.loss_grad_global(xc, po32)

    def rel(a_, b_):
        return float(np.linalg.norm((np.asarray(a_, np.float64) - b_).ravel()) / np.linalg.norm(b_.ravel()))
    rl, rg, ra, r32 = abs(loss - lo) / abs(lo), rel(g, go), rel(g, gm), rel(g32, go)
    c2["oracle_f64"] = {"loss": lo, "loss_rel": rl, "grad_rel_l2": rg, "grad_rel_l2_on_our_masks": ra,
                        "oracle_f32_grad_rel_l2": r32, "seconds": time.time() - t0,
                        "bounds": {"loss_rel": 1e-5, "grad_rel_l2": max(1e-3, 1.5 * r32),
                                   "grad_rel_l2_on_our_masks": 5e-6}}
    print(f"C2 vs f64 oracle: loss rel {rl:.2e}; grad rel-L2 {rg:.2e} (oracle's own f32 path {r32:.2e}); "
          f"on our ReLU masks {ra:.2e} ({time.time() - t0:.0f} s CPU)", flush=True)
    assert rl <= 1e-5 and ra <= 5e-6 and rg <= max(1e-3, 1.5 * r32), (rl, rg, ra, r32)
obj = objective_for(p)
x0 = torch.from_numpy(u).cuda()
minimize(obj, x0, LBFGSConfig(history_size=100, max_iters=3))  # module load / first binds
torch.cuda.synchronize()
t0 = time.perf_counter()
x, tr = minimize(obj, x0, LBFGSConfig(history_size=100, max_iters=c["iters"]))
torch.cuda.synchronize()
dt = time.perf_counter() - t0
its = len(tr.losses) - 1
c2.update({"iters": its, "evals": tr.evals, "seconds": dt, "iters_per_s": its / dt,
           "ms_per_iter": 1e3 * dt / its, "first_loss": tr.losses[0], "final_loss": tr.losses[-1]})
print("C2", json.dumps(c2), flush=True)
res["c2"] = c2
del p, obj, x, x0
torch.cuda.empty_cache()

# ---------------------------------------------------------------- C3
c = workloads.CONFIGS["c3"]
H, W = c["content"]
u = workloads.synth_content(H, W, 1)
v = workloads.synth_style(*c["style"], 2)
cfg = spst.RunConfig(n_scales=c["n_scales"], mode="fast", extractor=spec)
marks = {}


def progress(scale, it, loss, gnorm):
    now = time.perf_counter()
    m = marks.setdefault(scale, {"first": now, "iters": 0, "loss0": loss})
    m["last"], m["iters"], m["loss"] = now, it, loss


torch.cuda.synchronize()
t0 = time.perf_counter()
out = spst.multiscale_transfer(u, v, cfg, progress=progress)
torch.cuda.synchronize()
total = time.perf_counter() - t0
dims = spst.scale_dims((H, W), c["n_scales"])
rows, prev = [], t0
for s in sorted(marks):
    m = marks[s]
    rows.append({"scale": s, "dims": list(dims[s - 1]), "iters": m["iters"],
                 "ms_per_iter": 1e3 * (m["last"] - m["first"]) / max(1, m["iters"] - 1),
                 "seconds": m["last"] - prev, "first_loss": m["loss0"], "final_loss": m["loss"]})
    prev = m["last"]
res["c3"] = {"content": [H, W], "style": list(c["style"]), "schedule": list(spst.make_schedule(c["n_scales"], "fast").iters),
             "total_seconds": total, "scales": rows, "output_finite": bool(np.isfinite(out).all()),
             "note": "first multiscale run of the process (includes one-time binds / pool growth per scale)"}
print("C3", json.dumps(res["c3"]), flush=True)
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
with open(a.out, "w") as f:
    json.dump(res, f, indent=1)
