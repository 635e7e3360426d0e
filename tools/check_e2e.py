"""End-to-end device check against the reference's golden outputs (tests/golden)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_13459_b200 as spst  # noqa: E402
from paper_2212_13459_b200.spec import tinynet  # noqa: E402

G = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def rel(a, b):
    return float(np.linalg.norm((np.asarray(a, np.float64) - b).ravel()) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def tiny():
    d = np.load(os.path.join(G, "tinynet.npz"))
    spec = tinynet(0)
    for k in range(3):
        u, v, x = d[f"case{k}_u"], d[f"case{k}_v"], d[f"case{k}_x"]
        block, margin = d[f"case{k}_geom"]
        w = spst.default_loss_weights(spec)
        t0 = time.time()
        p = spst.build_problem(u, v, spec, w, block=int(block), margin=int(margin))
        loss, g = spst.loss_grad(x, p)
        dt = time.time() - t0
        gl = d[f"case{k}_grad_global"]
        ref_loss = d[f"case{k}_loss"][1]
        print(f"tiny case{k} {u.shape}: loss rel {abs(loss - ref_loss) / abs(ref_loss):.3e}  grad relL2 {rel(g, gl):.3e}"
              f"  ({dt:.2f}s)")
        st = spst.stats_pass(x, spec, block=int(block), margin=int(margin))
        for t in spec.style_taps:
            print(f"   {t}: gram rel {rel(st[t].gram, d[f'case{k}_{t}_gram']):.2e} mean {rel(st[t].mean, d[f'case{k}_{t}_mean']):.2e}"
                  f" std {rel(st[t].std, d[f'case{k}_{t}_std']):.2e}")


def vgg():
    path = os.path.join(G, "vgg19.npz")
    if not os.path.exists(path):
        print("no vgg golden")
        return
    d = np.load(path)
    spec = spst.calibrated_vgg19(0)
    u, v = d["c1_u"], d["c1_v"]
    w = spst.default_loss_weights(spec, lambda_c=float(d["c1_lambda_c"][0]))
    t0 = time.time()
    p = spst.build_problem(u, v, spec, w)
    torch.cuda.synchronize()
    print(f"vgg build_problem {time.time() - t0:.2f}s")
    for t in spec.style_taps:
        print(f"   style {t}: gram rel {rel(p.style_stats[t].gram, d[f'c1_style_{t}_gram']):.2e} "
              f"mean {rel(p.style_stats[t].mean, d[f'c1_style_{t}_mean']):.2e} std {rel(p.style_stats[t].std, d[f'c1_style_{t}_std']):.2e}")
    for rep in range(3):
        t0 = time.time()
        loss, g = spst.loss_grad(u, p)
        torch.cuda.synchronize()
        dt = time.time() - t0
    l64 = d["c1_loss64"][0]
    g64 = d["c1_grad64"].astype(np.float64)
    g32 = d["c1_grad32"].astype(np.float64)
    print(f"vgg c1 x0: loss rel {abs(loss - l64) / l64:.3e}  grad relL2 vs f64 {rel(g, g64):.3e}  "
          f"(reference f32 vs f64: {rel(g32, g64):.3e}; ours vs ref f32 {rel(g, g32):.3e})  {dt * 1e3:.1f} ms")
    x1 = d["c1_x1"]
    loss1, g1 = spst.loss_grad(x1, p)
    print(f"vgg c1 x1: loss rel {abs(loss1 - d['c1_loss64_x1'][0]) / d['c1_loss64_x1'][0]:.3e}  grad relL2 {rel(g1, d['c1_grad64_x1'].astype(np.float64)):.3e}")
    # ragged
    wr = spst.default_loss_weights(spec, lambda_c=float(d["r_lambda_c"][0]))
    pr = spst.build_problem(d["r_u"], d["r_v"], spec, wr)
    lr, gr = spst.loss_grad(d["r_x"], pr)
    print(f"vgg ragged 72x88: loss rel {abs(lr - d['r_loss64'][0]) / d['r_loss64'][0]:.3e} grad relL2 {rel(gr, d['r_grad64']):.3e}")
    # L-BFGS 3 iterations (losses vs reference f32 trajectory)
    x, tr = spst.minimize(spst.pipeline.objective_for(p), torch.from_numpy(u).cuda(), spst.LBFGSConfig(history_size=100, max_iters=3))
    print("lbfgs losses ours", tr.losses, "\n             ref ", d["c1_lbfgs_losses"].tolist(), "evals", tr.evals)


if __name__ == "__main__":
    tiny()
    vgg()
