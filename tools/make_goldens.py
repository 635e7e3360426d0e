"""Generate golden vectors from the REAL reference implementation (build container only).

    PYTHONPATH=/root/reference/pkg/src python tools/make_goldens.py

Writes tests/golden/*.npz. The reference (pure NumPy) is imported read-only; nothing here
runs on the GPU box, which only reads the committed fixtures.  Every fixture records the
inputs, the reference outputs, and for VGG-19 the sha256 of the calibrated weights so the box
can check it regenerates the identical network.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import tilestyle as ts  # noqa: E402
from tilestyle import extractor as rex, lbfgs as rlb, localized as rloc, pipeline as rpipe  # noqa: E402
from tilestyle import stats as rst, tensorops as rto, tiling as rti  # noqa: E402
from tilestyle import metrics as rme  # noqa: E402

from paper_2212_13459_b200 import spec as myspec  # noqa: E402
from paper_2212_13459_b200.workloads import synth_content, synth_style  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
os.makedirs(OUT, exist_ok=True)


def weights_sha(spec) -> str:
    h = hashlib.sha256()
    for l in spec.layers:
        if l.kind == "conv":
            h.update(np.ascontiguousarray(l.weight, dtype=np.float64).tobytes())
            h.update(np.ascontiguousarray(l.bias, dtype=np.float64).tobytes())
    return h.hexdigest()


def to_ref_spec(myspec_obj, ref_base):
    """Bind our calibrated weights into the reference's own unbound spec object."""
    from dataclasses import replace
    layers = []
    mine = {l.name: l for l in myspec_obj.layers}
    for l in ref_base.layers:
        if l.kind == "conv":
            layers.append(replace(l, weight=mine[l.name].weight.copy(), bias=mine[l.name].bias.copy()))
        else:
            layers.append(l)
    return replace(ref_base, layers=tuple(layers))


def save(name, **arrays):
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB)")


def kernels():
    rng = np.random.default_rng(1234)
    d = {}
    x = rng.standard_normal((5, 9, 11))
    w = rng.standard_normal((7, 5, 3, 3))
    b = rng.standard_normal(7)
    g = rng.standard_normal((7, 9, 11))
    d.update(conv_x=x, conv_w=w, conv_b=b, conv_y=rto.conv2d_forward(x, w, b, 1, 1), conv_g=g,
             conv_gx=rto.conv2d_backward_input(g, x.shape, w, 1, 1))
    p = rng.standard_normal((3, 9, 7))
    gp = rng.standard_normal((3, 4, 3))
    d.update(pool_x=p, pool_avg=rto.avgpool_forward(p, 2), pool_max=rto.maxpool_forward(p, 2), pool_g=gp,
             pool_avg_bwd=rto.avgpool_backward(gp, p.shape, 2), pool_max_bwd=rto.maxpool_backward(gp, p, 2))
    img = rng.random((37, 29, 3)).astype(np.float32)
    d.update(img=img, down3=rto.resize_down(img, 3), down8=rto.resize_down(img, 8),
             bil=rto.resize_bilinear(img, (53, 41)), up2=rto.resize_up2(img), up2t=rto.resize_up2(img, (73, 57)))
    padded = rto.pad_to_multiple(img, 16)
    gpad = rng.standard_normal(padded.shape).astype(np.float32)
    d.update(pad16=padded, gpad=gpad, fold=rto.fold_padding_gradient(gpad, img.shape[:2]))
    feats = rng.random((6, 10, 12))
    acc = rst.StatsAccumulator(6)
    acc.accumulate(feats)
    st = acc.finalize()
    ref = rst.compute_stats(rng.random((6, 8, 8)))
    tw = rst.TapWeights(0.3, 20.0, 7.0)
    terms, sg = rst.style_layer_loss_grad(feats, st, ref, tw)
    d.update(st_feats=feats, st_gram=st.gram, st_mean=st.mean, st_std=st.std, ref_gram=ref.gram,
             ref_mean=ref.mean, ref_std=ref.std, tw=np.array([tw.gram, tw.mean, tw.std]),
             sg_terms=np.array(terms), sg_grad=sg)
    save("kernels.npz", **d)


def tiny_cases():
    spec = ts.tinynet(0)
    mine = myspec.tinynet(0)
    diffs = [float(np.abs(a.weight - b.weight).max()) for a, b in zip(spec.layers, mine.layers) if a.kind == "conv"]
    print("tinynet weight max diff (ours vs reference):", max(diffs))
    d = {"tiny_w_" + l.name: l.weight for l in spec.layers if l.kind == "conv"}
    d.update({"tiny_b_" + l.name: l.bias for l in spec.layers if l.kind == "conv"})
    rng = np.random.default_rng(1234)
    cases = [(96, 96, 32, 16), (70, 53, 32, 16), (48, 48, 512, 16)]
    for k, (H, W, block, margin) in enumerate(cases):
        u = rng.random((H, W, 3))
        v = rng.random((H - 10, W + 7, 3)) * 0.6 + 0.2 * np.sin(np.arange(W + 7) / 5.0)[None, :, None]
        x = np.clip(u + 0.1 * rng.standard_normal(u.shape), 0, 1)
        w = rst.default_loss_weights(spec)
        p = rloc.build_problem(u, v, spec, w, block=block, margin=margin)
        lb, gb = rloc.loss_grad(x, p)
        lg, gg = rloc.loss_grad_global(x, p)
        sx = rloc.stats_pass(x, spec, block=block, margin=margin)
        d[f"case{k}_u"], d[f"case{k}_v"], d[f"case{k}_x"] = u, v, x
        d[f"case{k}_geom"] = np.array([block, margin])
        d[f"case{k}_loss"] = np.array([lb, lg])
        d[f"case{k}_grad"], d[f"case{k}_grad_global"] = gb, gg
        for t in spec.style_taps:
            d[f"case{k}_{t}_gram"] = sx[t].gram
            d[f"case{k}_{t}_mean"] = sx[t].mean
            d[f"case{k}_{t}_std"] = sx[t].std
            d[f"case{k}_{t}_n"] = np.array([sx[t].n_p])
            d[f"case{k}_style_{t}_gram"] = p.style_stats[t].gram
            d[f"case{k}_style_{t}_mean"] = p.style_stats[t].mean
            d[f"case{k}_style_{t}_std"] = p.style_stats[t].std
    # an f32 run of case 0 (pipeline dtype)
    u, v, x = (d["case0_u"].astype(np.float32), d["case0_v"].astype(np.float32), d["case0_x"].astype(np.float32))
    p = rloc.build_problem(u, v, spec, rst.default_loss_weights(spec), block=32, margin=16)
    l32, g32 = rloc.loss_grad(x, p)
    d["case0_loss_f32"], d["case0_grad_f32"] = np.array([l32]), g32
    # short L-BFGS trajectory (f32, like the pipeline) on case 0
    losses = []
    xs = []
    xr, tr = rlb.minimize(lambda a: rloc.loss_grad(a, p), x, rlb.LBFGSConfig(history_size=10, max_iters=5),
                          callback=lambda it, xi, l, gn: xs.append(xi.copy()))
    d["case0_lbfgs_losses"] = np.array(tr.losses)
    d["case0_lbfgs_x5"] = xr
    save("tinynet.npz", **d)


def lbfgs_cases():
    d = {}

    def quad(a):
        return lambda x: (float(np.sum((x - a) ** 2)), 2.0 * (x - a))

    def rosen(z):
        x, y = z
        return float((1 - x) ** 2 + 100 * (y - x ** 2) ** 2), np.array(
            [-2 * (1 - x) - 400 * x * (y - x ** 2), 200 * (y - x ** 2)])

    rng = np.random.default_rng(7)
    a = rng.standard_normal(20)
    x, tr = rlb.minimize(quad(a), np.zeros(20), rlb.LBFGSConfig(history_size=5, max_iters=30))
    d.update(quad_a=a, quad_x=x, quad_losses=np.array(tr.losses), quad_gn=np.array(tr.grad_norms))
    x, tr = rlb.minimize(rosen, np.array([-1.2, 1.0]), rlb.LBFGSConfig(history_size=10, max_iters=200))
    d.update(rosen_x=x, rosen_losses=np.array(tr.losses))
    # two-loop on a random admissible state
    st = rlb.LBFGSState()
    ss, ys = [], []
    for _ in range(4):
        s = rng.standard_normal(12)
        y = s + 0.3 * rng.standard_normal(12)
        st.push(s, y, m=3)
        ss.append(s)
        ys.append(y)
    g = rng.standard_normal(12)
    d.update(tl_s=np.array(ss), tl_y=np.array(ys), tl_g=g, tl_d=rlb.two_loop_direction(g, st))
    sched = [rpipe.make_schedule(n, m).iters for n, m in [(4, "fast"), (4, "baseline"), (6, "fast")]]
    d["sched_fast4"], d["sched_base4"], d["sched_fast6"] = [np.array(s) for s in sched]
    d["dims_4"] = np.array(rpipe.scale_dims((6048, 8064), 4))
    d["dims_3_odd"] = np.array(rpipe.scale_dims((1001, 777), 3))
    save("lbfgs_pipeline.npz", **d)


def vgg_cases():
    spec_mine = myspec.calibrated_vgg19(0)
    spec = to_ref_spec(spec_mine, rex.vgg19("avg"))
    d = {"weights_sha256": np.frombuffer(weights_sha(spec_mine).encode(), dtype=np.uint8)}
    print("margin_for_exact_gradient(VGG19) =", rti.margin_for_exact_gradient(spec))
    # C1: 256^2 single-scale transfer (BASELINE configs[0])
    u = synth_content(256, 256, 1)
    v = synth_style(256, 256, 2)
    cfg = rpipe.RunConfig(n_scales=1, extractor=spec)
    w = rpipe._weights_for_scale(cfg, spec, (256, 256))
    d["c1_u"], d["c1_v"], d["c1_lambda_c"] = u, v, np.array([w.lambda_c])
    t0 = time.time()
    p64 = rloc.build_problem(u.astype(np.float64), v.astype(np.float64), spec, w)
    x0 = u.astype(np.float64)
    l64, g64 = rloc.loss_grad_global(x0, p64)
    print(f"VGG f64 loss_grad_global 256^2: {time.time() - t0:.1f}s loss={l64}")
    for t in spec.style_taps:
        d[f"c1_style_{t}_gram"] = p64.style_stats[t].gram.astype(np.float32)
        d[f"c1_style_{t}_mean"] = p64.style_stats[t].mean
        d[f"c1_style_{t}_std"] = p64.style_stats[t].std
    sx = rloc.stats_pass(x0, spec)
    for t in spec.style_taps:
        d[f"c1_x0_{t}_gram"] = sx[t].gram.astype(np.float32)
        d[f"c1_x0_{t}_mean"] = sx[t].mean
        d[f"c1_x0_{t}_std"] = sx[t].std
        d[f"c1_x0_terms_{t}"] = np.array(rst.style_loss_terms(sx[t], p64.style_stats[t], w.style[t]))
    d["c1_loss64"], d["c1_grad64"] = np.array([l64]), g64.astype(np.float32)
    # the reference's own f32 path at the same x (its f32-vs-f64 gap bounds any fp32-class engine)
    p32 = rloc.build_problem(u, v, spec, w)
    l32, g32 = rloc.loss_grad(u.copy(), p32)
    d["c1_loss32"], d["c1_grad32"] = np.array([l32]), g32
    rel = np.linalg.norm(g32 - g64) / np.linalg.norm(g64)
    print(f"reference f32 vs f64 at x0: loss rel {abs(l32 - l64) / abs(l64):.2e}, grad rel-L2 {rel:.2e}")
    # a second point along the steepest-descent direction (first L-BFGS trial point)
    x1 = (u - (1.0 / np.abs(g32).max()) * g32).astype(np.float32)
    l1, g1 = rloc.loss_grad_global(x1.astype(np.float64), p64)
    d["c1_x1"], d["c1_loss64_x1"], d["c1_grad64_x1"] = x1, np.array([l1]), g1.astype(np.float32)
    # first reference f32 L-BFGS iterations (losses; iterates are chaotic beyond ~5)
    t0 = time.time()
    xr, tr = rlb.minimize(lambda a: rloc.loss_grad(a, p32), u.copy(), rlb.LBFGSConfig(history_size=100, max_iters=3))
    print(f"reference 3 L-BFGS iters 256^2 f32: {time.time() - t0:.1f}s losses={tr.losses}")
    d["c1_lbfgs_losses"] = np.array(tr.losses)
    # ragged small VGG case (replicate padding + fold): 72 x 88 -> padded 80 x 96
    rng = np.random.default_rng(5)
    us = synth_content(72, 88, 3)
    vs = synth_style(64, 64, 4)
    xs = np.clip(us + 0.05 * rng.standard_normal(us.shape), 0, 1)
    ws = rpipe._weights_for_scale(cfg, spec, (72, 88))
    ps = rloc.build_problem(us.astype(np.float64), vs.astype(np.float64), spec, ws)
    ls, gs = rloc.loss_grad_global(xs, ps)
    d.update(r_u=us, r_v=vs, r_x=xs, r_lambda_c=np.array([ws.lambda_c]), r_loss64=np.array([ls]), r_grad64=gs)
    save("vgg19.npz", **d)


def metrics_cases():
    """Reference metrics.py: psnr (24-31), ssim (55-73), gram_distance (76-89)."""
    d = {}
    rng = np.random.default_rng(11)
    pairs = {
        "rand": (rng.random((64, 80, 3)), None),
        "min11": (rng.random((11, 11, 3)), None),
        "gray": (rng.random((40, 53)), None),
        "synth": (synth_content(151, 129, 5).astype(np.float64), None),
    }
    for k, (a, _) in pairs.items():
        b = np.clip(a + 0.07 * rng.standard_normal(a.shape), 0.0, 1.0)
        if k == "synth":
            b = synth_style(151, 129, 6).astype(np.float64)
        d[f"{k}_a"], d[f"{k}_b"] = a, b
        d[f"{k}_psnr"] = np.array([rme.psnr(a, b)])
        d[f"{k}_ssim"] = np.array([rme.ssim(a, b)])
    # f32 inputs: the reference weights the luma in f32 (NumPy weak scalars)
    a32 = synth_content(97, 131, 7)
    b32 = np.clip(a32 + 0.05 * rng.standard_normal(a32.shape).astype(np.float32), 0, 1).astype(np.float32)
    d["f32_a"], d["f32_b"] = a32, b32
    d["f32_psnr"], d["f32_ssim"] = np.array([rme.psnr(a32, b32)]), np.array([rme.ssim(a32, b32)])
    a = d["rand_a"]
    d["same_psnr"], d["same_ssim"] = np.array([rme.psnr(a, a)]), np.array([rme.ssim(a, a)])
    # blockwise Gram distance on TinyNet (unweighted and weighted)
    spec = ts.tinynet(0)
    x = rng.random((70, 53, 3))
    v = rng.random((64, 64, 3)) * 0.5 + 0.25
    d["gd_x"], d["gd_v"] = x, v
    d["gd_plain"] = np.array([rme.gram_distance(x, v, spec, block=32, margin=16)])
    w = {t: 1.0 / (i + 1) for i, t in enumerate(spec.style_taps)}
    d["gd_weighted"] = np.array([rme.gram_distance(x, v, spec, block=32, margin=16, weights=w)])
    d["gd_weights"] = np.array([w[t] for t in spec.style_taps])
    save("metrics.npz", **d)


def vgg_lbfgs5():
    """The reference f32 path's first 5 L-BFGS iterations at C1 (final image and losses)."""
    spec_mine = myspec.calibrated_vgg19(0)
    spec = to_ref_spec(spec_mine, rex.vgg19("avg"))
    u = synth_content(256, 256, 1)
    v = synth_style(256, 256, 2)
    cfg = rpipe.RunConfig(n_scales=1, extractor=spec)
    w = rpipe._weights_for_scale(cfg, spec, (256, 256))
    p32 = rloc.build_problem(u, v, spec, w)
    t0 = time.time()
    xr, tr = rlb.minimize(lambda a: rloc.loss_grad(a, p32), u.copy(), rlb.LBFGSConfig(history_size=100, max_iters=5))
    print(f"reference 5 L-BFGS iters 256^2 f32: {time.time() - t0:.1f}s losses={tr.losses}")
    save("vgg19_lbfgs5.npz", x5=xr, losses=np.array(tr.losses))


def vgg_iterates():
    """Fixed same-x points for the gradient error budget: the reference f32 L-BFGS iterates
    x1..x5 at C1 (history 100) and, at each, the reference's own f64 gradient
    (loss_grad_global) and f32 gradient (loss_grad) -- the precision envelope of SURVEY 8(a) a20."""
    spec_mine = myspec.calibrated_vgg19(0)
    spec = to_ref_spec(spec_mine, rex.vgg19("avg"))
    u = synth_content(256, 256, 1)
    v = synth_style(256, 256, 2)
    cfg = rpipe.RunConfig(n_scales=1, extractor=spec)
    w = rpipe._weights_for_scale(cfg, spec, (256, 256))
    p32 = rloc.build_problem(u, v, spec, w)
    p64 = rloc.build_problem(u.astype(np.float64), v.astype(np.float64), spec, w)
    its = []
    rlb.minimize(lambda a: rloc.loss_grad(a, p32), u.copy(), rlb.LBFGSConfig(history_size=100, max_iters=5),
                 callback=lambda it, xi, loss, gn: its.append(np.array(xi, dtype=np.float32, copy=True)))
    d = {}
    for k, xi in enumerate([u] + its):
        l64, g64 = rloc.loss_grad_global(xi.astype(np.float64), p64)
        l32, g32 = rloc.loss_grad(xi.copy(), p32)
        rel = np.linalg.norm(g32 - g64) / np.linalg.norm(g64)
        print(f"iterate {k}: loss64 {l64:.6e}, reference f32 vs f64 grad rel-L2 {rel:.2e}")
        d[f"x{k}"], d[f"loss64_{k}"], d[f"grad64_{k}"] = xi, np.array([l64]), g64.astype(np.float32)
        d[f"loss32_{k}"], d[f"grad32_{k}"] = np.array([l32]), g32.astype(np.float32)
    save("vgg19_iterates.npz", **d)


def pipeline_cases():
    """Reference multiscale_transfer / texture_synthesize (pipeline.py:232-260) on TinyNet:
    2 scales x 3 L-BFGS iterations (history 5), f32 -- short enough that the final image is
    comparable (SURVEY 8d protocol 3)."""
    spec = ts.tinynet(0)
    rng = np.random.default_rng(21)
    u = synth_content(96, 80, 7)
    v = synth_style(64, 72, 8)
    orig = rpipe.make_schedule
    rpipe.make_schedule = lambda n, m="baseline": rpipe.Schedule(n, (3,) * n, (5,) * n, m)
    try:
        cfg = rpipe.RunConfig(n_scales=2, mode="fast", extractor=spec, block=32, margin=16)
        seen = []
        x = rpipe.multiscale_transfer(u, v, cfg, progress=lambda s, it, l, g: seen.append((s, it, l, g)))
        cfg_t = rpipe.RunConfig(n_scales=2, extractor=spec, block=32, margin=16, lambda_c=0.0, seed=3)
        seen_t = []
        xt = rpipe.texture_synthesize(v, cfg_t, progress=lambda s, it, l, g: seen_t.append((s, it, l, g)))
    finally:
        rpipe.make_schedule = orig
    save("pipeline.npz", u=u, v=v, ms_x=x, ms_trace=np.array(seen, dtype=np.float64),
         ts_x=xt, ts_trace=np.array(seen_t, dtype=np.float64))


def pipeline_vgg_cases():
    """The same drivers on the flagship network: calibrated VGG-19, content 128x160 / style
    96x112, f32, history 5.  multiscale_transfer runs 2 scales x 1 iteration, texture_synthesize
    2 scales x 3: with the content term, VGG-19 L-BFGS trajectories of any two fp32-class
    implementations part after a step or two at ReLU near-ties (the reference's own f32 run
    stays within 2.3e-4 of its f64 run here while ours parts at iteration 1; mean |diff| 9e-3
    after 2 x 3 iterations), so the image comparison is made where the protocol's 1/255 bar
    is meaningful."""
    spec = to_ref_spec(myspec.calibrated_vgg19(0), rex.vgg19("avg"))
    u = synth_content(128, 160, 11)
    v = synth_style(96, 112, 12)
    orig = rpipe.make_schedule
    try:
        t0 = time.time()
        rpipe.make_schedule = lambda n, m="baseline": rpipe.Schedule(n, (1,) * n, (5,) * n, m)
        cfg = rpipe.RunConfig(n_scales=2, mode="fast", extractor=spec)
        seen = []
        x = rpipe.multiscale_transfer(u, v, cfg, progress=lambda s, it, l, g: seen.append((s, it, l, g)))
        rpipe.make_schedule = lambda n, m="baseline": rpipe.Schedule(n, (3,) * n, (5,) * n, m)
        cfg_t = rpipe.RunConfig(n_scales=2, extractor=spec, lambda_c=0.0, seed=3)
        seen_t = []
        xt = rpipe.texture_synthesize(v, cfg_t, progress=lambda s, it, l, g: seen_t.append((s, it, l, g)))
        print(f"VGG pipeline goldens: {time.time() - t0:.1f}s")
    finally:
        rpipe.make_schedule = orig
    save("pipeline_vgg.npz", u=u, v=v, ms_x=x, ms_trace=np.array(seen, dtype=np.float64),
         ts_x=xt, ts_trace=np.array(seen_t, dtype=np.float64))


def api_cases():
    """Per-tap public helpers: forward_taps (extractor.py:171-197), style_layer_loss_grad and
    content_loss_grad (stats.py:127-174) on TinyNet and the calibrated VGG-19."""
    rng = np.random.default_rng(31)
    d = {}
    tiny = ts.tinynet(0)
    xt = rng.random((3, 64, 48)).astype(np.float32)
    taps = rex.forward_taps(xt, tiny)
    d["tiny_x"] = xt
    for t, v in taps.items():
        d[f"tiny_tap_{t}"] = v
    spec = to_ref_spec(myspec.calibrated_vgg19(0), rex.vgg19("avg"))
    xv = synth_content(64, 80, 9).transpose(2, 0, 1).copy()
    tv = rex.forward_taps(xv, spec)
    d["vgg_x"] = xv
    for t, v in tv.items():
        d[f"vgg_tap_{t}"] = v
    # style_layer_loss_grad on a slab of a tap with the image's global stats vs another image's
    V = tv["relu3_1"]
    acc = rst.StatsAccumulator(V.shape[0])
    acc.accumulate(V)
    sx = acc.finalize()
    tv2 = rex.forward_taps(synth_style(64, 80, 10).transpose(2, 0, 1).copy(), spec)
    acc2 = rst.StatsAccumulator(V.shape[0])
    acc2.accumulate(tv2["relu3_1"])
    sr = acc2.finalize()
    w = rst.TapWeights(1.0 / 256 ** 2, 1e3 / 256 ** 2, 1e3 / 256 ** 2)
    slab = V[:, 3:11, 5:17].copy()
    terms, g = rst.style_layer_loss_grad(slab, sx, sr, w)
    d.update(sg_slab=slab, sg_G=sx.gram, sg_mu=sx.mean, sg_sd=sx.std, sg_n=np.array([sx.n_p]),
             sg_Gr=sr.gram, sg_mur=sr.mean, sg_sdr=sr.std, sg_w=np.array([w.gram, w.mean, w.std]),
             sg_terms=np.array(terms), sg_grad=g)
    # degenerate channel: std 0 with a nonzero reference std -> zero std column + warning
    sd0 = sx.std.copy()
    sd0[7] = 0.0
    sxd = rst.LayerStats(gram=sx.gram, mean=sx.mean, std=sd0, n_p=sx.n_p)
    import warnings as _w
    with _w.catch_warnings(record=True) as rec:
        _w.simplefilter("always")
        termsd, gd = rst.style_layer_loss_grad(slab.astype(np.float64), sxd, sr, w)
    d.update(sgd_sd=sd0, sgd_terms=np.array(termsd), sgd_grad=gd, sgd_warned=np.array([len(rec)]))
    # content_loss_grad
    Vr = tv2["relu4_2"]
    Vx = tv["relu4_2"]
    cl, cg = rst.content_loss_grad(Vx, Vr, 0.37)
    d.update(cl_V=Vx, cl_Vr=Vr, cl_loss=np.array([cl]), cl_grad=cg)
    save("api.npz", **d)


def block_cases():
    """Reference Algorithm 1 on block grids whose margin is BELOW the exact margin (the result
    then depends on the grid: reference test_localized.py:72-78), plus stats_pass at non-style
    relu taps (localized.py:162-184 with taps=...)."""
    d = {}
    tiny = ts.tinynet(0)
    rng = np.random.default_rng(41)
    u = rng.random((150, 137, 3))
    v = rng.random((96, 80, 3)) * 0.6 + 0.2
    x = np.clip(u + 0.1 * rng.standard_normal(u.shape), 0, 1)
    w = rst.default_loss_weights(tiny)
    for m in (0, 8):
        p = rloc.build_problem(u, v, tiny, w, block=64, margin=m)
        l, g = rloc.loss_grad(x, p)
        d[f"tiny_m{m}_loss"], d[f"tiny_m{m}_grad"] = np.array([l]), g
        st = rloc.stats_pass(x, tiny, block=64, margin=m)
        for t in tiny.style_taps:
            d[f"tiny_m{m}_{t}_gram"], d[f"tiny_m{m}_{t}_mean"] = st[t].gram, st[t].mean
    lg, gg = rloc.loss_grad_global(x, rloc.build_problem(u, v, tiny, w, block=64, margin=0))
    d["tiny_global_loss"], d["tiny_global_grad"] = np.array([lg]), gg
    d.update(tiny_u=u, tiny_v=v, tiny_x=x)
    st = rloc.stats_pass(x, tiny, block=64, margin=16, taps=("relu1", "relu3"))
    for t in ("relu1", "relu3"):
        d[f"tiny_taps_{t}_gram"], d[f"tiny_taps_{t}_std"] = st[t].gram, st[t].std
    spec = to_ref_spec(myspec.calibrated_vgg19(0), rex.vgg19("avg"))
    uv = synth_content(96, 112, 12)
    vv = synth_style(80, 80, 13)
    xv = np.clip(uv + 0.05 * rng.standard_normal(uv.shape), 0, 1).astype(np.float32)
    wv = rpipe._weights_for_scale(rpipe.RunConfig(n_scales=1, extractor=spec), spec, (96, 112))
    p = rloc.build_problem(uv, vv, spec, wv, block=48, margin=16)
    l, g = rloc.loss_grad(xv, p)
    d.update(vgg_u=uv, vgg_v=vv, vgg_x=xv, vgg_lambda_c=np.array([wv.lambda_c]), vgg_m16_loss=np.array([l]),
             vgg_m16_grad=g)
    st = rloc.stats_pass(xv, spec, block=512, margin=256, taps=("relu4_2", "relu1_1"))
    for t in ("relu4_2", "relu1_1"):
        d[f"vgg_taps_{t}_gram"], d[f"vgg_taps_{t}_mean"], d[f"vgg_taps_{t}_std"] = st[t].gram, st[t].mean, st[t].std
    save("blocks.npz", **d)


def maxpool_cases():
    """vgg19(pooling="max") (extractor.py:321) and a max-pool TinyNet through the reference
    Algorithm 1 (first-argmax ties, tensorops.py:113-129): f64 and f32 loss / gradient."""
    from dataclasses import replace as _rep
    d = {}
    rng = np.random.default_rng(51)
    tiny = ts.tinynet(0)
    tiny = _rep(tiny, layers=tuple(_rep(l, pool="max") if l.kind == "pool" else l for l in tiny.layers))
    u, v = rng.random((64, 80, 3)), rng.random((48, 48, 3))
    x = np.clip(u + 0.1 * rng.standard_normal(u.shape), 0, 1)
    w = rst.default_loss_weights(tiny)
    p = rloc.build_problem(u, v, tiny, w, block=512, margin=16)
    l, g = rloc.loss_grad_global(x, p)
    d.update(tiny_u=u, tiny_v=v, tiny_x=x, tiny_loss=np.array([l]), tiny_grad=g)
    spec = to_ref_spec(myspec.calibrated_vgg19(0), rex.vgg19("max"))
    uv, vv = synth_content(160, 192, 14), synth_style(128, 128, 15)
    wv = rpipe._weights_for_scale(rpipe.RunConfig(n_scales=1, extractor=spec), spec, (160, 192))
    p64 = rloc.build_problem(uv.astype(np.float64), vv.astype(np.float64), spec, wv)
    p32 = rloc.build_problem(uv, vv, spec, wv)
    d.update(vgg_u=uv, vgg_v=vv, vgg_lambda_c=np.array([wv.lambda_c]))
    for t in spec.style_taps:
        d[f"vgg_style_{t}_gram"] = p64.style_stats[t].gram
    xs = [uv, np.clip(uv + 0.03 * rng.standard_normal(uv.shape), 0, 1).astype(np.float32)]
    for k, xk in enumerate(xs):
        l64, g64 = rloc.loss_grad_global(xk.astype(np.float64), p64)
        l32, g32 = rloc.loss_grad(xk.copy(), p32)
        print(f"max-pool VGG point {k}: reference f32 vs f64 grad rel-L2 "
              f"{np.linalg.norm(g32 - g64) / np.linalg.norm(g64):.2e}")
        d.update({f"vgg_x{k}": xk, f"vgg_loss64_{k}": np.array([l64]), f"vgg_grad64_{k}": g64.astype(np.float32),
                  f"vgg_grad32_{k}": g32})
    save("maxpool.npz", **d)


if __name__ == "__main__":
    which = sys.argv[1:] or ["kernels", "tiny", "lbfgs", "vgg", "metrics", "lbfgs5", "iterates", "pipeline", "pipeline_vgg", "api", "blocks", "maxpool"]
    if "maxpool" in which:
        maxpool_cases()
    if "blocks" in which:
        block_cases()
    if "api" in which:
        api_cases()
    if "iterates" in which:
        vgg_iterates()
    if "pipeline" in which:
        pipeline_cases()
    if "pipeline_vgg" in which:
        pipeline_vgg_cases()
    if "metrics" in which:
        metrics_cases()
    if "lbfgs5" in which:
        vgg_lbfgs5()
    if "kernels" in which:
        kernels()
    if "tiny" in which:
        tiny_cases()
    if "lbfgs" in which:
        lbfgs_cases()
    if "vgg" in which:
        vgg_cases()
