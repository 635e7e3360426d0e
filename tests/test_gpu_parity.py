"""Parity of the device hot path with the reference (golden vectors) and the oracle.

Tolerances (north_star): per-layer Gram and loss within 1e-3 relative; image gradient within
1e-3 relative L2 vs the f64 path at the same x.  Where a ReLU-mask flip makes the reference's
OWN f32 path miss 1e-3 against f64 (a discontinuity of the gradient, SURVEY.md §0 finding 2),
the bar is max(1e-3, 1.5 x the reference-f32 gap at that x); the VGG tests assert exactly
that, plus fp32-class arithmetic on our own ReLU pattern, and write their per-point tables to
profiles/.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import spst_oracle as O  # noqa: E402
import paper_2212_13459_b200 as spst  # noqa: E402
from paper_2212_13459_b200.pipeline import objective_for  # noqa: E402
from conftest import golden, rel_l2  # noqa: E402


# ---------------------------------------------------------------- TinyNet (reference test net)
@pytest.mark.parametrize("k", [0, 1, 2])
def test_tinynet_loss_grad_stats_vs_reference(tiny_spec, k):
    d = golden("tinynet.npz")
    u, v, x = d[f"case{k}_u"], d[f"case{k}_v"], d[f"case{k}_x"]
    block, margin = (int(a) for a in d[f"case{k}_geom"])
    p = spst.build_problem(u, v, tiny_spec, spst.default_loss_weights(tiny_spec), block=block, margin=margin)
    for t in tiny_spec.style_taps:
        assert rel_l2(p.style_stats[t].gram, d[f"case{k}_style_{t}_gram"]) <= 1e-5
    loss, g = spst.loss_grad(x, p)
    assert g.dtype == x.dtype and g.shape == x.shape
    assert abs(loss - d[f"case{k}_loss"][1]) <= 1e-5 * abs(d[f"case{k}_loss"][1])
    assert rel_l2(g, d[f"case{k}_grad"]) <= 1e-5          # blockwise reference == global
    lg, gg = spst.loss_grad_global(x, p)
    assert rel_l2(gg, d[f"case{k}_grad_global"]) <= 1e-5
    st = spst.stats_pass(x, tiny_spec, block=block, margin=margin)
    for t in tiny_spec.style_taps:
        assert st[t].n_p == int(d[f"case{k}_{t}_n"][0])
        assert rel_l2(st[t].gram, d[f"case{k}_{t}_gram"]) <= 1e-5
        assert rel_l2(st[t].mean, d[f"case{k}_{t}_mean"]) <= 1e-5
        assert rel_l2(st[t].std, d[f"case{k}_{t}_std"]) <= 1e-5


def test_tinynet_identity_problem_has_zero_loss(tiny_spec):
    """Reference test_localized.py:47-53: content = style = x gives loss 0 and zero gradient
    (here: up to fp32-class rounding of the statistics)."""
    v = np.random.default_rng(1).random((64, 64, 3))
    p = spst.build_problem(v, v, tiny_spec, spst.default_loss_weights(tiny_spec), block=64, margin=16)
    loss, g = spst.loss_grad(v, p)
    p2 = spst.build_problem(v, np.random.default_rng(2).random((64, 64, 3)), tiny_spec,
                            spst.default_loss_weights(tiny_spec), block=64, margin=16)
    l2, g2 = spst.loss_grad(v, p2)
    assert loss <= 1e-9 * l2
    assert np.abs(g).max() <= 1e-5 * np.abs(g2).max()


def test_tinynet_style_only_and_errors(tiny_spec):
    rng = np.random.default_rng(4)
    u, v, x = (rng.random((64, 80, 3)) for _ in range(3))
    w0 = spst.LossWeights(0.0, dict(spst.default_loss_weights(tiny_spec).style))
    p = spst.build_problem(None, v, tiny_spec, w0, block=64, margin=16)
    net = O.onet_from_spec(tiny_spec)
    po = O.build_problem(None, v, net, (0.0, O.default_weights(net)[1]), 64, 16)
    lo, go = O.loss_grad_global(x[:, :80][:64], po) if False else O.loss_grad_global(v, po)
    loss, g = spst.loss_grad(v, p)
    assert abs(loss - lo) <= 1e-5 * abs(lo) + 1e-12
    with pytest.raises(spst.ConfigError):
        spst.build_problem(None, v, tiny_spec, spst.default_loss_weights(tiny_spec), block=64, margin=16)
    pc = spst.build_problem(u, v, tiny_spec, spst.default_loss_weights(tiny_spec), block=64, margin=16)
    with pytest.raises(spst.ConfigError):
        spst.loss_grad(rng.random((128, 128, 3)), pc)


def test_tinynet_fd_directional(tiny_spec):
    """Reference test_localized.py:90-98: the gradient's directional derivative matches central
    differences of the (f64) reference loss, eps = 1e-5."""
    rng = np.random.default_rng(9)
    u, v, x = (rng.random((64, 64, 3)) for _ in range(3))
    p = spst.build_problem(u, v, tiny_spec, spst.default_loss_weights(tiny_spec), block=64, margin=16)
    loss, g = spst.loss_grad(x, p)
    net = O.onet_from_spec(tiny_spec)
    po = O.build_problem(u, v, net, O.default_weights(net), 64, 16)
    for _ in range(3):
        d = rng.standard_normal(x.shape)
        d /= np.linalg.norm(d)
        eps = 1e-5
        num = (O.loss_grad_global(x + eps * d, po)[0] - O.loss_grad_global(x - eps * d, po)[0]) / (2 * eps)
        assert abs(float(np.vdot(g, d)) - num) <= 1e-5 * abs(num)


def test_threads_and_repeat_bit_identical(tiny_spec):
    """Reference test_localized.py:118-125 (threads=1 vs 4 bit-identical): the device path uses
    fixed-order reductions, so repeated evaluations are bit-identical."""
    rng = np.random.default_rng(5)
    u, v, x = (rng.random((96, 96, 3)).astype(np.float32) for _ in range(3))
    p1 = spst.build_problem(u, v, tiny_spec, spst.default_loss_weights(tiny_spec), block=64, margin=16, threads=1)
    l1, g1 = spst.loss_grad(x, p1)
    p4 = spst.build_problem(u, v, tiny_spec, spst.default_loss_weights(tiny_spec), block=64, margin=16, threads=4)
    l4, g4 = spst.loss_grad(x, p4)
    assert l1 == l4
    np.testing.assert_array_equal(g1, g4)


# ---------------------------------------------------------------- VGG-19 (the benchmark network)
@pytest.fixture(scope="module")
def vgg_c1(vgg_spec):
    d = golden("vgg19.npz")
    w = spst.default_loss_weights(vgg_spec, lambda_c=float(d["c1_lambda_c"][0]))
    p = spst.build_problem(d["c1_u"], d["c1_v"], vgg_spec, w)
    return d, p


def test_vgg19_style_stats_vs_reference(vgg_spec, vgg_c1):
    d, p = vgg_c1
    for t in vgg_spec.style_taps:
        assert rel_l2(p.style_stats[t].gram, d[f"c1_style_{t}_gram"]) <= 1e-4
        assert rel_l2(p.style_stats[t].mean, d[f"c1_style_{t}_mean"]) <= 1e-4
        assert rel_l2(p.style_stats[t].std, d[f"c1_style_{t}_std"]) <= 1e-4
    st = spst.stats_pass(d["c1_u"], vgg_spec)
    for t in vgg_spec.style_taps:
        assert rel_l2(st[t].gram, d[f"c1_x0_{t}_gram"]) <= 1e-4


def _table_out(name, rows):
    """Per-point parity table -> profiles/ (and gpurun_out/ when present, to bring it back)."""
    import json
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for d in ("profiles", "gpurun_out"):
        path = os.path.join(root, d)
        if os.path.isdir(path):
            with open(os.path.join(path, name), "w") as f:
                json.dump(rows, f, indent=1)


def test_vgg19_same_x_gradient_north_star_bar(vgg_spec, vgg_c1):
    """North-star gradient bar at the reference's own C1 points: x0 = u and its f32 L-BFGS
    iterates x1..x5 (tests/golden/vgg19_iterates.npz, real reference f64 and f32 gradients).

    * loss within 1e-5 of f64 (north star: 1e-3);
    * plain image gradient vs f64 within max(1e-3, 1.5 x the reference f32-vs-f64 gap at that x);
    * arithmetic (f64 network evaluated on OUR ReLU pattern) within 5e-6 -- fp32-class;
    * every unit whose ReLU sign differs from f64 is a near-tie, |pre| <= 1e-5 rms.
    """
    d, p = vgg_c1
    it = golden("vgg19_iterates.npz")
    net = O.onet_from_spec(vgg_spec)
    lam = float(d["c1_lambda_c"][0])
    po = O.build_problem(d["c1_u"].astype(np.float64), d["c1_v"].astype(np.float64), net,
                         O.default_weights(net, lam), 512, 256)
    rows = []
    for k in range(6):
        x = it[f"x{k}"]
        loss, g = spst.loss_grad(x, p)
        g64, g32 = it[f"grad64_{k}"], it[f"grad32_{k}"]
        l64 = float(it[f"loss64_{k}"][0])
        masks = p.engine.relu_masks()
        dead = _degenerate_sets(p, vgg_spec, po, x)
        _, gm = O.loss_grad_global(x.astype(np.float64), po, masks=masks)
        flips, tie = _flips(masks, _f64_preacts(po, x))
        row = dict(point=k, loss_rel=abs(loss - l64) / l64, plain=rel_l2(g, g64), ref_f32_gap=rel_l2(g32, g64),
                   arith=rel_l2(g, gm), flips=flips, flip_max_pre_over_rms=tie, degenerate=dead)
        row["bar"] = max(1e-3, 1.5 * row["ref_f32_gap"])
        rows.append(row)
        print(f"x{k}: loss rel {row['loss_rel']:.1e}; grad vs f64 {row['plain']:.2e} (bar {row['bar']:.2e}, "
              f"reference f32 {row['ref_f32_gap']:.2e}); arithmetic {row['arith']:.2e}; flips {flips} "
              f"(max |pre|/rms {tie:.1e})")
    _table_out("parity_c1_iterates.json", rows)
    for r in rows:
        assert r["loss_rel"] <= 1e-5, r
        assert r["arith"] <= 5e-6, r
        assert r["flip_max_pre_over_rms"] <= 1e-5, r
        assert r["plain"] <= r["bar"], r
        # the degenerate-std channel sets (stats.py:158-162) are the oracle's, tap by tap
        for t, (ours, ref) in r["degenerate"].items():
            assert ours == ref, (r["point"], t, ours, ref)


def _degenerate_sets(p, spec, po, x):
    """{tap: (our channels with std < 1e-8, the f64 oracle's)} at the last forward / at x."""
    eng = p.engine
    xp = O.pad_edge16(x.astype(np.float64), po.net.deepest_stride())
    taps, _ = O.run_forward(np.ascontiguousarray(xp.transpose(2, 0, 1)), po.net)
    out = {}
    for i, t in enumerate(eng.style_taps):
        S, sv = eng.tap_sums(i)
        ours = spst.stats.finalize_sums(S.cpu().numpy(), sv.cpu().numpy(), eng.owned_pixels(i)).std
        ref = O.stats_of(taps[t]).std
        out[t] = (sorted(np.flatnonzero(ours < 1e-8).tolist()), sorted(np.flatnonzero(ref < 1e-8).tolist()))
    return out


def test_vgg19_loss_grad_vs_reference_f64(vgg_c1):
    """x0 and the steepest-descent trial point x1 of vgg19.npz (reference f64 loss_grad_global)."""
    d, p = vgg_c1
    loss, g = spst.loss_grad(d["c1_u"], p)
    assert abs(loss - d["c1_loss64"][0]) <= 1e-5 * d["c1_loss64"][0]
    gap32 = rel_l2(d["c1_grad32"], d["c1_grad64"])
    assert rel_l2(g, d["c1_grad64"]) <= max(1e-3, 1.5 * gap32)
    loss1, g1 = spst.loss_grad(d["c1_x1"], p)
    assert abs(loss1 - d["c1_loss64_x1"][0]) <= 1e-5 * d["c1_loss64_x1"][0]
    err1 = rel_l2(g1, d["c1_grad64_x1"])
    print(f"x0: grad vs f64 {rel_l2(g, d['c1_grad64']):.2e} (reference f32 {gap32:.2e}); x1: {err1:.2e}")
    assert err1 <= 1e-3


def test_vgg19_ragged_dims_vs_reference_f64(vgg_spec):
    d = golden("vgg19.npz")
    w = spst.default_loss_weights(vgg_spec, lambda_c=float(d["r_lambda_c"][0]))
    p = spst.build_problem(d["r_u"], d["r_v"], vgg_spec, w)
    loss, g = spst.loss_grad(d["r_x"], p)
    assert g.shape == (72, 88, 3)
    assert abs(loss - d["r_loss64"][0]) <= 1e-5 * d["r_loss64"][0]
    # replicate padding + fold on ragged dims; arithmetic on our ReLU pattern, flips near-ties
    net = O.onet_from_spec(vgg_spec)
    po = O.build_problem(d["r_u"].astype(np.float64), d["r_v"].astype(np.float64), net,
                         O.default_weights(net, float(d["r_lambda_c"][0])), 512, 256)
    masks = p.engine.relu_masks()
    _, gm = O.loss_grad_global(d["r_x"].astype(np.float64), po, masks=masks)
    flips, tie = _flips(masks, _f64_preacts(po, d["r_x"]))
    err, arith = rel_l2(g, d["r_grad64"]), rel_l2(g, gm)
    print(f"ragged: grad rel-L2 vs f64 {err:.2e}; vs f64-on-our-masks {arith:.2e}; ReLU flips {flips} "
          f"(max |pre|/rms {tie:.1e})")
    assert arith <= 5e-6
    assert tie <= 1e-5
    assert err <= 1e-3


def test_vgg19_lbfgs_same_x_first_five_iterates(vgg_spec, vgg_c1):
    """Run OUR L-BFGS 5 iterations; at each of our iterates evaluate the f64 oracle (and the
    oracle's f32 path for the precision envelope) and compare gradients and losses.

    Our iterates are not the reference's, so the oracle-f32 envelope at a given iterate is a
    single draw of which near-tie ReLU units an f32 path happens to flip.  An iterate may
    therefore exceed max(1e-3, 1.5 x that gap) only when the excess is entirely due to flips
    of units within 1e-6 x rms of zero -- decisions below fp32 resolution -- with the
    arithmetic on our own ReLU pattern still within 5e-6.  (The reference's own iterates in
    test_vgg19_same_x_gradient_north_star_bar get the bar with no such exception.)"""
    d, p = vgg_c1
    iterates = []
    x0 = torch.from_numpy(d["c1_u"]).cuda()
    x, tr = spst.minimize(objective_for(p), x0, spst.LBFGSConfig(history_size=100, max_iters=5),
                          callback=lambda it, xi, l, gn: iterates.append(xi.cpu().numpy().copy()))
    np.testing.assert_allclose(tr.losses[:4], d["c1_lbfgs_losses"], rtol=2e-3)
    net = O.onet_from_spec(vgg_spec)
    lam = float(d["c1_lambda_c"][0])
    po = O.build_problem(d["c1_u"].astype(np.float64), d["c1_v"].astype(np.float64), net,
                         O.default_weights(net, lam), 512, 256)
    po32 = O.build_problem(d["c1_u"], d["c1_v"], net, O.default_weights(net, lam), 512, 256)
    rows = []
    for it, xi in enumerate(iterates, start=1):
        lo, go = O.loss_grad_global(xi.astype(np.float64), po)
        _, g32 = O.loss_grad_global(xi, po32)
        loss, g = spst.loss_grad(xi, p)
        masks = p.engine.relu_masks()
        lm, gm = O.loss_grad_global(xi.astype(np.float64), po, masks=masks)
        flips, tie = _flips(masks, _f64_preacts(po, xi))
        err, gap, arith = rel_l2(g, go), rel_l2(g32, go), rel_l2(g, gm)
        rows.append(dict(iterate=it, loss_rel=abs(loss - lo) / lo, plain=err, oracle_f32_gap=gap, arith=arith,
                         flips=flips, flip_max_pre_over_rms=tie, bar=max(1e-3, 1.5 * gap)))
        print(f"iterate {it}: loss rel {abs(loss - lo) / lo:.2e}, grad rel-L2 vs f64 {err:.2e} "
              f"(oracle-f32 {gap:.2e}); vs f64-on-our-masks {arith:.2e}; ReLU flips {flips} "
              f"(max |pre|/rms {tie:.1e})")
    _table_out("parity_c1_own_iterates.json", rows)
    for r in rows:
        assert r["loss_rel"] <= 1e-5, r
        assert r["arith"] <= 5e-6, r
        assert r["flip_max_pre_over_rms"] <= 1e-5, r
        assert r["plain"] <= r["bar"] or r["flip_max_pre_over_rms"] <= 1e-6, r


def _flips(masks, pre):
    """(number of units whose ReLU sign differs from f64, max |pre_f64| / rms(pre) over them)."""
    n, worst = 0, 0.0
    for name, m in masks.items():
        pf = pre[name]
        h, w = min(m.shape[1], pf.shape[1]), min(m.shape[2], pf.shape[2])
        diff = m[:, :h, :w] != (pf[:, :h, :w] > 0)
        if diff.any():
            rms = float(np.sqrt(np.mean(pf[:, :h, :w] ** 2)))
            n += int(diff.sum())
            worst = max(worst, float(np.abs(pf[:, :h, :w][diff]).max()) / rms)
    return n, worst


def _f64_preacts(po, xi):
    """f64 pre-activations of every ReLU at x (for counting mask flips)."""
    net = po.net
    xp = O.pad_edge16(xi.astype(np.float64), net.deepest_stride())
    _, saved = O.run_forward(np.ascontiguousarray(xp.transpose(2, 0, 1)), net, keep=True)
    return {l.name: saved[i] for i, l in enumerate(net.layers[:net.last() + 1]) if l.kind == "relu"}


# ---------------------------------------------------------------- L-BFGS semantics on device
def test_two_loop_matches_reference():
    d = golden("lbfgs_pipeline.npz")
    st = spst.LBFGSState()
    for s, y in zip(d["tl_s"], d["tl_y"]):
        st.push(s, y, 3)
    assert len(st.s_hist) == 3
    np.testing.assert_allclose(spst.two_loop_direction(d["tl_g"], st), d["tl_d"], rtol=1e-12)
    g = np.random.default_rng(0).standard_normal(12)
    np.testing.assert_allclose(spst.two_loop_direction(g, spst.LBFGSState()), -g)
    e1 = np.zeros(3)
    e1[0] = 1
    s1 = spst.LBFGSState()
    assert s1.push(e1, e1, 5)
    np.testing.assert_allclose(spst.two_loop_direction(e1, s1), -e1)
    s2 = spst.LBFGSState()
    assert not s2.push(np.array([1.0, 0]), np.array([0.0, 1.0]), 5)  # curvature rejection


def test_minimize_reference_trajectories():
    d = golden("lbfgs_pipeline.npz")
    a = d["quad_a"]
    x, tr = spst.minimize(lambda z: (float(np.sum((z - a) ** 2)), 2.0 * (z - a)), np.zeros(20),
                          spst.LBFGSConfig(history_size=5, max_iters=30))
    np.testing.assert_allclose(x, d["quad_x"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(tr.losses, d["quad_losses"], rtol=1e-8, atol=1e-20)

    def rosen(z):
        x0, y0 = z
        return float((1 - x0) ** 2 + 100 * (y0 - x0 ** 2) ** 2), np.array(
            [-2 * (1 - x0) - 400 * x0 * (y0 - x0 ** 2), 200 * (y0 - x0 ** 2)])

    x, tr = spst.minimize(rosen, np.array([-1.2, 1.0]), spst.LBFGSConfig(history_size=10, max_iters=200))
    assert np.abs(x - 1.0).max() <= 1e-8
    assert all(b <= a_ for a_, b in zip(tr.losses, tr.losses[1:]))  # monotone trace


def test_minimize_nonfinite_keeps_last_x():
    """Reference test_lbfgs.py:114-121: NaN loss raises NonFiniteError carrying the last
    finite iterate."""
    c = np.array([1.0, 3.0, 10.0, 0.5])
    calls = []

    def f(z):
        calls.append(1)
        if len(calls) > 4:
            return float("nan"), np.zeros_like(z)
        return float(np.sum(c * z ** 2)), 2 * c * z

    with pytest.raises(spst.NonFiniteError) as ei:
        spst.minimize(f, np.ones(4), spst.LBFGSConfig(max_iters=10))
    assert ei.value.x is not None and np.all(np.isfinite(ei.value.x))


def test_first_step_scaled_by_inf_norm():
    seen = []

    def f(z):
        seen.append(np.array(z))
        return float(0.5 * np.sum(z ** 2)), z.copy()

    spst.minimize(f, np.array([0.0, 8.0]), spst.LBFGSConfig(max_iters=1))
    np.testing.assert_allclose(seen[1], [0.0, 8.0] - (1 / 8) * np.array([0.0, 8.0]))


# ---------------------------------------------------------------- driver
def test_multiscale_transfer_small(tiny_spec):
    rng = np.random.default_rng(11)
    u = rng.random((96, 80, 3)).astype(np.float32)
    v = rng.random((64, 64, 3)).astype(np.float32)
    seen = []
    cfg = spst.RunConfig(n_scales=2, mode="fast", extractor=tiny_spec, block=64, margin=16)
    from dataclasses import replace
    import paper_2212_13459_b200.pipeline as pl
    sched = pl.make_schedule
    pl.make_schedule = lambda n, m="baseline": pl.Schedule(n, (4,) * n, (5,) * n, m)
    try:
        x = spst.multiscale_transfer(u, v, cfg, progress=lambda s, it, l, g: seen.append((s, it, l)))
    finally:
        pl.make_schedule = sched
    assert x.shape == u.shape and x.dtype == np.float32
    for s in (1, 2):
        ls = [l for (ss, it, l) in seen if ss == s]
        assert len(ls) == 4 and all(b <= a for a, b in zip(ls, ls[1:]))


def test_texture_synthesis_deterministic(tiny_spec):
    import paper_2212_13459_b200.pipeline as pl
    v = np.random.default_rng(2).random((64, 64, 3)).astype(np.float32)
    cfg = spst.RunConfig(n_scales=1, extractor=tiny_spec, block=64, margin=16, lambda_c=0.0, seed=3)
    sched = pl.make_schedule
    pl.make_schedule = lambda n, m="baseline": pl.Schedule(n, (3,) * n, (5,) * n, m)
    try:
        a = spst.texture_synthesize(v, cfg)
        b = spst.texture_synthesize(v, cfg)
    finally:
        pl.make_schedule = sched
    np.testing.assert_array_equal(a, b)


# ---------------------------------------------------------------- final image after 5 iterations
# SURVEY.md §8(d) parity protocol (3): on <= 5-iteration runs the final image matches the
# reference's to a mean absolute difference of at most 1/255.
def test_tinynet_five_iterations_final_image(tiny_spec):
    d = golden("tinynet.npz")
    u, v, x = (d[f"case0_{k}"].astype(np.float32) for k in ("u", "v", "x"))
    p = spst.build_problem(u, v, tiny_spec, spst.default_loss_weights(tiny_spec), block=32, margin=16)
    x5, tr = spst.minimize(objective_for(p), torch.from_numpy(x).cuda(), spst.LBFGSConfig(history_size=10, max_iters=5))
    x5 = x5.cpu().numpy() if isinstance(x5, torch.Tensor) else x5
    np.testing.assert_allclose(tr.losses, d["case0_lbfgs_losses"], rtol=1e-4)
    assert float(np.mean(np.abs(x5 - d["case0_lbfgs_x5"]))) <= 1.0 / 255


def test_vgg19_five_iterations_final_image(vgg_c1):
    d, p = vgg_c1
    ref = golden("vgg19_lbfgs5.npz")
    x5, tr = spst.minimize(objective_for(p), torch.from_numpy(d["c1_u"]).cuda(),
                           spst.LBFGSConfig(history_size=100, max_iters=5))
    x5 = x5.cpu().numpy() if isinstance(x5, torch.Tensor) else x5
    np.testing.assert_allclose(tr.losses, ref["losses"], rtol=2e-3)
    mad = float(np.mean(np.abs(x5 - ref["x5"])))
    print(f"VGG C1 5 iterations: final-image mean |diff| {mad:.2e} (bar {1 / 255:.2e})")
    assert mad <= 1.0 / 255


def test_device_nonfinite_keeps_last_x(tiny_spec):
    """Reference lbfgs.py:92-96 on the DEVICE objective: an evaluation whose activation range
    cannot be represented (here: an Inf pixel in the trial point) fails inside the native
    forward with SPST_ERR_NONFINITE; minimize re-raises NonFiniteError carrying the last
    finite iterate."""
    rng = np.random.default_rng(3)
    u, v = (rng.random((48, 48, 3)).astype(np.float32) for _ in range(2))
    p = spst.build_problem(u, v, tiny_spec, spst.default_loss_weights(tiny_spec), block=64, margin=16)
    base = objective_for(p)
    calls = []

    class Poisoned:
        lazy = True

        def loss(self, x_dev):
            calls.append(1)
            if len(calls) == 4:
                x_dev = x_dev.clone()
                x_dev[5, 7, 1] = float("inf")
            return base.loss(x_dev)

        def grad(self, out):
            return base.grad(out)

    with pytest.raises(spst.NonFiniteError) as ei:
        spst.minimize(Poisoned(), torch.from_numpy(u).cuda(), spst.LBFGSConfig(max_iters=10))
    x = ei.value.x
    assert x is not None and bool(torch.isfinite(torch.as_tensor(x)).all())
    # the engine is usable afterwards
    loss, g = spst.loss_grad(u, p)
    assert np.isfinite(loss) and np.isfinite(g).all()
