"""Pin the CPU oracle (oracle/spst_oracle.py) to the reference's own outputs.

The golden vectors in tests/golden were produced by running the real reference package
(tools/make_goldens.py); these tests never need a GPU."""

import numpy as np
import pytest

import spst_oracle as O
from conftest import golden, rel_l2


def test_dense_kernels_match_reference():
    d = golden("kernels.npz")
    np.testing.assert_allclose(O.conv3x3(d["conv_x"], d["conv_w"], d["conv_b"]), d["conv_y"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(O.conv3x3_input_grad(d["conv_g"], d["conv_w"]), d["conv_gx"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(O.pool2_fwd(d["pool_x"], "avg"), d["pool_avg"], rtol=1e-14)
    np.testing.assert_allclose(O.pool2_fwd(d["pool_x"], "max"), d["pool_max"], rtol=0)
    np.testing.assert_allclose(O.pool2_bwd(d["pool_g"], d["pool_x"], "avg"), d["pool_avg_bwd"], rtol=1e-14)
    np.testing.assert_array_equal(O.pool2_bwd(d["pool_g"], d["pool_x"], "max"), d["pool_max_bwd"])


def test_resampling_and_padding_match_reference():
    d = golden("kernels.npz")
    img = d["img"]
    np.testing.assert_allclose(O.area_down(img, 3), d["down3"], rtol=2e-6)
    np.testing.assert_allclose(O.area_down(img, 8), d["down8"], rtol=2e-6)
    np.testing.assert_allclose(O.bilinear(img, 53, 41), d["bil"], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(O.bilinear(img, 74, 58), d["up2"], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(O.bilinear(img, 73, 57), d["up2t"], rtol=1e-6, atol=1e-7)
    np.testing.assert_array_equal(O.pad_edge16(img, 16), d["pad16"])
    np.testing.assert_allclose(O.fold_pad_grad(d["gpad"], 37, 29), d["fold"], rtol=1e-6, atol=1e-6)


def test_stats_and_style_gradient_match_reference():
    d = golden("kernels.npz")
    st = O.stats_of(d["st_feats"])
    np.testing.assert_allclose(st.gram, d["st_gram"], rtol=1e-13)
    np.testing.assert_allclose(st.mean, d["st_mean"], rtol=1e-13)
    np.testing.assert_allclose(st.std, d["st_std"], rtol=1e-12)
    ref = O.OStats(d["ref_gram"], d["ref_mean"], d["ref_std"], 64)
    w = O.OW(*d["tw"])
    np.testing.assert_allclose(O.style_terms(st, ref, w), d["sg_terms"], rtol=1e-12)
    np.testing.assert_allclose(O.style_feature_grad(d["st_feats"], st, ref, w), d["sg_grad"], rtol=1e-12, atol=1e-16)


def _tiny_onet(d):
    from paper_2212_13459_b200.spec import tinynet
    spec = tinynet(0)
    net = O.onet_from_spec(spec)
    # use the reference's own tinynet weights (identical to ours to 1e-16, see make_goldens)
    layers = []
    for l in net.layers:
        if l.kind == "conv":
            l = O.OLayer("conv", l.name, l.cin, l.cout, w=d["tiny_w_" + l.name], b=d["tiny_b_" + l.name])
        layers.append(l)
    return O.ONet(tuple(layers), net.style_taps, net.content_tap)


@pytest.mark.parametrize("k", [0, 1, 2])
def test_tinynet_algorithm1_matches_reference(k):
    d = golden("tinynet.npz")
    net = _tiny_onet(d)
    u, v, x = d[f"case{k}_u"], d[f"case{k}_v"], d[f"case{k}_x"]
    block, margin = (int(a) for a in d[f"case{k}_geom"])
    p = O.build_problem(u, v, net, O.default_weights(net), block, margin)
    for t in net.style_taps:
        np.testing.assert_allclose(p.style[t].gram, d[f"case{k}_style_{t}_gram"], rtol=1e-10, atol=1e-14)
    lb, gb = O.loss_grad(x, p)
    lg, gg = O.loss_grad_global(x, p)
    assert abs(lb - d[f"case{k}_loss"][0]) <= 1e-10 * abs(d[f"case{k}_loss"][0])
    assert abs(lg - d[f"case{k}_loss"][1]) <= 1e-10 * abs(d[f"case{k}_loss"][1])
    assert rel_l2(gb, d[f"case{k}_grad"]) <= 1e-10
    assert rel_l2(gg, d[f"case{k}_grad_global"]) <= 1e-10
    sx = O.stats_pass(x, net, block, margin)
    for t in net.style_taps:
        np.testing.assert_allclose(sx[t].gram, d[f"case{k}_{t}_gram"], rtol=1e-10, atol=1e-14)
        assert sx[t].n_p == int(d[f"case{k}_{t}_n"][0])


def test_tinynet_lbfgs_trajectory_matches_reference():
    d = golden("tinynet.npz")
    net = _tiny_onet(d)
    u, v, x = (d["case0_u"].astype(np.float32), d["case0_v"].astype(np.float32), d["case0_x"].astype(np.float32))
    p = O.build_problem(u, v, net, O.default_weights(net), 32, 16)
    l32, g32 = O.loss_grad(x, p)
    assert abs(l32 - d["case0_loss_f32"][0]) <= 1e-5 * abs(l32)
    assert rel_l2(g32, d["case0_grad_f32"]) <= 1e-4
    xr, losses, _ = O.minimize(lambda a: O.loss_grad(a, p), x, m=10, max_iters=5)
    np.testing.assert_allclose(losses, d["case0_lbfgs_losses"], rtol=1e-3)


def test_lbfgs_and_schedule_match_reference():
    d = golden("lbfgs_pipeline.npz")
    a = d["quad_a"]
    x, losses, gn = O.minimize(lambda z: (float(np.sum((z - a) ** 2)), 2.0 * (z - a)), np.zeros(20), m=5,
                               max_iters=30)
    np.testing.assert_allclose(x, d["quad_x"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(losses, d["quad_losses"], rtol=1e-10, atol=1e-20)

    def rosen(z):
        x0, y0 = z
        return float((1 - x0) ** 2 + 100 * (y0 - x0 ** 2) ** 2), np.array(
            [-2 * (1 - x0) - 400 * x0 * (y0 - x0 ** 2), 200 * (y0 - x0 ** 2)])

    x, losses, _ = O.minimize(rosen, np.array([-1.2, 1.0]), m=10, max_iters=200)
    np.testing.assert_allclose(x, d["rosen_x"], rtol=1e-10)
    h = O.OHistory()
    for s, y in zip(d["tl_s"], d["tl_y"]):
        h.push(s, y, 3)
    np.testing.assert_allclose(O.direction(d["tl_g"], h), d["tl_d"], rtol=1e-12)
    assert O.schedule(4, "fast")[0] == tuple(d["sched_fast4"])
    assert O.schedule(4, "baseline")[0] == tuple(d["sched_base4"])
    assert O.schedule(6, "fast")[0] == tuple(d["sched_fast6"])
    assert [tuple(t) for t in d["dims_4"]] == O.scale_dims(6048, 8064, 4)
    assert [tuple(t) for t in d["dims_3_odd"]] == O.scale_dims(1001, 777, 3)


def test_vgg19_oracle_matches_reference_at_x0():
    import os
    from conftest import GOLDEN
    if not os.path.exists(os.path.join(GOLDEN, "vgg19.npz")):
        pytest.skip("vgg19 golden not generated")
    d = golden("vgg19.npz")
    from paper_2212_13459_b200.spec import calibrated_vgg19
    import hashlib
    spec = calibrated_vgg19(0)
    h = hashlib.sha256()
    for l in spec.layers:
        if l.kind == "conv":
            h.update(np.ascontiguousarray(l.weight, dtype=np.float64).tobytes())
            h.update(np.ascontiguousarray(l.bias, dtype=np.float64).tobytes())
    assert h.hexdigest() == bytes(d["weights_sha256"]).decode(), "calibrated VGG-19 weights differ from the golden run"
    net = O.onet_from_spec(spec)
    us, vs, xs = d["r_u"], d["r_v"], d["r_x"]
    lam = float(d["r_lambda_c"][0])
    p = O.build_problem(us.astype(np.float64), vs.astype(np.float64), net, O.default_weights(net, lam), 512, 256)
    loss, g = O.loss_grad_global(xs, p)
    assert abs(loss - d["r_loss64"][0]) <= 1e-9 * abs(d["r_loss64"][0])
    assert rel_l2(g, d["r_grad64"]) <= 1e-9
