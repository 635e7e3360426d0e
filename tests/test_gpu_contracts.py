"""API contracts of the drop-in that are not numerics of the hot path: odd-sized L-BFGS state
(16-byte-aligned history slots), per-problem content targets, copies handed to callbacks,
float64 resampling and the float64 precision warning."""

import warnings

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import spst_oracle as O  # noqa: E402
import paper_2212_13459_b200 as spst  # noqa: E402
from paper_2212_13459_b200.pipeline import objective_for  # noqa: E402
from conftest import golden, rel_l2  # noqa: E402


def test_minimize_odd_sized_image_history_alignment(tiny_spec):
    """37 x 41 x 3 = 4551 floats: slot k of a (m+1) x numel history ring would start off a
    16-byte boundary; minimize must run its float4 vector kernels on every slot."""
    rng = np.random.default_rng(8)
    u, v = rng.random((37, 41, 3)).astype(np.float32), rng.random((40, 40, 3)).astype(np.float32)
    p = spst.build_problem(u, v, tiny_spec, spst.default_loss_weights(tiny_spec), block=64, margin=16)
    x, tr = spst.minimize(objective_for(p), torch.from_numpy(u).cuda(), spst.LBFGSConfig(history_size=3, max_iters=6))
    torch.cuda.synchronize()
    assert x.shape == (37, 41, 3) and bool(torch.isfinite(x).all())
    assert all(b <= a for a, b in zip(tr.losses, tr.losses[1:])) and tr.losses[-1] < tr.losses[0]


def test_two_problems_same_dims_keep_their_content_targets(tiny_spec):
    rng = np.random.default_rng(9)
    u1, u2, v, x = (rng.random((48, 48, 3)).astype(np.float32) for _ in range(4))
    w = spst.default_loss_weights(tiny_spec)
    p1 = spst.build_problem(u1, v, tiny_spec, w, block=64, margin=16)
    l1, g1 = spst.loss_grad(x, p1)
    p2 = spst.build_problem(u2, v, tiny_spec, w, block=64, margin=16)  # same dims, same engine
    l2, g2 = spst.loss_grad(x, p2)
    l1b, g1b = spst.loss_grad(x, p1)
    assert l1b == l1 and np.array_equal(g1b, g1)
    assert l2 != l1
    net = O.onet_from_spec(tiny_spec)
    po2 = O.build_problem(u2.astype(np.float64), v.astype(np.float64), net, O.default_weights(net), 64, 16)
    lo2, go2 = O.loss_grad_global(x.astype(np.float64), po2)
    assert abs(l2 - lo2) <= 1e-5 * lo2 and rel_l2(g2, go2) <= 1e-5


def test_callback_gets_its_own_copy(tiny_spec):
    rng = np.random.default_rng(10)
    u, v = rng.random((48, 48, 3)).astype(np.float32), rng.random((48, 48, 3)).astype(np.float32)
    p = spst.build_problem(u, v, tiny_spec, spst.default_loss_weights(tiny_spec), block=64, margin=16)
    seen = []
    x, tr = spst.minimize(objective_for(p), torch.from_numpy(u).cuda(), spst.LBFGSConfig(max_iters=4),
                          callback=lambda it, xi, l, g: seen.append(xi))
    assert len(seen) == 4 and all(a.data_ptr() != b.data_ptr() for a, b in zip(seen, seen[1:]))
    assert torch.equal(seen[-1], x)


def test_resample_float64_path():
    d = golden("kernels.npz")
    img = d["img"].astype(np.float64) * 0.9 + 0.05
    down = spst.resize_down(img, 3)
    assert down.dtype == np.float64
    assert np.max(np.abs(down - O.area_down(img, 3))) <= 1e-13
    bil = spst.resize_bilinear(img, (53, 41))
    assert bil.dtype == np.float64
    assert np.max(np.abs(bil - O.bilinear(img, 53, 41))) <= 1e-13


def test_float64_inputs_warn(tiny_spec):
    rng = np.random.default_rng(12)
    u, v = rng.random((48, 48, 3)), rng.random((48, 48, 3))
    p = spst.build_problem(u.astype(np.float32), v.astype(np.float32), tiny_spec,
                           spst.default_loss_weights(tiny_spec), block=64, margin=16)
    with pytest.warns(spst.PrecisionWarning):
        loss, g = spst.loss_grad(u, p)
    assert g.dtype == np.float64
    with warnings.catch_warnings():
        warnings.simplefilter("error", spst.PrecisionWarning)
        spst.loss_grad(u.astype(np.float32), p)


def test_fp16_precision_mode_is_opt_in(vgg_spec):
    """SURVEY.md §7 step 3 precision knob: one-pass fp16 convs run (loss within ~1e-2, gradient
    visibly coarser than the fp32-class default); the default mode is restored and exact again."""
    d = golden("vgg19.npz")
    w = spst.default_loss_weights(vgg_spec, lambda_c=float(d["c1_lambda_c"][0]))
    p = spst.build_problem(d["c1_u"], d["c1_v"], vgg_spec, w)
    x = golden("vgg19_iterates.npz")["x2"]
    g64 = golden("vgg19_iterates.npz")["grad64_2"]
    l64 = float(golden("vgg19_iterates.npz")["loss64_2"][0])
    assert spst.get_precision() == "fp16x3"
    try:
        spst.set_precision("fp16")
        lf, gf = spst.loss_grad(x, p)
    finally:
        spst.set_precision("fp16x3")
    l3, g3 = spst.loss_grad(x, p)
    ef, e3 = rel_l2(gf, g64), rel_l2(g3, g64)
    print(f"fp16: loss rel {abs(lf - l64) / l64:.1e}, grad {ef:.1e}; fp16x3: loss rel {abs(l3 - l64) / l64:.1e}, "
          f"grad {e3:.1e}")
    assert abs(lf - l64) <= 1e-2 * l64 and ef < 1.0
    assert abs(l3 - l64) <= 1e-5 * l64 and e3 <= 1e-3 and ef > 10 * e3
    with pytest.raises(ValueError):
        spst.set_precision("bf16")
