"""Device window evaluation (the per-rank unit of the multi-GPU path) on one GPU: a 2x2 grid of
owned rectangles with a receptive-field halo, evaluated by four engines in one process, their
statistics summed in rank order (what the fixed-order reduction does across ranks), must
reproduce the whole-image loss and gradient."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2212_13459_b200 as spst  # noqa: E402
from paper_2212_13459_b200.device import Engine  # noqa: E402
from paper_2212_13459_b200.distributed import DeviceWindowEngine, grid_windows  # noqa: E402
from paper_2212_13459_b200.spec import tap_geometry  # noqa: E402
from paper_2212_13459_b200.tiling import margin_for_exact_gradient  # noqa: E402
from conftest import rel_l2  # noqa: E402


@pytest.mark.parametrize("net,shape,grid", [("tiny", (150, 137), (2, 2)), ("vgg", (360, 200), (2, 1)),
                                            ("vgg", (392, 424), (2, 2)), ("vggmax", (392, 424), (2, 2))])
def test_device_windows_equal_whole_image(net, shape, grid, tiny_spec, vgg_spec):
    spec = {"tiny": tiny_spec, "vgg": vgg_spec}.get(net) or spst.calibrated_vgg19(0, pooling="max")
    rng = np.random.default_rng(3)
    h, w = shape
    u = rng.random((h, w, 3)).astype(np.float32)
    v = rng.random((120, 110, 3)).astype(np.float32)
    x = np.clip(u + 0.1 * rng.standard_normal(u.shape), 0, 1).astype(np.float32)
    weights = spst.default_loss_weights(spec, lambda_c=1e-3)
    p = spst.build_problem(u, v, spec, weights)
    loss_ref, g_ref = spst.loss_grad(x, p)

    s = spec.deepest_stride()
    Hp, Wp = h + (-h) % s, w + (-w) % s
    wins = grid_windows(Hp, Wp, s, margin_for_exact_gradient(spec), *grid)
    engines = [DeviceWindowEngine(Engine(spec)) for _ in wins]
    ud, xd = torch.from_numpy(u).cuda(), torch.from_numpy(x).cuda()
    for e, wd in zip(engines, wins):
        e.bind(h, w, *wd.bind_args())
        e.forward_block(ud[wd.gr0:min(wd.gr1, h), wd.gc0:min(wd.gc1, w)], (wd.gr0, wd.gc0))
        e.capture_content()
        for i, t in enumerate(spec.style_taps):
            e.set_style_ref(i, p.style_stats[t], weights.style[t])
        e.forward_block(xd[wd.gr0:min(wd.gr1, h), wd.gc0:min(wd.gc1, w)], (wd.gr0, wd.gc0))
    T = len(spec.style_taps)
    for i in range(T):  # the reduction: owned partials summed in rank order, written back
        S = engines[0].tap_sums(i)[0].clone()
        sv = engines[0].tap_sums(i)[1].clone()
        for e in engines[1:]:
            S += e.tap_sums(i)[0]
            sv += e.tap_sums(i)[1]
        for e in engines:
            e.tap_sums(i)[0].copy_(S)
            e.tap_sums(i)[1].copy_(sv)
    counts = [(Hp // tap_geometry(spec, t).stride) * (Wp // tap_geometry(spec, t).stride) for t in spec.style_taps]
    terms = [e.finalize(counts)[0] for e in engines]
    for t in terms[1:]:
        np.testing.assert_array_equal(terms[0], t)
    content = sum(float(e.content_sqdiff().item()) for e in engines)
    loss = float(terms[0].sum()) + weights.lambda_c * content
    assert abs(loss - loss_ref) <= 1e-6 * abs(loss_ref)
    grad = torch.zeros((h, w, 3), device="cuda")
    for e, wd in zip(engines, wins):
        r0, r1, c0, c1 = min(wd.or0, h), min(wd.or1, h), min(wd.oc0, w), min(wd.oc1, w)
        blk = torch.empty((r1 - r0, c1 - c0, 3), device="cuda")
        e.backward_block(2 * weights.lambda_c, blk, (r0, c0))
        grad[r0:r1, c0:c1] = blk
    err = rel_l2(grad.cpu().numpy(), g_ref)
    print(f"{net} {shape} grid {grid}: loss rel {abs(loss - loss_ref) / loss_ref:.1e}, grad rel-L2 {err:.1e}")
    assert err <= 1e-5
