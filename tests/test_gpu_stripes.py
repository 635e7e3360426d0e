"""Device stripe evaluation (the per-rank unit of the multi-GPU path) on one GPU: two stripes
with a receptive-field halo, evaluated by two engines in one process, their statistics
summed by hand (what the NCCL all-reduce does across ranks), must reproduce the whole-image
loss and gradient."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2212_13459_b200 as spst  # noqa: E402
from paper_2212_13459_b200.device import Engine  # noqa: E402
from paper_2212_13459_b200.distributed import DeviceStripeEngine  # noqa: E402
from paper_2212_13459_b200.spec import tap_geometry  # noqa: E402
from paper_2212_13459_b200.tiling import margin_for_exact_gradient, stripes  # noqa: E402
from conftest import rel_l2  # noqa: E402


@pytest.mark.parametrize("net,shape", [("tiny", (150, 137)), ("vgg", (360, 200))])
def test_two_device_stripes_equal_whole_image(net, shape, tiny_spec, vgg_spec):
    spec = tiny_spec if net == "tiny" else vgg_spec
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
    parts = stripes(Hp, s, margin_for_exact_gradient(spec), 2)
    engines = [DeviceStripeEngine(Engine(spec)) for _ in parts]
    ud, xd = torch.from_numpy(u).cuda(), torch.from_numpy(x).cuda()
    for e, st in zip(engines, parts):
        e.bind(h, w, (st.grid_r0, st.grid_r1), (st.own_r0, st.own_r1))
        e.forward_rows(ud[st.grid_r0:min(st.grid_r1, h)], st.grid_r0)
        e.capture_content()
        for i, t in enumerate(spec.style_taps):
            e.set_style_ref(i, p.style_stats[t], weights.style[t])
        e.forward_rows(xd[st.grid_r0:min(st.grid_r1, h)], st.grid_r0)
    T = len(spec.style_taps)
    # "all-reduce": sum owned-row partials over the two stripes, write back into both engines
    for i in range(T):
        S = sum(e.tap_sums(i)[0].clone() for e in engines)
        sv = sum(e.tap_sums(i)[1].clone() for e in engines)
        for e in engines:
            e.tap_sums(i)[0].copy_(S)
            e.tap_sums(i)[1].copy_(sv)
    counts = [(Hp // tap_geometry(spec, t).stride) * (Wp // tap_geometry(spec, t).stride) for t in spec.style_taps]
    terms = [e.finalize(counts)[0] for e in engines]
    np.testing.assert_array_equal(terms[0], terms[1])
    content = sum(float(e.content_sqdiff().item()) for e in engines)
    loss = float(terms[0].sum()) + weights.lambda_c * content
    assert abs(loss - loss_ref) <= 1e-6 * abs(loss_ref)
    grad = torch.zeros((h, w, 3), device="cuda")
    for e, st in zip(engines, parts):
        r0, r1 = min(st.own_r0, h), min(st.own_r1, h)
        shard = torch.empty((r1 - r0) * w * 3, device="cuda")
        e.backward_rows(2 * weights.lambda_c, shard, r0, w)
        grad[r0:r1] = shard.view(r1 - r0, w, 3)
    assert rel_l2(grad.cpu().numpy(), g_ref) <= 1e-5
