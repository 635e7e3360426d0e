"""Max pooling on the device (reference tensorops.py:113-129, extractor.py:321
vgg19(pooling="max")): the conv epilogue pools 2x2 windows to their maximum and stores the
first-argmax index (row-major in the window, ties to the first); the backward routes each
pooled gradient to that index.  Checked against fp64 at the kernel level and against the
reference's own Algorithm 1 (tests/golden/maxpool.npz)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2212_13459_b200 as spst  # noqa: E402
from paper_2212_13459_b200 import _native  # noqa: E402
from paper_2212_13459_b200.spec import with_pooling  # noqa: E402
from conftest import golden, rel_l2  # noqa: E402


def _debug_conv(mode, x, w, b):
    cin, cout = w.shape[1], w.shape[0]
    H, W = x.shape[1:]
    y = np.zeros((cout, H // 2, W // 2), np.float32)
    st = _native.lib().spst_debug_conv(0, mode, cin, cout, H, W, np.ascontiguousarray(x, np.float32).ctypes.data,
                                       np.ascontiguousarray(w, np.float64).ctypes.data,
                                       np.ascontiguousarray(b, np.float64).ctypes.data, y.ctypes.data)
    _native.check(st)
    return y


@pytest.mark.parametrize("cin,cout", [(64, 64), (128, 256), (512, 512)])
def test_maxpool_epilogue_vs_fp64(cin, cout):
    F = torch.nn.functional
    rng = np.random.default_rng(cin + cout)
    H, W = 18, 140
    x = rng.random((cin, H, W)).astype(np.float32)
    w = rng.normal(0, np.sqrt(2 / (9 * cin)), (cout, cin, 3, 3))
    b = rng.normal(0, 0.1, cout)
    a = torch.relu(F.conv2d(torch.from_numpy(x).double()[None], torch.from_numpy(w), torch.from_numpy(b),
                            padding=1)[0]).numpy()
    win = a.reshape(cout, H // 2, 2, W // 2, 2).transpose(0, 1, 3, 2, 4).reshape(cout, H // 2, W // 2, 4)
    y = _debug_conv(4, x, w, b)
    assert rel_l2(y, win.max(axis=3)) <= 2e-6
    idx = _debug_conv(5, x, w, b).astype(np.int64)
    ref = np.argmax(win, axis=3)  # first argmax (reference tensorops.py:121-123)
    srt = np.sort(win, axis=3)
    clear = (srt[..., 3] - srt[..., 2]) > 1e-5 * (np.abs(srt[..., 3]) + 1e-30)  # not a near-tie
    assert np.array_equal(idx[clear], ref[clear])
    zero = srt[..., 3] == 0  # all-zero ReLU windows: the first index, like np.argmax
    assert np.all(idx[zero] == 0)


def test_maxpool_tinynet_vs_reference():
    d = golden("maxpool.npz")
    spec = with_pooling(spst.tinynet(0), "max")
    p = spst.build_problem(d["tiny_u"], d["tiny_v"], spec, spst.default_loss_weights(spec), block=512, margin=16)
    loss, g = spst.loss_grad(d["tiny_x"], p)
    assert abs(loss - d["tiny_loss"][0]) <= 1e-5 * abs(d["tiny_loss"][0])
    assert rel_l2(g, d["tiny_grad"]) <= 1e-5


def test_maxpool_vgg19_vs_reference():
    d = golden("maxpool.npz")
    spec = spst.calibrated_vgg19(0, pooling="max")
    assert [l.pool for l in spec.layers if l.kind == "pool"] == ["max"] * 4
    w = spst.default_loss_weights(spec, lambda_c=float(d["vgg_lambda_c"][0]))
    p = spst.build_problem(d["vgg_u"], d["vgg_v"], spec, w)
    for t in spec.style_taps:
        assert rel_l2(p.style_stats[t].gram, d[f"vgg_style_{t}_gram"]) <= 1e-5
    for k in range(2):
        loss, g = spst.loss_grad(d[f"vgg_x{k}"], p)
        g64, g32 = d[f"vgg_grad64_{k}"], d[f"vgg_grad32_{k}"]
        err, gap = rel_l2(g, g64), rel_l2(g32, g64)
        print(f"max-pool VGG point {k}: loss rel {abs(loss - d[f'vgg_loss64_{k}'][0]) / d[f'vgg_loss64_{k}'][0]:.1e}, "
              f"grad vs f64 {err:.2e} (reference f32 {gap:.2e})")
        assert abs(loss - d[f"vgg_loss64_{k}"][0]) <= 1e-5 * d[f"vgg_loss64_{k}"][0]
        assert err <= max(1e-3, 1.5 * gap)
