"""Per-tap public helpers of the drop-in, checked against the reference's own outputs
(tests/golden/api.npz, written by tools/make_goldens.py from the real reference):
forward_taps (reference extractor.py:171-197), style_layer_loss_grad and content_loss_grad
(reference stats.py:127-174)."""

import warnings

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2212_13459_b200 as spst  # noqa: E402
from conftest import golden, rel_l2  # noqa: E402


def test_forward_taps_tinynet_vs_reference(tiny_spec):
    d = golden("api.npz")
    taps = spst.forward_taps(d["tiny_x"], tiny_spec)
    assert set(taps) == set(tiny_spec.taps)
    for t, v in taps.items():
        ref = d[f"tiny_tap_{t}"]
        assert v.shape == ref.shape and v.dtype == np.float32
        assert rel_l2(v, ref) <= 1e-6, (t, rel_l2(v, ref))


def test_forward_taps_vgg19_vs_reference(vgg_spec):
    d = golden("api.npz")
    taps = spst.forward_taps(d["vgg_x"], vgg_spec)
    for t in vgg_spec.taps:
        ref = d[f"vgg_tap_{t}"]
        err = rel_l2(taps[t], ref)
        print(f"forward_taps {t}: rel-L2 {err:.2e}")
        assert taps[t].shape == ref.shape
        assert err <= 1e-5, (t, err)
    # CUDA tensors in -> CUDA tensors out
    tt = spst.forward_taps(torch.from_numpy(d["vgg_x"]).cuda(), vgg_spec)
    assert tt["relu1_1"].is_cuda and rel_l2(tt["relu1_1"].cpu().numpy(), d["vgg_tap_relu1_1"]) <= 1e-5


def test_forward_taps_errors(tiny_spec):
    with pytest.raises(spst.ShapeError):
        spst.forward_taps(np.zeros((4, 16, 16), np.float32), tiny_spec)
    with pytest.raises(spst.GeometryError):
        spst.forward_taps(np.zeros((3, 2, 16), np.float32), tiny_spec)
    with pytest.raises(NotImplementedError):
        spst.forward_taps(np.zeros((3, 16, 16), np.float32), tiny_spec, save_for_backward=True)
    with pytest.raises(NotImplementedError):
        spst.forward_taps(np.zeros((3, 18, 16), np.float32), tiny_spec)


def _stats(d, sd_key="sg_sd"):
    n = int(d["sg_n"][0])
    return (spst.LayerStats(d["sg_G"], d["sg_mu"], d[sd_key], n),
            spst.LayerStats(d["sg_Gr"], d["sg_mur"], d["sg_sdr"], n))


def test_style_layer_loss_grad_vs_reference():
    d = golden("api.npz")
    sx, sr = _stats(d)
    w = spst.TapWeights(*d["sg_w"])
    terms, g = spst.style_layer_loss_grad(d["sg_slab"], sx, sr, w)
    np.testing.assert_allclose(terms, d["sg_terms"], rtol=1e-12)
    assert g.dtype == np.float32 and g.shape == d["sg_slab"].shape
    assert rel_l2(g, d["sg_grad"]) <= 1e-6, rel_l2(g, d["sg_grad"])
    with pytest.raises(spst.ShapeError):
        spst.style_layer_loss_grad(d["sg_slab"][:5], sx, sr, w)


def test_style_layer_loss_grad_degenerate_column():
    d = golden("api.npz")
    sx, sr = _stats(d, "sgd_sd")
    w = spst.TapWeights(*d["sg_w"])
    assert int(d["sgd_warned"][0]) == 1
    with pytest.warns(spst.DegenerateStdWarning):
        terms, g = spst.style_layer_loss_grad(d["sg_slab"].astype(np.float64), sx, sr, w)
    assert g.dtype == np.float64
    np.testing.assert_allclose(terms, d["sgd_terms"], rtol=1e-12)
    assert rel_l2(g, d["sgd_grad"]) <= 1e-12


def test_content_loss_grad_vs_reference():
    d = golden("api.npz")
    loss, g = spst.content_loss_grad(d["cl_V"], d["cl_Vr"], 0.37)
    assert abs(loss - d["cl_loss"][0]) <= 1e-9 * abs(d["cl_loss"][0])
    assert rel_l2(g, d["cl_grad"]) <= 1e-7
    with pytest.raises(spst.ShapeError):
        spst.content_loss_grad(d["cl_V"], d["cl_Vr"][:, :2], 1.0)
