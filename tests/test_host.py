"""Host-side logic (no GPU): specs and geometry, tiling and stripes, stats bookkeeping,
formats, schedules.  Known-answer tests follow the reference suite."""

import hashlib
import os

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from paper_2212_13459_b200 import errors, formats
from paper_2212_13459_b200.pipeline import make_schedule, scale_dims, synthesis_scales_for, _weights_for_scale, RunConfig
from paper_2212_13459_b200.spec import (ExtractorSpec, LayerSpec, conv, load_weights, relu, save_weights, tap_geometry,
                                        tinynet, vgg19)
from paper_2212_13459_b200.stats import (LayerStats, StatsAccumulator, TapWeights, default_loss_weights,
                                         finalize_sums, load_stats, save_stats, style_loss_terms, LossWeights)
from paper_2212_13459_b200.tiling import (BlockGrid, feature_inner_crop, margin_for_exact_gradient, partition,
                                          stripes)
from conftest import golden


# ---------------------------------------------------------------- spec / geometry
def test_vgg19_taps_strides_widths():
    s = vgg19()
    geo = {t: tap_geometry(s, t) for t in s.taps}
    assert [geo[f"relu{g}_1"].stride for g in range(1, 6)] == [1, 2, 4, 8, 16]
    assert [geo[f"relu{g}_1"].channels for g in range(1, 6)] == [64, 128, 256, 512, 512]
    assert geo["relu4_2"].stride == 8 and geo["relu4_2"].channels == 512
    assert s.deepest_stride() == 16
    assert margin_for_exact_gradient(s) == 160


def test_tinynet_exact_margin_and_weights_match_reference():
    t = tinynet(0)
    assert margin_for_exact_gradient(t) == 16
    d = golden("tinynet.npz")
    for l in t.layers:
        if l.kind == "conv":
            np.testing.assert_allclose(l.weight, d["tiny_w_" + l.name], rtol=0, atol=1e-14)
            np.testing.assert_allclose(l.bias, d["tiny_b_" + l.name], rtol=0, atol=1e-14)


def test_calibrated_vgg19_is_the_golden_network(vgg_spec):
    d = golden("vgg19.npz")
    h = hashlib.sha256()
    for l in vgg_spec.layers:
        if l.kind == "conv":
            h.update(np.ascontiguousarray(l.weight, dtype=np.float64).tobytes())
            h.update(np.ascontiguousarray(l.bias, dtype=np.float64).tobytes())
    assert h.hexdigest() == bytes(d["weights_sha256"]).decode()


def test_spec_validation_errors():
    with pytest.raises(errors.GeometryError):
        LayerSpec("conv", "c", in_ch=3, out_ch=4, k=2, pad=0)
    with pytest.raises(errors.GeometryError):
        LayerSpec("conv", "c", in_ch=3, out_ch=4, k=3, pad=0)
    with pytest.raises(errors.GeometryError):
        LayerSpec("pool", "p", k=2, pool="median")
    with pytest.raises(KeyError):
        ExtractorSpec((conv("c1", 3, 8), relu("r1")), ("nope",), "r1")
    with pytest.raises(errors.GeometryError):
        ExtractorSpec((conv("c1", 3, 8), relu("r1")), ("c1",), "r1")


# ---------------------------------------------------------------- tiling
def test_partition_kat():
    blocks = partition(BlockGrid(1024, 1024, block=512, margin=256, stride=16))
    assert len(blocks) == 4
    b = blocks[0]
    assert (b.padded.x0, b.padded.y0, b.padded.w, b.padded.h) == (0, 0, 768, 768)
    assert b.present_margin == (0, 0, 256, 256)
    b = blocks[3]
    assert (b.padded.x0, b.padded.y0) == (256, 256)


def test_feature_inner_crop_kat():
    blocks = partition(BlockGrid(1024, 1024, block=512, margin=256, stride=16))
    c = feature_inner_crop(blocks[3], tap_geometry(vgg19(), "relu3_1"))
    assert (c.x0, c.y0, c.w, c.h) == (64, 64, 128, 128)


def test_grid_validation():
    with pytest.raises(errors.GeometryError):
        BlockGrid(100, 100, block=8, margin=0, stride=16)
    with pytest.raises(errors.GeometryError):
        BlockGrid(100, 100, block=64, margin=8, stride=16)
    with pytest.raises(errors.GeometryError):
        BlockGrid(0, 100, block=64, margin=16, stride=16)


@settings(max_examples=200, deadline=None)
@given(st.integers(1, 40), st.integers(1, 40), st.integers(1, 6), st.integers(0, 4))
def test_partition_cover_disjoint(hu, wu, bu, mu):
    s = 16
    H, W = hu * s, wu * s
    blocks = partition(BlockGrid(H, W, block=bu * s, margin=mu * s, stride=s))
    cover = np.zeros((H, W), np.int32)
    for b in blocks:
        cover[b.inner.y0:b.inner.y1, b.inner.x0:b.inner.x1] += 1
        assert b.padded.x0 >= 0 and b.padded.y0 >= 0 and b.padded.x1 <= W and b.padded.y1 <= H
    assert np.all(cover == 1)


@settings(max_examples=100, deadline=None)
@given(st.integers(1, 400), st.integers(1, 9), st.sampled_from([0, 16, 160]))
def test_stripes_cover_owned_rows(units, n, halo):
    Hp = units * 16
    ss = stripes(Hp, 16, halo, n)
    own = np.zeros(Hp, np.int32)
    for s in ss:
        own[s.own_r0:s.own_r1] += 1
        assert s.grid_r0 == max(0, s.own_r0 - halo) and s.grid_r1 == min(Hp, s.own_r1 + halo)
        assert s.own_r0 % 16 == 0 and s.own_r1 % 16 == 0 and s.own_r1 > s.own_r0
    assert np.all(own == 1)


# ---------------------------------------------------------------- stats
def test_stats_finalize_kats():
    acc = StatsAccumulator(2)
    acc.accumulate(np.array([[[3.0]], [[0.0]]]))
    st1 = acc.finalize()
    np.testing.assert_array_equal(st1.gram, [[9.0, 0.0], [0.0, 0.0]])
    assert st1.n_p == 1
    a, b = StatsAccumulator(2), StatsAccumulator(2)
    f = np.random.default_rng(0).random((2, 4, 6))
    a.accumulate(f[:, :2])
    b.accumulate(f[:, 2:])
    a.merge(b)
    whole = StatsAccumulator(2)
    whole.accumulate(f)
    np.testing.assert_allclose(a.finalize().gram, whole.finalize().gram, rtol=1e-14)
    with pytest.raises(errors.EmptyError):
        StatsAccumulator(3).finalize()
    # two-point variance: values 1 and 3 -> mean 2, std 1
    s = finalize_sums(np.array([[1.0 + 9.0]]), np.array([4.0]), 2)
    assert s.std[0] == pytest.approx(1.0)


def test_default_weights_and_terms():
    w = default_loss_weights(vgg19())
    assert w.style["relu1_1"].gram == pytest.approx(1 / 64 ** 2)
    assert w.style["relu5_1"].mean == pytest.approx(1e3 / 512 ** 2)
    a = LayerStats(np.eye(2), np.zeros(2), np.ones(2), 4)
    b = LayerStats(2 * np.eye(2), np.ones(2), np.zeros(2), 4)
    assert style_loss_terms(a, b, TapWeights(1.0, 2.0, 3.0)) == pytest.approx((2.0, 4.0, 6.0))
    with pytest.warns(UserWarning):
        LossWeights(0.0, {"t": TapWeights(0.0, 0.0, 0.0)})
    with pytest.raises(errors.ShapeError):
        LossWeights(-1.0, {})


def test_per_element_content_weight():
    s = vgg19()
    w = _weights_for_scale(RunConfig(extractor=s), s, (256, 256))
    assert w.lambda_c == pytest.approx(1.0 / (512 * 32 * 32))
    assert float(golden("vgg19.npz")["c1_lambda_c"][0]) == pytest.approx(w.lambda_c)


# ---------------------------------------------------------------- formats
def test_nstw1_roundtrip_and_errors(tmp_path):
    t = tinynet(0)
    p = tmp_path / "w.nstw"
    save_weights(p, t)
    t2 = load_weights(p, tinynet(1))
    for a, b in zip(t.layers, t2.layers):
        if a.kind == "conv":
            np.testing.assert_array_equal(a.weight, b.weight)
    (tmp_path / "bad.nstw").write_bytes(b"NOPE!")
    with pytest.raises(errors.FormatError):
        formats.read_records(tmp_path / "bad.nstw")
    raw = p.read_bytes()
    (tmp_path / "trunc.nstw").write_bytes(raw[:-7])
    with pytest.raises(errors.FormatError):
        formats.read_records(tmp_path / "trunc.nstw")
    st = {"relu1": LayerStats(np.eye(3), np.ones(3), np.ones(3) * 2, 17)}
    save_stats(tmp_path / "s.nstw", st)
    back = load_stats(tmp_path / "s.nstw")
    assert back["relu1"].n_p == 17
    np.testing.assert_array_equal(back["relu1"].gram, np.eye(3))


def test_nstw1_reads_reference_written_file(tmp_path):
    """Byte compatibility: a file written by the reference layout parses identically."""
    import struct
    rec = np.arange(6, dtype=np.float32).reshape(2, 3)
    buf = b"NSTW1" + struct.pack("<I", 1) + b"a" + struct.pack("<BI", 0, 2) + struct.pack("<2I", 2, 3) + rec.tobytes()
    (tmp_path / "r.nstw").write_bytes(buf)
    out = formats.read_records(tmp_path / "r.nstw")
    np.testing.assert_array_equal(out["a"], rec)


# ---------------------------------------------------------------- schedules
def test_schedule_and_dims_kats():
    d = golden("lbfgs_pipeline.npz")
    assert make_schedule(4, "fast").iters == (600, 200, 66, 30) == tuple(d["sched_fast4"])
    assert make_schedule(4, "baseline").iters == (600, 300, 300, 300) == tuple(d["sched_base4"])
    assert make_schedule(6, "fast").iters == tuple(d["sched_fast6"])
    assert make_schedule(3).histories == (100, 10, 10)
    assert scale_dims((6048, 8064), 4) == [tuple(x) for x in d["dims_4"]]
    assert scale_dims((6048, 8064), 4)[0] == (756, 1008)
    assert scale_dims((1001, 777), 3) == [tuple(x) for x in d["dims_3_odd"]]
    assert synthesis_scales_for((600, 800)) == 2
    with pytest.raises(errors.ConfigError):
        make_schedule(0)
    with pytest.raises(errors.ConfigError):
        make_schedule(2, "turbo")


# Names re-exported by the reference package (reference __init__.py:3-17); the drop-in must
# provide every one of them.
REFERENCE_PUBLIC_NAMES = (
    "ConfigError", "DegenerateStdWarning", "EmptyError", "FormatError", "GeometryError", "NonFiniteError",
    "ShapeError", "ExtractorSpec", "LayerSpec", "Preprocess", "TapGeometry", "forward_taps", "load_weights",
    "save_weights", "tap_geometry", "tinynet", "vgg19", "LBFGSConfig", "LBFGSState", "minimize",
    "two_loop_direction", "TransferProblem", "build_problem", "loss_grad", "loss_grad_global", "stats_pass",
    "track_activations", "IdentityReport", "gram_distance", "identity_test", "psnr", "ssim", "RunConfig",
    "Schedule", "make_schedule", "multiscale_transfer", "scale_dims", "texture_synthesize", "LayerStats",
    "LossWeights", "StatsAccumulator", "TapWeights", "content_loss_grad", "default_loss_weights",
    "style_layer_loss_grad", "resize_bilinear", "resize_down", "resize_up2", "Block", "BlockGrid", "Rect",
    "feature_inner_crop", "margin_for_exact_gradient", "partition", "__version__")


def test_every_reference_public_name_is_exported():
    import paper_2212_13459_b200 as spst
    missing = [n for n in REFERENCE_PUBLIC_NAMES if not hasattr(spst, n)]
    assert not missing, missing
