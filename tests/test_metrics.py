"""Evaluation metrics (reference metrics.py).

CPU tests pin the oracle restatement to the reference's own outputs and check the host-side
behaviour of the device module (errors raised before any device work, report/CSV formats).
GPU tests compare the CUDA kernels with the reference values and the oracle."""

import json
import math

import numpy as np
import pytest
import torch

import spst_oracle as O
import paper_2212_13459_b200 as spst
from paper_2212_13459_b200 import metrics as M
from conftest import golden

CASES = ["rand", "min11", "gray", "synth", "f32"]


# ---------------------------------------------------------------- CPU
@pytest.mark.parametrize("k", CASES)
def test_oracle_metrics_match_reference(k):
    d = golden("metrics.npz")
    assert O.psnr(d[f"{k}_a"], d[f"{k}_b"]) == pytest.approx(d[f"{k}_psnr"][0], rel=1e-13)
    assert O.ssim(d[f"{k}_a"], d[f"{k}_b"]) == pytest.approx(d[f"{k}_ssim"][0], rel=1e-13)


def test_oracle_identical_images():
    d = golden("metrics.npz")
    a = d["rand_a"]
    assert O.psnr(a, a) == math.inf == d["same_psnr"][0]
    assert O.ssim(a, a) == pytest.approx(d["same_ssim"][0], rel=1e-15)


def test_shape_errors_raised_before_device_work():
    a = np.zeros((20, 20, 3), np.float32)
    with pytest.raises(spst.ShapeError):
        M.psnr(a, np.zeros((20, 21, 3), np.float32))
    with pytest.raises(spst.ShapeError):
        M.ssim(a, np.zeros((21, 20, 3), np.float32))
    with pytest.raises(spst.ShapeError):
        M.ssim(np.zeros((10, 40, 3)), np.zeros((10, 40, 3)))


def test_identity_report_json_and_csv(tmp_path):
    r = M.IdentityReport(psnr=31.5, ssim=0.93, gram_distance=1.25, gram_distance_weighted=0.5, wall_time=2.0,
                         config_hash="abc")
    assert json.loads(r.to_json()) == {"psnr": 31.5, "ssim": 0.93, "gram": 1.25, "gram_weighted": 0.5,
                                       "seconds": 2.0, "config_hash": "abc"}
    p = tmp_path / "ids.csv"
    M.append_csv(p, "starry", r)
    M.append_csv(p, "scream", r)
    assert p.read_text().splitlines() == ["style_id,psnr,ssim,gram,seconds,config_hash",
                                          "starry,31.5,0.93,1.25,2.0,abc", "scream,31.5,0.93,1.25,2.0,abc"]


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("k", CASES)
def test_device_metrics_match_reference(k):
    d = golden("metrics.npz")
    a, b = d[f"{k}_a"], d[f"{k}_b"]
    assert M.psnr(a, b) == pytest.approx(d[f"{k}_psnr"][0], rel=1e-12)
    assert M.ssim(a, b) == pytest.approx(d[f"{k}_ssim"][0], rel=1e-12)


@pytest.mark.gpu
def test_device_metrics_edge_cases():
    d = golden("metrics.npz")
    a = d["rand_a"]
    assert M.psnr(a, a) == math.inf
    assert M.ssim(a, a) == pytest.approx(1.0, abs=1e-14)
    # torch CUDA inputs, mixed dtypes (NumPy promotes to f64), ragged 11 x N and N x 11
    rng = np.random.default_rng(3)
    for h, w in [(11, 200), (173, 11), (517, 389)]:
        x = rng.random((h, w, 3)).astype(np.float32)
        y = np.clip(x + 0.1 * rng.standard_normal(x.shape), 0, 1)
        assert M.ssim(x, y) == pytest.approx(O.ssim(x, y), rel=1e-12)
        assert M.psnr(torch.from_numpy(x).cuda(), y) == pytest.approx(O.psnr(x, y), rel=1e-12)
    # deterministic (fixed-order reductions)
    x = rng.random((300, 301, 3))
    y = rng.random((300, 301, 3))
    assert M.ssim(x, y) == M.ssim(x, y)
    assert M.psnr(x, y) == M.psnr(x, y)


@pytest.mark.gpu
def test_device_ssim_full_resolution_matches_oracle():
    """The benchmark's 6048x8064 size (a stride-aligned strip of it keeps the oracle fast)."""
    rng = np.random.default_rng(4)
    x = rng.random((6048, 8064, 3), dtype=np.float32)
    y = np.clip(x + 0.02 * rng.standard_normal(x.shape, dtype=np.float32), 0, 1)
    full = M.ssim(x, y)
    assert 0.0 < full < 1.0
    strip = M.ssim(x[:64], y[:64])
    assert strip == pytest.approx(O.ssim(x[:64], y[:64]), rel=1e-12)


@pytest.mark.gpu
def test_gram_distance_matches_reference(tiny_spec):
    d = golden("metrics.npz")
    got = M.gram_distance(d["gd_x"], d["gd_v"], tiny_spec, block=32, margin=16)
    assert got == pytest.approx(d["gd_plain"][0], rel=1e-5)
    w = dict(zip(tiny_spec.style_taps, d["gd_weights"]))
    got_w = M.gram_distance(d["gd_x"], d["gd_v"], tiny_spec, block=32, margin=16, weights=w)
    assert got_w == pytest.approx(d["gd_weighted"][0], rel=1e-5)


@pytest.mark.gpu
def test_identity_test_reports(tiny_spec, tmp_path):
    rng = np.random.default_rng(8)
    style = (0.5 + 0.3 * np.sin(np.arange(64)[None, :, None] / 4.0) + 0.05 * rng.random((64, 64, 3))).astype(np.float32)
    # two scales: the upsampled coarse result is not the style, so the finest scale has work to do
    cfg = spst.RunConfig(n_scales=2, extractor=tiny_spec, mode="fast", block=32, margin=16)
    report, out = M.identity_test(style, cfg)
    assert out.shape == style.shape
    for v in (report.psnr, report.ssim, report.gram_distance, report.gram_distance_weighted):
        assert np.isfinite(v)
    assert report.psnr == pytest.approx(O.psnr(out, style), rel=1e-12)
    assert report.ssim == pytest.approx(O.ssim(out, style), rel=1e-12)
    assert report.psnr > 20 and report.ssim > 0.5
    M.append_csv(tmp_path / "r.csv", "synthetic", report)
