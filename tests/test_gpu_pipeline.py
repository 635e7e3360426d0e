"""Drivers against the reference's own runs (tests/golden/pipeline.npz, written by
tools/make_goldens.py from the real reference): multiscale_transfer and texture_synthesize
(reference pipeline.py:232-260) on TinyNet, 2 scales x 3 L-BFGS iterations (history 5).
SURVEY.md §8(d) parity protocol (3): on runs this short the final image matches the
reference's to a mean absolute difference of at most 1/255."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2212_13459_b200 as spst  # noqa: E402
import paper_2212_13459_b200.pipeline as pl  # noqa: E402
from conftest import golden  # noqa: E402


@pytest.fixture
def short_schedule():
    orig = pl.make_schedule
    pl.make_schedule = lambda n, m="baseline": pl.Schedule(n, (3,) * n, (5,) * n, m)
    try:
        yield
    finally:
        pl.make_schedule = orig


def _check_trace(seen, ref):
    ref = np.asarray(ref)
    assert len(seen) == len(ref)
    for (s, it, l, g), (rs, rit, rl, rg) in zip(seen, ref):
        assert (s, it) == (int(rs), int(rit))
        assert abs(l - rl) <= 2e-3 * abs(rl), (s, it, l, rl)


def test_multiscale_transfer_vs_reference(tiny_spec, short_schedule):
    d = golden("pipeline.npz")
    cfg = spst.RunConfig(n_scales=2, mode="fast", extractor=tiny_spec, block=32, margin=16)
    seen = []
    x = spst.multiscale_transfer(d["u"], d["v"], cfg, progress=lambda s, it, l, g: seen.append((s, it, l, g)))
    assert x.shape == d["ms_x"].shape and x.dtype == np.float32
    _check_trace(seen, d["ms_trace"])
    mad = float(np.mean(np.abs(x - d["ms_x"])))
    print(f"multiscale_transfer: final-image mean |diff| vs reference {mad:.2e} (bar {1 / 255:.2e})")
    assert mad <= 1.0 / 255


def test_texture_synthesize_vs_reference(tiny_spec, short_schedule):
    d = golden("pipeline.npz")
    cfg = spst.RunConfig(n_scales=2, extractor=tiny_spec, block=32, margin=16, lambda_c=0.0, seed=3)
    seen = []
    x = spst.texture_synthesize(d["v"], cfg, progress=lambda s, it, l, g: seen.append((s, it, l, g)))
    assert x.shape == d["ts_x"].shape
    _check_trace(seen, d["ts_trace"])
    mad = float(np.mean(np.abs(x - d["ts_x"])))
    print(f"texture_synthesize: final-image mean |diff| vs reference {mad:.2e} (bar {1 / 255:.2e})")
    assert mad <= 1.0 / 255


def test_multiscale_and_texture_vgg19_vs_reference(vgg_spec):
    """The flagship network through both drivers (tests/golden/pipeline_vgg.npz: the reference's
    own calibrated-VGG-19 runs, content 128x160): multiscale_transfer 2 scales x 1 iteration,
    texture_synthesize 2 scales x 3 (tools/make_goldens.py pipeline_vgg_cases says why the
    content run is kept to one step per scale)."""
    d = golden("pipeline_vgg.npz")
    orig = pl.make_schedule
    try:
        pl.make_schedule = lambda n, m="baseline": pl.Schedule(n, (1,) * n, (5,) * n, m)
        cfg = spst.RunConfig(n_scales=2, mode="fast", extractor=vgg_spec)
        seen = []
        x = spst.multiscale_transfer(d["u"], d["v"], cfg, progress=lambda s, it, l, g: seen.append((s, it, l, g)))
        pl.make_schedule = lambda n, m="baseline": pl.Schedule(n, (3,) * n, (5,) * n, m)
        cfg_t = spst.RunConfig(n_scales=2, extractor=vgg_spec, lambda_c=0.0, seed=3)
        seen_t = []
        xt = spst.texture_synthesize(d["v"], cfg_t, progress=lambda s, it, l, g: seen_t.append((s, it, l, g)))
    finally:
        pl.make_schedule = orig
    _check_trace(seen, d["ms_trace"])
    _check_trace(seen_t, d["ts_trace"])
    mad = float(np.mean(np.abs(x - d["ms_x"])))
    mad_t = float(np.mean(np.abs(xt - d["ts_x"])))
    print(f"VGG-19 multiscale_transfer / texture_synthesize: final-image mean |diff| vs reference "
          f"{mad:.2e} / {mad_t:.2e} (bar {1 / 255:.2e})")
    assert mad <= 1.0 / 255 and mad_t <= 1.0 / 255
