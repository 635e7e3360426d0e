"""Windowed evaluation (engine spst_bind_window): the reference's block grid reproduced block
by block when its margin is below the exact margin (reference localized.py:227-280; the result
then depends on the grid, test_localized.py:72-78), memory-bounded halo tiles when the image
does not fit, and stats_pass at any tap of the spec (localized.py:162-184).  Goldens:
tests/golden/blocks.npz, written by tools/make_goldens.py from the real reference."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2212_13459_b200 as spst  # noqa: E402
from conftest import golden, rel_l2  # noqa: E402


@pytest.mark.parametrize("m", [0, 8])
def test_tinynet_inexact_margin_matches_reference_blocks(tiny_spec, m):
    d = golden("blocks.npz")
    w = spst.default_loss_weights(tiny_spec)
    p = spst.build_problem(d["tiny_u"], d["tiny_v"], tiny_spec, w, block=64, margin=m)
    assert len(p.windows) == len(spst.partition(p.grid)) > 1
    loss, g = spst.loss_grad(d["tiny_x"], p)
    ref = d[f"tiny_m{m}_grad"]
    print(f"margin {m}: loss rel {abs(loss - d[f'tiny_m{m}_loss'][0]) / d[f'tiny_m{m}_loss'][0]:.1e}, "
          f"grad rel-L2 vs reference blocks {rel_l2(g, ref):.1e} "
          f"(vs the global gradient {rel_l2(ref, d['tiny_global_grad']):.1e})")
    assert abs(loss - d[f"tiny_m{m}_loss"][0]) <= 1e-5 * d[f"tiny_m{m}_loss"][0]
    assert rel_l2(g, ref) <= 1e-5
    if m == 0:  # the whole-image entry point ignores the grid (golden problem: margin-0 style stats)
        lg, gg = spst.loss_grad_global(d["tiny_x"], p)
        assert abs(lg - d["tiny_global_loss"][0]) <= 1e-5 * d["tiny_global_loss"][0]
        assert rel_l2(gg, d["tiny_global_grad"]) <= 1e-5
    st = spst.stats_pass(d["tiny_x"], tiny_spec, block=64, margin=m)
    for t in tiny_spec.style_taps:
        assert rel_l2(st[t].gram, d[f"tiny_m{m}_{t}_gram"]) <= 1e-5
        assert rel_l2(st[t].mean, d[f"tiny_m{m}_{t}_mean"]) <= 1e-5


def test_vgg19_inexact_margin_matches_reference_blocks(vgg_spec):
    d = golden("blocks.npz")
    w = spst.default_loss_weights(vgg_spec, lambda_c=float(d["vgg_lambda_c"][0]))
    p = spst.build_problem(d["vgg_u"], d["vgg_v"], vgg_spec, w, block=48, margin=16)
    loss, g = spst.loss_grad(d["vgg_x"], p)
    err = rel_l2(g, d["vgg_m16_grad"])
    print(f"VGG block 48 margin 16 ({len(p.windows)} blocks): loss rel "
          f"{abs(loss - d['vgg_m16_loss'][0]) / d['vgg_m16_loss'][0]:.1e}, grad rel-L2 {err:.1e}")
    assert abs(loss - d["vgg_m16_loss"][0]) <= 1e-5 * d["vgg_m16_loss"][0]
    assert err <= 1e-3


def test_stats_pass_at_any_spec_tap(tiny_spec, vgg_spec):
    d = golden("blocks.npz")
    st = spst.stats_pass(d["tiny_x"], tiny_spec, block=64, margin=16, taps=("relu1", "relu3"))
    for t in ("relu1", "relu3"):
        assert rel_l2(st[t].gram, d[f"tiny_taps_{t}_gram"]) <= 1e-5
        assert rel_l2(st[t].std, d[f"tiny_taps_{t}_std"]) <= 1e-5
    st = spst.stats_pass(d["vgg_x"], vgg_spec, taps=("relu4_2", "relu1_1"))  # relu4_2: the content tap
    for t in ("relu4_2", "relu1_1"):
        assert rel_l2(st[t].gram, d[f"vgg_taps_{t}_gram"]) <= 1e-5, t
        assert rel_l2(st[t].mean, d[f"vgg_taps_{t}_mean"]) <= 1e-5, t
        assert rel_l2(st[t].std, d[f"vgg_taps_{t}_std"]) <= 1e-5, t
    with pytest.raises(NotImplementedError):
        spst.stats_pass(d["vgg_x"], vgg_spec, taps=("conv1_1",))


def test_memory_bounded_tiles_equal_whole_image(vgg_spec, monkeypatch):
    """Exact margin, image 'too big' for the device (SPST_MAX_WINDOW_PX = 448^2 < 640 x 512): 128-px tiles
    with the 160-px exact margin, evaluated in two passes, give the whole-image loss and
    gradient, and the bound workspace stays at one tile's."""
    from paper_2212_13459_b200 import workloads
    u = workloads.synth_content(640, 512, 21)
    v = workloads.synth_style(256, 256, 22)
    x = np.clip(u + 0.03 * np.random.default_rng(2).standard_normal(u.shape), 0, 1).astype(np.float32)
    w = spst.default_loss_weights(vgg_spec, lambda_c=1e-4)
    p = spst.build_problem(u, v, vgg_spec, w)
    assert len(p.windows) == 1
    with spst.track_activations() as m1:
        l1, g1 = spst.loss_grad(x, p)
    monkeypatch.setenv("SPST_MAX_WINDOW_PX", str(448 ** 2))
    pw = spst.build_problem(u, v, vgg_spec, w)
    assert len(pw.windows) == 20  # 128-px tiles of the 640 x 512 image
    with spst.track_activations() as m2:
        l2, g2 = spst.loss_grad(x, pw)
    print(f"20 tiles vs whole image: loss rel {abs(l2 - l1) / l1:.1e}, grad rel-L2 {rel_l2(g2, g1):.1e}; "
          f"peak workspace {m2.peak / 1e6:.0f} MB vs {m1.peak / 1e6:.0f} MB whole")
    assert abs(l2 - l1) <= 1e-5 * l1
    assert rel_l2(g2, g1) <= 1e-4
    assert m2.peak < m1.peak
