"""Size-independent properties of the hot path at BASELINE.json's full size (config C4's last
scale: content 6048x8064, style 4226x5319, VGG-19 to relu5_1), where the f64 oracle cannot run.

* the gradient is the derivative of the loss: central differences of our own loss along two
  directions agree with <g, d> (the loss is evaluated fp32-class, so the step is chosen to make
  the loss change ~1e-3 of the loss, far above its rounding, and the O(eps^2) term cancels);
* the memory-bounded windowed evaluation (two passes over halo tiles, as the reference's
  blockwise Algorithm 1 with the exact margin) equals the one-window evaluation.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2212_13459_b200 as spst  # noqa: E402
from paper_2212_13459_b200 import workloads  # noqa: E402
from paper_2212_13459_b200.pipeline import RunConfig, _weights_for_scale, objective_for  # noqa: E402
from conftest import rel_l2  # noqa: E402


@pytest.fixture(scope="module")
def c4():
    c = workloads.CONFIGS["c4"]
    H, W = c["content"]
    spec = spst.calibrated_vgg19(0)
    u = workloads.synth_content(H, W, 1)
    v = workloads.synth_style(*c["style"], 2)
    return spec, u, v, _weights_for_scale(RunConfig(extractor=spec), spec, (H, W))


def test_c4_gradient_is_the_derivative_of_the_loss(c4):
    spec, u, v, w = c4
    p = spst.build_problem(u, v, spec, w)
    obj = objective_for(p)
    rng = np.random.default_rng(5)
    x = torch.from_numpy(np.clip(u + 0.02 * rng.standard_normal(u.shape), 0, 1).astype(np.float32)).cuda()
    loss = obj.loss(x)
    g = torch.empty_like(x)
    obj.grad(g)
    assert np.isfinite(loss) and bool(torch.isfinite(g).all())
    gn = float(torch.linalg.vector_norm(g.double()))
    r = torch.from_numpy(rng.standard_normal(u.shape).astype(np.float32)).cuda()
    for name, d in (("gradient", g / gn), ("random", r / torch.linalg.vector_norm(r))):
        gd = float((g.double() * d.double()).sum())
        eps = 1e-3 * loss / gn  # loss change ~1e-3 of the loss along the gradient direction
        lp = obj.loss((x + eps * d).contiguous())
        lm = obj.loss((x - eps * d).contiguous())
        fd = (lp - lm) / (2 * eps)
        err = abs(fd - gd) / gn
        print(f"{name}: <g,d> {gd:.6e}  central difference {fd:.6e}  |diff|/|g| {err:.1e}")
        assert err <= 2e-3, (name, gd, fd)


def test_c4_memory_bounded_windows_equal_one_window(c4, monkeypatch):
    spec, u, v, w = c4
    rng = np.random.default_rng(6)
    x = np.clip(u + 0.02 * rng.standard_normal(u.shape), 0, 1).astype(np.float32)
    p = spst.build_problem(u, v, spec, w)
    assert len(p.windows) == 1
    l1, g1 = spst.loss_grad(x, p)
    del p
    monkeypatch.setenv("SPST_MAX_WINDOW_PX", str(4000 * 4500))
    pw = spst.build_problem(u, v, spec, w)
    assert len(pw.windows) > 1
    l2, g2 = spst.loss_grad(x, pw)
    print(f"{len(pw.windows)} windows vs one: loss rel {abs(l2 - l1) / l1:.1e}, grad rel-L2 {rel_l2(g2, g1):.1e}")
    assert abs(l2 - l1) <= 1e-5 * l1
    assert rel_l2(g2, g1) <= 1e-4
