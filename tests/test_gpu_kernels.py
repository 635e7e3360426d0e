"""Kernel-level numerics on the B200 through the C ABI (tensor-core conv / Gram, vector and
resampling kernels) vs fp64 references (torch fp64 for the convs, the oracle otherwise)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import spst_oracle as O  # noqa: E402
from paper_2212_13459_b200 import _native  # noqa: E402
import paper_2212_13459_b200 as spst  # noqa: E402
from conftest import golden, rel_l2  # noqa: E402

# every conv shape of VGG-19 (reduced spatial size) + TinyNet-like odd channel counts
SHAPES = [(64, 64), (64, 128), (128, 128), (128, 256), (256, 256), (256, 512), (512, 512), (8, 16), (16, 32)]


def _debug_conv(mode, x, w, b):
    cin, cout = w.shape[1], w.shape[0]
    H, W = x.shape[1:]
    ny = cout if mode != 2 else cin
    shape = (ny, H // 2, W // 2) if mode == 1 else (ny, H, W)
    y = np.zeros(shape, np.float32)
    x = np.ascontiguousarray(x, np.float32)
    w = np.ascontiguousarray(w, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    st = _native.lib().spst_debug_conv(0, mode, cin, cout, H, W, x.ctypes.data, w.ctypes.data, b.ctypes.data,
                                       y.ctypes.data)
    _native.check(st)
    return y


@pytest.mark.parametrize("cin,cout", SHAPES)
def test_conv_forward_relu_pool_backward_vs_fp64(cin, cout):
    F = torch.nn.functional
    rng = np.random.default_rng(cin * 1000 + cout)
    H, W = 18, 140  # ragged 128-px column block, odd row pair count
    x = rng.random((cin, H, W)).astype(np.float32)
    w = rng.normal(0, np.sqrt(2 / (9 * cin)), (cout, cin, 3, 3))
    b = rng.normal(0, 0.1, cout)
    xt, wt, bt = torch.from_numpy(x).double()[None], torch.from_numpy(w), torch.from_numpy(b)
    pre = F.conv2d(xt, wt, bt, padding=1)[0]
    y = _debug_conv(0, x, w, b)
    assert rel_l2(y, torch.relu(pre).numpy()) <= 2e-6
    yp = _debug_conv(1, x, w, b)
    assert rel_l2(yp, F.avg_pool2d(torch.relu(pre)[None], 2)[0].numpy()) <= 2e-6
    m = _debug_conv(3, x, w, b)
    assert np.mean(m != (pre > 0).numpy()) <= 1e-5  # mask flips only at |pre| ~ 1e-7
    g = rng.standard_normal((cout, H, W)).astype(np.float32)
    gx = _debug_conv(2, g, w, b)
    ref = F.conv_transpose2d(torch.from_numpy(g).double()[None], wt, padding=1)[0].numpy()
    assert rel_l2(gx, ref) <= 2e-6


def test_conv_matches_reference_kernel_golden():
    """Reference conv2d_forward / conv2d_backward_input known answers (tensorops.py:33-74)."""
    d = golden("kernels.npz")
    y = _debug_conv(0, d["conv_x"], d["conv_w"], d["conv_b"])
    np.testing.assert_allclose(y, np.maximum(d["conv_y"], 0), rtol=1e-5, atol=1e-5)
    gx = _debug_conv(2, d["conv_g"], d["conv_w"], d["conv_b"])
    np.testing.assert_allclose(gx, d["conv_gx"], rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("C,P", [(64, 5000), (128, 70000), (256, 9000), (512, 17000), (16, 300)])
def test_gram_vs_fp64(C, P):
    rng = np.random.default_rng(C + P)
    f = rng.random((C, P)).astype(np.float32)
    S = np.zeros((C, C))
    _native.check(_native.lib().spst_debug_gram(0, C, P, f.ctypes.data, S.ctypes.data))
    ref = f.astype(np.float64) @ f.astype(np.float64).T
    assert np.abs(S - ref).max() <= 2e-6 * np.abs(ref).max()
    np.testing.assert_array_equal(S, S.T)


def test_resampling_matches_reference_golden():
    from paper_2212_13459_b200 import resample
    d = golden("kernels.npz")
    img = d["img"]
    np.testing.assert_allclose(resample.resize_down(img, 3), d["down3"], rtol=2e-6, atol=1e-7)
    np.testing.assert_allclose(resample.resize_down(img, 8), d["down8"], rtol=2e-6, atol=1e-7)
    np.testing.assert_allclose(resample.resize_bilinear(img, (53, 41)), d["bil"], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(resample.resize_up2(img), d["up2"], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(resample.resize_up2(img, (73, 57)), d["up2t"], rtol=1e-6, atol=1e-7)
    # the reference test anchors: 6048x8064 / 8 -> 756x1008, factor 1 identity, constant image
    assert resample.resize_down(np.zeros((6048, 8064, 3), np.float32), 8).shape == (756, 1008, 3)
    c = np.full((20, 30, 3), 0.5, np.float32)
    np.testing.assert_array_equal(resample.resize_down(c, 4), np.full((5, 8, 3), 0.5, np.float32))
    np.testing.assert_array_equal(resample.resize_down(img, 1), img)
    np.testing.assert_allclose(resample.resize_up2(np.full((1, 1, 3), 0.25, np.float32)), np.full((2, 2, 3), 0.25))


def test_vector_kernels_f32_f64():
    from paper_2212_13459_b200.lbfgs import _Vec
    rng = np.random.default_rng(3)
    for dt in (torch.float32, torch.float64):
        a = torch.from_numpy(rng.standard_normal(100003)).to("cuda", dt)
        b = torch.from_numpy(rng.standard_normal(100003)).to("cuda", dt)
        v = _Vec(dt, a.device)
        d = v.dots((a, b), (a, a))
        an, bn = a.double().cpu().numpy(), b.double().cpu().numpy()
        assert d[0] == pytest.approx(float(an @ bn), rel=1e-12, abs=1e-9)
        assert d[1] == pytest.approx(float(an @ an), rel=1e-12)
        assert v.absmax(a) == pytest.approx(float(np.abs(an).max()))
        out = torch.empty_like(a)
        v.axpy(a, b, 0.37, out)
        ref = (a + torch.tensor(0.37, dtype=dt) * b).cpu().numpy()
        np.testing.assert_array_equal(out.cpu().numpy(), ref)
        s, y = torch.empty_like(a), torch.empty_like(a)
        ys, ss, yy = v.sy(a, b, b, a, s, y)
        sn, yn = s.double().cpu().numpy(), y.double().cpu().numpy()
        np.testing.assert_array_equal(sn, (a - b).cpu().numpy())
        assert ys == pytest.approx(float(yn @ sn), rel=1e-12)
        assert ss == pytest.approx(float(sn @ sn), rel=1e-12)


# ---------------------------------------------------------------- measurement hooks
@pytest.mark.gpu
def test_launch_counter_and_timer(tiny_spec):
    """spst_launch_count counts our kernels; the engine's launch timer brackets the tensor-core
    launches of an evaluation with events and reports algorithmic FLOPs (bench.py's roofline)."""
    from paper_2212_13459_b200 import _native as nat
    rng = np.random.default_rng(0)
    u, v, x = (rng.random((64, 96, 3)).astype(np.float32) for _ in range(3))
    p = spst.build_problem(u, v, tiny_spec, spst.default_loss_weights(tiny_spec))
    spst.loss_grad(x, p)  # warm (range exponents known)
    eng = p.engine
    n0 = int(nat.lib().spst_launch_count())
    eng.timing_enable(True)
    spst.loss_grad(x, p)
    t = eng.timing_read()
    eng.timing_enable(False)
    n1 = int(nat.lib().spst_launch_count())
    assert n1 - n0 >= 10
    assert set(t) <= {"conv3x3_tc<128>", "conv3x3_tc<64>", "gram_tc"} and "conv3x3_tc<64>" in t
    for ms, flops, n in t.values():
        assert ms > 0 and n > 0 and flops >= 0
    # disabled timer records nothing
    eng.timing_enable(False)
    spst.loss_grad(x, p)
    assert eng.timing_read() == {}


@pytest.mark.parametrize("dtype,n,m", [(torch.float32, 100003, 100), (torch.float64, 4099, 7), (torch.float32, 2_300_001, 10)])
def test_two_loop_native_equals_step_by_step(dtype, n, m):
    """spst_vec_two_loop (one cooperative launch) must equal the step-by-step kernels bit for
    bit (the step path is what multi-GPU runs use, with an all-reduce per dot product)."""
    from paper_2212_13459_b200.lbfgs import LBFGSState, _two_loop, _Vec
    g0 = torch.Generator(device="cuda").manual_seed(n + m)
    st = LBFGSState()
    for _ in range(m):
        s = torch.randn(n, dtype=dtype, device="cuda", generator=g0)
        y = s + 0.3 * torch.randn(n, dtype=dtype, device="cuda", generator=g0)
        assert st.push(s, y, m)
    g = torch.randn(n, dtype=dtype, device="cuda", generator=g0)
    vec = _Vec(dtype, g.device)
    d_native = _two_loop(g, st, vec, torch.empty_like(g))
    d_steps = _two_loop(g, st, vec, torch.empty_like(g), allreduce=lambda t, op="sum": t)
    torch.cuda.synchronize()
    assert torch.equal(d_native, d_steps)
    assert torch.isfinite(d_native).all()
