"""CPU oracle for the localized Gatys transfer hot path — TEST INFRASTRUCTURE ONLY.

This module is a from-scratch NumPy restatement of the reference package `tilestyle`
(arXiv 2212.13459, "SPST"), used as the *checker* for the CUDA path:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
  ``--impl reference`` legs may import it;
* the product package ``paper_2212_13459_b200`` never imports it and has no CPU fallback.

Parity pinning: ``tools/make_goldens.py`` runs the real reference (importable read-only in
the build container from /root/reference/pkg/src) and writes ``tests/golden/*.npz``;
``tests/test_oracle_golden.py`` checks every function below against those vectors, so the
oracle is pinned to the reference's own outputs (not just to its description).

Every function cites the reference file:line it restates (paths relative to
/root/reference/pkg/src/tilestyle/).  Conventions follow the reference: images are HWC,
feature maps CHW, convolution is cross-correlation with zero "same" padding.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------------------------------
# network description (extractor.py:21-106, 318-345)
# ----------------------------------------------------------------------------------------


@dataclass(frozen=True)
class OLayer:
    kind: str            # "conv" | "relu" | "pool"
    name: str
    cin: int = 0
    cout: int = 0
    pool: str = "avg"
    w: np.ndarray | None = None   # (cout, cin, 3, 3)
    b: np.ndarray | None = None


@dataclass(frozen=True)
class ONet:
    layers: tuple
    style_taps: tuple
    content_tap: str
    order: str = "rgb"
    mean: tuple = (0.0, 0.0, 0.0)
    scale: tuple = (1.0, 1.0, 1.0)

    def index(self, name):
        for i, l in enumerate(self.layers):
            if l.name == name:
                return i
        raise KeyError(name)

    @property
    def taps(self):
        return tuple(dict.fromkeys((*self.style_taps, self.content_tap)))

    def last(self):
        return max(self.index(t) for t in self.taps)

    def geometry(self, tap):
        """(stride, rf_radius, channels) — extractor.py:217-237."""
        jump, rad, ch = 1, 0, 3
        for l in self.layers[: self.index(tap) + 1]:
            if l.kind == "conv":
                rad += jump
                ch = l.cout
            elif l.kind == "pool":
                jump *= 2
        return jump, rad, ch

    def deepest_stride(self):
        return max(self.geometry(t)[0] for t in self.taps)


def onet_from_spec(spec) -> ONet:
    """Adapt any tilestyle-like spec (reference or product) into the oracle's description."""
    layers = []
    for l in spec.layers:
        if l.kind == "conv":
            if getattr(l, "k", 3) != 3 or getattr(l, "stride", 1) != 1:
                raise ValueError("oracle restates 3x3 stride-1 convs only")
            layers.append(OLayer("conv", l.name, l.in_ch, l.out_ch,
                                 w=np.asarray(l.weight, np.float64), b=np.asarray(l.bias, np.float64)))
        elif l.kind == "relu":
            layers.append(OLayer("relu", l.name))
        else:
            if getattr(l, "k", 2) != 2:
                raise ValueError("oracle restates 2x2 pools only")
            layers.append(OLayer("pool", l.name, pool=l.pool))
    pre = spec.preprocess
    return ONet(tuple(layers), tuple(spec.style_taps), spec.content_tap,
                pre.channel_order, tuple(pre.mean), tuple(pre.scale))


# ----------------------------------------------------------------------------------------
# dense kernels (tensorops.py)
# ----------------------------------------------------------------------------------------

def conv3x3(x, w, b):
    """Cross-correlation, pad 1, stride 1, + bias (tensorops.py:33-55).

    Restated as a sum of nine shifted 1x1 contractions over a zero-padded copy.
    """
    c, h, wd = x.shape
    xp = np.zeros((c, h + 2, wd + 2), dtype=x.dtype)
    xp[:, 1:-1, 1:-1] = x
    wt = w.astype(x.dtype, copy=False)
    out = np.empty((w.shape[0], h, wd), dtype=x.dtype)
    acc = None
    for dy in range(3):
        for dx in range(3):
            win = xp[:, dy:dy + h, dx:dx + wd].reshape(c, -1)
            term = wt[:, :, dy, dx] @ win
            acc = term if acc is None else acc + term
    out[:] = acc.reshape(-1, h, wd)
    out += b.astype(x.dtype, copy=False)[:, None, None]
    return out


def conv3x3_input_grad(g, w):
    """Adjoint of conv3x3 wrt its input (tensorops.py:58-74): transposed taps, scattered."""
    o, h, wd = g.shape
    wt = w.astype(g.dtype, copy=False)
    gp = np.zeros((w.shape[1], h + 2, wd + 2), dtype=g.dtype)
    gf = g.reshape(o, -1)
    for dy in range(3):
        for dx in range(3):
            gp[:, dy:dy + h, dx:dx + wd] += (wt[:, :, dy, dx].T @ gf).reshape(-1, h, wd)
    return np.ascontiguousarray(gp[:, 1:-1, 1:-1])


def pool2_fwd(x, kind):
    """2x2 stride-2 pooling, floor dims (tensorops.py:91-101, 113-115)."""
    c, h, w = x.shape
    oh, ow = h // 2, w // 2
    if oh == 0 or ow == 0:
        raise ValueError("pool window larger than input")
    q = x[:, :2 * oh, :2 * ow].reshape(c, oh, 2, ow, 2)
    return q.mean(axis=(2, 4)) if kind == "avg" else q.max(axis=(2, 4))


def pool2_bwd(g, x_in, kind):
    """Adjoint of pool2_fwd (tensorops.py:104-110, 118-129): avg spreads g/4, max routes to
    the first row-major argmax; the ragged remainder row/col gets zero."""
    c, h, w = x_in.shape
    oh, ow = g.shape[1:]
    out = np.zeros((c, h, w), dtype=g.dtype)
    if kind == "avg":
        up = g / 4
        for i in range(2):
            for j in range(2):
                out[:, i:2 * oh:2, j:2 * ow:2] = up
        return out
    win = x_in[:, :2 * oh, :2 * ow].reshape(c, oh, 2, ow, 2).transpose(0, 1, 3, 2, 4).reshape(c, oh, ow, 4)
    arg = np.argmax(win, axis=3)
    for k in range(4):
        i, j = divmod(k, 2)
        out[:, i:2 * oh:2, j:2 * ow:2] = np.where(arg == k, g, 0)
    return out


def pad_edge16(img, m):
    """Replicate-pad right/bottom to a multiple of m (tensorops.py:201-209)."""
    h, w = img.shape[:2]
    ph, pw = (-h) % m, (-w) % m
    if ph == 0 and pw == 0:
        return img
    rows = np.concatenate([img, np.repeat(img[-1:], ph, axis=0)], axis=0) if ph else img
    return np.concatenate([rows, np.repeat(rows[:, -1:], pw, axis=1)], axis=1) if pw else rows


def fold_pad_grad(g, h, w):
    """Sum replicated-pixel gradients back onto the last row/col (tensorops.py:212-229)."""
    out = g[:h, :w].copy()
    if g.shape[0] > h:
        out[h - 1] += g[h:, :w].sum(axis=0)
    if g.shape[1] > w:
        out[:, w - 1] += g[:h, w:].sum(axis=1)
    if g.shape[0] > h and g.shape[1] > w:
        out[h - 1, w - 1] += g[h:, w:].sum(axis=(0, 1))
    return out


def area_down(img, f):
    """Box mean with ragged right/bottom boxes, out dims ceil (tensorops.py:136-155)."""
    if f == 1:
        return img.copy()
    h, w = img.shape[:2]
    oh, ow = -(-h // f), -(-w // f)
    acc = np.zeros((oh, ow) + img.shape[2:], dtype=np.float64)
    for i in range(oh):
        rs = img[i * f:min((i + 1) * f, h)].sum(axis=0, dtype=np.float64)
        for j in range(ow):
            acc[i, j] = rs[j * f:min((j + 1) * f, w)].sum(axis=0)
    bh = np.minimum(f, h - np.arange(oh) * f)
    bw = np.minimum(f, w - np.arange(ow) * f)
    area = (bh[:, None] * bw[None, :]).astype(np.float64)
    if img.ndim == 3:
        area = area[:, :, None]
    return (acc / area).astype(img.dtype)


def bilinear(img, oh, ow):
    """Half-pixel-centred bilinear with clamped sources (tensorops.py:158-185)."""
    h, w = img.shape[:2]

    def taps(n_in, n_out):
        s = (np.arange(n_out, dtype=np.float64) + 0.5) * (n_in / n_out) - 0.5
        s = np.clip(s, 0.0, n_in - 1.0)
        i0 = np.floor(s).astype(np.int64)
        return i0, np.minimum(i0 + 1, n_in - 1), (s - i0).astype(img.dtype)

    y0, y1, ty = taps(h, oh)
    x0, x1, tx = taps(w, ow)
    ex = (slice(None),) + (None,) * (img.ndim - 1)
    r = img[y0] * (1 - ty[ex]) + img[y1] * ty[ex]
    ex2 = (None, slice(None)) + (None,) * (img.ndim - 2)
    return (r[:, x0] * (1 - tx[ex2]) + r[:, x1] * tx[ex2]).astype(img.dtype)


# ----------------------------------------------------------------------------------------
# forward with taps / backward to pixels (extractor.py:151-214)
# ----------------------------------------------------------------------------------------

_PERM = {"rgb": (0, 1, 2), "bgr": (2, 1, 0)}


def preprocess(x_chw, net):
    perm = list(_PERM[net.order])
    m = np.asarray(net.mean, dtype=x_chw.dtype)[:, None, None]
    s = np.asarray(net.scale, dtype=x_chw.dtype)[:, None, None]
    return (x_chw[perm] - m) / s


def preprocess_adjoint(g, net):
    perm = list(_PERM[net.order])
    s = np.asarray(net.scale, dtype=g.dtype)[:, None, None]
    out = np.empty_like(g)
    out[perm] = g / s
    return out


def run_forward(x_chw, net, keep=False, masks=None):
    """Returns (taps, saved layer inputs or None). Stops at the deepest tap
    (extractor.py:171-197).  `masks` ({relu name: bool array}) forces the ReLU activation
    pattern (test hook: the f64 network evaluated on another engine's masks)."""
    names = set(net.taps)
    cur = preprocess(x_chw, net)
    taps, saved = {}, []
    for l in net.layers[: net.last() + 1]:
        if keep:
            saved.append(cur if masks is None or l.name not in masks else np.where(masks[l.name], 1.0, -1.0))
        if l.kind == "conv":
            cur = conv3x3(cur, l.w, l.b)
        elif l.kind == "relu":
            cur = np.maximum(cur, 0) if masks is None or l.name not in masks else cur * masks[l.name]
        else:
            cur = pool2_fwd(cur, l.pool)
        if l.name in names:
            taps[l.name] = cur
    return taps, (saved if keep else None)


def run_backward(tap_grads, saved, net):
    """Reverse pass from tap gradients to preprocessed-input gradient, then through the
    preprocessing (extractor.py:200-214)."""
    g = None
    for i in range(net.last(), -1, -1):
        l = net.layers[i]
        if l.name in tap_grads:
            g = tap_grads[l.name].copy() if g is None else g + tap_grads[l.name]
        if g is None:
            continue
        if l.kind == "conv":
            g = conv3x3_input_grad(g, l.w)
        elif l.kind == "relu":
            g = g * (saved[i] > 0)
        else:
            g = pool2_bwd(g, saved[i], l.pool)
    return preprocess_adjoint(g, net)


# ----------------------------------------------------------------------------------------
# statistics and feature-space gradients (stats.py)
# ----------------------------------------------------------------------------------------

STD_EPS = 1e-8


@dataclass
class OStats:
    gram: np.ndarray
    mean: np.ndarray
    std: np.ndarray
    n_p: int


class OAcc:
    """f64 running sums S=FF^T, s=sum F, n (stats.py:34-66)."""

    def __init__(self, c):
        self.S = np.zeros((c, c))
        self.s = np.zeros(c)
        self.n = 0

    def add(self, f):
        flat = f.reshape(f.shape[0], -1).astype(np.float64)
        self.S += flat @ flat.T
        self.s += flat.sum(axis=1)
        self.n += flat.shape[1]

    def merge(self, o):
        self.S += o.S
        self.s += o.s
        self.n += o.n

    def done(self):
        if self.n == 0:
            raise ValueError("empty accumulator")
        g = self.S / self.n
        mu = self.s / self.n
        return OStats(g, mu, np.sqrt(np.maximum(np.diagonal(g) - mu ** 2, 0.0)), self.n)


def stats_of(f):
    a = OAcc(f.shape[0])
    a.add(f)
    return a.done()


@dataclass(frozen=True)
class OW:
    gram: float
    mean: float
    std: float


def default_weights(net, lambda_c=1.0, factor=1e3):
    """stats.py:98-110."""
    out = {}
    for t in net.style_taps:
        c = net.geometry(t)[2]
        out[t] = OW(1.0 / c ** 2, factor / c ** 2, factor / c ** 2)
    return lambda_c, out


def style_terms(sx, sr, w):
    """stats.py:117-124."""
    return (w.gram * float(np.sum((sx.gram - sr.gram) ** 2)),
            w.mean * float(np.sum((sx.mean - sr.mean) ** 2)),
            w.std * float(np.sum((sx.std - sr.std) ** 2)))


def style_feature_grad(V, sx, sr, w):
    """Pointwise feature gradient given global stats (stats.py:127-165)."""
    dt = V.dtype
    n = sx.n_p
    out = np.zeros_like(V)
    if w.gram:
        d = (sx.gram - sr.gram).astype(dt)
        out += (4.0 * w.gram / n) * (d @ V.reshape(V.shape[0], -1)).reshape(V.shape)
    if w.mean:
        out += (2.0 * w.mean / n) * (sx.mean - sr.mean).astype(dt)[:, None, None]
    if w.std:
        dead = sx.std < STD_EPS
        ratio = np.where(dead, 0.0, (sx.std - sr.std) / np.where(dead, 1.0, sx.std)).astype(dt)
        out += (2.0 * w.std / n) * (V - sx.mean.astype(dt)[:, None, None]) * ratio[:, None, None]
    return out


# ----------------------------------------------------------------------------------------
# tiling (tiling.py:39-104, localized.py:116-120)
# ----------------------------------------------------------------------------------------

@dataclass(frozen=True)
class OBlock:
    ix: int
    iy: int
    iw: int
    ih: int
    px: int
    py: int
    pw: int
    ph: int
    left: int
    top: int


def blocks_of(H, W, block, margin):
    """Row-major inner rects tiling H x W, padded by the clipped margin (tiling.py:57-72)."""
    out = []
    for y0 in range(0, H, block):
        ih = min(block, H - y0)
        for x0 in range(0, W, block):
            iw = min(block, W - x0)
            l, t = min(margin, x0), min(margin, y0)
            r, b = min(margin, W - x0 - iw), min(margin, H - y0 - ih)
            out.append(OBlock(x0, y0, iw, ih, x0 - l, y0 - t, iw + l + r, ih + t + b, l, t))
    return out


def inner_crop(blk, stride):
    """Tap-space crop (tiling.py:75-88)."""
    return (blk.left // stride, blk.top // stride, -(-blk.iw // stride), -(-blk.ih // stride))


def exact_margin(net):
    """tiling.py:91-104."""
    s = net.deepest_stride()
    rf = max(net.geometry(t)[1] for t in net.taps)
    need = rf + s * ((rf + s - 1) // s)
    return -(-need // s) * s


def padded_dims(net, h, w):
    s = net.deepest_stride()
    return h + (-h) % s, w + (-w) % s


# ----------------------------------------------------------------------------------------
# Algorithm 1 (localized.py:162-311)
# ----------------------------------------------------------------------------------------

def _tile(xp, b):
    return np.ascontiguousarray(xp[b.py:b.py + b.ph, b.px:b.px + b.pw].transpose(2, 0, 1))


def _crop(t, c):
    x0, y0, w, h = c
    return t[:, y0:y0 + h, x0:x0 + w]


def stats_pass(img, net, block=512, margin=256, taps=None):
    """Blockwise global statistics (localized.py:162-184); blocks merged in order."""
    taps = tuple(taps) if taps is not None else net.style_taps
    s = net.deepest_stride()
    if block % s or margin % s or block < s:
        raise ValueError("block/margin must be multiples of the deepest stride")
    H, W = padded_dims(net, *img.shape[:2])
    xp = pad_edge16(img, s)
    tot = {t: OAcc(net.geometry(t)[2]) for t in taps}
    for b in blocks_of(H, W, block, margin):
        feats, _ = run_forward(_tile(xp, b), net)
        for t in taps:
            tot[t].add(_crop(feats[t], inner_crop(b, net.geometry(t)[0])))
    return {t: tot[t].done() for t in taps}


@dataclass
class OProblem:
    net: ONet
    lambda_c: float
    tw: dict
    H: int
    W: int
    block: int
    margin: int
    style: dict
    content_tiles: list | None
    content_img: np.ndarray | None
    _full: np.ndarray | None = field(default=None, repr=False)

    def content_full(self):
        if self._full is None:
            xp = pad_edge16(self.content_img, self.net.deepest_stride())
            self._full = run_forward(np.ascontiguousarray(xp.transpose(2, 0, 1)), self.net)[0][self.net.content_tap]
        return self._full


def build_problem(u, v, net, weights, block=512, margin=256, style_stats=None):
    """localized.py:187-220. weights = (lambda_c, {tap: OW})."""
    lam, tw = weights
    st = style_stats if style_stats is not None else stats_pass(v, net, block, margin)
    ref = u if lam > 0 else (u if u is not None else v)
    if lam > 0 and u is None:
        raise ValueError("content image required")
    H, W = padded_dims(net, *ref.shape[:2])
    tiles = None
    if lam > 0:
        up = pad_edge16(u, net.deepest_stride())
        tiles = [run_forward(_tile(up, b), net)[0][net.content_tap] for b in blocks_of(H, W, block, margin)]
    return OProblem(net, lam, tw, H, W, block, margin, st, tiles, u)


def loss_grad(x, p):
    """Two-pass blockwise loss and pixel gradient (localized.py:227-280)."""
    net = p.net
    h, w = x.shape[:2]
    if padded_dims(net, h, w) != (p.H, p.W):
        raise ValueError("image does not match the problem grid")
    s = net.deepest_stride()
    xp = pad_edge16(x, s)
    sx = stats_pass(x, net, p.block, p.margin)
    total = 0.0
    for t in net.style_taps:
        total += sum(style_terms(sx[t], p.style[t], p.tw[t]))
    gpad = np.zeros((p.H, p.W, 3), dtype=x.dtype)
    closs = 0.0
    ct = net.content_tap
    for i, b in enumerate(blocks_of(p.H, p.W, p.block, p.margin)):
        feats, saved = run_forward(_tile(xp, b), net, keep=True)
        tg = {t: style_feature_grad(feats[t], sx[t], p.style[t], p.tw[t]) for t in net.style_taps}
        if p.lambda_c > 0:
            diff = feats[ct] - p.content_tiles[i].astype(x.dtype, copy=False)
            closs += p.lambda_c * float(np.sum(_crop(diff, inner_crop(b, net.geometry(ct)[0])).astype(np.float64) ** 2))
            cg = (2.0 * p.lambda_c) * diff
            tg[ct] = tg[ct] + cg if ct in tg else cg
        gb = run_backward(tg, saved, net)
        gpad[b.iy:b.iy + b.ih, b.ix:b.ix + b.iw] = gb[:, b.top:b.top + b.ih, b.left:b.left + b.iw].transpose(1, 2, 0)
    return total + closs, fold_pad_grad(gpad, h, w)


def loss_grad_global(x, p, masks=None):
    """Single-pass whole-image oracle (localized.py:283-311). `masks`: see run_forward."""
    net = p.net
    h, w = x.shape[:2]
    xp = pad_edge16(x, net.deepest_stride())
    feats, saved = run_forward(np.ascontiguousarray(xp.transpose(2, 0, 1)), net, keep=True, masks=masks)
    total = 0.0
    tg = {}
    for t in net.style_taps:
        sx = stats_of(feats[t])
        total += sum(style_terms(sx, p.style[t], p.tw[t]))
        tg[t] = style_feature_grad(feats[t], sx, p.style[t], p.tw[t])
    ct = net.content_tap
    if p.lambda_c > 0:
        diff = feats[ct] - p.content_full().astype(x.dtype, copy=False)
        total += p.lambda_c * float(np.sum(diff.astype(np.float64) ** 2))
        cg = (2.0 * p.lambda_c) * diff
        tg[ct] = tg[ct] + cg if ct in tg else cg
    g = run_backward(tg, saved, net)
    return total, fold_pad_grad(np.ascontiguousarray(g.transpose(1, 2, 0)), h, w)


# ----------------------------------------------------------------------------------------
# L-BFGS (lbfgs.py:18-142)
# ----------------------------------------------------------------------------------------

CURVATURE_REJECT = 1e-10


class OHistory:
    def __init__(self):
        self.s, self.y, self.rho = [], [], []

    def push(self, s, y, m):
        ys = float(np.vdot(y, s))
        if ys <= CURVATURE_REJECT * float(np.linalg.norm(s.ravel()) * np.linalg.norm(y.ravel())):
            return False
        self.s.append(s)
        self.y.append(y)
        self.rho.append(1.0 / ys)
        while len(self.s) > m:
            self.drop()
        return True

    def drop(self):
        if self.s:
            del self.s[0], self.y[0], self.rho[0]


def direction(g, hist):
    q = g.copy()
    alpha = [0.0] * len(hist.s)
    for i in reversed(range(len(hist.s))):
        alpha[i] = hist.rho[i] * float(np.vdot(hist.s[i], q))
        q -= alpha[i] * hist.y[i]
    if hist.s:
        q *= float(np.vdot(hist.s[-1], hist.y[-1])) / float(np.vdot(hist.y[-1], hist.y[-1]))
    for i in range(len(hist.s)):
        beta = hist.rho[i] * float(np.vdot(hist.y[i], q))
        q += (alpha[i] - beta) * hist.s[i]
    return -q


def minimize(f, x0, m=10, max_iters=100, c1=1e-4, shrink=0.5, max_evals=25, grad_tol=1e-9,
             callback=None, eval_log=None):
    """Returns (x, losses, grad_norms). eval_log (list) receives every trial x if given."""
    x = np.array(x0, copy=True)
    loss, g = f(x)
    if not np.isfinite(loss):
        raise FloatingPointError("non-finite loss")
    losses, gn = [float(loss)], [float(np.abs(g).max())]
    hist = OHistory()
    for it in range(max_iters):
        gmax = float(np.abs(g).max())
        if gmax <= grad_tol:
            break
        d = direction(g, hist)
        gd = float(np.vdot(g, d))
        if gd >= 0:
            d = -g
            gd = float(np.vdot(g, d))
        t = 1.0 if hist.s else 1.0 / gmax
        ok = False
        for _ in range(max_evals):
            xt = x + t * d
            if eval_log is not None:
                eval_log.append(xt)
            lt, gt = f(xt)
            if not np.isfinite(lt):
                raise FloatingPointError("non-finite loss")
            if lt <= loss + c1 * t * gd:
                ok = True
                break
            t *= shrink
        if ok:
            hist.push(xt - x, gt - g, m)
            x, loss, g = xt, float(lt), gt
        else:
            hist.drop()
        losses.append(loss)
        gn.append(float(np.abs(g).max()))
        if callback is not None:
            callback(it + 1, x, loss, gn[-1])
    return x, losses, gn


# ----------------------------------------------------------------------------------------
# multiscale driver pieces (pipeline.py:50-69, 170-181)
# ----------------------------------------------------------------------------------------

def schedule(n, mode="baseline"):
    its = [600]
    for _ in range(n - 1):
        its.append(300 if mode == "baseline" else max(its[-1] // 3, 30))
    return tuple(its), (100,) + (10,) * (n - 1)


def scale_dims(h, w, n):
    return [(-(-h // 2 ** (n - s)), -(-w // 2 ** (n - s))) for s in range(1, n + 1)]


def lambda_for_scale(net, dims, lam=1.0):
    """Per-element content normalisation (pipeline.py:170-181)."""
    s_, _, c = net.geometry(net.content_tap)
    ph, pw = padded_dims(net, *dims)
    return lam / (c * (ph // s_) * (pw // s_))


# ----------------------------------------------------------------------------------------
# evaluation metrics (metrics.py:17-73)
# ----------------------------------------------------------------------------------------
def psnr(a, b):
    """metrics.py:24-31: 10 log10(1 / mean((a-b)^2)) in f64, +inf when identical."""
    err = np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64)
    mse = float(np.mean(err * err))
    return math.inf if mse == 0.0 else -10.0 * math.log10(mse)


def luma(img):
    """metrics.py:34-38 (Rec. 601).  The weights are Python floats, so an f32 image is weighted
    in f32 (NumPy weak-scalar promotion) and only then widened."""
    img = np.asarray(img)
    if img.ndim == 2:
        return img.astype(np.float64)
    dt = img.dtype.type if img.dtype in (np.float32, np.float64) else np.float64
    w = [dt(c) for c in (0.299, 0.587, 0.114)]
    x = img.astype(dt, copy=False)
    return ((w[0] * x[..., 0] + w[1] * x[..., 1]) + w[2] * x[..., 2]).astype(np.float64)


def ssim(a, b, win=11, sigma=1.5, k1=0.01, k2=0.03):
    """metrics.py:41-73: mean SSIM map of the luma, separable Gaussian window in valid mode."""
    t = np.arange(win, dtype=np.float64) - (win - 1) / 2.0
    g = np.exp(-t * t / (2.0 * sigma * sigma))
    g /= g.sum()

    def blur(f):  # valid-mode separable filter, rows then columns
        h, w = f.shape
        rows = sum(g[j] * f[j:h - win + 1 + j, :] for j in range(win))
        return sum(g[j] * rows[:, j:w - win + 1 + j] for j in range(win))

    x, y = luma(a), luma(b)
    mx, my = blur(x), blur(y)
    vx, vy, cxy = blur(x * x) - mx * mx, blur(y * y) - my * my, blur(x * y) - mx * my
    c1, c2 = k1 * k1, k2 * k2
    smap = ((2 * mx * my + c1) * (2 * cxy + c2)) / ((mx * mx + my * my + c1) * (vx + vy + c2))
    return float(smap.mean())
