"""Algorithm 1 on the device: global statistics, transfer loss and pixel gradient.

Drop-in for the reference localized module (reference localized.py:116-311): same names,
signatures, return types and errors.  The reference evaluates the loss block by block on CPU
(two passes over margin-padded blocks) so its memory stays bounded; with a margin of at least
``margin_for_exact_gradient`` its result equals the whole-image gradient (localized.py:1-14).

The device evaluates a list of WINDOWS, each a padded rectangle evaluated as one zero-padded
image that owns an inner rectangle (statistics, content loss and gradient are restricted to
the owned pixels; engine binding ``spst_bind_window``):

* exact margin and the padded image fits the device: ONE window, the whole image -- one
  forward (activations, masks and Gram partials kept resident), finalize, one backward; no
  halo recomputation and no second forward;
* exact margin but the image does not fit (beyond ~2x the C4 area on one B200): halo-padded
  tiles sized to the free memory, two passes like the reference -- memory bounded by a tile;
* a margin below the exact margin: the reference's own block grid, block by block, so the
  grid-dependent result is reproduced (reference test_localized.py:72-78).

Multi-GPU runs give each rank one window (``distributed.py``).
"""

from __future__ import annotations

import math
import os
import warnings
from contextlib import contextmanager
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from .device import Engine, engine_for, require_cuda
from .errors import ConfigError, DegenerateStdWarning, PrecisionWarning
from .spec import ExtractorSpec, tap_geometry
from .stats import LayerStats, LossWeights, finalize_sums
from .tiling import BlockGrid, margin_for_exact_gradient, partition


# ------------------------------------------------------------------------------------------
# activation accounting (reference localized.py:39-77): reports device workspace bytes
# ------------------------------------------------------------------------------------------

class ActivationMeter:
    def __init__(self):
        self.current = 0
        self.peak = 0

    def add(self, nbytes: int) -> None:
        self.current += nbytes
        self.peak = max(self.peak, self.current)

    def release(self, nbytes: int) -> None:
        self.current -= nbytes


_active_meter: ActivationMeter | None = None


@contextmanager
def track_activations():
    global _active_meter
    meter = ActivationMeter()
    prev, _active_meter = _active_meter, meter
    try:
        yield meter
    finally:
        _active_meter = prev


def _meter(engine: Engine):
    if _active_meter is not None:
        n = engine.workspace_bytes()
        _active_meter.add(n)
        _active_meter.release(n)


# ------------------------------------------------------------------------------------------
# geometry + problem
# ------------------------------------------------------------------------------------------

def make_grid(spec: ExtractorSpec, h: int, w: int, block: int, margin: int) -> BlockGrid:
    """Grid over the stride-padded dims of an h x w image (localized.py:116-120)."""
    s = spec.deepest_stride()
    return BlockGrid(image_h=h + (-h) % s, image_w=w + (-w) % s, block=block, margin=margin, stride=s)


def _is_exact(spec, grid: BlockGrid) -> bool:
    return len(partition(grid)) == 1 or grid.margin >= margin_for_exact_gradient(spec)


_BPP: dict = {}


def _bytes_per_px(eng) -> float:
    """Bound workspace of the engine per padded pixel, measured once by binding a 512^2 probe
    (VGG-19: ~1.65 KB)."""
    hit = _BPP.get(id(eng))
    if hit is None:
        prev = eng.bound
        eng.bind(512, 512)
        hit = _BPP[id(eng)] = eng.workspace_bytes() / (512 * 512)
        if prev is not None:
            eng.bind(prev[0], prev[1], *prev[2:])
    return hit


def _window_budget_px(eng) -> int:
    env = os.environ.get("SPST_MAX_WINDOW_PX")
    if env:
        return int(env)
    free, _ = torch.cuda.mem_get_info(eng.device)
    held = eng.workspace_bytes()  # the current binding is released before a new one
    return int(0.8 * (free + held) / _bytes_per_px(eng))


def plan_windows(spec, grid: BlockGrid, eng) -> list:
    """Windows (grid rows, owned rows, grid cols, owned cols) in padded-image coordinates."""
    Hp, Wp = grid.image_h, grid.image_w
    if _is_exact(spec, grid):
        budget = _window_budget_px(eng)
        if Hp * Wp <= budget:
            return [((0, Hp), (0, Hp), (0, Wp), (0, Wp))]
        m = margin_for_exact_gradient(spec)
        s = spec.deepest_stride()
        block = max(s, (int(math.sqrt(budget)) - 2 * m) // s * s)
        blocks = partition(BlockGrid(Hp, Wp, block, m, s))
    else:
        blocks = partition(grid)
    return [((b.padded.y0, b.padded.y1), (b.inner.y0, b.inner.y1), (b.padded.x0, b.padded.x1),
             (b.inner.x0, b.inner.x1)) for b in blocks]


class DeviceContentStore:
    """Content-tap features of u live in HBM (never spilled): inside the engine for a
    whole-image problem, one target per window otherwise (reference ContentStore,
    localized.py:84-109)."""
    spilled = False

    def __init__(self):
        self.targets = None  # per-window (device bytes, scale) in windowed mode


@dataclass
class TransferProblem:
    extractor: ExtractorSpec
    weights: LossWeights
    grid: BlockGrid
    style_stats: dict
    content_store: DeviceContentStore | None
    content_image: np.ndarray | None
    threads: int = 1
    engine: Engine | None = field(default=None, repr=False)
    windows: list = field(default_factory=list, repr=False)
    _content_epoch: int = field(default=-1, repr=False)
    _refs_epoch: int = field(default=-1, repr=False)

    @property
    def has_content(self) -> bool:
        return self.weights.lambda_c > 0

    @property
    def windowed(self) -> bool:
        return len(self.windows) > 1


# ------------------------------------------------------------------------------------------
# host <-> device helpers
# ------------------------------------------------------------------------------------------

def to_device_image(x, device=None) -> torch.Tensor:
    """(h, w, 3) image as a contiguous float32 CUDA tensor (uploads numpy inputs)."""
    require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    if isinstance(x, torch.Tensor):
        t = x.to(device=dev, dtype=torch.float32)
    else:
        a = np.asarray(x)
        if a.ndim != 3 or a.shape[2] != 3:
            from .errors import ShapeError
            raise ShapeError(f"image must be (h, w, 3), got {a.shape}")
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev, non_blocking=False)
    return t.contiguous()


def _tap_counts(spec, Hp, Wp, taps):
    return [(Hp // tap_geometry(spec, t).stride) * (Wp // tap_geometry(spec, t).stride) for t in taps]


def _window_sums(eng, x_dev, h, w, windows, n_taps):
    """Forward of every window in order; per-tap owned-pixel sums added in window order (f64 on
    the device: the block-order merge of reference localized.py:180-183)."""
    tot = None
    for win in windows:
        eng.bind(h, w, *_bind_args(win))
        eng.forward(x_dev)
        _meter(eng)
        part = [eng.tap_sums(i) for i in range(n_taps)]
        if tot is None:
            tot = [(S.clone(), sv.clone()) for S, sv in part]
        else:
            for (S, sv), (a, b) in zip(tot, part):
                S += a
                sv += b
    return tot


def _bind_args(win):
    (g0, g1), (o0, o1), (c0, c1), (oc0, oc1) = win
    return (g0, g1), (o0, o1), (c0, c1), (oc0, oc1)


_TAP_SPECS: dict = {}


def _spec_for_taps(spec: ExtractorSpec, taps: tuple) -> ExtractorSpec:
    """A spec whose style taps are `taps` (the engine computes statistics at style taps)."""
    if set(taps) <= set(spec.style_taps):
        return spec
    kinds = {l.name: l.kind for l in spec.layers}
    bad = [t for t in taps if kinds.get(t) != "relu"]
    if bad:
        raise NotImplementedError(f"device statistics are computed at relu outputs only, not {bad}")
    key = (id(spec), taps)
    hit = _TAP_SPECS.get(key)
    if hit is None or hit[0] is not spec:
        hit = _TAP_SPECS[key] = (spec, replace(spec, style_taps=tuple(taps)))
    return hit[1]


# ------------------------------------------------------------------------------------------
# public API
# ------------------------------------------------------------------------------------------

def stats_pass(img, spec: ExtractorSpec, block: int = 512, margin: int = 256, threads: int = 1,
               taps=None) -> dict:
    """Global per-tap statistics of img (localized.py:162-184), at any relu taps."""
    taps = tuple(taps) if taps is not None else tuple(spec.style_taps)
    _warn_f64(img)
    h, w = int(img.shape[0]), int(img.shape[1])
    grid = make_grid(spec, h, w, block, margin)
    run_spec = _spec_for_taps(spec, taps)
    eng = engine_for(run_spec)
    with eng.lock:
        windows = plan_windows(spec, grid, eng)
        x_dev = to_device_image(img, eng.device)
        tot = _window_sums(eng, x_dev, h, w, windows, len(eng.style_taps))
        counts = _tap_counts(spec, grid.image_h, grid.image_w, eng.style_taps)
        out = {}
        for t in taps:
            i = eng.style_taps.index(t)
            S, sv = tot[i]
            out[t] = finalize_sums(S.cpu().numpy().copy(), sv.cpu().numpy().copy(), counts[i])
    return out


def build_problem(content_img, style_img, spec: ExtractorSpec, weights: LossWeights, block: int = 512,
                  margin: int = 256, threads: int = 1, content_budget_bytes: int = 256 << 20,
                  style_stats: dict | None = None) -> TransferProblem:
    """Style statistics of v + content features of u (localized.py:187-220)."""
    if style_stats is None:
        style_stats = stats_pass(style_img, spec, block=block, margin=margin, threads=threads)
    for t in spec.style_taps:
        if style_stats[t].channels != tap_geometry(spec, t).channels:
            raise ConfigError(f"style stats for {t} have {style_stats[t].channels} channels, "
                              f"tap has {tap_geometry(spec, t).channels}")
    if weights.lambda_c > 0:
        if content_img is None:
            raise ConfigError("content image required when the content weight is nonzero")
        ref = content_img
        store = DeviceContentStore()
    else:
        ref = content_img if content_img is not None else style_img
        store = None
    grid = make_grid(spec, ref.shape[0], ref.shape[1], block, margin)
    p = TransferProblem(extractor=spec, weights=weights, grid=grid, style_stats=style_stats,
                        content_store=store, content_image=content_img, threads=threads)
    p.engine = engine_for(spec)
    with p.engine.lock:
        p.windows = plan_windows(spec, grid, p.engine)
        if p.windowed and p.has_content:  # one content target per window (reference ContentStore tiles)
            u_dev = to_device_image(content_img, p.engine.device)
            h, w = int(content_img.shape[0]), int(content_img.shape[1])
            targets = []
            for win in p.windows:
                p.engine.bind(h, w, *_bind_args(win))
                p.engine.forward(u_dev)
                p.engine.capture_content()
                targets.append(p.engine.content_target())
            store.targets = targets
        _prepare(p)
    return p


def _prepare(p: TransferProblem, h=None, w=None, whole=False):
    """Bind the engine (whole-image problems), (re)capture content, install style references."""
    eng = p.engine
    if h is None:
        ref = p.content_image if p.content_image is not None else None
        if ref is not None:
            h, w = ref.shape[:2]
        else:
            h, w = p.grid.image_h, p.grid.image_w
    if not p.windowed or whole:
        eng.bind(int(h), int(w))
        # the engine holds ONE content target: re-capture when this problem's target is not the
        # one resident (another problem of the same dims may have captured its own since)
        if p.has_content and (p._content_epoch != eng.bind_epoch or getattr(eng, "_content_problem", None) is not p):
            eng.forward(to_device_image(p.content_image, eng.device))
            eng.capture_content()
            p._content_epoch = eng.bind_epoch
            eng._content_problem = p
    if getattr(eng, "_active_problem", None) is not p or p._refs_epoch != eng.bind_epoch or p.windowed:
        for i, t in enumerate(eng.style_taps):
            eng.set_style_ref(i, p.style_stats[t], p.weights.style[t])
        eng._active_problem = p
        p._refs_epoch = eng.bind_epoch


def _check_dims(x, p: TransferProblem):
    h, w = int(x.shape[0]), int(x.shape[1])
    g = make_grid(p.extractor, h, w, p.grid.block, p.grid.margin)
    if (g.image_h, g.image_w) != (p.grid.image_h, p.grid.image_w):
        raise ConfigError(f"image {h}x{w} does not match the problem grid {p.grid.image_h}x{p.grid.image_w}")
    return h, w


def _warn_degenerate(degenerate):
    if any(degenerate):
        warnings.warn("zero-std channel with nonzero reference std; its gradient column is zeroed",
                      DegenerateStdWarning, stacklevel=4)


class Evaluation:
    """Loss (and lazily the gradient) of one x on one problem — the line-search unit.

    Whole-image problems: one forward + finalize for the loss, one backward for the gradient.
    Windowed problems (reference localized.py:227-280, two passes): the loss pass forwards every
    window and merges the statistics; the gradient pass re-runs each window's forward, installs
    the global statistics, and back-propagates its owned pixels."""

    def __init__(self, p: TransferProblem, whole: bool = False):
        self.p = p
        self.whole = whole or not p.windowed
        self._x = None
        self._global = None

    def loss(self, x_dev: torch.Tensor) -> float:
        p, eng = self.p, self.p.engine
        h, w = int(x_dev.shape[0]), int(x_dev.shape[1])
        _prepare(p, h, w, whole=self.whole)
        if self.whole:
            eng.forward(x_dev)
            _meter(eng)
            counts = eng.owned_counts()
            content = eng.content_sqdiff() if p.has_content else None
            if content is not None:  # copied behind the pass: read after finalize's one sync
                cpin = eng.pinned_scalar()
                cpin.copy_(content, non_blocking=True)
            terms, degenerate = eng.finalize(counts)
            _warn_degenerate(degenerate)
            total = float(terms.sum())
            if content is not None:
                if eng.forward_redone():  # the forward was re-run in careful mode
                    cval = float(eng.content_sqdiff().item())
                else:
                    cval = float(cpin[0])
                total += p.weights.lambda_c * cval
            return total
        # windowed: pass 1 (statistics of every window, content loss of every owned crop)
        T = len(eng.style_taps)
        tot, closs = None, None
        for wi, win in enumerate(p.windows):
            eng.bind(h, w, *_bind_args(win))
            eng.forward(x_dev)
            _meter(eng)
            part = [eng.tap_sums(i) for i in range(T)]
            tot = [(S.clone(), sv.clone()) for S, sv in part] if tot is None else tot
            if wi:
                for (S, sv), (a, b) in zip(tot, part):
                    S += a
                    sv += b
            if p.has_content:
                eng.set_content_target(p.content_store.targets[wi])
                c = eng.content_sqdiff().clone()
                closs = c if closs is None else closs + c
        self._global = tot
        self._x = x_dev
        terms, degenerate = self._finalize_global()
        _warn_degenerate(degenerate)
        total = float(terms.sum())
        if closs is not None:
            total += p.weights.lambda_c * float(closs.item())
        return total

    def _finalize_global(self):
        eng, p = self.p.engine, self.p
        for i, (S, sv) in enumerate(self._global):
            dS, ds = eng.tap_sums(i)
            dS.copy_(S)
            ds.copy_(sv)
        return eng.finalize(_tap_counts(p.extractor, p.grid.image_h, p.grid.image_w, eng.style_taps))

    def grad(self, out: torch.Tensor, defer: bool = False) -> torch.Tensor:
        """Gradient of the last ``loss`` point into ``out``.  defer=True (whole-image problems):
        launch only; ``grad_resolve`` settles the backward's range check."""
        p, eng = self.p, self.p.engine
        two_lambda = 2.0 * p.weights.lambda_c if p.has_content else 0.0
        if self.whole:
            eng.backward(two_lambda, out, defer=defer)
            return out
        # windowed: pass 2 (reference localized.py:246-278)
        x_dev = self._x
        h, w = int(x_dev.shape[0]), int(x_dev.shape[1])
        for wi, win in enumerate(p.windows):
            eng.bind(h, w, *_bind_args(win))
            eng.forward(x_dev)
            self._finalize_global()
            if p.has_content:
                eng.set_content_target(p.content_store.targets[wi])
            eng.backward(two_lambda, out)
        return out

    def grad_resolve(self) -> bool:
        """Settle a deferred gradient; True if it was rewritten (work launched on it is stale)."""
        return self.p.engine.backward_resolve() if self.whole else False


def loss_grad(x, p: TransferProblem):
    """Transfer loss and its pixel gradient on the problem's block grid (localized.py:227-280).

    numpy in -> (float, numpy of x's dtype); CUDA tensor in -> (float, float32 CUDA tensor).
    """
    return _loss_grad(x, p, whole=False)


def _warn_f64(x):
    dt = x.dtype if isinstance(x, torch.Tensor) else np.asarray(x).dtype
    if dt in (np.float64, torch.float64):
        warnings.warn("float64 input: the device network runs in fp32-class arithmetic (fp16x3 operands, "
                      "compensated fp32 accumulation, f64 statistics); results are returned as float64",
                      PrecisionWarning, stacklevel=3)


def _loss_grad(x, p: TransferProblem, whole: bool):
    _check_dims(x, p)
    _warn_f64(x)
    with p.engine.lock:
        x_dev = to_device_image(x, p.engine.device)
        ev = Evaluation(p, whole=whole)
        loss = ev.loss(x_dev)
        g = torch.empty_like(x_dev)
        ev.grad(g)
    if isinstance(x, torch.Tensor):
        return loss, g
    return loss, g.cpu().numpy().astype(np.asarray(x).dtype, copy=False)


def loss_grad_global(x, p: TransferProblem):
    """Single-pass whole-image evaluation (localized.py:283-311): independent of the block grid,
    equal to ``loss_grad`` whenever the margin is exact."""
    return _loss_grad(x, p, whole=True)
