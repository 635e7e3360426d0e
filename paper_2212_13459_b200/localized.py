"""Algorithm 1 on the device: global statistics, exact transfer loss and pixel gradient.

Drop-in for the reference localized module (reference localized.py:116-311): same names,
signatures, return types and errors.  The reference evaluates the loss block by block on
CPU (two passes over margin-padded blocks) so its memory stays bounded; with a margin of at
least ``margin_for_exact_gradient`` its result equals the whole-image gradient
(localized.py:1-14).  A B200 holds the whole 6048x8064 working set (~80 GB) in HBM, so the
device path evaluates the padded image in ONE forward (activations, masks and Gram partials
kept resident), finalises the global statistics, and runs ONE backward — no halo
recomputation and no second forward.  Multi-GPU runs split the rows into halo-padded stripes
(``distributed.py``); that is where the block/margin geometry reappears.
"""

from __future__ import annotations

import warnings
from contextlib import contextmanager
from dataclasses import dataclass, field

import numpy as np
import torch

from .device import Engine, engine_for, require_cuda
from .errors import ConfigError, DegenerateStdWarning
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


def _check_exact(spec, grid: BlockGrid):
    if len(partition(grid)) > 1 and grid.margin < margin_for_exact_gradient(spec):
        raise NotImplementedError(
            f"margin {grid.margin} is below the exact margin {margin_for_exact_gradient(spec)}: the reference "
            "result then depends on the block grid; the device path evaluates exact (whole-image) gradients only")


class DeviceContentStore:
    """Content-tap features of u live in HBM inside the engine (never spilled)."""
    spilled = False


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
    _content_epoch: int = field(default=-1, repr=False)
    _refs_epoch: int = field(default=-1, repr=False)

    @property
    def has_content(self) -> bool:
        return self.weights.lambda_c > 0


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


def _sums_to_stats(engine: Engine, t_index: int, count: int) -> LayerStats:
    S, s = engine.tap_sums(t_index)
    return finalize_sums(S.cpu().numpy().copy(), s.cpu().numpy().copy(), count)


# ------------------------------------------------------------------------------------------
# public API
# ------------------------------------------------------------------------------------------

def stats_pass(img, spec: ExtractorSpec, block: int = 512, margin: int = 256, threads: int = 1,
               taps=None) -> dict:
    """Global per-tap statistics of img (localized.py:162-184)."""
    taps = tuple(taps) if taps is not None else tuple(spec.style_taps)
    h, w = int(img.shape[0]), int(img.shape[1])
    grid = make_grid(spec, h, w, block, margin)
    _check_exact(spec, grid)
    eng = engine_for(spec)
    missing = [t for t in taps if t not in eng.style_taps]
    if missing:
        raise NotImplementedError(f"device statistics are computed at the style taps only, not {missing}")
    with eng.lock:
        eng.bind(h, w)
        eng.forward(to_device_image(img, eng.device))
        _meter(eng)
        out = {}
        for t in taps:
            i = eng.style_taps.index(t)
            out[t] = _sums_to_stats(eng, i, eng.owned_pixels(i))
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
    _check_exact(spec, grid)
    p = TransferProblem(extractor=spec, weights=weights, grid=grid, style_stats=style_stats,
                        content_store=store, content_image=content_img, threads=threads)
    p.engine = engine_for(spec)
    _prepare(p)
    return p


def _prepare(p: TransferProblem, h=None, w=None):
    """Bind the engine to the problem grid, (re)capture content and style references."""
    eng = p.engine
    if h is None:
        ref = p.content_image if p.content_image is not None else None
        if ref is not None:
            h, w = ref.shape[:2]
        else:
            s = p.extractor.deepest_stride()
            h, w = p.grid.image_h, p.grid.image_w
    eng.bind(int(h), int(w))
    # the engine holds ONE content target: re-capture when this problem's target is not the one
    # resident (another problem of the same dims may have captured its own since)
    if p.has_content and (p._content_epoch != eng.bind_epoch or getattr(eng, "_content_problem", None) is not p):
        eng.forward(to_device_image(p.content_image, eng.device))
        eng.capture_content()
        p._content_epoch = eng.bind_epoch
        eng._content_problem = p
    if getattr(eng, "_active_problem", None) is not p or p._refs_epoch != eng.bind_epoch:
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


class Evaluation:
    """Loss (and lazily the gradient) of one x on one problem — the line-search unit."""

    def __init__(self, p: TransferProblem):
        self.p = p

    def loss(self, x_dev: torch.Tensor) -> float:
        p, eng = self.p, self.p.engine
        h, w = int(x_dev.shape[0]), int(x_dev.shape[1])
        _prepare(p, h, w)
        eng.forward(x_dev)
        _meter(eng)
        counts = [eng.owned_pixels(i) for i in range(len(eng.style_taps))]
        content = eng.content_sqdiff() if p.has_content else None  # read after finalize's one sync
        terms, degenerate = eng.finalize(counts)
        if any(degenerate):
            warnings.warn("zero-std channel with nonzero reference std; its gradient column is zeroed",
                          DegenerateStdWarning, stacklevel=3)
        total = float(terms.sum())
        if content is not None:
            total += p.weights.lambda_c * float(content.item())
        return total

    def grad(self, out: torch.Tensor) -> torch.Tensor:
        p = self.p
        p.engine.backward(2.0 * p.weights.lambda_c if p.has_content else 0.0, out)
        return out


def loss_grad(x, p: TransferProblem):
    """Exact transfer loss and its pixel gradient (localized.py:227-280).

    numpy in -> (float, numpy of x's dtype); CUDA tensor in -> (float, float32 CUDA tensor).
    """
    _check_dims(x, p)
    with p.engine.lock:
        x_dev = to_device_image(x, p.engine.device)
        ev = Evaluation(p)
        loss = ev.loss(x_dev)
        g = torch.empty_like(x_dev)
        ev.grad(g)
    if isinstance(x, torch.Tensor):
        return loss, g
    return loss, g.cpu().numpy().astype(np.asarray(x).dtype, copy=False)


def loss_grad_global(x, p: TransferProblem):
    """Single-pass whole-image evaluation (localized.py:283-311) — on the device this is the
    same computation as ``loss_grad``."""
    return loss_grad(x, p)
