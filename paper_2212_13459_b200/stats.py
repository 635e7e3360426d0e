"""Style statistics records, loss weights and the host-side accumulator API.

Mirrors the reference stats module's public data model (reference stats.py:22-124,
181-200): ``LayerStats``, ``StatsAccumulator`` (f64 merge/finalize), ``TapWeights``,
``LossWeights``, ``default_loss_weights``, ``style_loss_terms`` and the stats file format.
On the device path the per-pixel work (Gram contraction, feature gradients) runs in
libspst.so; what remains here is the O(C^2) host bookkeeping of finalised statistics.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np

from . import formats
from .errors import EmptyError, ShapeError

STD_EPS = 1e-8  # stats.py:19


@dataclass(frozen=True)
class LayerStats:
    gram: np.ndarray   # (n_c, n_c)
    mean: np.ndarray   # (n_c,)
    std: np.ndarray    # (n_c,)
    n_p: int

    @property
    def channels(self) -> int:
        return self.mean.shape[0]


def finalize_sums(S: np.ndarray, s: np.ndarray, n: int) -> LayerStats:
    """G = S/n, mu = s/n, std = sqrt(max(diag G - mu^2, 0)) (stats.py:59-66)."""
    if n == 0:
        raise EmptyError("no feature pixels accumulated")
    gram = S / n
    mean = s / n
    var = np.maximum(np.diagonal(gram) - mean ** 2, 0.0)
    return LayerStats(gram=gram, mean=mean, std=np.sqrt(var), n_p=int(n))


class StatsAccumulator:
    """Streaming f64 sums (stats.py:34-66); device partials merge into it."""

    def __init__(self, channels: int):
        self.channels = channels
        self.sum_outer = np.zeros((channels, channels))
        self.sum = np.zeros(channels)
        self.count = 0

    def accumulate(self, features: np.ndarray) -> None:
        if features.ndim != 3 or features.shape[0] != self.channels:
            raise ShapeError(f"expected ({self.channels},h,w) features, got {features.shape}")
        flat = features.reshape(self.channels, -1).astype(np.float64, copy=False)
        self.sum_outer += flat @ flat.T
        self.sum += flat.sum(axis=1)
        self.count += flat.shape[1]

    def add_sums(self, S: np.ndarray, s: np.ndarray, n: int) -> None:
        self.sum_outer += S
        self.sum += s
        self.count += int(n)

    def merge(self, other: "StatsAccumulator") -> None:
        if other.channels != self.channels:
            raise ShapeError(f"cannot merge {other.channels}-channel stats into {self.channels}")
        self.add_sums(other.sum_outer, other.sum, other.count)

    def finalize(self) -> LayerStats:
        return finalize_sums(self.sum_outer, self.sum, self.count)


@dataclass(frozen=True)
class TapWeights:
    gram: float
    mean: float
    std: float


@dataclass(frozen=True)
class LossWeights:
    lambda_c: float
    style: dict

    def __post_init__(self):
        vals = [self.lambda_c] + [v for w in self.style.values() for v in (w.gram, w.mean, w.std)]
        if any(v < 0 for v in vals):
            raise ShapeError("loss weights must be >= 0")
        if not any(v > 0 for v in vals):
            warnings.warn("all loss weights are zero; the objective is identically 0", stacklevel=2)


def default_loss_weights(spec, lambda_c: float = 1.0, mean_std_factor: float = 1e3) -> LossWeights:
    """w_gram = 1/n_c^2, w_mean = w_std = factor/n_c^2 (stats.py:98-110)."""
    from .spec import tap_geometry
    style = {}
    for t in spec.style_taps:
        c = tap_geometry(spec, t).channels
        style[t] = TapWeights(1.0 / c ** 2, mean_std_factor / c ** 2, mean_std_factor / c ** 2)
    return LossWeights(lambda_c=lambda_c, style=style)


def style_loss_terms(sx: LayerStats, sr: LayerStats, w: TapWeights) -> tuple:
    """(w_g |G-G_ref|^2, w_m |mu-mu_ref|^2, w_s |std-std_ref|^2) (stats.py:117-124)."""
    if sx.channels != sr.channels:
        raise ShapeError(f"stats have {sx.channels} vs {sr.channels} channels")
    return (w.gram * float(np.sum((sx.gram - sr.gram) ** 2)),
            w.mean * float(np.sum((sx.mean - sr.mean) ** 2)),
            w.std * float(np.sum((sx.std - sr.std) ** 2)))


def save_stats(path, stats: dict) -> None:
    recs = {}
    for tap, s in stats.items():
        recs[f"{tap}.gram"] = s.gram
        recs[f"{tap}.mean"] = s.mean
        recs[f"{tap}.std"] = s.std
        recs[f"{tap}.n_p"] = np.array([s.n_p], dtype=np.float64)
    formats.write_records(path, recs)


def load_stats(path) -> dict:
    recs = formats.read_records(path)
    out = {}
    for tap in sorted({k.rsplit(".", 1)[0] for k in recs}):
        out[tap] = LayerStats(recs[f"{tap}.gram"], recs[f"{tap}.mean"], recs[f"{tap}.std"],
                              int(recs[f"{tap}.n_p"][0]))
    return out


# ------------------------------------------------------------------------------------------
# per-slab feature gradients (reference stats.py:127-174) on the device
# ------------------------------------------------------------------------------------------

def _dev(a, dtype):
    import torch
    from .device import require_cuda
    require_cuda()
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def _io_dtype(V):
    import torch
    if isinstance(V, torch.Tensor):
        return torch.float64 if V.dtype == torch.float64 else torch.float32
    return torch.float64 if np.asarray(V).dtype == np.float64 else torch.float32


def _back(t, like):
    import torch
    if isinstance(like, torch.Tensor):
        return t
    return t.cpu().numpy()


def style_layer_loss_grad(V, stats_x: LayerStats, stats_ref: LayerStats, w: TapWeights) -> tuple:
    """Loss terms and the feature gradient of the augmented style loss on a slab V of the
    image whose GLOBAL statistics are ``stats_x`` (stats.py:127-165):

        gram (4 w_g / n_p) (G - G_ref) V,  mean (2 w_m / n_p)(mu - mu_ref),
        std  (2 w_s / n_p)(V - mu)(std - std_ref) / std   (column zeroed if std < 1e-8).

    The three terms are one affine map V -> A V + r.V + b (A = (4 w_g/n_p)(G - G_ref),
    r = (2 w_s/n_p) ratio, b = (2 w_m/n_p)(mu - mu_ref) - r mu), evaluated by
    ``spst_feature_affine`` on the device."""
    import torch
    from . import _native as nat
    from .errors import DegenerateStdWarning
    if V.ndim != 3 or V.shape[0] != stats_x.channels:
        raise ShapeError(f"expected ({stats_x.channels},h,w) features, got {tuple(V.shape)}")
    terms = style_loss_terms(stats_x, stats_ref, w)
    C = stats_x.channels
    n_p = float(stats_x.n_p)
    A = (4.0 * w.gram / n_p) * (stats_x.gram - stats_ref.gram) if w.gram else np.zeros((C, C))
    b = (2.0 * w.mean / n_p) * (stats_x.mean - stats_ref.mean) if w.mean else np.zeros(C)
    r = np.zeros(C)
    if w.std:
        std = stats_x.std
        degenerate = std < STD_EPS
        if np.any(degenerate & (stats_ref.std > STD_EPS)):
            warnings.warn("zero-std channel with nonzero reference std; its gradient column is zeroed",
                          DegenerateStdWarning, stacklevel=2)
        ratio = np.where(degenerate, 0.0, (std - stats_ref.std) / np.where(degenerate, 1.0, std))
        r = (2.0 * w.std / n_p) * ratio
        b = b - r * stats_x.mean
    dt = _io_dtype(V)
    Vd = _dev(V, dt)
    out = torch.empty_like(Vd)
    P = int(Vd[0].numel())
    s = torch.cuda.current_stream()
    Ad, rd, bd = _dev(A, dt), _dev(r, dt), _dev(b, dt)  # held until the call returns (no aliasing)
    nat.check(nat.lib().spst_feature_affine(1 if dt == torch.float64 else 0, nat.ptr(Ad), nat.ptr(rd), nat.ptr(bd),
                                            C, P, nat.ptr(Vd), nat.ptr(out), s.cuda_stream), None,
              "spst_feature_affine")
    return terms, _back(out, V)


def content_loss_grad(V, V_ref, lambda_c: float) -> tuple:
    """lambda_c sum (V - V_ref)^2 (f64, fixed order) and its gradient 2 lambda_c (V - V_ref)
    (stats.py:168-174)."""
    import torch
    from . import _native as nat
    if tuple(V.shape) != tuple(V_ref.shape):
        raise ShapeError(f"content features {tuple(V.shape)} vs reference {tuple(V_ref.shape)}")
    dt = _io_dtype(V)
    a, b = _dev(V, dt), _dev(V_ref, dt)
    f64 = 1 if dt == torch.float64 else 0
    n = a.numel()
    s = torch.cuda.current_stream()
    part = torch.empty(nat.lib().spst_vec_partials() + 8, dtype=torch.float64, device="cuda")
    acc = torch.zeros(1, dtype=torch.float64, device="cuda")
    nat.check(nat.lib().spst_metric_sqdiff(f64, nat.ptr(a), nat.ptr(b), n, nat.ptr(part), nat.ptr(acc),
                                           s.cuda_stream), None, "spst_metric_sqdiff")
    g = torch.empty_like(a)
    nat.check(nat.lib().spst_vec_scaled_diff(f64, nat.ptr(a), nat.ptr(b), 2.0 * float(lambda_c), n, nat.ptr(g),
                                             s.cuda_stream), None, "spst_vec_scaled_diff")
    loss = float(lambda_c) * float(acc.item())
    return loss, _back(g, V)
