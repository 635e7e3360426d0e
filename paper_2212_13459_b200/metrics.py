"""Quantitative evaluation on device: PSNR, SSIM, blockwise Gram distance, identity test.

Mirrors the reference metrics.py (same names, constants, argument meaning and errors):
``psnr`` (metrics.py:24-31), ``ssim`` (55-73), ``gram_distance`` (76-89), ``IdentityReport``
(92-106), ``identity_test`` (109-137), ``append_csv`` (140-148).  PSNR and SSIM run as CUDA
kernels (``spst_metric_sqdiff`` / ``spst_metric_ssim``: f64 arithmetic, fixed-order
reductions); ``gram_distance`` reuses the device ``stats_pass``.  There is no CPU path.
"""

from __future__ import annotations

import json
import math
import os
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .device import require_cuda
from .errors import ShapeError
from .localized import stats_pass

LUMA_WEIGHTS = (0.299, 0.587, 0.114)  # Rec. 601
SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
SSIM_K1 = 0.01
SSIM_K2 = 0.03


def _to_device(img) -> torch.Tensor:
    """Contiguous CUDA tensor in the image's own float dtype (f32/f64; others widen to f64)."""
    require_cuda()
    t = img if isinstance(img, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(img))
    if t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float64)
    return t.to("cuda", non_blocking=False).contiguous()


def _pair(a, b):
    ta, tb = _to_device(a), _to_device(b)
    if ta.dtype != tb.dtype:  # NumPy promotes mixed f32/f64 to f64
        ta, tb = ta.to(torch.float64), tb.to(torch.float64)
    return ta, tb


def _scratch(device):
    nb = nat.lib().spst_vec_partials()
    return (torch.empty(nb, dtype=torch.float64, device=device), torch.empty(1, dtype=torch.float64, device=device))


def psnr(a, b) -> float:
    """10*log10(1/MSE) on [0,1] images; +inf for identical inputs."""
    if tuple(a.shape) != tuple(b.shape):
        raise ShapeError(f"psnr dims differ: {tuple(a.shape)} vs {tuple(b.shape)}")
    ta, tb = _pair(a, b)
    n = ta.numel()
    if n == 0:
        return math.nan  # np.mean of an empty array
    part, out = _scratch(ta.device)
    s = torch.cuda.current_stream(ta.device)
    nat.check(nat.lib().spst_metric_sqdiff(1 if ta.dtype == torch.float64 else 0, nat.ptr(ta), nat.ptr(tb), n,
                                           nat.ptr(part), nat.ptr(out), s.cuda_stream), None, "spst_metric_sqdiff")
    mse = float(out.item()) / n
    if mse == 0.0:
        return math.inf
    return 10.0 * math.log10(1.0 / mse)


def ssim(a, b) -> float:
    """Mean local SSIM on luma: 11x11 Gaussian window (sigma 1.5), K1/K2 = 0.01/0.03."""
    if tuple(a.shape) != tuple(b.shape):
        raise ShapeError(f"ssim dims differ: {tuple(a.shape)} vs {tuple(b.shape)}")
    if min(a.shape[0], a.shape[1]) < SSIM_WINDOW:
        raise ShapeError(f"ssim needs min side >= {SSIM_WINDOW}, got {tuple(a.shape[:2])}")
    if len(a.shape) == 3 and a.shape[2] != 3:
        raise ShapeError(f"ssim expects (h, w) or (h, w, 3) images, got {tuple(a.shape)}")
    ta, tb = _to_device(a), _to_device(b)  # each luma in its own dtype (reference _luma)
    h, w = int(a.shape[0]), int(a.shape[1])
    c = 1 if len(a.shape) == 2 else 3
    part, out = _scratch(ta.device)
    s = torch.cuda.current_stream(ta.device)
    mask = (1 if ta.dtype == torch.float64 else 0) | (2 if tb.dtype == torch.float64 else 0)
    nat.check(nat.lib().spst_metric_ssim(mask, nat.ptr(ta), nat.ptr(tb), h, w, c,
                                         nat.ptr(part), nat.ptr(out), s.cuda_stream), None, "spst_metric_ssim")
    return float(out.item()) / ((h - SSIM_WINDOW + 1) * (w - SSIM_WINDOW + 1))


def gram_distance(x, v, spec, block: int = 512, margin: int = 256, weights: dict | None = None,
                  threads: int = 1) -> float:
    """Weighted squared Frobenius distance between the Gram matrices of x and v, summed over
    the style taps (reference metrics.py:76-89).  Both images go through the device
    ``stats_pass`` on the given grid; ``weights`` ({tap: w}) defaults to 1 per tap."""
    grams = [stats_pass(img, spec, block=block, margin=margin, threads=threads) for img in (x, v)]
    return sum((1.0 if weights is None else weights[t]) * float(np.sum((grams[0][t].gram - grams[1][t].gram) ** 2))
               for t in spec.style_taps)


@dataclass(frozen=True)
class IdentityReport:
    """Identity-test record (reference metrics.py:92-106); JSON keys as the reference writes them."""
    psnr: float
    ssim: float
    gram_distance: float
    gram_distance_weighted: float
    wall_time: float
    config_hash: str

    _JSON_KEYS = (("psnr", "psnr"), ("ssim", "ssim"), ("gram", "gram_distance"),
                  ("gram_weighted", "gram_distance_weighted"), ("seconds", "wall_time"),
                  ("config_hash", "config_hash"))

    def to_json(self) -> str:
        return json.dumps({key: getattr(self, attr) for key, attr in self._JSON_KEYS})


def identity_test(style, cfg, progress=None) -> tuple:
    """Style transfer of a painting onto itself, scored by PSNR/SSIM/Gram distance
    (reference metrics.py:109-137).  Returns (IdentityReport, output image); the Gram distance
    is given unweighted and with the run's per-tap Gram weights."""
    from .pipeline import multiscale_transfer
    from .stats import default_loss_weights

    start = time.perf_counter()
    out = multiscale_transfer(style, style, cfg, progress=progress)
    seconds = time.perf_counter() - start
    spec = cfg.extractor
    lw = cfg.weights if cfg.weights is not None else default_loss_weights(spec, mean_std_factor=cfg.mean_std_factor)
    tap_w = {tap: sw.gram for tap, sw in lw.style.items()}
    target = style.astype(out.dtype, copy=False)
    geo = dict(block=cfg.block, margin=cfg.margin, threads=cfg.threads)
    return IdentityReport(psnr=psnr(out, target), ssim=ssim(out, target),
                          gram_distance=gram_distance(out, target, spec, **geo),
                          gram_distance_weighted=gram_distance(out, target, spec, weights=tap_w, **geo),
                          wall_time=seconds, config_hash=cfg.config_hash), out


CSV_COLUMNS = ("style_id", "psnr", "ssim", "gram", "seconds", "config_hash")


def append_csv(path, style_id: str, report: IdentityReport) -> None:
    """One row per identity test; the header is written when the file is created
    (reference metrics.py:140-148)."""
    fields = (style_id, report.psnr, report.ssim, report.gram_distance, report.wall_time, report.config_hash)
    row = ",".join(str(f) for f in fields) + "\n"
    fresh = not os.path.exists(path)
    with open(path, "a") as fh:
        fh.write((",".join(CSV_COLUMNS) + "\n" if fresh else "") + row)
