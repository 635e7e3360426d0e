"""Image resampling on the device (reference tensorops.py:136-185).

``resize_down``: area mean over f x f boxes with ragged right/bottom boxes, output dims
ceil(in/f).  ``resize_bilinear``: half-pixel-centred bilinear with clamped sources.
``resize_up2``: bilinear x2 or to an explicit target (absorbs ceil drift).  numpy in ->
numpy out; CUDA tensor in -> CUDA tensor out.  Images are (h, w) or (h, w, c); f64 images are
resampled in f64 (the reference's dtype="f64" path), everything else in f32.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native as nat
from .device import require_cuda
from .errors import ShapeError


def _prep(img):
    require_cuda()
    is_t = isinstance(img, torch.Tensor)
    t = img if is_t else torch.from_numpy(np.ascontiguousarray(np.asarray(img)))
    dtype = t.dtype
    work = torch.float64 if dtype == torch.float64 else torch.float32  # f64 images resample in f64
    t = t.to(device="cuda", dtype=work).contiguous()
    squeeze = t.ndim == 2
    if squeeze:
        t = t[:, :, None]
    if t.ndim != 3:
        raise ShapeError(f"image must be (h, w) or (h, w, c), got {tuple(img.shape)}")
    return t, is_t, dtype, squeeze


def _finish(out, is_t, dtype, squeeze):
    if squeeze:
        out = out[:, :, 0]
    if is_t:
        return out if out.dtype == dtype else out.to(dtype)
    return out.cpu().numpy().astype(np.dtype(str(dtype).replace("torch.", "")), copy=False)


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def resize_down(img, factor: int):
    if factor < 1:
        raise ShapeError(f"resize_down factor must be >= 1, got {factor}")
    t, is_t, dtype, sq = _prep(img)
    if factor == 1:
        return _finish(t.clone(), is_t, dtype, sq)
    h, w, c = t.shape
    out = torch.empty((-(-h // factor), -(-w // factor), c), dtype=t.dtype, device=t.device)
    nat.check(nat.lib().spst_resize_down_typed(int(t.dtype == torch.float64), nat.ptr(t), h, w, c, factor,
                                               nat.ptr(out), _stream()), None, "spst_resize_down")
    return _finish(out, is_t, dtype, sq)


def resize_bilinear(img, out_hw: tuple):
    oh, ow = int(out_hw[0]), int(out_hw[1])
    if oh < 1 or ow < 1:
        raise ShapeError(f"bilinear target must be >= 1x1, got {oh}x{ow}")
    t, is_t, dtype, sq = _prep(img)
    h, w, c = t.shape
    out = torch.empty((oh, ow, c), dtype=t.dtype, device=t.device)
    nat.check(nat.lib().spst_resize_bilinear_typed(int(t.dtype == torch.float64), nat.ptr(t), h, w, c, oh, ow,
                                                   nat.ptr(out), _stream()), None, "spst_resize_bilinear")
    return _finish(out, is_t, dtype, sq)


def resize_up2(img, target_hw: tuple | None = None):
    h, w = img.shape[:2]
    return resize_bilinear(img, target_hw if target_hw is not None else (2 * h, 2 * w))
