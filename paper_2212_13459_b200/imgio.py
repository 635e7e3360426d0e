"""Image I/O used by the driver's checkpoints (reference imgio.py:17-63): 8-bit decode/encode
and the 16-bit PNG checkpoint view.  Host-side file format code (out of the hot path)."""

from __future__ import annotations

import numpy as np

from .errors import FormatError


def _cv2():
    import cv2
    return cv2


def decode(path) -> np.ndarray:
    """8-bit PNG/JPEG -> (h, w, 3) float32 RGB in [0, 1]."""
    img = _cv2().imread(str(path), _cv2().IMREAD_COLOR)
    if img is None:
        raise FormatError(f"{path}: cannot decode image")
    return (img[:, :, ::-1].astype(np.float32) / 255.0)


def encode(path, img: np.ndarray) -> None:
    a = np.clip(np.asarray(img, dtype=np.float64), 0.0, 1.0)
    out = np.round(a * 255.0).astype(np.uint8)
    if not _cv2().imwrite(str(path), np.ascontiguousarray(out[:, :, ::-1])):
        raise FormatError(f"{path}: cannot encode image")


def save_png16(path, img: np.ndarray) -> None:
    a = np.clip(np.asarray(img, dtype=np.float64), 0.0, 1.0)
    out = np.round(a * 65535.0).astype(np.uint16)
    if not _cv2().imwrite(str(path), np.ascontiguousarray(out[:, :, ::-1])):
        raise FormatError(f"{path}: cannot write 16-bit PNG")


def load_png16(path, dtype="f32") -> np.ndarray:
    img = _cv2().imread(str(path), _cv2().IMREAD_UNCHANGED)
    if img is None or img.dtype != np.uint16:
        raise FormatError(f"{path}: not a 16-bit PNG")
    return (img[:, :, ::-1].astype(np.float64) / 65535.0).astype(np.float32 if dtype == "f32" else np.float64)
