"""Synthetic benchmark / parity workloads (BASELINE.json configs).

Content u: smooth bilinear-upsampled field + fine grain (generalises the reference test
helper make_painting, tests/oracles.py:86-92, to h x w).  Style v: coloured oriented
sinusoid with 5 % grain — deliberately different statistics from u so G(x) - G_ref is not
pure cancellation (SURVEY.md §0 finding 4).  Both float32 in [0, 1], seeded.
"""

from __future__ import annotations

import math

import numpy as np


def _bilinear_np(img, oh, ow):
    h, w = img.shape[:2]

    def axis(n_in, n_out):
        s = np.clip((np.arange(n_out) + 0.5) * (n_in / n_out) - 0.5, 0.0, n_in - 1.0)
        i0 = np.floor(s).astype(np.int64)
        return i0, np.minimum(i0 + 1, n_in - 1), s - i0

    y0, y1, ty = axis(h, oh)
    x0, x1, tx = axis(w, ow)
    r = img[y0] * (1 - ty)[:, None, None] + img[y1] * ty[:, None, None]
    return r[:, x0] * (1 - tx)[None, :, None] + r[:, x1] * tx[None, :, None]


def synth_content(h: int, w: int, seed: int = 1) -> np.ndarray:
    r = np.random.default_rng(seed)
    base = _bilinear_np(r.random((max(h // 8, 1), max(w // 8, 1), 3)), h, w)
    return np.clip(base + 0.15 * (r.random((h, w, 3)) - 0.5), 0.0, 1.0).astype(np.float32)


def synth_style(h: int, w: int, seed: int = 2) -> np.ndarray:
    r = np.random.default_rng(seed)
    yy, xx = np.meshgrid(np.arange(h, dtype=np.float64) / max(h, 1), np.arange(w, dtype=np.float64) / max(w, 1),
                         indexing="ij")
    phase = r.uniform(0.0, 2 * math.pi, 3)
    amp = np.array([1.0, 0.7, 0.4])
    img = 0.5 + 0.45 * np.sin(2 * math.pi * (7 * xx[..., None] + 3 * yy[..., None]) + phase) * amp
    img = img + 0.05 * r.standard_normal((h, w, 3))
    return np.clip(img, 0.0, 1.0).astype(np.float32)


CONFIGS = {
    # BASELINE.json configs[0]: single scale 256^2, 10 iterations (CPU-runnable reference case)
    "c1": dict(content=(256, 256), style=(256, 256), n_scales=1, iters=10),
    # configs[1]: single scale 1512x2016 content, 1024^2 style, 100 iterations
    "c2": dict(content=(1512, 2016), style=(1024, 1024), n_scales=1, iters=100),
    # configs[2]: two scales 756x1008 -> 3024x4032
    "c3": dict(content=(3024, 4032), style=(2113, 2660), n_scales=3, iters=None),
    # configs[3]: full 4-scale UHR transfer, the metric's resolution
    "c4": dict(content=(6048, 8064), style=(4226, 5319), n_scales=4, iters=None),
    # the coarsest scale of c4 (600 iterations of the fast and baseline schedules)
    "c4s1": dict(content=(756, 1008), style=(529, 665), n_scales=1, iters=600),
}
