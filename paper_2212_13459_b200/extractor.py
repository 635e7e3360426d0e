"""Device ``forward_taps`` (reference extractor.py:171-197).

The reference runs preprocess + every layer up to the deepest tap on a (3, h, w) array and
returns the tensors recorded at the tap layers.  Here the same forward runs in libspst.so
(the tcgen05 conv chain of ``loss_grad``) and the tap features are unpacked from the engine's
HL16 tap buffers into f32 on the device.

Differences from the reference, both raised loudly:
* ``save_for_backward=True`` -- the device forward keeps 1-bit ReLU masks, not the per-layer
  inputs the reference saves for ``backward_to_input`` (NotImplementedError);
* inputs whose sides are not multiples of the deepest stride -- the reference floors the
  ragged rows at each pool; the device grid is stride-aligned (NotImplementedError).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from .device import engine_for, require_cuda
from .errors import GeometryError, ShapeError
from .spec import ExtractorSpec, tap_geometry


def _stage_of(spec: ExtractorSpec) -> dict:
    """relu layer name -> conv stage index of the device engine."""
    out, k = {}, 0
    for i, l in enumerate(spec.layers[:spec.deepest_tap_index() + 1]):
        if l.kind == "conv":
            out[spec.layers[i + 1].name] = k
            k += 1
    return out


def forward_taps(x, spec: ExtractorSpec, save_for_backward: bool = False):
    """Tap map {layer name: (C, h/s, w/s) features} of a (3, h, w) image (extractor.py:171-197).

    numpy in -> numpy of x's dtype; CUDA tensor in -> float32 CUDA tensors."""
    if x.ndim != 3 or x.shape[0] != 3:
        raise ShapeError(f"extractor input must be (3,h,w), got {tuple(x.shape)}")
    stride = spec.deepest_stride()
    h, w = int(x.shape[1]), int(x.shape[2])
    if h < stride or w < stride:
        raise GeometryError(f"input {h}x{w} smaller than one feature pixel at the deepest tap (stride {stride})")
    if save_for_backward:
        raise NotImplementedError("the device forward keeps 1-bit ReLU masks, not per-layer inputs; "
                                  "use loss_grad for gradients")
    if h % stride or w % stride:
        raise NotImplementedError(f"device forward_taps needs sides that are multiples of the deepest stride "
                                  f"{stride} (got {h}x{w}); pad with pad_to_multiple first")
    require_cuda()
    eng = engine_for(spec)
    stage = _stage_of(spec)
    is_t = isinstance(x, torch.Tensor)
    with eng.lock:
        img = (x.permute(1, 2, 0) if is_t else torch.from_numpy(np.ascontiguousarray(np.asarray(x).transpose(1, 2, 0),
                                                                                       dtype=np.float32)))
        img = img.to(device=f"cuda:{eng.device}", dtype=torch.float32).contiguous()
        eng.bind(h, w)
        eng.forward(img)
        out = {}
        for t in spec.taps:
            g = tap_geometry(spec, t)
            buf = torch.empty((g.channels, h // g.stride, w // g.stride), dtype=torch.float32,
                              device=f"cuda:{eng.device}")
            eng.stream()
            eng._check(nat.lib().spst_stage_features(eng._h, stage[t], nat.ptr(buf)), "spst_stage_features")
            out[t] = buf
        torch.cuda.current_stream(eng.device).synchronize()
    if is_t:
        return out
    dt = np.asarray(x).dtype if np.asarray(x).dtype in (np.float32, np.float64) else np.float32
    return {t: v.cpu().numpy().astype(dt, copy=False) for t, v in out.items()}
