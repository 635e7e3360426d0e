"""Device engine: one libspst context per (extractor spec, device).

``Engine`` owns the native context (weights staged in tensor-core layouts, HBM workspace)
and exposes the steps of Algorithm 1 (reference localized.py:162-311) as device calls:
``forward`` (activations, masks, per-tap Gram / channel sums), ``finalize`` (global
statistics, loss terms, closed-form feature gradients), ``backward`` (pixel gradient).
PyTorch is used only for device memory and the stream; every FLOP runs in libspst.so.
"""

from __future__ import annotations

import ctypes
import threading
import weakref

import numpy as np
import torch

from . import _native as nat
from .errors import ShapeError
from .spec import check_device_supported, tap_geometry

_KIND = {"conv": 0, "relu": 1}


class _DevView:
    """Expose a raw device pointer to torch via __cuda_array_interface__."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape),
                                         "typestr": typestr, "version": 3}


def device_view(ptr, shape, dtype="<f8"):
    return torch.as_tensor(_DevView(ptr, shape, dtype), device="cuda")


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2212_13459_b200 requires a CUDA (sm_100a) device; there is no CPU path")


class Engine:
    """Native SPST context for one extractor spec on one device."""

    def __init__(self, spec, device: int = 0):
        require_cuda()
        check_device_supported(spec)
        if not spec.has_weights():
            raise ShapeError("extractor has no weights bound")
        self.spec = spec
        self.device = device
        L = nat.lib()
        layers = spec.layers[:spec.deepest_tap_index() + 1]
        n = len(layers)
        kinds = (ctypes.c_int * n)()
        cin = (ctypes.c_int * n)()
        cout = (ctypes.c_int * n)()
        wp = (ctypes.POINTER(ctypes.c_double) * n)()
        bp = (ctypes.POINTER(ctypes.c_double) * n)()
        self._keep = []
        for i, l in enumerate(layers):
            if l.kind == "pool":
                kinds[i] = 2 if l.pool == "avg" else 3
            else:
                kinds[i] = _KIND[l.kind]
            if l.kind == "conv":
                cin[i], cout[i] = l.in_ch, l.out_ch
                w = np.ascontiguousarray(l.weight, dtype=np.float64)
                b = np.ascontiguousarray(l.bias, dtype=np.float64)
                self._keep += [w, b]
                wp[i] = w.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
                bp[i] = b.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        idx = spec.layer_index()
        self.style_taps = tuple(spec.style_taps)
        st = (ctypes.c_int * max(1, len(self.style_taps)))(*[idx[t] for t in self.style_taps])
        pre = spec.preprocess
        mean = (ctypes.c_double * 3)(*pre.mean)
        scale = (ctypes.c_double * 3)(*pre.scale)
        handle = ctypes.c_void_p()
        with torch.cuda.device(device):
            status = L.spst_create(device, n, kinds, cin, cout, wp, bp, len(self.style_taps), st,
                                   idx[spec.content_tap], 1 if pre.channel_order == "bgr" else 0, mean, scale,
                                   ctypes.byref(handle))
        self._h = handle.value
        if status != nat.OK:
            msg = L.spst_last_error(self._h).decode() if self._h else ""
            if self._h:
                L.spst_destroy(self._h)
                self._h = None
            nat.check(status, None, f"spst_create: {msg}")
        self._finalizer = weakref.finalize(self, L.spst_destroy, self._h)
        self._check(L.spst_set_precision(self._h, _PRECISION_MODES[_precision]), "spst_set_precision")
        self.geom = {t: tap_geometry(spec, t) for t in spec.taps}
        self.bound = None
        self.bind_epoch = 0
        self.lock = threading.RLock()
        self._terms = np.zeros(3 * max(1, len(self.style_taps)))
        self._deg = (ctypes.c_int * max(1, len(self.style_taps)))()
        self._content_out = None
        self.last_forward_key = None

    # ------------------------------------------------------------------ plumbing
    def _check(self, status, what):
        nat.check(status, self._h, what)

    def stream(self):
        s = torch.cuda.current_stream(self.device)
        nat.lib().spst_set_stream(self._h, ctypes.c_void_p(s.cuda_stream))
        return s

    # ------------------------------------------------------------------ geometry
    def bind(self, h, w, grid=None, own=None, gcols=None, ocols=None):
        """Bind image dims and the evaluated window (padded-image coordinates): rows grid / own,
        columns gcols / ocols (defaults: the whole padded image, owned entirely)."""
        s = self.spec.deepest_stride()
        Hp, Wp = h + (-h) % s, w + (-w) % s
        grid = tuple(grid or (0, Hp))
        own = tuple(own or grid)
        gcols = tuple(gcols or (0, Wp))
        ocols = tuple(ocols or gcols)
        key = (h, w, grid, own, gcols, ocols)
        if self.bound == key:
            return
        with torch.cuda.device(self.device):
            self._check(nat.lib().spst_bind_window(self._h, h, w, grid[0], grid[1], gcols[0], gcols[1], own[0],
                                                   own[1], ocols[0], ocols[1]), "spst_bind_window")
        self.bound = key
        self.bind_epoch += 1
        self.last_forward_key = None
        self._content_out = torch.zeros(1, dtype=torch.float64, device=f"cuda:{self.device}")

    def window_dims(self):
        """(rows, columns) of the bound window's padded grid."""
        a, b = ctypes.c_int(), ctypes.c_int()
        nat.lib().spst_window_dims(self._h, ctypes.byref(a), ctypes.byref(b))
        return a.value, b.value

    def unbind(self):
        with torch.cuda.device(self.device):
            nat.lib().spst_unbind(self._h)
        self.bound = None
        self.bind_epoch += 1

    def padded_dims(self):
        a, b = ctypes.c_int(), ctypes.c_int()
        nat.lib().spst_padded_dims(self._h, ctypes.byref(a), ctypes.byref(b))
        return a.value, b.value

    def owned_pixels(self, t_index):
        c, st, n = ctypes.c_int(), ctypes.c_int(), ctypes.c_longlong()
        self._check(nat.lib().spst_tap_info(self._h, t_index, ctypes.byref(c), ctypes.byref(st), ctypes.byref(n)),
                    "spst_tap_info")
        return n.value

    def owned_counts(self):
        """owned_pixels of every style tap (cached per binding)."""
        if getattr(self, "_counts_epoch", None) != self.bind_epoch:
            self._counts = [self.owned_pixels(i) for i in range(len(self.style_taps))]
            self._counts_epoch = self.bind_epoch
        return self._counts

    def pinned_scalar(self):
        """A pinned host f64[1] for asynchronous scalar read-backs on the engine stream."""
        if getattr(self, "_pin1", None) is None:
            self._pin1 = torch.empty(1, dtype=torch.float64).pin_memory()
        return self._pin1

    def workspace_bytes(self):
        return int(nat.lib().spst_workspace_bytes(self._h))

    # ------------------------------------------------------------------ passes
    def forward(self, x_dev, origin=(0, 0)):
        """x_dev: float32 CUDA tensor of image rows/columns starting at global pixel `origin`
        ((h, w, 3) for the whole image; any (rows, cols, 3) block covering the window's image
        pixels otherwise)."""
        self.stream()
        pitch = int(x_dev.shape[1])
        ptr = nat.ptr(x_dev) - 12 * (origin[0] * pitch + origin[1])
        with torch.cuda.device(self.device):
            self._check(nat.lib().spst_forward_pitched(self._h, ctypes.c_void_p(ptr), pitch, 1), "spst_forward")

    def tap_sums(self, t_index):
        """Device f64 views (S: C x C, s: C) of this device's owned-row sums for style tap t."""
        S, s = ctypes.c_void_p(), ctypes.c_void_p()
        self._check(nat.lib().spst_stats_ptrs(self._h, t_index, ctypes.byref(S), ctypes.byref(s)), "spst_stats_ptrs")
        C = self.geom[self.style_taps[t_index]].channels
        return device_view(S.value, (C, C)), device_view(s.value, (C,))

    def set_style_ref(self, t_index, stats, w):
        g = np.ascontiguousarray(stats.gram, dtype=np.float64)
        m = np.ascontiguousarray(stats.mean, dtype=np.float64)
        d = np.ascontiguousarray(stats.std, dtype=np.float64)
        P = ctypes.POINTER(ctypes.c_double)
        self._check(nat.lib().spst_set_style_ref(self._h, t_index, g.ctypes.data_as(P), m.ctypes.data_as(P),
                                                  d.ctypes.data_as(P), float(w.gram), float(w.mean), float(w.std)),
                    "spst_set_style_ref")

    def finalize(self, counts):
        """Global statistics -> per-tap (gram, mean, std) loss terms [T, 3] and degenerate flags."""
        n = (ctypes.c_longlong * max(1, len(counts)))(*[int(c) for c in counts])
        terms = (ctypes.c_double * len(self._terms))()
        self._check(nat.lib().spst_finalize(self._h, n, terms, self._deg), "spst_finalize")
        T = len(self.style_taps)
        return np.array(terms[:3 * T]).reshape(T, 3), [bool(self._deg[i]) for i in range(T)]

    def capture_content(self):
        self._check(nat.lib().spst_capture_content(self._h), "spst_capture_content")

    def content_sqdiff(self):
        """Device f64 scalar: sum over owned rows of (V - V_u)^2 at the content tap."""
        self._check(nat.lib().spst_content_sqdiff(self._h, nat.ptr(self._content_out)), "spst_content_sqdiff")
        return self._content_out

    def relu_masks(self):
        """{relu layer name: bool (C, H, W)} of the last forward (test/diagnostic hook)."""
        out = {}
        convs = [i for i, l in enumerate(self.spec.layers[:self.spec.deepest_tap_index() + 1]) if l.kind == "conv"]
        Hl, Wp = self.window_dims()
        for k, li in enumerate(convs):
            stride = 2 ** sum(1 for l in self.spec.layers[:li] if l.kind == "pool")
            C = self.spec.layers[li].out_ch
            buf = np.zeros((C, Hl // stride, Wp // stride), dtype=np.uint8)
            self._check(nat.lib().spst_debug_mask(self._h, k, buf.ctypes.data), "spst_debug_mask")
            out[self.spec.layers[li + 1].name] = buf.astype(bool)
        return out

    def stage_outputs(self):
        """{relu layer name: f32 (C, H, W)} stored relu outputs of the last forward (diagnostics;
        bind with SPST_DEBUG_STORE_ALL=1 to keep the non-tap pool stages too)."""
        out = {}
        convs = [i for i, l in enumerate(self.spec.layers[:self.spec.deepest_tap_index() + 1]) if l.kind == "conv"]
        Hl, Wp = self.window_dims()
        for k, li in enumerate(convs):
            stride = 2 ** sum(1 for l in self.spec.layers[:li] if l.kind == "pool")
            buf = np.zeros((self.spec.layers[li].out_ch, Hl // stride, Wp // stride), dtype=np.float32)
            if nat.lib().spst_debug_stage_out(self._h, k, buf.ctypes.data) == nat.OK:
                out[self.spec.layers[li + 1].name] = buf
        return out

    TIMER_CLASSES = ("conv3x3_tc<128>", "conv3x3_tc<64>", "gram_tc", "unused")

    def timing_enable(self, on=True):
        """Bracket every tensor-core launch with CUDA events on the engine stream (resets totals)."""
        self._check(nat.lib().spst_timing_enable(self._h, 1 if on else 0), "spst_timing_enable")

    def timing_read(self):
        """{class: (device ms, algorithmic FLOPs, launches)} since timing_enable."""
        ms, fl, n = (ctypes.c_double * 4)(), (ctypes.c_double * 4)(), (ctypes.c_longlong * 4)()
        self._check(nat.lib().spst_timing_read(self._h, ms, fl, n), "spst_timing_read")
        return {c: (ms[i], fl[i], n[i]) for i, c in enumerate(self.TIMER_CLASSES) if n[i]}

    def backward(self, two_lambda, grad_dev, origin=(0, 0), defer=False):
        """Writes the owned pixels' gradient into grad_dev (a float32 (rows, cols, 3) CUDA block
        whose first pixel is global pixel `origin`).  defer=True returns right after the launch;
        ``backward_resolve`` then settles the pass's range check (one synchronisation)."""
        self.stream()
        pitch = int(grad_dev.shape[1])
        ptr = nat.ptr(grad_dev) - 12 * (origin[0] * pitch + origin[1])
        with torch.cuda.device(self.device):
            fn = nat.lib().spst_backward_async if defer else nat.lib().spst_backward_pitched
            self._check(fn(self._h, float(two_lambda), ctypes.c_void_p(ptr), pitch), "spst_backward")

    def backward_resolve(self) -> bool:
        """Settle a deferred backward; True if it had to be re-run (the gradient was rewritten)."""
        r = ctypes.c_int()
        self._check(nat.lib().spst_backward_resolve(self._h, ctypes.byref(r)), "spst_backward_resolve")
        return bool(r.value)

    def forward_redone(self) -> bool:
        """True if the last finalize re-ran the forward (work launched behind it is stale)."""
        return bool(nat.lib().spst_forward_redone(self._h))

    def content_target(self):
        """(device uint8 copy of the bound window's content target, its scale)."""
        buf, n, sc = ctypes.c_void_p(), ctypes.c_longlong(), ctypes.c_float()
        self._check(nat.lib().spst_content_target(self._h, ctypes.byref(buf), ctypes.byref(n), ctypes.byref(sc)),
                    "spst_content_target")
        self.stream()
        return device_view(buf.value, (n.value,), "|u1").clone(), sc.value

    def set_content_target(self, t):
        buf, scale = t
        self.stream()
        self._check(nat.lib().spst_set_content_target(self._h, ctypes.c_void_p(buf.data_ptr()), float(scale)),
                    "spst_set_content_target")


_ENGINES: dict = {}

_PRECISION_MODES = {"fp16x3": 0, "fp16": 1}
_precision = "fp16x3"


def set_precision(mode: str) -> None:
    """Tensor-core precision of the conv layers for every engine (existing and future):
    "fp16x3" (default: hi/lo split operands, three MMA passes, fp32-class, meets the parity
    bar) or "fp16" (one pass, ~3x less tensor work, ~1e-3 relative per layer -- an opt-in speed
    mode for previews; it does not meet the gradient parity bar).  SURVEY.md §7 step 3."""
    global _precision
    if mode not in _PRECISION_MODES:
        raise ValueError(f"precision must be one of {sorted(_PRECISION_MODES)}, got {mode!r}")
    _precision = mode
    for _, eng in _ENGINES.values():
        eng._check(nat.lib().spst_set_precision(eng._h, _PRECISION_MODES[mode]), "spst_set_precision")


def get_precision() -> str:
    return _precision


def engine_for(spec, device: int | None = None) -> Engine:
    """One engine per (spec object, device); keeps the spec alive to pin its id."""
    require_cuda()
    dev = torch.cuda.current_device() if device is None else device
    key = (id(spec), dev)
    hit = _ENGINES.get(key)
    if hit is not None and hit[0] is spec:
        return hit[1]
    if len(_ENGINES) >= 4:
        _ENGINES.pop(next(iter(_ENGINES)))
    eng = Engine(spec, dev)
    _ENGINES[key] = (spec, eng)
    return eng


def clear_engines():
    _ENGINES.clear()
