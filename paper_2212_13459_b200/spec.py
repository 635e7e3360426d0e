"""Feature-extractor description, receptive-field geometry and weight binding.

Drop-in for the reference extractor module's data model (reference extractor.py:21-106,
217-345): same class names, fields, validation errors and stock specs, so user code that
builds or loads an ``ExtractorSpec`` works unchanged.  Evaluation itself is not here: the
device runtime (``device.py`` -> libspst.so) executes the spec.

Also provides ``calibrated_vgg19`` — the seeded, activation-calibrated VGG-19 weights the
benchmark and parity tests use (the reference ships no VGG weights, and plain
He-init leaves dead channels).
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from . import formats
from .errors import FormatError, GeometryError, ShapeError

HEADER_RECORD = "__header__"


@dataclass(frozen=True)
class LayerSpec:
    """One layer; ``kind`` is "conv", "relu" or "pool" (extractor.py:21-42)."""
    kind: str
    name: str
    in_ch: int = 0
    out_ch: int = 0
    k: int = 0
    stride: int = 1
    pad: int = 0
    pool: str = "avg"
    weight: np.ndarray | None = field(default=None, repr=False, compare=False)
    bias: np.ndarray | None = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        if self.kind == "conv":
            if self.k % 2 == 0:
                raise GeometryError(f"{self.name}: conv kernel must be odd, got {self.k}")
            if self.pad != (self.k - 1) // 2:
                raise GeometryError(f"{self.name}: conv pad must be (k-1)/2 for same geometry")
        elif self.kind == "pool" and self.pool not in ("avg", "max"):
            raise GeometryError(f"{self.name}: pool kind must be avg or max, got {self.pool!r}")


def conv(name, in_ch, out_ch, k=3, stride=1):
    return LayerSpec("conv", name, in_ch=in_ch, out_ch=out_ch, k=k, stride=stride, pad=(k - 1) // 2)


def relu(name):
    return LayerSpec("relu", name)


def pool(name, k=2, kind="avg"):
    return LayerSpec("pool", name, k=k, pool=kind)


@dataclass(frozen=True)
class Preprocess:
    """Per-channel normalisation before the first layer (extractor.py:58-62)."""
    channel_order: str = "rgb"
    mean: tuple = (0.0, 0.0, 0.0)
    scale: tuple = (1.0, 1.0, 1.0)


@dataclass(frozen=True)
class TapGeometry:
    stride: int
    rf_radius: int
    channels: int


@dataclass(frozen=True)
class ExtractorSpec:
    layers: tuple
    style_taps: tuple
    content_tap: str
    preprocess: Preprocess = Preprocess()

    def __post_init__(self):
        idx = self.layer_index()
        for tap in (*self.style_taps, self.content_tap):
            if tap not in idx:
                raise KeyError(f"tap {tap!r} names no layer")
            if self.layers[idx[tap]].kind != "relu":
                raise GeometryError(f"tap {tap!r} must point at a relu layer")

    def layer_index(self) -> dict:
        return {l.name: i for i, l in enumerate(self.layers)}

    @property
    def taps(self) -> tuple:
        return tuple(dict.fromkeys((*self.style_taps, self.content_tap)))

    def deepest_tap_index(self) -> int:
        idx = self.layer_index()
        return max(idx[t] for t in self.taps)

    def deepest_stride(self) -> int:
        return max(tap_geometry(self, t).stride for t in self.taps)

    def max_rf_radius(self) -> int:
        return max(tap_geometry(self, t).rf_radius for t in self.taps)

    def has_weights(self) -> bool:
        return all(l.weight is not None for l in self.layers if l.kind == "conv")


def tap_geometry(spec, tap: str) -> TapGeometry:
    """Stride / conv-support radius / channels of a tap (extractor.py:217-237)."""
    idx = spec.layer_index()
    if tap not in idx:
        raise KeyError(f"unknown tap {tap!r}")
    jump, radius, ch = 1, 0, 3
    for l in spec.layers[:idx[tap] + 1]:
        if l.kind == "conv":
            radius += jump * (l.k - 1) // 2
            jump *= l.stride
            ch = l.out_ch
        elif l.kind == "pool":
            jump *= l.k
    return TapGeometry(stride=jump, rf_radius=radius, channels=ch)


# ------------------------------------------------------------------------------------------
# weight files (extractor.py:244-280)
# ------------------------------------------------------------------------------------------

def save_weights(path, spec: ExtractorSpec) -> None:
    pre = spec.preprocess
    recs = {HEADER_RECORD: np.array([pre.channel_order == "bgr", *pre.mean, *pre.scale], dtype=np.float64)}
    for l in spec.layers:
        if l.kind != "conv":
            continue
        if l.weight is None:
            raise FormatError(f"{l.name}: cannot save unbound conv weights")
        recs[f"{l.name}.weight"] = l.weight
        recs[f"{l.name}.bias"] = l.bias
    formats.write_records(path, recs)


def load_weights(path, spec: ExtractorSpec) -> ExtractorSpec:
    recs = formats.read_records(path)
    head = recs.get(HEADER_RECORD)
    if head is None or head.shape != (7,):
        raise FormatError(f"{path}: missing or malformed preprocessing header")
    pre = Preprocess("bgr" if head[0] else "rgb", tuple(head[1:4]), tuple(head[4:7]))
    out = []
    for l in spec.layers:
        if l.kind != "conv":
            out.append(l)
            continue
        try:
            w, b = recs[f"{l.name}.weight"], recs[f"{l.name}.bias"]
        except KeyError as e:
            raise FormatError(f"{path}: missing record for layer {l.name}") from e
        want = (l.out_ch, l.in_ch, l.k, l.k)
        if w.shape != want or b.shape != (l.out_ch,):
            raise FormatError(f"{path}: layer {l.name} has weight {w.shape} / bias {b.shape}, "
                              f"expected {want} / ({l.out_ch},)")
        out.append(replace(l, weight=w, bias=b))
    return replace(spec, layers=tuple(out), preprocess=pre)


# ------------------------------------------------------------------------------------------
# stock specs (extractor.py:287-345)
# ------------------------------------------------------------------------------------------

_VGG19_GROUPS = ((64, 2), (128, 2), (256, 4), (512, 4), (512, 4))
VGG_PREPROCESS = Preprocess("rgb", (0.485, 0.456, 0.406), (0.229, 0.224, 0.225))


def vgg19(pooling: str = "avg") -> ExtractorSpec:
    """Unbound VGG-19 up to relu5_1: style taps relu{g}_1, content tap relu4_2."""
    layers, cin = [], 3
    for g, (width, n) in enumerate(_VGG19_GROUPS, start=1):
        for j in range(1, n + 1):
            layers += [conv(f"conv{g}_{j}", cin, width), relu(f"relu{g}_{j}")]
            cin = width
            if g == 5:
                break
        if g < 5:
            layers.append(pool(f"pool{g}", 2, pooling))
        else:
            break
    return ExtractorSpec(tuple(layers), tuple(f"relu{g}_1" for g in range(1, 6)), "relu4_2", VGG_PREPROCESS)


def _conv_np(x, w):
    """f64 3x3 same-conv used only for weight calibration on a small probe (host setup)."""
    c, h, wd = x.shape
    xp = np.pad(x, ((0, 0), (1, 1), (1, 1)))
    cols = np.stack([xp[:, dy:dy + h, dx:dx + wd] for dy in range(3) for dx in range(3)], axis=1)
    return np.einsum("ocyx,cyxhw->ohw", w.reshape(w.shape[0], c, 3, 3),
                     cols.reshape(c, 3, 3, h, wd), optimize=False)


def _calibrate(rng, dims, probe, pool_after, names):
    """TinyNet recipe (extractor.py:296-312): He draw, unit pre-activation std per channel on
    the probe, bias 0.2 - mean, then relu (+ 2x2 avg pool) to feed the next layer."""
    layers, cur = [], probe
    for (cin, cout), pool_here, (cname, rname, pname) in zip(dims, pool_after, names):
        w = rng.normal(0.0, np.sqrt(2.0 / (cin * 9)), size=(cout, cin, 3, 3))
        pre = _conv_np(cur, w)
        sd = pre.reshape(cout, -1).std(axis=1)
        w /= sd[:, None, None, None]
        pre /= sd[:, None, None]
        b = 0.2 - pre.reshape(cout, -1).mean(axis=1)
        layers += [replace(conv(cname, cin, cout), weight=w, bias=b), relu(rname)]
        cur = np.maximum(pre + b[:, None, None], 0)
        if pool_here:
            layers.append(pool(pname, 2, "avg"))
            c, h, wd = cur.shape
            cur = cur[:, :h // 2 * 2, :wd // 2 * 2].reshape(c, h // 2, 2, wd // 2, 2).mean(axis=(2, 4))
    return layers


def with_pooling(spec: ExtractorSpec, pooling: str) -> ExtractorSpec:
    """The same network (weights included) with every pool layer set to `pooling`
    ("avg" or "max", reference extractor.py:321 vgg19(pooling=...))."""
    if pooling not in ("avg", "max"):
        raise ShapeError(f"pooling must be avg or max, got {pooling!r}")
    return replace(spec, layers=tuple(replace(l, pool=pooling) if l.kind == "pool" else l for l in spec.layers))


def calibrated_vgg19(seed: int = 0, probe: int = 64, pooling: str = "avg") -> ExtractorSpec:
    """VGG-19 with seeded, activation-calibrated weights: per conv, draw
    N(0, 2/(9 C_in)) from default_rng(seed) in layer order, normalise each channel's
    pre-activation std on a seeded probe (rng.random, preprocessed), bias = 0.2 - mean.
    The weights are calibrated through average pooling; ``pooling="max"`` then swaps the pool
    kind (identical weights)."""
    base = vgg19("avg")
    rng = np.random.default_rng(seed)
    img = rng.random((3, probe, probe))
    pre = base.preprocess
    x = (img - np.asarray(pre.mean)[:, None, None]) / np.asarray(pre.scale)[:, None, None]
    convs = [l for l in base.layers if l.kind == "conv"]
    dims, pools, names = [], [], []
    names_all = [l.name for l in base.layers]
    for l in convs:
        i = names_all.index(l.name)
        has_pool = i + 2 < len(base.layers) and base.layers[i + 2].kind == "pool"
        dims.append((l.in_ch, l.out_ch))
        pools.append(has_pool)
        names.append((l.name, base.layers[i + 1].name, base.layers[i + 2].name if has_pool else ""))
    layers = _calibrate(rng, dims, x, pools, names)
    out = replace(base, layers=tuple(layers))
    return out if pooling == "avg" else with_pooling(out, pooling)


def tinynet(seed: int = 0) -> ExtractorSpec:
    """Three-conv desk-scale extractor (extractor.py:287-315): strides 1/2/4, taps at every
    relu, content relu2; weights calibrated on a seeded 48x48 probe."""
    rng = np.random.default_rng(seed)
    probe = rng.random((3, 48, 48))
    layers = _calibrate(rng, [(3, 8), (8, 16), (16, 32)], probe, [True, True, False],
                        [("conv1", "relu1", "pool1"), ("conv2", "relu2", "pool2"), ("conv3", "relu3", "")])
    return ExtractorSpec(tuple(layers), ("relu1", "relu2", "relu3"), "relu2")


def check_device_supported(spec) -> None:
    """The device path covers (conv3x3 s1 -> relu [-> avg / max pool 2]) chains up to the deepest tap."""
    for l in spec.layers[:spec.deepest_tap_index() + 1]:
        if l.kind == "conv" and (l.k != 3 or l.stride != 1):
            raise ShapeError(f"{l.name}: device path supports 3x3 stride-1 convs only")
        if l.kind == "pool" and l.k != 2:
            raise ShapeError(f"{l.name}: device path supports 2x2 pools only")
