"""Measure the round-toward-zero bias of the tensor-core accumulation (GPU box; test infra).

    SPST_RZ_KAPPA=0 python tools/rz_calibrate.py   # raw bias -> fitted kappas
    python tools/rz_calibrate.py                                         # residual with the defaults

One tcgen05 conv layer (relu-like input, one K-chunk per TMEM group as in the forward) and the
two Gram kernels (64 and 256 channels) are compared with float64 on the same operands; the
signed relative error (mean of (ours - f64) * sign(f64) / mean |f64|) is the systematic part
the compensation in conv_tc.cu / gram_tc.cu removes.  With the compensation disabled it gives
kappa = -bias / w (w from rz_weight: 5 for a forward conv chunk, 8.5 for a 2-stage Gram
accumulator)."""

from __future__ import annotations

import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def conv64(x, w):
    C, H, W = x.shape
    xp = np.pad(x, ((0, 0), (1, 1), (1, 1)))
    out = np.zeros((w.shape[0], H, W))
    for dy in range(3):
        for dx in range(3):
            out += np.einsum("oc,chw->ohw", w[:, :, dy, dx], xp[:, dy:dy + H, dx:dx + W])
    return out


def main():
    from paper_2212_13459_b200 import _native as nat
    L = nat.lib()
    rng = np.random.default_rng(7)
    res = {"env": {k: v for k, v in os.environ.items() if k.startswith("SPST_")}}
    # conv: relu-like 256-channel input (half zeros), He weights, no bias
    for cin, cout, hw in ((256, 256, 32), (64, 128, 64)):
        x = np.maximum(rng.standard_normal((cin, hw, hw)), 0).astype(np.float32)
        w = rng.standard_normal((cout, cin, 3, 3)) * np.sqrt(2.0 / (9 * cin))
        b = np.zeros(cout)
        y = np.zeros((cout, hw, hw), np.float32)
        st = L.spst_debug_conv(0, 0, cin, cout, hw, hw, x.ctypes.data, w.ctypes.data, b.ctypes.data, y.ctypes.data)
        assert st == 0, st
        ref = conv64(x.astype(np.float64), w)
        pos = ref > 0
        bias = float(np.sum((y[pos] - ref[pos])) / np.sum(np.abs(ref[pos])))
        rel = float(np.linalg.norm(y[pos] - ref[pos]) / np.linalg.norm(ref[pos]))
        res[f"conv_{cin}x{cout}"] = {"bias": bias, "rel_l2": rel, "kappa_fit": -bias / 5.0}
    # Gram: relu-like features
    for C in (64, 256):
        P = 65536
        f = (np.maximum(rng.standard_normal((C, P)), 0) * rng.random((C, 1))).astype(np.float32)
        S = np.zeros((C, C))
        st = L.spst_debug_gram(0, C, P, f.ctypes.data, S.ctypes.data)
        assert st == 0, st
        f64 = f.astype(np.float64)
        ref = f64 @ f64.T
        d = np.eye(C, dtype=bool)
        bd = float(np.mean((S[d] - ref[d]) / ref[d]))
        off = ~d & (np.abs(ref) > 0)
        bo = float(np.sum((S[off] - ref[off]) * np.sign(ref[off])) / np.sum(np.abs(ref[off])))
        res[f"gram_{C}"] = {"diag_bias": bd, "off_bias": bo, "rel_l2": float(np.linalg.norm(S - ref) / np.linalg.norm(ref)),
                            "kappa_same_fit": -bd / 8.5, "kappa_off_fit": -bo / 8.5}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
