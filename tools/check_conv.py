"""GPU smoke of the tensor-core conv + Gram kernels against torch fp64 (debug hooks)."""
import ctypes, sys, time
import numpy as np
import torch
import torch.nn.functional as F
sys.path.insert(0, ".")
from paper_2212_13459_b200 import _native as nat

L = nat.lib()
rng = np.random.default_rng(0)
worst = 0.0
for (cin, cout, H, W) in [(64, 64, 20, 150), (64, 128, 9, 40), (128, 128, 7, 131), (256, 256, 6, 64), (512, 512, 4, 33), (64, 64, 256, 256)]:
    x = rng.random((cin, H, W)).astype(np.float32)
    w = rng.normal(0, np.sqrt(2 / (9 * cin)), (cout, cin, 3, 3))
    b = rng.normal(0, 0.1, cout)
    for mode in (0, 1, 2, 3):
        if mode == 1 and (H % 2 or W % 2):
            continue
        xin = x if mode != 2 else rng.standard_normal((cout, H, W)).astype(np.float32)
        ny = cout if mode != 2 else cin
        shape = (ny, H // 2, W // 2) if mode == 1 else (ny, H, W)
        y = np.zeros(shape, np.float32)
        st = L.spst_debug_conv(0, mode, cin, cout, H, W, xin.ctypes.data, w.ctypes.data, b.ctypes.data, y.ctypes.data)
        if st != 0:
            print("status", st); sys.exit(1)
        xt = torch.from_numpy(xin).double()[None]
        wt = torch.from_numpy(w)
        if mode == 2:
            ref = F.conv_transpose2d(xt, wt, padding=1)[0]
        else:
            pre = F.conv2d(xt, wt, torch.from_numpy(b), padding=1)[0]
            ref = (pre > 0).double() if mode == 3 else torch.relu(pre)
            if mode == 1:
                ref = F.avg_pool2d(ref[None], 2)[0]
        ref = ref.numpy()
        if mode == 3:
            err = float(np.mean(ref != y))
        else:
            err = float(np.linalg.norm(ref - y) / max(np.linalg.norm(ref), 1e-30))
        worst = max(worst, err if mode != 3 else 0)
        print(f"conv cin={cin} cout={cout} {H}x{W} mode={mode} rel_err={err:.3e}")
for (C, P) in [(64, 5000), (128, 20000), (256, 9000), (512, 17000), (512, 1000)]:
    f = rng.random((C, P)).astype(np.float32)
    S = np.zeros((C, C))
    st = L.spst_debug_gram(0, C, P, f.ctypes.data, S.ctypes.data)
    ref = f.astype(np.float64) @ f.astype(np.float64).T
    err = np.abs(S - ref).max() / np.abs(ref).max()
    worst = max(worst, err)
    print(f"gram C={C} P={P} status={st} max rel err={err:.3e}")
print("WORST", worst)
