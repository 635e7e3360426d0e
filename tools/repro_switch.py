"""Problem switch on one engine: the first gradient after another problem's evaluations."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2212_13459_b200 as spst
spec = spst.calibrated_vgg19(0)
rng = np.random.default_rng(3)
h, w = 360, 200
u = rng.random((h, w, 3)).astype(np.float32)
v = rng.random((120, 110, 3)).astype(np.float32)
x = np.clip(u + 0.1 * rng.standard_normal(u.shape), 0, 1).astype(np.float32)
pA = spst.build_problem(u, v, spec, spst.default_loss_weights(spec, lambda_c=1e-3))
print("A", spst.loss_grad(x, pA)[0], flush=True)
d = np.load(os.path.join(ROOT, "tests/golden/vgg19.npz"))
it = np.load(os.path.join(ROOT, "tests/golden/vgg19_iterates.npz"))
pB = spst.build_problem(d["c1_u"], d["c1_v"], spec, spst.default_loss_weights(spec, lambda_c=float(d["c1_lambda_c"][0])))
for k in range(3):
    l, g = spst.loss_grad(it["x0"], pB)
    print("B", k, l, np.linalg.norm(g - it["grad64_0"]) / np.linalg.norm(it["grad64_0"]), flush=True)
