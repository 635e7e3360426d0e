"""One native two-loop (m=10) at the 6048x8064 vector length, for an ncu capture of
two_loop_coop_kernel:  ncu --set full -k regex:two_loop_coop -c 1 python tools/two_loop_ncu.py
Algorithmic bytes: (2m+1) fused steps, each reading q, v, w and writing q (the first reads g
and writes q, the last has no w): (8m + 2) x N x 4 B."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_13459_b200.lbfgs import LBFGSState, _two_loop, _Vec  # noqa: E402

n, m = 6048 * 8064 * 3, 10
gen = torch.Generator(device="cuda").manual_seed(1)
st = LBFGSState()
for _ in range(m):
    s = torch.randn(n, device="cuda", generator=gen)
    st.push(s, s + 0.3 * torch.randn(n, device="cuda", generator=gen), m)
g = torch.randn(n, device="cuda", generator=gen)
vec, out = _Vec(torch.float32, g.device), torch.empty_like(g)
_two_loop(g, st, vec, out, None)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    _two_loop(g, st, vec, out, None)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"two-loop m={m} n={n}: {ms:.2f} ms, {(8 * m + 2) * n * 4 / ms / 1e6:.0f} GB/s algorithmic")
