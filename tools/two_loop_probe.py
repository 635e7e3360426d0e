import sys, time, torch
sys.path.insert(0, "/root/repo")
from paper_2212_13459_b200 import _native as nat
from paper_2212_13459_b200.lbfgs import LBFGSState, _two_loop, _Vec
for n, m in [(2_300_000, 100), (2_300_000, 10), (146_000_000, 10)]:
    g0 = torch.Generator(device="cuda").manual_seed(1)
    st = LBFGSState()
    for _ in range(m):
        s = torch.randn(n, device="cuda", generator=g0); y = s + 0.3 * torch.randn(n, device="cuda", generator=g0)
        st.push(s, y, m)
    g = torch.randn(n, device="cuda", generator=g0); vec = _Vec(torch.float32, g.device); out = torch.empty_like(g)
    for name, ar in [("native", None), ("steps", lambda t, op="sum": t)]:
        _two_loop(g, st, vec, out, ar); torch.cuda.synchronize()
        c0 = nat.lib().spst_launch_count(); t = time.perf_counter()
        for _ in range(5): _two_loop(g, st, vec, out, ar)
        torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 5
        print(f"n={n} m={m} {name}: {dt*1e3:.2f} ms, launches/call {(nat.lib().spst_launch_count()-c0)/5:.0f}")
    del st, g, out
    torch.cuda.empty_cache()
