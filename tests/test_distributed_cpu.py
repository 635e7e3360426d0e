"""Multi-rank host logic of the sharded transfer on CPU (gloo, world_size 2-4).

The device Engine is replaced by an oracle-backed window engine with the same interface, so
this checks the decomposition itself: 2-D grid / halo geometry, the fixed-order statistics
reduction, the content-loss reduction, owned-rectangle gradient assembly with the
replicate-pad fold, sharded L-BFGS scalars -- against the single-process whole-image oracle."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleWindowEngine:
    """CPU stand-in for DeviceWindowEngine (test infrastructure, uses the oracle): evaluates the
    bound window as one zero-padded image of replicate-clamped pixels, owns a rectangle."""

    def __init__(self, net):
        import spst_oracle as O
        self.O = O
        self.net = net
        self.refs = {}

    def bind(self, h, w, grid, own, gcols, ocols):
        s = self.net.deepest_stride()
        self.h, self.w = h, w
        self.Hp, self.Wp = h + (-h) % s, w + (-w) % s
        self.grid, self.own, self.gcols, self.ocols = grid, own, gcols, ocols

    def _crop(self, t, stride):
        (g0, _), (o0, o1), (c0, _), (q0, q1) = self.grid, self.own, self.gcols, self.ocols
        return t[:, (o0 - g0) // stride:(o1 - g0) // stride, (q0 - c0) // stride:(q1 - c0) // stride]

    def forward_block(self, block, origin):
        O = self.O
        (g0, g1), (c0, c1) = self.grid, self.gcols
        b = block.numpy().astype(np.float64)
        ys = [min(y, self.h - 1) - origin[0] for y in range(g0, g1)]
        xs = [min(x, self.w - 1) - origin[1] for x in range(c0, c1)]
        loc = b[np.ix_(ys, xs)]
        self.feats, self.saved = O.run_forward(np.ascontiguousarray(loc.transpose(2, 0, 1)), self.net, keep=True)
        self.sums = []
        for t in self.net.style_taps:
            F = self._crop(self.feats[t], self.net.geometry(t)[0])
            flat = F.reshape(F.shape[0], -1)
            self.sums.append((torch.from_numpy(flat @ flat.T), torch.from_numpy(flat.sum(axis=1))))

    def tap_sums(self, i):
        return self.sums[i]

    def set_style_ref(self, i, stats, w):
        self.refs[self.net.style_taps[i]] = (self.O.OStats(stats.gram, stats.mean, stats.std, stats.n_p),
                                             self.O.OW(w.gram, w.mean, w.std))

    def finalize(self, counts):
        O = self.O
        self.stats_x, terms = {}, []
        for i, t in enumerate(self.net.style_taps):
            S, s = self.sums[i]
            n = counts[i]
            g = S.numpy() / n
            mu = s.numpy() / n
            sx = O.OStats(g, mu, np.sqrt(np.maximum(np.diagonal(g) - mu ** 2, 0)), n)
            self.stats_x[t] = sx
            terms.append(O.style_terms(sx, *self.refs[t]))
        return np.array(terms), [False] * len(terms)

    def capture_content(self):
        self.Vu = self.feats[self.net.content_tap].copy()

    def content_sqdiff(self):
        ct = self.net.content_tap
        d = self._crop(self.feats[ct] - self.Vu, self.net.geometry(ct)[0])
        return torch.tensor([float(np.sum(d ** 2))], dtype=torch.float64)

    def backward_block(self, two_lambda, out, origin):
        O = self.O
        tg = {t: O.style_feature_grad(self.feats[t], self.stats_x[t], *self.refs[t]) for t in self.net.style_taps}
        ct = self.net.content_tap
        if two_lambda:
            cg = two_lambda * (self.feats[ct] - self.Vu)
            tg[ct] = tg[ct] + cg if ct in tg else cg
        g = O.run_backward(tg, self.saved, self.net).transpose(1, 2, 0)  # window grid (Hl, Wl, 3)
        (g0, _), (o0, o1), (c0, _), (q0, q1) = self.grid, self.own, self.gcols, self.ocols
        loc = g[o0 - g0:o1 - g0, q0 - c0:q1 - c0]          # owned padded rectangle
        ri, ci = min(o1, self.h) - o0, min(q1, self.w) - q0  # its image part
        res = loc[:ri, :ci].copy()
        if o1 > self.h:  # replicate-pad rows fold onto the last image row (tensorops.py:212-229)
            res[-1] += loc[ri:, :ci].sum(axis=0)
        if q1 > self.w:
            res[:, -1] += loc[:ri, ci:].sum(axis=1)
        if o1 > self.h and q1 > self.w:
            res[-1, -1] += loc[ri:, ci:].sum(axis=(0, 1))
        assert tuple(origin) == (o0, q0)
        out.copy_(torch.from_numpy(res))


def _worker(rank, world, port, case, q, grid=None, repeat=1):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import spst_oracle as O
    from paper_2212_13459_b200.distributed import ShardedProblem
    from paper_2212_13459_b200.spec import tinynet
    from paper_2212_13459_b200.stats import default_loss_weights
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        spec = tinynet(0)
        net = O.onet_from_spec(spec)
        rng = np.random.default_rng(7)
        h, w, halo = case
        u, v, x = rng.random((h, w, 3)), rng.random((h + 13, w - 5, 3)), rng.random((h, w, 3))
        wts = default_loss_weights(spec)
        sp = ShardedProblem(u, v, spec, wts, OracleWindowEngine(net), halo=halo, grid=grid)
        xs = sp.shard_of(x).double()
        out = []
        for _ in range(repeat):
            loss = sp.loss(xs)
            g = torch.empty_like(xs)
            sp.grad(g)
            out.append((loss, sp.gather_image(g).numpy()))
        # sharded scalar reductions used by L-BFGS (dot products / max|g|) equal the global ones
        dot = sp.allreduce(torch.tensor([float(xs @ g)], dtype=torch.float64))
        mx = sp.allreduce(torch.tensor([float(g.abs().max())], dtype=torch.float64), op="max")
        if rank == 0:
            q.put((out[0][0], out[0][1], (float(dot), float(mx)), sp.windows, sp.grid_shape, out))
    except Exception as e:  # surface worker failures immediately
        q.put(e)
        raise
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(case, world=2, grid=None, repeat=1):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q, grid, repeat)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=600)
    if isinstance(out, Exception):
        raise out
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def _global_oracle(case):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import spst_oracle as O
    from paper_2212_13459_b200.spec import tinynet
    net = O.onet_from_spec(tinynet(0))
    rng = np.random.default_rng(7)
    h, w, _ = case
    u, v, x = rng.random((h, w, 3)), rng.random((h + 13, w - 5, 3)), rng.random((h, w, 3))
    p = O.build_problem(u, v, net, O.default_weights(net), 4096, 16)
    return O.loss_grad_global(x, p), p, x


@pytest.mark.parametrize("case", [(96, 80, 16), (77, 90, 16)])
def test_two_ranks_equal_whole_image(case):
    loss, grad, _, wins, shape, _ = _run(case, grid=(2, 1))
    assert len(wins) == 2 and shape == (2, 1)
    (lo, go), p, x = _global_oracle(case)
    assert abs(loss - lo) <= 1e-10 * abs(lo)
    assert np.linalg.norm(grad - go) <= 1e-10 * np.linalg.norm(go)


def test_four_ranks_2x2_grid_equal_whole_image():
    """2-D rank grid: owned rectangles with a halo on every interior side; the
    window of each rank needs pixels from all three other ranks (corner exchange)."""
    case = (77, 90, 16)
    loss, grad, _, wins, shape, _ = _run(case, world=4, grid=(2, 2))
    assert shape == (2, 2) and len({(w.oc0, w.oc1) for w in wins}) == 2
    (lo, go), _, _ = _global_oracle(case)
    assert abs(loss - lo) <= 1e-10 * abs(lo)
    assert np.linalg.norm(grad - go) <= 1e-10 * np.linalg.norm(go)


def test_three_ranks_halo_wider_than_a_stripe():
    """Halo exchange when a neighbour's rectangle is thinner than the halo: rank 0's window needs
    pixels from rank 2 as well as rank 1 (point-to-point from every rank that owns them)."""
    case = (48, 40, 32)
    loss, grad, _, wins, _, _ = _run(case, world=3, grid=(3, 1))
    assert wins[1].or1 - wins[1].or0 < 32 and wins[0].gr1 > wins[1].or1
    (lo, go), _, _ = _global_oracle(case)
    assert abs(loss - lo) <= 1e-10 * abs(lo)
    assert np.linalg.norm(grad - go) <= 1e-10 * np.linalg.norm(go)


def test_two_rank_lbfgs_reductions_match_global():
    """Sharded L-BFGS scalars: sum of per-rank dot products and max of per-rank max|g|."""
    case = (96, 80, 16)
    loss, grad, (dot, mx), _, _, _ = _run(case, grid=(1, 2))
    (lo, go), _, x = _global_oracle(case)
    assert dot == pytest.approx(float(np.vdot(x, go)), rel=1e-10)
    assert mx == pytest.approx(float(np.abs(go).max()), rel=1e-12)


def test_fixed_order_reduction_is_deterministic():
    """Repeated evaluations give bit-identical losses and gradients (statistics reduced by an
    all-gather and an ordered sum, not the collective's own order)."""
    _, _, _, _, _, outs = _run((77, 90, 16), world=4, grid=(2, 2), repeat=2)
    assert outs[0][0] == outs[1][0]
    np.testing.assert_array_equal(outs[0][1], outs[1][1])


def test_small_image_is_replicated():
    """No split brings a rank's window under 60 % of a small image: every rank evaluates the
    whole image (no data-path collective) and the result is the global one."""
    case = (40, 40, 16)
    loss, grad, _, wins, shape, _ = _run(case, world=2)
    assert shape == (0, 0)
    (lo, go), _, _ = _global_oracle(case)
    assert abs(loss - lo) <= 1e-10 * abs(lo)
    assert np.linalg.norm(grad - go) <= 1e-10 * np.linalg.norm(go)


def test_zero_halo_is_visibly_wrong():
    """Reference test_localized.py:72-78 analogue: without the receptive-field halo the sharded
    gradient is not the whole-image gradient."""
    case = (96, 80, 0)
    loss, grad, _, _, _, _ = _run(case, grid=(2, 1))
    (lo, go), _, _ = _global_oracle(case)
    assert np.linalg.norm(grad - go) >= 1e-3 * np.linalg.norm(go)


def test_choose_grid_prefers_2x4_at_8_gpus():
    sys.path.insert(0, ROOT)
    from paper_2212_13459_b200.distributed import choose_grid, grid_windows
    assert choose_grid(6048, 8064, 16, 160, 8) == (2, 4)
    assert choose_grid(6048, 8064, 16, 160, 4) == (2, 2)
    assert choose_grid(6048, 8064, 16, 160, 1) == (1, 1)
    assert choose_grid(256, 256, 16, 160, 8) == (0, 0)
    ws = grid_windows(6048, 8064, 16, 160, 2, 4)
    own = sum((w.or1 - w.or0) * (w.oc1 - w.oc0) for w in ws)
    assert own == 6048 * 8064
    assert max(w.area for w in ws) == (3024 + 160) * (2016 + 320)
