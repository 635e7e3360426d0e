"""Multi-rank host logic of the sharded transfer on CPU (gloo, world_size 2).

The device Engine is replaced by an oracle-backed stripe engine with the same interface, so
this checks the decomposition itself: stripe/halo geometry, the statistics all-reduce, the
content-loss reduction, owned-row gradient assembly with the replicate-pad fold, sharded
L-BFGS dot products — against the single-process whole-image oracle."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleStripeEngine:
    """CPU stand-in for DeviceStripeEngine (test infrastructure, uses the oracle)."""

    def __init__(self, net):
        import spst_oracle as O
        self.O = O
        self.net = net
        self.refs = {}

    def bind(self, h, w, grid, own):
        s = self.net.deepest_stride()
        self.h, self.w = h, w
        self.Hp, self.Wp = h + (-h) % s, w + (-w) % s
        self.grid, self.own = grid, own

    def forward_rows(self, rows, row0):
        O, g0, g1 = self.O, self.grid[0], self.grid[1]
        r = rows.numpy().astype(np.float64)
        idx = [min(gr, self.h - 1) - row0 for gr in range(g0, g1)]
        loc = r[idx]
        loc = np.concatenate([loc, np.repeat(loc[:, -1:], self.Wp - self.w, axis=1)], axis=1)
        self.feats, self.saved = O.run_forward(np.ascontiguousarray(loc.transpose(2, 0, 1)), self.net, keep=True)
        self.sums = []
        for t in self.net.style_taps:
            st = self.net.geometry(t)[0]
            F = self.feats[t][:, (self.own[0] - g0) // st:(self.own[1] - g0) // st]
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
        st = self.net.geometry(self.net.content_tap)[0]
        g0 = self.grid[0]
        d = (self.feats[self.net.content_tap] - self.Vu)[:, (self.own[0] - g0) // st:(self.own[1] - g0) // st]
        return torch.tensor([float(np.sum(d ** 2))], dtype=torch.float64)

    def backward_rows(self, two_lambda, out, own_row0, w):
        O = self.O
        tg = {t: O.style_feature_grad(self.feats[t], self.stats_x[t], *self.refs[t]) for t in self.net.style_taps}
        ct = self.net.content_tap
        if two_lambda:
            cg = two_lambda * (self.feats[ct] - self.Vu)
            tg[ct] = tg[ct] + cg if ct in tg else cg
        g = O.run_backward(tg, self.saved, self.net).transpose(1, 2, 0)  # (Hl, Wp, 3)
        g0 = self.grid[0]
        r0, r1 = own_row0, min(self.own[1], self.h)
        res = np.zeros((r1 - r0, w, 3))
        for gr in range(r0, r1):
            row = g[gr - g0].copy()
            if gr == self.h - 1:
                for extra in range(self.h, self.Hp):
                    row += g[extra - g0]
            res[gr - r0] = row[:w]
            res[gr - r0, w - 1] += row[w:].sum(axis=0)
        out.view(r1 - r0, w, 3).copy_(torch.from_numpy(res))


def _worker(rank, world, port, case, q):
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
        sp = ShardedProblem(u, v, spec, wts, OracleStripeEngine(net), halo=halo)
        xs = sp.shard_of(x).double()
        loss = sp.loss(xs)
        g = torch.empty_like(xs)
        sp.grad(g)
        full = sp.gather_image(g)
        # sharded scalar reductions used by L-BFGS (dot products / max|g|) equal the global ones
        dot = sp.allreduce(torch.tensor([float(xs @ g)], dtype=torch.float64))
        mx = sp.allreduce(torch.tensor([float(g.abs().max())], dtype=torch.float64), op="max")
        if rank == 0:
            q.put((loss, full.numpy(), (float(dot), float(mx)), sp.stripes))
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


def _run(case, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
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
def test_two_rank_stripes_equal_whole_image(case):
    loss, grad, losses, st = _run(case)
    assert len(st) == 2 and st[0].own_r1 == st[1].own_r0
    (lo, go), p, x = _global_oracle(case)
    assert abs(loss - lo) <= 1e-10 * abs(lo)
    assert np.linalg.norm(grad - go) <= 1e-10 * np.linalg.norm(go)


def test_three_ranks_halo_wider_than_a_stripe():
    """Halo exchange when a neighbour's stripe is thinner than the halo: rank 0's window needs
    rows from rank 2 as well as rank 1 (point-to-point from every rank that owns them)."""
    case = (48, 40, 32)
    loss, grad, _, st = _run(case, world=3)
    assert len(st) == 3 and st[1].own_r1 - st[1].own_r0 < 32 and st[0].grid_r1 > st[1].own_r1
    (lo, go), _, _ = _global_oracle(case)
    assert abs(loss - lo) <= 1e-10 * abs(lo)
    assert np.linalg.norm(grad - go) <= 1e-10 * np.linalg.norm(go)


def test_two_rank_lbfgs_reductions_match_global():
    """Sharded L-BFGS scalars: sum of per-rank dot products and max of per-rank max|g|."""
    case = (96, 80, 16)
    loss, grad, (dot, mx), _ = _run(case)
    (lo, go), _, x = _global_oracle(case)
    assert dot == pytest.approx(float(np.vdot(x, go)), rel=1e-10)
    assert mx == pytest.approx(float(np.abs(go).max()), rel=1e-12)


def test_zero_halo_is_visibly_wrong():
    """Reference test_localized.py:72-78 analogue: without the receptive-field halo the stripe
    gradient is not the whole-image gradient."""
    case = (96, 80, 0)
    loss, grad, _, _ = _run(case)
    (lo, go), _, _ = _global_oracle(case)
    assert np.linalg.norm(grad - go) >= 1e-3 * np.linalg.norm(go)
