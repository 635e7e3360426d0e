"""Multi-GPU Algorithm 1: one image split into a 2-D grid of owned rectangles, one process per GPU.

Decomposition.  The padded image is cut into ry x rx owned rectangles
(sides are multiples of the deepest stride; ``choose_grid`` picks the factorisation of the
world size with the smallest per-rank window -- 2x4 for 8 GPUs at 6048x8064).  Each rank
evaluates its rectangle plus a receptive-field halo of ``margin_for_exact_gradient`` pixels
(160 for VGG-19) as one zero-padded window (engine ``spst_bind_window``), so its owned pixels
see exactly the whole-image activations (reference localized.py:1-14 -- the argument that makes
the reference's blockwise gradient exact).  The only global coupling of the loss is the per-tap
statistics, so per evaluation the data-path exchange is:

  * the x halo: each rank receives the parts of its window owned by other ranks point-to-point
    (``halo_window``; up to 8 neighbours on a 2-D grid, more when a neighbour is thinner than
    the halo);
  * the statistics: every style tap's owned partials S = sum F F^T, s = sum F (611,776 f64 for
    VGG-19) and the content distance, packed in ONE buffer and reduced in FIXED RANK ORDER
    (all-gather, then an ordered sum on every rank: the result does not depend on the
    collective's internal order, SURVEY.md §5 "determinism").

L-BFGS runs on each rank's owned pixels of x / g / s / y; its dot products and max|g| are
scalars reduced the same fixed-order way (``allreduce``).  Each rank writes only its owned
gradient pixels, so no gradient all-gather is needed.  Images too small to gain from splitting
(a rank's window would exceed 60 % of the image) are replicated instead: every rank evaluates
the whole image and no data-path collective runs.

The per-rank engine is the device ``Engine`` (``DeviceWindowEngine``); tests substitute a CPU
oracle engine with the same interface to check this host logic with the gloo backend.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .spec import tap_geometry
from .stats import finalize_sums
from .tiling import margin_for_exact_gradient


def init(local_rank: int | None = None, backend: str | None = None):
    """Initialise the default process group from torchrun's env (MASTER_ADDR=127.0.0.1)."""
    if not dist.is_initialized():
        if backend is None:  # SPST_DIST_BACKEND: functional multi-rank checks on one device (gloo)
            backend = os.environ.get("SPST_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl" and local_rank is not None:
            torch.cuda.set_device(local_rank)
        dist.init_process_group(backend)
        if backend == "nccl":
            # create the communicator eagerly with a collective every rank joins: the first
            # NCCL call of a group must not be a batch_isend_irecv that only some ranks issue
            dist.all_reduce(torch.zeros(1, device=torch.cuda.current_device()))
    return dist.group.WORLD


def world_size(group=None) -> int:
    return dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1


# ------------------------------------------------------------------------------------------
# geometry
# ------------------------------------------------------------------------------------------

@dataclass(frozen=True)
class Window:
    """A rank's share of the padded grid (padded-image coordinates): it evaluates rows
    [gr0, gr1) x columns [gc0, gc1) as one zero-padded image and owns [or0, or1) x [oc0, oc1)."""
    gr0: int
    gr1: int
    or0: int
    or1: int
    gc0: int
    gc1: int
    oc0: int
    oc1: int

    @property
    def area(self) -> int:
        return (self.gr1 - self.gr0) * (self.gc1 - self.gc0)

    def bind_args(self):
        return (self.gr0, self.gr1), (self.or0, self.or1), (self.gc0, self.gc1), (self.oc0, self.oc1)


def _split(n_px: int, stride: int, parts: int) -> list:
    units = n_px // stride
    return [round(i * units / parts) * stride for i in range(parts + 1)]


def grid_windows(Hp: int, Wp: int, stride: int, halo: int, ry: int, rx: int) -> list:
    """ry x rx owned rectangles (row-major rank order) with `halo`-pixel windows."""
    if ry > Hp // stride or rx > Wp // stride:
        raise ValueError(f"a {Hp}x{Wp} grid has {Hp // stride}x{Wp // stride} stride cells, cannot split {ry}x{rx}")
    rb, cb = _split(Hp, stride, ry), _split(Wp, stride, rx)
    out = []
    for i in range(ry):
        for j in range(rx):
            o0, o1, c0, c1 = rb[i], rb[i + 1], cb[j], cb[j + 1]
            out.append(Window(max(0, o0 - halo), min(Hp, o1 + halo), o0, o1,
                              max(0, c0 - halo), min(Wp, c1 + halo), c0, c1))
    return out


def choose_grid(Hp: int, Wp: int, stride: int, halo: int, n: int) -> tuple:
    """(ry, rx) with ry * rx = n minimising the largest rank window ((0, 0): replicate -- no
    factorisation brings a window under 60 % of the image)."""
    best, best_area = (0, 0), None
    for ry in range(1, n + 1):
        if n % ry:
            continue
        rx = n // ry
        if ry > Hp // stride or rx > Wp // stride:
            continue
        area = max(w.area for w in grid_windows(Hp, Wp, stride, halo, ry, rx))
        if best_area is None or area < best_area:
            best, best_area = (ry, rx), area
    if best_area is None or (n > 1 and best_area > 0.6 * Hp * Wp):
        return (0, 0)
    return best


# ------------------------------------------------------------------------------------------
# sharded problem
# ------------------------------------------------------------------------------------------

class ShardedProblem:
    """2-D grid sharded transfer problem (one rank's view)."""

    def __init__(self, u, v, spec, weights, engine, group=None, halo: int | None = None, grid=None,
                 style_stats: dict | None = None):
        self.spec = spec
        self.weights = weights
        self.engine = engine
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_available() and dist.is_initialized() else 0
        self.world = world_size(group)
        self.s = spec.deepest_stride()
        self.halo = margin_for_exact_gradient(spec) if halo is None else halo
        ref = u if u is not None else v
        self.h, self.w = int(ref.shape[0]), int(ref.shape[1])
        self.Hp = self.h + (-self.h) % self.s
        self.Wp = self.w + (-self.w) % self.s
        ry, rx = grid if grid is not None else choose_grid(self.Hp, self.Wp, self.s, self.halo, self.world)
        self.replicated = ry == 0
        if self.replicated:
            self.windows = [Window(0, self.Hp, 0, self.Hp, 0, self.Wp, 0, self.Wp)] * self.world
        else:
            if ry * rx != self.world:
                raise ValueError(f"grid {ry}x{rx} does not match world size {self.world}")
            self.windows = grid_windows(self.Hp, self.Wp, self.s, self.halo, ry, rx)
        self.grid_shape = (ry, rx)
        self.me = self.windows[self.rank]
        # owned pixels of the unpadded image, per rank: (r0, r1, c0, c1)
        self.owned = [(min(wd.or0, self.h), min(wd.or1, self.h), min(wd.oc0, self.w), min(wd.oc1, self.w))
                      for wd in self.windows]
        self.own = self.owned[self.rank]
        self.max_shard = max((b - a) * (d - c) for a, b, c, d in self.owned) * 3
        self.style_stats = style_stats if style_stats is not None else self._sharded_stats(v)
        self._content = weights.lambda_c > 0
        self._bind()
        if self._content:
            self.engine.forward_block(self._block_of(u, self.me), (self.me.gr0, self.me.gc0))
            self.engine.capture_content()
        for i, t in enumerate(spec.style_taps):
            self.engine.set_style_ref(i, self.style_stats[t], weights.style[t])
        self.counts = [(self.Hp // tap_geometry(spec, t).stride) * (self.Wp // tap_geometry(spec, t).stride)
                       for t in spec.style_taps]

    # ------------------------------------------------------------------ helpers
    def _bind(self):
        self.engine.bind(self.h, self.w, *self.me.bind_args())

    def _block_of(self, img, wd: Window, h=None, w=None):
        """Image pixels of window wd (clipped to the image) as a contiguous block."""
        h = self.h if h is None else h
        w = self.w if w is None else w
        a = img[wd.gr0:min(wd.gr1, h), wd.gc0:min(wd.gc1, w)]
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
        return t.contiguous()

    def _gloo_cuda(self, t) -> bool:
        return t.is_cuda and dist.get_backend(self.group) == "gloo"

    def allreduce(self, t, op="sum"):
        """Sum (or max) over ranks in FIXED rank order: all-gather, then an ordered reduction on
        every rank (the result does not depend on the collective's internal order)."""
        if self.world == 1 or self.replicated:
            return t
        stage = self._gloo_cuda(t)
        src = t.cpu() if stage else t.contiguous()
        parts = [torch.empty_like(src) for _ in range(self.world)]
        dist.all_gather(parts, src, group=self.group)
        acc = parts[0].clone()
        for p in parts[1:]:
            if op == "max":
                torch.maximum(acc, p, out=acc)
            else:
                acc += p
        t.copy_(acc.to(t.device) if stage else acc)
        return t

    def _sharded_stats(self, v):
        """Global style statistics of v: each rank reduces its own rectangle of v's grid."""
        s = self.s
        vh, vw = int(v.shape[0]), int(v.shape[1])
        vHp, vWp = vh + (-vh) % s, vw + (-vw) % s
        ry, rx = choose_grid(vHp, vWp, s, self.halo, self.world)
        if ry == 0:  # small style image: every rank computes it whole, no exchange
            wd = Window(0, vHp, 0, vHp, 0, vWp, 0, vWp)
        else:
            wd = grid_windows(vHp, vWp, s, self.halo, ry, rx)[self.rank]
        self.engine.bind(vh, vw, *wd.bind_args())
        self.engine.forward_block(self._block_of(v, wd, vh, vw), (wd.gr0, wd.gc0))
        sums = [self.engine.tap_sums(i) for i in range(len(self.spec.style_taps))]
        if ry != 0 and self.world > 1:
            flat = [t for pr in sums for t in pr]
            buf = torch.cat([t.reshape(-1) for t in flat])
            self._ordered_sum(buf)
            off = 0
            for t in flat:
                t.copy_(buf[off:off + t.numel()].view_as(t))
                off += t.numel()
        out = {}
        for i, t in enumerate(self.spec.style_taps):
            g = tap_geometry(self.spec, t).stride
            S, sv = sums[i]
            out[t] = finalize_sums(S.cpu().numpy().astype(np.float64), sv.cpu().numpy().astype(np.float64),
                                   (vHp // g) * (vWp // g))
        return out

    def _ordered_sum(self, buf):
        stage = self._gloo_cuda(buf)
        src = buf.cpu() if stage else buf
        parts = [torch.empty_like(src) for _ in range(self.world)]
        dist.all_gather(parts, src, group=self.group)
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p
        buf.copy_(acc.to(buf.device) if stage else acc)

    def _reduce(self, parts, extra=None):
        """One fixed-order reduction of every tap's (S, s) partials (+ the content distance)."""
        if self.world == 1 or self.replicated:
            return
        flat = [t for pr in parts for t in pr] + ([extra] if extra is not None else [])
        buf = torch.cat([t.reshape(-1) for t in flat])
        self._ordered_sum(buf)
        off = 0
        for t in flat:
            n = t.numel()
            t.copy_(buf[off:off + n].view_as(t))
            off += n

    def shard_of(self, x):
        """This rank's owned pixels of a full image, flattened (the L-BFGS vector shard)."""
        a, b, c, d = self.own
        t = x[a:b, c:d] if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x[a:b, c:d]))
        if hasattr(self.engine, "device_of"):  # the device engine computes on float32 vectors
            t = t.to(self.engine.device_of(), torch.float32)
        return t.contiguous().reshape(-1).clone()

    def _shard_view(self, shard, k=None):
        a, b, c, d = self.owned[self.rank if k is None else k]
        return shard[:(b - a) * (d - c) * 3].view(b - a, d - c, 3)

    def gather_image(self, shard):
        """Full (h, w, 3) image from every rank's shard (all-gather of padded shards) -- for
        results, scale changes and checkpoints; the evaluation itself only exchanges halos."""
        if self.replicated or self.world == 1:
            return self._shard_view(shard).clone()
        stage = self._gloo_cuda(shard)
        buf = torch.zeros(self.max_shard, dtype=shard.dtype, device="cpu" if stage else shard.device)
        buf[:shard.numel()] = shard.cpu() if stage else shard
        parts = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(parts, buf, group=self.group)
        img = torch.empty((self.h, self.w, 3), dtype=shard.dtype, device=shard.device)
        for k, p in enumerate(parts):
            a, b, c, d = self.owned[k]
            if b > a and d > c:
                img[a:b, c:d] = self._shard_view(p, k).to(shard.device)
        return img

    # ------------------------------------------------------------------ objective
    def halo_window(self, shard):
        """This rank's window pixels of x: its own shard plus the parts of the window owned by
        other ranks, exchanged point-to-point (each rank sends exactly the pixels of its
        owned rectangle that another rank's window covers).  At 8 ranks (2x4) of 6048x8064
        this moves the 160-px frame of a 3024x2016 rectangle per rank instead of an all-gather
        of the image."""
        me = self.me
        g0, g1, c0, c1 = me.gr0, min(me.gr1, self.h), me.gc0, min(me.gc1, self.w)
        win = torch.empty((g1 - g0, c1 - c0, 3), dtype=shard.dtype, device=shard.device)
        a, b, c, d = self.own
        mine = self._shard_view(shard)
        win[a - g0:b - g0, c - c0:d - c0] = mine
        if self.world > 1 and not self.replicated:
            stage = self._gloo_cuda(shard)
            ops, landed = [], []
            for j, wd in enumerate(self.windows):
                if j == self.rank:
                    continue
                ja, jb, jc, jd = self.owned[j]
                r0, r1, q0, q1 = max(g0, ja), min(g1, jb), max(c0, jc), min(c1, jd)  # j's pixels I need
                if r1 > r0 and q1 > q0:
                    buf = torch.empty((r1 - r0, q1 - q0, 3), dtype=shard.dtype,
                                      device="cpu" if stage else shard.device)
                    landed.append(((r0 - g0, r1 - g0, q0 - c0, q1 - c0), buf))
                    ops.append(dist.P2POp(dist.irecv, buf, j, group=self.group))
                wr0, wr1, wc0, wc1 = wd.gr0, min(wd.gr1, self.h), wd.gc0, min(wd.gc1, self.w)
                s0, s1, t0, t1 = max(wr0, a), min(wr1, b), max(wc0, c), min(wc1, d)  # my pixels j needs
                if s1 > s0 and t1 > t0:
                    src = mine[s0 - a:s1 - a, t0 - c:t1 - c].contiguous()
                    ops.append(dist.P2POp(dist.isend, src.cpu() if stage else src, j, group=self.group))
            if ops:
                for req in dist.batch_isend_irecv(ops):
                    req.wait()
            for (y0, y1, x0, x1), buf in landed:
                win[y0:y1, x0:x1] = buf.to(win.device)
        return win

    def loss(self, x_shard) -> float:
        self._bind()
        self.engine.forward_block(self.halo_window(x_shard), (self.me.gr0, self.me.gc0))
        parts = [self.engine.tap_sums(i) for i in range(len(self.spec.style_taps))]
        c = self.engine.content_sqdiff() if self._content else None
        self._reduce(parts, c)
        terms, _ = self.engine.finalize(self.counts)
        total = float(np.sum(terms))
        if self._content:
            total += self.weights.lambda_c * float(c.item())
        return total

    def grad(self, out_shard):
        a, b, c, d = self.own
        self.engine.backward_block(2.0 * self.weights.lambda_c if self._content else 0.0,
                                   self._shard_view(out_shard), (a, c))
        return out_shard

    def objective(self):
        return _ShardObjective(self)


class _ShardObjective:
    lazy = True

    def __init__(self, sp: ShardedProblem):
        self.sp = sp

    def loss(self, x_shard):
        return self.sp.loss(x_shard)

    def grad(self, out):
        return self.sp.grad(out)


def build_sharded_problem(u, v, spec, weights, group=None, style_stats=None, grid=None):
    """Device version: one Engine per rank bound to its window."""
    from .device import engine_for
    return ShardedProblem(u, v, spec, weights, DeviceWindowEngine(engine_for(spec)), group=group,
                          style_stats=style_stats, grid=grid)


class DeviceWindowEngine:
    """Adapter giving the device Engine the window interface (image blocks addressed by their
    global origin)."""

    def __init__(self, engine):
        self.e = engine

    def device_of(self):
        return torch.device("cuda", self.e.device)

    def bind(self, h, w, grid, own, gcols, ocols):
        self.e.bind(h, w, grid, own, gcols, ocols)

    def forward_block(self, block, origin):
        block = block.to(self.device_of(), torch.float32).contiguous()
        self._block = block  # keep alive for the duration of the pass
        self.e.forward(block, origin=origin)

    def tap_sums(self, i):
        return self.e.tap_sums(i)

    def set_style_ref(self, i, stats, w):
        self.e.set_style_ref(i, stats, w)

    def finalize(self, counts):
        return self.e.finalize(counts)

    def capture_content(self):
        self.e.capture_content()

    def content_sqdiff(self):
        return self.e.content_sqdiff()

    def backward_block(self, two_lambda, out_block, origin):
        self.e.backward(two_lambda, out_block, origin=origin)
