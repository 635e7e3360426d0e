"""Multi-GPU Algorithm 1: one image split into row stripes, one process per GPU.

Decomposition.  The padded image is cut into N owned row stripes (rows
are multiples of the deepest stride); each rank evaluates its stripe plus a receptive-field
halo of ``margin_for_exact_gradient`` rows (160 for VGG-19) as one zero-padded image, so its
owned rows see exactly the whole-image activations (reference localized.py:1-14 — the same
argument that makes the reference's blockwise gradient exact).  The only global coupling of
the loss is the per-tap statistics, so per evaluation the data-path exchange is:

  * all-reduce (sum, f64) of each style tap's owned-row partials S = sum F F^T and s = sum F
    (5 taps x (C^2 + C) = 611,776 values) between the forward and the gradient pass,
    fused with the content squared distance into ONE f64 buffer and one collective,
  * the x halo: each rank receives its neighbours' rows within the halo point-to-point
    (``halo_window``).

L-BFGS runs on each rank's owned rows of x / g / s / y; its dot products and max|g| are
all-reduced scalars (``allreduce``).  Each rank writes only its owned gradient rows, so no
gradient all-gather is needed.

The per-stripe engine is the device ``Engine``; tests substitute a CPU oracle engine with the
same interface to check this host logic with the gloo backend.
"""

from __future__ import annotations

import os

import numpy as np
import torch
import torch.distributed as dist

from .spec import tap_geometry
from .stats import finalize_sums
from .tiling import margin_for_exact_gradient, stripes


def init(local_rank: int | None = None, backend: str | None = None):
    """Initialise the default process group from torchrun's env (MASTER_ADDR=127.0.0.1)."""
    if not dist.is_initialized():
        if backend is None:  # SPST_DIST_BACKEND: functional multi-rank checks on one device (gloo)
            backend = os.environ.get("SPST_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl" and local_rank is not None:
            torch.cuda.set_device(local_rank)
        dist.init_process_group(backend)
    return dist.group.WORLD


class ShardedProblem:
    """Row-stripe sharded transfer problem (one rank's view)."""

    def __init__(self, u, v, spec, weights, engine, group=None, halo: int | None = None):
        self.spec = spec
        self.weights = weights
        self.engine = engine
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.s = spec.deepest_stride()
        self.halo = margin_for_exact_gradient(spec) if halo is None else halo
        self.h, self.w = int(u.shape[0]) if u is not None else int(v.shape[0]), \
            int(u.shape[1]) if u is not None else int(v.shape[1])
        self.Hp = self.h + (-self.h) % self.s
        self.Wp = self.w + (-self.w) % self.s
        self.stripes = stripes(self.Hp, self.s, self.halo, self.world)
        if len(self.stripes) < self.world:
            raise ValueError(f"image has {self.Hp // self.s} stride rows, cannot split {self.world} ways")
        self.me = self.stripes[self.rank]
        # rows of x this rank owns (unpadded image rows)
        self.own_rows = (min(self.me.own_r0, self.h), min(self.me.own_r1, self.h))
        self.all_own_rows = [(min(st.own_r0, self.h), min(st.own_r1, self.h)) for st in self.stripes]
        self.max_rows = max(b - a for a, b in self.all_own_rows)
        self.style_stats = self._sharded_stats(v)
        self._content = weights.lambda_c > 0
        if self._content:
            self._bind(self.h, self.w)
            self.engine.forward_rows(self._rows_of(u, self.me.grid_r0, self.me.grid_r1, self.h), self.me.grid_r0)
            self.engine.capture_content()
        self._bind(self.h, self.w)
        for i, t in enumerate(spec.style_taps):
            self.engine.set_style_ref(i, self.style_stats[t], weights.style[t])
        self.counts = [(self.Hp // tap_geometry(spec, t).stride) * (self.Wp // tap_geometry(spec, t).stride)
                       for t in spec.style_taps]

    # ------------------------------------------------------------------ helpers
    def _bind(self, h, w):
        self.engine.bind(h, w, (self.me.grid_r0, self.me.grid_r1), (self.me.own_r0, self.me.own_r1))

    @staticmethod
    def _rows_of(img, r0, r1, h):
        a = img[r0:min(r1, h)]
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
        return t.contiguous()

    def allreduce(self, t, op="sum"):
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM, group=self.group)
        return t

    def _sharded_stats(self, v):
        """Global style statistics of v: each rank reduces its own stripe of v's grid."""
        s = self.s
        vh, vw = int(v.shape[0]), int(v.shape[1])
        vHp = vh + (-vh) % s
        vst = stripes(vHp, s, self.halo, self.world)
        if len(vst) < self.world:  # tiny style image: every rank computes it whole, no exchange
            self.engine.bind(vh, vw, (0, vHp), (0, vHp))
            self.engine.forward_rows(self._rows_of(v, 0, vHp, vh), 0)
            sums = [self.engine.tap_sums(i) for i in range(len(self.spec.style_taps))]
        else:
            me = vst[self.rank]
            self.engine.bind(vh, vw, (me.grid_r0, me.grid_r1), (me.own_r0, me.own_r1))
            self.engine.forward_rows(self._rows_of(v, me.grid_r0, me.grid_r1, vh), me.grid_r0)
            sums = [self.engine.tap_sums(i) for i in range(len(self.spec.style_taps))]
            for S, sv in sums:
                self.allreduce(S)
                self.allreduce(sv)
        out = {}
        vWp = vw + (-vw) % s
        for i, t in enumerate(self.spec.style_taps):
            g = tap_geometry(self.spec, t).stride
            S, sv = sums[i]
            out[t] = finalize_sums(S.cpu().numpy().astype(np.float64), sv.cpu().numpy().astype(np.float64),
                                   (vHp // g) * (vWp // g))
        return out

    def shard_of(self, x):
        """This rank's owned rows of a full image, flattened (the L-BFGS vector shard)."""
        a, b = self.own_rows
        t = x[a:b] if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x[a:b]))
        if hasattr(self.engine, "device_of"):  # the device engine computes on float32 vectors
            t = t.to(self.engine.device_of(), torch.float32)
        return t.contiguous().reshape(-1).clone()

    def gather_image(self, shard):
        """Full (h, w, 3) image from every rank's shard (all-gather of padded shards) — for
        results and checkpoints; the evaluation itself only exchanges halo rows."""
        buf = torch.zeros(self.max_rows * self.w * 3, dtype=shard.dtype, device=shard.device)
        buf[:shard.numel()] = shard
        if self.world > 1:
            parts = [torch.empty_like(buf) for _ in range(self.world)]
            dist.all_gather(parts, buf, group=self.group)
        else:
            parts = [buf]
        img = torch.empty((self.h, self.w, 3), dtype=shard.dtype, device=shard.device)
        for (a, b), p in zip(self.all_own_rows, parts):
            if b > a:
                img[a:b] = p[:(b - a) * self.w * 3].view(b - a, self.w, 3)
        return img

    # ------------------------------------------------------------------ objective
    def halo_window(self, shard):
        """This rank's grid rows [grid_r0, min(grid_r1, h)) of x: its own shard plus the
        neighbours' rows inside the halo, exchanged point-to-point (each rank sends exactly the
        rows of its owned stripe that another rank's grid window covers; a neighbour thinner
        than the halo is covered by the rank beyond it).  Per evaluation at 8 stripes of
        6048x8064 this moves 2 x 160 rows (31 MB) per rank instead of an all-gather of 7/8 of
        the image (512 MB)."""
        g0, g1 = self.me.grid_r0, min(self.me.grid_r1, self.h)
        a, b = self.own_rows
        win = torch.empty((g1 - g0, self.w, 3), dtype=shard.dtype, device=shard.device)
        win[a - g0:b - g0] = shard[:(b - a) * self.w * 3].view(b - a, self.w, 3)
        if self.world > 1:
            mine = shard[:(b - a) * self.w * 3].view(b - a, self.w, 3)
            # gloo moves host memory only (functional multi-rank runs on one device)
            stage = shard.is_cuda and dist.get_backend(self.group) == "gloo"
            ops, landed = [], []
            for j, st in enumerate(self.stripes):
                if j == self.rank:
                    continue
                ja, jb = self.all_own_rows[j]
                r0, r1 = max(g0, ja), min(g1, jb)          # rows of j's stripe that I need
                if r1 > r0:
                    dst = win[r0 - g0:r1 - g0]
                    buf = torch.empty(dst.shape, dtype=dst.dtype) if stage else dst
                    landed.append((dst, buf))
                    ops.append(dist.P2POp(dist.irecv, buf, j, group=self.group))
                q0, q1 = max(st.grid_r0, a), min(min(st.grid_r1, self.h), b)  # my rows j needs
                if q1 > q0:
                    src = mine[q0 - a:q1 - a]
                    ops.append(dist.P2POp(dist.isend, src.cpu() if stage else src.contiguous(), j,
                                          group=self.group))
            if ops:
                for req in dist.batch_isend_irecv(ops):
                    req.wait()
            for dst, buf in landed:
                if buf is not dst:
                    dst.copy_(buf)
        return win

    def _reduce_statistics(self, with_content: bool):
        """One all-reduce of every style tap's (S, s) partials (and the content distance) as a
        single f64 buffer — one collective per evaluation instead of 2T + 1."""
        parts = [t for i in range(len(self.spec.style_taps)) for t in self.engine.tap_sums(i)]
        c = self.engine.content_sqdiff() if with_content else None
        if self.world > 1:
            flat = torch.cat([t.reshape(-1) for t in parts] + ([c.reshape(-1)] if c is not None else []))
            self.allreduce(flat)
            off = 0
            for t in parts + ([c] if c is not None else []):
                n = t.numel()
                t.copy_(flat[off:off + n].view_as(t))
                off += n
        return c

    def loss(self, x_shard) -> float:
        self.engine.forward_rows(self.halo_window(x_shard), self.me.grid_r0)
        c = self._reduce_statistics(self._content)
        terms, _ = self.engine.finalize(self.counts)
        total = float(np.sum(terms))
        if self._content:
            total += self.weights.lambda_c * float(c.item())
        return total

    def grad(self, out_shard):
        self.engine.backward_rows(2.0 * self.weights.lambda_c if self._content else 0.0, out_shard,
                                  self.own_rows[0], self.w)
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


def build_sharded_problem(u, v, spec, weights, group=None):
    """Device version: one Engine per rank bound to its stripe."""
    from .device import engine_for
    return ShardedProblem(u, v, spec, weights, DeviceStripeEngine(engine_for(spec)), group=group)


class DeviceStripeEngine:
    """Adapter giving the device Engine the stripe interface (row-offset image pointers)."""

    def __init__(self, engine):
        self.e = engine

    def device_of(self):
        return torch.device("cuda", self.e.device)

    def bind(self, h, w, grid, own):
        self.e.bind(h, w, grid, own)
        self.w = w

    def forward_rows(self, rows, row0):
        rows = rows.to(self.device_of(), torch.float32).contiguous()
        self._rows = rows  # keep alive for the duration of the pass
        self.e.forward(_Shifted(rows, -row0 * self.w * 3))

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

    def backward_rows(self, two_lambda, out_shard, own_row0, w):
        self.e.backward(two_lambda, _Shifted(out_shard, -own_row0 * w * 3))


class _Shifted:
    """A float32 tensor viewed from `offset` elements before its start (row-offset pointers
    for the C ABI, which indexes images by global row)."""

    def __init__(self, t, offset):
        self.t = t
        self.offset = offset

    def data_ptr(self):
        return self.t.data_ptr() + 4 * self.offset
