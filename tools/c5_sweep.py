"""Config C5 (BASELINE.json configs[4]): tile-size and halo sweep at 6048x8064 —
the statistics exchange against conv time, at 1/2/4/8 GPUs.

    python tools/c5_sweep.py [--out gpurun_out/c5_sweep.json] [--reps 3]

Two decompositions of one evaluation (forward + statistics + backward to the image) of the C4
last-scale problem, every piece timed on the device with CUDA events on the engine's stream:

* square tiles T in {256, 512, 1024, 2048} with the exact halo (160 px, reference
  ``margin_for_exact_gradient``; the reference grid is ``partition(BlockGrid(H, W, T, 160))``,
  tiling.py:57-72): every window of the grid is evaluated as one zero-padded image whose owned
  rows are the tile's inner rows; windows are grouped by their clipped dims and each distinct
  size is timed once.  The sum over windows is what one GPU spends per evaluation with that
  tiling (halo recompute included); ``halo_factor`` = window area / image area.
* row stripes for N = 1, 2, 4, 8 (``tiling.stripes``, the decomposition ``distributed.py``
  shards over): the slowest stripe's evaluation time is the per-rank compute of an N-GPU
  evaluation.  The per-evaluation exchange is counted in bytes (5 style taps' S and s partials
  in f64 = 611,776 values plus the content scalar, as one all-reduce; the x halo rows received
  point-to-point) and converted to time with a stated NVLink bandwidth model — this run has one GPU, so the
  exchange itself is not measured.

Diagnostic tool; not a bench line.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_13459_b200 as spst  # noqa: E402
from paper_2212_13459_b200 import workloads  # noqa: E402
from paper_2212_13459_b200.device import Engine, clear_engines  # noqa: E402
from paper_2212_13459_b200.distributed import DeviceStripeEngine  # noqa: E402
from paper_2212_13459_b200.pipeline import RunConfig, _weights_for_scale  # noqa: E402
from paper_2212_13459_b200.spec import tap_geometry  # noqa: E402
from paper_2212_13459_b200.tiling import BlockGrid, margin_for_exact_gradient, partition, stripes  # noqa: E402

FLOP_PER_PX = 1514240
NVLINK_GBS = 900.0      # NVLink 5 per direction per GPU (B200); bandwidth model only
COLL_LAT_US = 20.0      # per-collective latency assumed for the model (NCCL small-message)

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/c5_sweep.json")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--tiles", default="256,512,1024,2048")
a = ap.parse_args()

H, W = workloads.CONFIGS["c4"]["content"]
sh, sw = workloads.CONFIGS["c4"]["style"]
spec = spst.calibrated_vgg19(0)
halo = margin_for_exact_gradient(spec)
s = spec.deepest_stride()
u = workloads.synth_content(H, W, 1)
v = workloads.synth_style(sh, sw, 2)
weights = _weights_for_scale(RunConfig(extractor=spec), spec, (H, W))
t0 = time.time()
p = spst.build_problem(u, v, spec, weights)
style_stats = {t: p.style_stats[t] for t in spec.style_taps}
del p
clear_engines()
torch.cuda.empty_cache()
print(f"style statistics {time.time() - t0:.1f} s", flush=True)

rng = np.random.default_rng(5)
x = np.clip(u + 0.02 * rng.standard_normal(u.shape), 0, 1).astype(np.float32)
ud, xd = torch.from_numpy(u).cuda(), torch.from_numpy(x).cuda()
eng = DeviceStripeEngine(Engine(spec))


def time_window(r0, r1, c0, c1, own0, own1):
    """Device ms of one evaluation of the window [r0,r1) x [c0,c1) (padded-grid coords) owning
    window rows [own0, own1)."""
    h, w = min(r1, H) - r0, min(c1, W) - c0
    Hp = h + (-h) % s
    uw = ud[r0:r0 + h, c0:c0 + w].contiguous()
    xw = xd[r0:r0 + h, c0:c0 + w].contiguous()
    eng.bind(h, w, (0, Hp), (own0, own1))
    eng.forward_rows(uw, 0)
    eng.capture_content()
    for i, t in enumerate(spec.style_taps):
        eng.set_style_ref(i, style_stats[t], weights.style[t])
    counts = [(H // tap_geometry(spec, t).stride) * (W // tap_geometry(spec, t).stride) for t in spec.style_taps]
    out = torch.empty((own1 - own0) * w * 3, device="cuda")

    def one():
        eng.forward_rows(xw, 0)
        eng.finalize(counts)
        float(eng.content_sqdiff().item())
        eng.backward_rows(2 * weights.lambda_c, out, own0, w)

    one()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = eng.e.stream()  # the engine launches on torch's current stream of its device
    e0.record(cur)
    for _ in range(a.reps):
        one()
    e1.record(cur)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps


res = {"workload": "C5: tile/halo sweep at 6048x8064 (C4 last scale, VGG-19 to relu5_1, calibrated seed 0)",
       "halo": halo, "device": torch.cuda.get_device_name(0), "reps": a.reps, "tiles": [], "stripes": []}
full_ms = None

# ---- row stripes at N = 1, 2, 4, 8 (the multi-GPU decomposition)
stat_values = sum(tap_geometry(spec, t).channels ** 2 + tap_geometry(spec, t).channels for t in spec.style_taps)
for n in (1, 2, 4, 8):
    parts = stripes(H, s, halo, n)
    times = []
    for st in parts if n <= 2 else [parts[0], parts[len(parts) // 2]]:  # edge + interior (others repeat)
        ms = time_window(st.grid_r0, st.grid_r1, 0, W, st.own_r0 - st.grid_r0, st.own_r1 - st.grid_r0)
        times.append({"grid_rows": [st.grid_r0, st.grid_r1], "own_rows": [st.own_r0, st.own_r1], "ms": ms})
    worst = max(t["ms"] for t in times)
    if n == 1:
        full_ms = worst
    # the exchange per evaluation (distributed.py): one fused f64 all-reduce of the statistics
    # (ring: 2(N-1)/N of the buffer per GPU) and the point-to-point halo rows of x
    me = max(parts, key=lambda st: st.grid_r1 - st.grid_r0)
    halo_bytes = ((me.grid_r1 - me.grid_r0) - (me.own_r1 - me.own_r0)) * W * 3 * 4 if n > 1 else 0
    stat_bytes = 8 * (stat_values + 1)
    ar_us = (2 * (n - 1) / n * stat_bytes / (NVLINK_GBS * 1e3) + COLL_LAT_US) if n > 1 else 0.0
    hx_us = (halo_bytes / (NVLINK_GBS * 1e3) + COLL_LAT_US) if n > 1 else 0.0
    halo_rows = sum(st.grid_r1 - st.grid_r0 for st in parts)
    comm_ms = (ar_us + hx_us) / 1e3
    res["stripes"].append({
        "gpus": n, "per_rank_eval_ms": worst, "stripes_timed": times,
        "halo_factor": halo_rows / H,
        "stats_allreduce_bytes": stat_bytes, "stats_allreduce_model_us": ar_us,
        "x_halo_bytes_per_rank": halo_bytes, "x_halo_model_us": hx_us,
        "comm_share_model": comm_ms / (worst + comm_ms),
        "projected_evals_per_s": 1e3 / (worst + comm_ms),
        "projected_speedup_vs_1": (full_ms / (worst + comm_ms)) if full_ms else None,
    })
    print(json.dumps(res["stripes"][-1]), flush=True)

# ---- 2-D rank grids (rows x cols): the per-rank window of the slowest (interior) rank.  The
# engine owns row ranges only, so the column halo's statistics are counted too (Gram work is
# 2 % of an evaluation) — a timing model for the next decomposition, not a parity path.
res["grid2d"] = []
for gr, gc in ((1, 2), (2, 2), (2, 4)):
    rs, cs = stripes(H, s, halo, gr), stripes(W, s, halo, gc)
    worst = 0.0
    for st_r in {rs[0], rs[len(rs) // 2]}:
        for st_c in {cs[0], cs[len(cs) // 2]}:
            ms = time_window(st_r.grid_r0, st_r.grid_r1, st_c.grid_r0, st_c.grid_r1,
                             st_r.own_r0 - st_r.grid_r0, st_r.own_r1 - st_r.grid_r0)
            worst = max(worst, ms)
    area = sum((a.grid_r1 - a.grid_r0) * (b.grid_r1 - b.grid_r0) for a in rs for b in cs)
    res["grid2d"].append({"gpus": gr * gc, "grid": [gr, gc], "per_rank_eval_ms": worst,
                          "halo_factor": area / (H * W), "projected_speedup_vs_1": full_ms / worst})
    print(json.dumps(res["grid2d"][-1]), flush=True)

# ---- square tiles with the exact halo on one GPU (the reference's grid)
for T in (int(t) for t in a.tiles.split(",")):
    blocks = partition(BlockGrid(H, W, T, halo, s))
    groups = {}
    for b in blocks:
        key = (b.padded.h, b.padded.w, b.present_margin[1], b.inner.h)
        groups.setdefault(key, []).append(b)
    total, win_px, per = 0.0, 0, []
    for (ph, pw, top, ih), bl in sorted(groups.items()):
        b = bl[0]
        ms = time_window(b.padded.y0, b.padded.y1, b.padded.x0, b.padded.x1, top, top + ih)
        total += ms * len(bl)
        win_px += ph * pw * len(bl)
        per.append({"window": [ph, pw], "count": len(bl), "ms": ms})
    res["tiles"].append({"tile": T, "blocks": len(blocks), "distinct_windows": len(groups),
                         "halo_factor": win_px / (H * W), "eval_ms_one_gpu": total,
                         "vs_whole_image": total / full_ms if full_ms else None, "windows": per})
    print(json.dumps({k: v for k, v in res["tiles"][-1].items() if k != "windows"}), flush=True)

res["whole_image_eval_ms"] = full_ms
res["whole_image_algorithmic_tflops"] = FLOP_PER_PX * H * W / (full_ms * 1e-3) / 1e12
res["model"] = (f"exchange time = bytes / {NVLINK_GBS:.0f} GB/s + {COLL_LAT_US:.0f} us per exchange (one fused "
                "statistics all-reduce, one batch of point-to-point halo rows); not measured (1 GPU)")
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
with open(a.out, "w") as f:
    json.dump(res, f, indent=1)
print("wrote", a.out)
