"""Config C5 (BASELINE.json configs[4]): tile-size and halo sweep at 6048x8064 —
the statistics exchange against conv time, at 1/2/4/8 GPUs.

    python tools/c5_sweep.py [--out gpurun_out/c5_sweep.json] [--reps 3]

Every piece is one evaluation (forward + statistics + backward to the image) of the C4
last-scale problem on ONE window (engine ``spst_bind_window``: a padded rectangle evaluated as
one zero-padded image that owns an inner rectangle), timed on the device with CUDA events:

* the multi-GPU decomposition of ``distributed.py`` for N = 1, 2, 4, 8 (``choose_grid``: 1x1,
  1x2, 2x2, 2x4 windows with the exact 160-px halo): the slowest rank's window is the per-rank
  compute of an N-GPU evaluation.  The per-evaluation exchange is counted in bytes (the
  statistics buffer, all-gathered and summed in rank order; the x halo received point-to-point)
  and converted to time with a stated NVLink model -- this run has one GPU, so the exchange
  itself is not measured;
* square tiles T in {256, 512, 1024, 2048} with the exact halo (the reference grid
  ``partition(BlockGrid(H, W, T, 160))``, tiling.py:57-72) on one GPU: windows grouped by their
  dims, each distinct window timed once; ``halo_factor`` = window area / image area.

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
from paper_2212_13459_b200.distributed import Window, choose_grid, grid_windows  # noqa: E402
from paper_2212_13459_b200.pipeline import RunConfig, _weights_for_scale  # noqa: E402
from paper_2212_13459_b200.spec import tap_geometry  # noqa: E402
from paper_2212_13459_b200.tiling import BlockGrid, margin_for_exact_gradient, partition  # noqa: E402

FLOP_PER_PX = 1514240
NVLINK_GBS = 900.0      # NVLink 5 per direction per GPU (B200); bandwidth model only
COLL_LAT_US = 20.0      # per-exchange latency assumed for the model (NCCL small-message)

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
eng = Engine(spec)
counts = [(H // tap_geometry(spec, t).stride) * (W // tap_geometry(spec, t).stride) for t in spec.style_taps]


def time_window(wd: Window):
    """Device ms of one evaluation of window wd (global padded coordinates)."""
    eng.bind(H, W, *wd.bind_args())
    eng.forward(ud)
    eng.capture_content()
    for i, t in enumerate(spec.style_taps):
        eng.set_style_ref(i, style_stats[t], weights.style[t])
    r0, r1, c0, c1 = wd.or0, min(wd.or1, H), wd.oc0, min(wd.oc1, W)
    out = torch.empty((r1 - r0, c1 - c0, 3), device="cuda")

    def one():
        eng.forward(xd)
        c = eng.content_sqdiff()
        eng.finalize(counts)
        float(c.item())
        eng.backward(2 * weights.lambda_c, out, origin=(r0, c0))

    one()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = eng.stream()
    e0.record(cur)
    for _ in range(a.reps):
        one()
    e1.record(cur)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps


res = {"workload": "C5: tile/halo sweep at 6048x8064 (C4 last scale, VGG-19 to relu5_1, calibrated seed 0)",
       "halo": halo, "device": torch.cuda.get_device_name(0), "reps": a.reps, "tiles": [], "ranks": []}
full_ms = None

# ---- the multi-GPU decomposition (distributed.py) at N = 1, 2, 4, 8
stat_values = sum(tap_geometry(spec, t).channels ** 2 + tap_geometry(spec, t).channels for t in spec.style_taps)
for n in (1, 2, 4, 8):
    ry, rx = choose_grid(H, W, s, halo, n)
    wins = grid_windows(H, W, s, halo, ry, rx)
    distinct = {}
    for wd in wins:
        distinct.setdefault((wd.gr1 - wd.gr0, wd.gc1 - wd.gc0), wd)
    times = [{"window": list(k), "ms": time_window(wd)} for k, wd in distinct.items()]
    worst = max(t["ms"] for t in times)
    if n == 1:
        full_ms = worst
    # exchange per evaluation: statistics all-gather (N-1 remote copies of the 4.9 MB buffer
    # into every rank) and the halo pixels of the largest window received point-to-point
    me = max(wins, key=lambda wd: wd.area)
    halo_bytes = (me.area - (me.or1 - me.or0) * (me.oc1 - me.oc0)) * 3 * 4 if n > 1 else 0
    stat_bytes = 8 * (stat_values + 1)
    ag_us = ((n - 1) * stat_bytes / (NVLINK_GBS * 1e3) + COLL_LAT_US) if n > 1 else 0.0
    hx_us = (halo_bytes / (NVLINK_GBS * 1e3) + COLL_LAT_US) if n > 1 else 0.0
    comm_ms = (ag_us + hx_us) / 1e3
    res["ranks"].append({
        "gpus": n, "grid": [ry, rx], "per_rank_eval_ms": worst, "windows_timed": times,
        "halo_factor": sum(wd.area for wd in wins) / (H * W),
        "stats_allgather_bytes_per_rank": (n - 1) * stat_bytes, "stats_model_us": ag_us,
        "x_halo_bytes_per_rank": halo_bytes, "x_halo_model_us": hx_us,
        "comm_share_model": comm_ms / (worst + comm_ms),
        "projected_speedup_vs_1": (full_ms / (worst + comm_ms)) if full_ms else None,
        "projected_efficiency": (full_ms / (worst + comm_ms) / n) if full_ms else None,
    })
    print(json.dumps(res["ranks"][-1]), flush=True)

# ---- square tiles with the exact halo on one GPU (the reference's grid)
for T in (int(t) for t in a.tiles.split(",")):
    blocks = partition(BlockGrid(H, W, T, halo, s))
    groups = {}
    for b in blocks:
        key = (b.padded.h, b.padded.w)
        groups.setdefault(key, []).append(b)
    total, win_px, per = 0.0, 0, []
    for (ph, pw), bl in sorted(groups.items()):
        b = bl[0]
        ms = time_window(Window(b.padded.y0, b.padded.y1, b.inner.y0, b.inner.y1,
                                b.padded.x0, b.padded.x1, b.inner.x0, b.inner.x1))
        total += ms * len(bl)
        win_px += ph * pw * len(bl)
        per.append({"window": [ph, pw], "count": len(bl), "ms": ms})
    res["tiles"].append({"tile": T, "blocks": len(blocks), "distinct_windows": len(groups),
                         "halo_factor": win_px / (H * W), "eval_ms_one_gpu": total,
                         "vs_whole_image": total / full_ms if full_ms else None, "windows": per})
    print(json.dumps({k: v for k, v in res["tiles"][-1].items() if k != "windows"}), flush=True)

res["whole_image_eval_ms"] = full_ms
res["whole_image_algorithmic_tflops"] = FLOP_PER_PX * H * W / (full_ms * 1e-3) / 1e12
res["model"] = (f"exchange time = bytes / {NVLINK_GBS:.0f} GB/s + {COLL_LAT_US:.0f} us per exchange (statistics "
                "all-gather, one batch of point-to-point halo pixels); not measured (1 GPU)")
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
with open(a.out, "w") as f:
    json.dump(res, f, indent=1)
print("wrote", a.out)
