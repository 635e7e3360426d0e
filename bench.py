"""Benchmark: L-BFGS iterations/s of the localized Gatys transfer at 6048x8064 (tiled VGG-19).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c4]

Metric (BASELINE.json): L-BFGS iters/s at 6048x8064.  Workload: the last scale of config C4
(6048x8064 content, 4226x5319 style, calibrated seeded VGG-19, history m=10, default loss
weights).  One step = one L-BFGS iteration (two-loop direction, Armijo line search with
loss-only trials, one gradient for the accepted point).  Inputs are synthetic (seeded
content/style with distinct statistics).  The working set (~80 GB) exceeds
L2, so no flush is needed between steps.

--impl reference: the reference algorithm's CPU implementation (oracle/spst_oracle.py, a
restatement of the pure-NumPy reference -- the reference itself cannot travel to the GPU box)
timed on the host cores.  --config c1 runs it END TO END (10 L-BFGS iterations at 256^2, no
extrapolation); the large configs time a bounded sample per step (one interior 512x512 padded
block of the reference's default 512/256 grid through both passes, style and content feature
gradients included), extrapolated by padded area and the evals/iteration.  Our arm's
cpu_baseline uses the same sample, and both arms print the same config dict.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FLOP_PER_PX = 1514240  # fwd + bwd-input + Gram + style-grad per padded px per eval


def peaks():
    try:
        with open(PEAKS) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p["bf16_tflops_sustained"], "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=5)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 2 + i and "Active" in s[2 + i]
                          and "Not" not in s[2 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.samples[0][1]) if self.samples[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ------------------------------------------------------------------------------------------
# our implementation
# ------------------------------------------------------------------------------------------
def run_ours(args):
    import torch
    rank, world, local = dist_env()
    # SPST_BENCH_DEVICE (with SPST_DIST_BACKEND=gloo): put every rank on one device for a
    # functional check of the multi-rank code path -- such a run has no performance meaning
    local = int(os.environ.get("SPST_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    import paper_2212_13459_b200 as spst
    from paper_2212_13459_b200 import workloads
    from paper_2212_13459_b200.pipeline import objective_for, _weights_for_scale, RunConfig
    spst.set_precision(args.precision)
    from paper_2212_13459_b200.lbfgs import LBFGSConfig, minimize

    cfgw = workloads.CONFIGS[args.config]
    H, W = cfgw["content"]
    sh, sw = cfgw["style"]
    spec = spst.calibrated_vgg19(0)
    u = workloads.synth_content(H, W, 1)
    v = workloads.synth_style(sh, sw, 2)
    weights = _weights_for_scale(RunConfig(extractor=spec), spec, (H, W))
    group = None
    if world > 1:
        from paper_2212_13459_b200 import distributed as dist_mod
        group = dist_mod.init(local)
    t_setup = time.time()
    if world > 1:
        problem = dist_mod.build_sharded_problem(u, v, spec, weights)
        objective = problem.objective()
        x = problem.shard_of(u)
        allreduce = problem.allreduce
    else:
        grid = dict(block=128, margin=160) if args.config == "c1" else {}  # C1: 2x2 tiles with halo
        problem = spst.build_problem(u, v, spec, weights, **grid)
        objective = objective_for(problem)
        x = torch.from_numpy(u).cuda()
        allreduce = None
    torch.cuda.synchronize()
    setup_s = time.time() - t_setup

    # one continuous L-BFGS run: W warm-up iterations (they also fill the history), then K
    # timed steady-state iterations, bracketed by CUDA events recorded from the per-iteration
    # callback (the barrier + synchronize on both sides are inside the callback)
    from paper_2212_13459_b200.lbfgs import Trace
    peak_hbm, peak_bf16, peak_sus, peak_kind = peaks()
    sampler = ClockSampler(local)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    marks = {}
    if world > 1:
        import torch.distributed as tdist

    # the native engine of this rank: its launch timer brackets every tensor-core launch with
    # CUDA events on the engine stream during the timed iterations (dominant-kernel roofline)
    eng = getattr(problem, "engine", None)
    eng = getattr(eng, "e", eng)
    if not hasattr(eng, "timing_enable"):
        eng = None

    def on_iter(it, xi, loss, gnorm):
        if it in (args.warmup, args.warmup + args.steps):
            torch.cuda.synchronize()
            if world > 1:
                tdist.barrier()
            if it == args.warmup:
                if eng is not None:
                    eng.timing_enable(True)
                sampler.start()
                marks["launch0"] = launch_count()
                e0.record()
            else:
                e1.record()
                marks["launch1"] = launch_count()
                if eng is not None:
                    marks["timer"] = eng.timing_read()
                    eng.timing_enable(False)
            marks[it] = None

    decomposition = (f"2-D grid {problem.grid_shape[0]}x{problem.grid_shape[1]} of halo-padded windows"
                     if world > 1 and not problem.replicated else
                     ("replicated" if world > 1 else "whole image, one window"))
    if args.warmup == 0:  # time from the start (includes L-BFGS's first evaluation)
        on_iter(0, None, None, None)
    x, tr_all = minimize(objective, x, LBFGSConfig(history_size=history_for(args.config),
                                                   max_iters=args.warmup + args.steps),
                         callback=on_iter, allreduce=allreduce)
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    clocks = sampler.stop()
    if args.warmup + args.steps not in marks:
        raise RuntimeError("L-BFGS stopped before the timed iterations completed")
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms = float(t.item())
    tr = tr_all
    iters = args.steps
    evals_per_iter = tr.evals / max(1, len(tr.losses) - 1)
    n_launch = marks["launch1"] - marks["launch0"]  # our kernels in the timed region (this rank)
    if world > 1:  # whole job
        t = torch.tensor([float(n_launch)], dtype=torch.float64, device="cuda")
        tdist.all_reduce(t)
        n_launch = int(t.item())

    # roofline of the dominant kernel (conv fwd/bwd): algorithmic FLOPs per eval / eval time
    Hp, Wp = H + (-H) % 16, W + (-W) % 16
    flops_eval = FLOP_PER_PX * Hp * Wp
    # every rank evaluates (the sharded objective all-reduces its statistics); slowest rank counts
    eval_ms = measure_eval(objective, x, torch)
    if world > 1:
        t = torch.tensor([eval_ms], dtype=torch.float64, device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        eval_ms = float(t.item())

    # e2e through the public API with host buffers: minimize() called on a pinned host
    # iterate (numpy in -> numpy out, H2D of x and D2H of the result inside the region)
    # (N > 1: every rank runs minimize on its own pinned host shard; the slowest rank's time
    # counts and the copied bytes are summed over ranks)
    xh = torch.empty_like(x, device="cpu").pin_memory()
    xh.copy_(x)
    xnp = xh.numpy()
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    t0 = time.time()
    xr, tr2 = minimize(objective, xnp, LBFGSConfig(history_size=history_for(args.config), max_iters=args.steps),
                       allreduce=allreduce)
    e2e_s = time.time() - t0
    nbytes = xnp.nbytes
    if world > 1:
        t = torch.tensor([e2e_s, float(nbytes)], dtype=torch.float64, device="cuda")
        tmax = t[:1].clone()
        tdist.all_reduce(tmax, op=tdist.ReduceOp.MAX)
        tsum = t[1:].clone()
        tdist.all_reduce(tsum)
        e2e_s, nbytes = float(tmax.item()), int(tsum.item())
    it2 = max(1, len(tr2.losses) - 1)
    e2e = {"value": it2 / e2e_s, "unit": "iters/s", "h2d_bytes_per_step": nbytes // it2,
           "d2h_bytes_per_step": nbytes // it2 + 8 * (tr2.evals // it2 + 1),
           # one cold minimize() call: L-BFGS's initial evaluation and its empty-history first
           # step are inside (the device-timed value is steady state, evals_per_iter there)
           "iters": it2, "evals": tr2.evals, "cold_start": True}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, H, W, sh, sw, evals_per_iter)

    if rank == 0:
        value = iters / (ms / 1e3)
        achieved = flops_eval / (eval_ms / 1e3) / 1e12 / world if eval_ms else None
        line = {
            "metric": metric_name(H, W),
            "value": value, "unit": "iters/s", "n_gpus": world, "steps": iters, "warmup": args.warmup,
            "ms_per_step": ms / iters, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": ("fp16x3 (fp16 hi/lo split operands, compensated fp32 accumulation) / f32 vectors"
                      if args.precision == "fp16x3" else "fp16 (one MMA pass, opt-in speed mode) / f32 vectors"),
            "data": "synthetic (seeded content/style, calibrated seeded VGG-19 weights)",
            "config": bench_config(args.config, H, W, sh, sw, world),
            "evals_per_iter": evals_per_iter, "setup_s": setup_s,
            "decomposition": decomposition,
            "roofline": dominant_roofline(marks.get("timer"), ms, peak_sus, peak_kind, flops_eval, eval_ms, world,
                                          args.config),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": n_launch,
            "clocks": clocks,
        }
        print(json.dumps(line))


def dominant_roofline(timer, step_region_ms, peak, peak_kind, flops_eval, eval_ms, world, config="c4"):
    """Roofline of the dominant kernel class from the engine's live launch timer: achieved =
    algorithmic FLOPs of its launches / their summed device time (CUDA events on the launching
    stream over the timed region); traffic = DRAM bytes per launch from the committed ncu
    capture (profiles/), or None."""
    whole = {"achieved_per_eval": (flops_eval / (eval_ms / 1e3) / 1e12 / world) if eval_ms else None,
             "algorithmic_flop_per_eval": flops_eval, "eval_ms": eval_ms}
    if not timer:
        return {"bound": "tensor", "kernel": "whole loss_grad eval (launch timer unavailable)",
                "achieved": whole["achieved_per_eval"], "peak": peak, "unit": "TFLOP/s",
                "frac": (whole["achieved_per_eval"] / peak) if whole["achieved_per_eval"] else None,
                "traffic": None, "peak_kind": peak_kind, **whole}
    name, (kms, kflops, n) = max(timer.items(), key=lambda kv: kv[1][0])
    achieved = kflops / (kms / 1e3) / 1e12
    traffic = None
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "dominant_traffic.json")) as f:
            tr = json.load(f)
        if tr.get("kernel_class") == name and config == tr.get("config", "c4"):  # captured on c4
            traffic = tr["dram_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        pass
    return {"bound": "tensor", "kernel": name, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_unit": "bytes DRAM per launch (ncu)",
            "peak_kind": f"bf16 dense sustained ({peak_kind})",
            "launches": n, "avg_launch_ms": kms / n, "algorithmic_flop_per_launch": kflops / n,
            "share_of_timed_region": kms / step_region_ms,
            "classes": {c: {"ms": v[0], "tflop": v[1] / 1e12, "launches": v[2]} for c, v in timer.items()},
            "note": "algorithmic FLOPs (real channels, 1 pass); the fp16x3 split executes 3 MMA passes, "
                    "so frac <= 1/3 by construction", **whole}


def measure_eval(objective, x, torch):
    """Average device time of one full loss+gradient evaluation (forward, stats, backward)."""
    g = torch.empty_like(x)
    objective.loss(x)
    objective.grad(g)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    n = 3
    e0.record()
    for _ in range(n):
        objective.loss(x)
        objective.grad(g)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def launch_count():
    """Kernels launched so far by libspst (every launch site counts itself)."""
    from paper_2212_13459_b200 import _native as nat
    return int(nat.lib().spst_launch_count())


# ------------------------------------------------------------------------------------------
# CPU baseline: the reference algorithm (oracle port) on the host cores
# ------------------------------------------------------------------------------------------
def history_for(config):
    """L-BFGS history of the config's (last) scale: 100 at a single-scale run's only scale,
    10 at later scales (reference pipeline.py:32-33)."""
    return 100 if config in ("c1", "c2", "c4s1") else 10


def bench_config(config, H, W, sh, sw, world):
    """The config dict both arms print (identical keys and values for the same workload)."""
    return {"workload": workload_name(config, H, W, sh, sw), "image": [H, W], "style": [sh, sw],
            "history": history_for(config), "n_gpus": world,
            "l2_flush": "not needed (working set >> 126 MB L2)" if H * W > 1 << 22 else
                        "not flushed (small config)"}


def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import spst_oracle as O  # test/baseline infrastructure only
    return O


def cpu_sample(H, W, sh, sw, side=512):
    """The reference algorithm (oracle port) on ONE interior padded block of the reference's
    default 512/256 grid, both passes of localized.py:227-280: pass-1 forward + statistics,
    pass-2 forward with saves, the style feature gradient at every style tap
    (style_layer_loss_grad, stats.py:127-165), the content term (stats.py:168-174) and the
    backward to the pixels.  Returns (seconds, padded-area factor of the whole grid)."""
    O = _oracle()
    from paper_2212_13459_b200 import spec as specmod
    from paper_2212_13459_b200 import workloads
    from paper_2212_13459_b200.tiling import BlockGrid, partition
    net = O.onet_from_spec(specmod.calibrated_vgg19(0))
    lam, tw = O.default_weights(net)
    blk = workloads.synth_content(side, side, 5)
    x = np.ascontiguousarray(blk.transpose(2, 0, 1))
    ref_feats, _ = O.run_forward(np.ascontiguousarray(workloads.synth_style(side, side, 6).transpose(2, 0, 1)), net)
    refs = {t: O.stats_of(ref_feats[t]) for t in net.style_taps}
    cont = ref_feats[net.content_tap]
    t0 = time.time()
    feats, _ = O.run_forward(x, net)                           # pass 1
    stats = {t: O.stats_of(feats[t]) for t in net.style_taps}
    feats, saved = O.run_forward(x, net, keep=True)            # pass 2
    tg = {t: O.style_feature_grad(feats[t], stats[t], refs[t], tw[t]) for t in net.style_taps}
    ct = net.content_tap
    cg = (2.0 * 1e-4) * (feats[ct] - cont)
    tg[ct] = tg[ct] + cg if ct in tg else cg
    O.run_backward(tg, saved, net)
    dt = time.time() - t0
    grid = BlockGrid(H + (-H) % 16, W + (-W) % 16, 512, 256, 16)
    area = sum(b.padded.w * b.padded.h for b in partition(grid))
    return dt, area / (side * side)


def cpu_baseline(args, H, W, sh, sw, evals_per_iter):
    cores = os.cpu_count()
    if args.config == "c1":
        return cpu_full_c1(args, steps=min(args.steps, 10))
    dt, factor = cpu_sample(H, W, sh, sw, args.cpu_block)
    iter_s = dt * factor * evals_per_iter
    return {"value": 1.0 / iter_s, "unit": "iters/s", "cores": cores, "kind": "port",
            "sample": f"one {args.cpu_block}x{args.cpu_block} padded block of the reference 512/256 grid through "
                      f"both passes incl. style/content feature gradients ({dt:.1f}s, f32 numpy, {cores} threads), "
                      f"extrapolated by padded area x{factor:.1f} and {evals_per_iter:.2f} evals/iter"}


def cpu_full_c1(args, steps=10, warmup=0):
    """C1 end to end on the host (no extrapolation): the reference algorithm (oracle port, f32)
    runs build_problem + L-BFGS (history 100) on 256^2 for warmup + steps iterations; the last
    `steps` iterations are timed."""
    O = _oracle()
    from paper_2212_13459_b200 import spec as specmod
    from paper_2212_13459_b200 import workloads
    from paper_2212_13459_b200.pipeline import RunConfig, _weights_for_scale
    spec = specmod.calibrated_vgg19(0)
    net = O.onet_from_spec(spec)
    u = workloads.synth_content(256, 256, 1)
    v = workloads.synth_style(256, 256, 2)
    lam = _weights_for_scale(RunConfig(extractor=spec), spec, (256, 256)).lambda_c
    # BASELINE.json configs[0]: "2x2 tiles with halo" -- block 128, margin 160 (the exact margin)
    p = O.build_problem(u, v, net, O.default_weights(net, lam), 128, 160)
    marks = {}
    t_start = time.time()

    def cb(it, x, loss, gn):
        if it == warmup:
            marks["t0"] = time.time()
        marks["last"] = (it, time.time())

    if warmup == 0:
        marks["t0"] = t_start
    _, losses, _ = O.minimize(lambda a: O.loss_grad(a, p), u, m=100, max_iters=warmup + steps, callback=cb)
    it_end, t_end = marks["last"]
    done = it_end - warmup
    return {"value": done / (t_end - marks["t0"]), "unit": "iters/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"C1 end to end: {done} timed L-BFGS iterations (of {warmup + steps}) of the reference "
                      f"algorithm at 256x256 on its 2x2 block grid (block 128, margin 160), f32 numpy, "
                      f"{os.cpu_count()} threads, no extrapolation"}


def metric_name(H, W):
    return f"L-BFGS iters/sec at {H}x{W} (tiled VGG-19)"


def workload_name(config, H, W, sh, sw):
    return (f"{config}: single-scale L-BFGS at {H}x{W} content, {sh}x{sw} style, VGG-19 to relu5_1, "
            f"m={history_for(config)}, default loss weights")


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfgw = __import__("paper_2212_13459_b200.workloads", fromlist=["CONFIGS"]).CONFIGS[args.config]
    H, W = cfgw["content"]
    sh, sw = cfgw["style"]
    if args.config == "c1":  # the one config the reference runs end to end in minutes
        r = cpu_full_c1(args, steps=args.steps, warmup=args.warmup)
        value = r["value"]
        last = r
    else:
        vals, last = [], None
        for i in range(args.warmup + args.steps):
            dt, factor = cpu_sample(H, W, sh, sw, args.cpu_block)
            v = 1.0 / (dt * factor * args.ref_evals_per_iter)
            if i >= args.warmup:
                vals.append(v)
            last = {"value": v, "unit": "iters/s", "cores": os.cpu_count(), "kind": "port",
                    "sample": f"one {args.cpu_block}x{args.cpu_block} padded block of the reference 512/256 grid "
                              f"through both passes incl. style/content feature gradients per step ({dt:.1f}s), "
                              f"extrapolated by padded area x{factor:.1f} and {args.ref_evals_per_iter:.2f} "
                              "evals/iter"}
        value = statistics.mean(vals) if vals else last["value"]
    line = {"metric": metric_name(H, W), "value": value, "unit": "iters/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / value,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded content/style, calibrated seeded VGG-19 weights)", "impl": "reference",
            "config": bench_config(args.config, H, W, sh, sw, world),
            "cpu_baseline": dict(last, value=value),
            "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--precision", default="fp16x3", choices=["fp16x3", "fp16"],
                    help="conv tensor-core precision (fp16: one-pass opt-in speed mode, not the parity mode)")
    # the reference's line search is restated exactly by ours, so trials per iteration are a
    # property of the problem: 1.08 is what our minimize measures at C4 (the reference itself
    # measured 1.8 at the 256^2 C1 config)
    ap.add_argument("--ref-evals-per-iter", type=float, default=1.08)
    ap.add_argument("--cpu-block", type=int, default=512, help="CPU sample block side (padded px), both arms")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
