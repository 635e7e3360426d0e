"""Gradient error budget of the device path at fixed same-x points (GPU box; test infrastructure).

    SPST_DEBUG_STORE_ALL=1 python tools/error_budget.py [--lib path/to/libspst_variant.so] [--out json]

Points: x0 = u and the reference's f32 L-BFGS iterates x1..x5 at C1 (tests/golden/vgg19_iterates.npz,
written by tools/make_goldens.py from the real reference), each with the reference f64 and f32
gradients.  At every point the device result is split into:

* plain     -- vs the reference f64 gradient (the north-star number);
* arith     -- vs the f64 oracle evaluated on OUR ReLU pattern (arithmetic only);
* bwd       -- vs the f64 oracle on our pattern AND with our statistics (G, mu, sigma)
               injected (forward features + backward arithmetic only);
* stats     -- arith minus bwd, i.e. what the statistics' rounding contributes;
* per-layer relu-output error vs the f64 network on our pattern, per-tap G / mu / sigma error,
  and the ReLU flips (count, max |pre|/rms).
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def oracle_eval(O, x, po, masks, sx_override=None):
    """loss_grad_global of the oracle on a forced ReLU pattern, optionally with given stats.
    Returns (loss, grad, relu outputs per relu layer, f64 stats per tap)."""
    net = po.net
    h, w = x.shape[:2]
    xp = O.pad_edge16(x.astype(np.float64), net.deepest_stride())
    cur = O.preprocess(np.ascontiguousarray(xp.transpose(2, 0, 1)), net)
    saved, relu_out, feats = [], {}, {}
    for l in net.layers[: net.last() + 1]:
        saved.append(cur if l.name not in masks else np.where(masks[l.name], 1.0, -1.0))
        if l.kind == "conv":
            cur = O.conv3x3(cur, l.w, l.b)
        elif l.kind == "relu":
            cur = cur * masks[l.name]
            relu_out[l.name] = cur
        else:
            cur = O.pool2_fwd(cur, l.pool)
        if l.name in net.taps:
            feats[l.name] = cur
    total, tg, sx_all = 0.0, {}, {}
    for t in net.style_taps:
        sx = O.stats_of(feats[t]) if sx_override is None else sx_override[t]
        sx_all[t] = O.stats_of(feats[t])
        total += sum(O.style_terms(sx, po.style[t], po.tw[t]))
        tg[t] = O.style_feature_grad(feats[t], sx, po.style[t], po.tw[t])
    ct = net.content_tap
    if po.lambda_c > 0:
        diff = feats[ct] - po.content_full()
        total += po.lambda_c * float(np.sum(diff ** 2))
        cg = (2.0 * po.lambda_c) * diff
        tg[ct] = tg[ct] + cg if ct in tg else cg
    g = O.run_backward(tg, saved, net)
    return total, O.fold_pad_grad(np.ascontiguousarray(g.transpose(1, 2, 0)), h, w), relu_out, sx_all


def f64_preacts(O, po, x):
    net = po.net
    xp = O.pad_edge16(x.astype(np.float64), net.deepest_stride())
    _, saved = O.run_forward(np.ascontiguousarray(xp.transpose(2, 0, 1)), net, keep=True)
    return {l.name: saved[i] for i, l in enumerate(net.layers[: net.last() + 1]) if l.kind == "relu"}


def flips(masks, pre):
    n, worst = 0, 0.0
    per = {}
    for name, m in masks.items():
        pf = pre[name]
        d = m != (pf > 0)
        if d.any():
            rms = float(np.sqrt(np.mean(pf ** 2)))
            n += int(d.sum())
            per[name] = int(d.sum())
            worst = max(worst, float(np.abs(pf[d]).max()) / rms)
    return n, worst, per


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=None)
    ap.add_argument("--out", default=None)
    ap.add_argument("--points", default="0,1,2,3,4,5")
    ap.add_argument("--diag", action="store_true", help="per-statistic breakdown at the last point")
    args = ap.parse_args()
    if args.lib:
        os.environ["SPST_LIB"] = os.path.abspath(args.lib)
    os.environ.setdefault("SPST_DEBUG_STORE_ALL", "1")
    import spst_oracle as O
    import paper_2212_13459_b200 as spst
    from paper_2212_13459_b200.stats import finalize_sums  # noqa: F401

    d = np.load(os.path.join(ROOT, "tests", "golden", "vgg19.npz"))
    it = np.load(os.path.join(ROOT, "tests", "golden", "vgg19_iterates.npz"))
    spec = spst.calibrated_vgg19(0)
    lam = float(d["c1_lambda_c"][0])
    p = spst.build_problem(d["c1_u"], d["c1_v"], spec, spst.default_loss_weights(spec, lambda_c=lam))
    net = O.onet_from_spec(spec)
    po = O.build_problem(d["c1_u"].astype(np.float64), d["c1_v"].astype(np.float64), net,
                         O.default_weights(net, lam), 512, 256)
    eng = p.engine
    rows = []
    for k in [int(v) for v in args.points.split(",")]:
        x = it[f"x{k}"]
        loss, g = spst.loss_grad(x, p)
        masks = eng.relu_masks()
        outs = eng.stage_outputs()
        # our statistics (owned sums -> G, mu, sigma in f64, as the device finalize uses them)
        ours = {}
        for i, t in enumerate(eng.style_taps):
            S, s = eng.tap_sums(i)
            n = eng.owned_pixels(i)
            S = S.cpu().numpy().astype(np.float64)
            s = s.cpu().numpy().astype(np.float64)
            G = S / n
            mu = s / n
            ours[t] = O.OStats(G, mu, np.sqrt(np.maximum(np.diagonal(G) - mu ** 2, 0.0)), n)
        lm, gm, relu64, st64 = oracle_eval(O, x, po, masks)
        # the device's style references are its own statistics of v (build_problem): inject
        # those too, so gb differs from g only by features + backward arithmetic
        po_ours = O.OProblem(**{**po.__dict__, "style": {t: O.OStats(st.gram, st.mean, st.std, st.n_p)
                                                          for t, st in p.style_stats.items()}})
        lb, gb, _, _ = oracle_eval(O, x, po_ours, masks, sx_override=ours)
        nfl, tie, per_fl = flips(masks, f64_preacts(O, po, x))
        row = {
            "point": k,
            "loss_rel_f64": abs(loss - float(it[f"loss64_{k}"][0])) / float(it[f"loss64_{k}"][0]),
            "plain": rel(g, it[f"grad64_{k}"]),
            "ref_f32_gap": rel(it[f"grad32_{k}"], it[f"grad64_{k}"]),
            "arith": rel(g, gm),
            "bwd_with_our_stats": rel(g, gb),
            "stats_only": rel(gb, gm),
            "flips": nfl, "flip_max_pre_over_rms": tie, "flips_per_layer": per_fl,
            "relu_out_rel": {n_: rel(outs[n_], relu64[n_][:, :outs[n_].shape[1], :outs[n_].shape[2]])
                             for n_ in outs},
            # signed (systematic) part: mean (ours - f64) sign(f64) / rms(f64)
            "relu_out_bias": {n_: float(np.mean((outs[n_] - relu64[n_]) * np.sign(relu64[n_]))
                                        / np.sqrt(np.mean(relu64[n_] ** 2))) for n_ in outs},
            "tap_stats": {},
        }
        for t in eng.style_taps:
            r, o = st64[t], ours[t]
            sr = po.style[t]
            row["tap_stats"][t] = {
                "G": rel(o.gram, r.gram), "mu": rel(o.mean, r.mean), "sd": rel(o.std, r.std),
                "G_minus_Gref": rel(o.gram - sr.gram, r.gram - sr.gram),
                "sd_minus_sdref": rel(o.std - sr.std, r.std - sr.std),
                "sd_max_relerr": float(np.max(np.abs(o.std - r.std) / np.maximum(r.std, 1e-30))),
                "Gdiag_bias": float(np.mean(np.diagonal(o.gram) - np.diagonal(r.gram)) / np.mean(np.diagonal(r.gram))),
            }
        if args.diag and k == int(args.points.split(",")[-1]):
            # which statistic moves the gradient: inject ours one quantity at a time
            for what in ("gram", "mean", "std"):
                mix = {t: O.OStats(ours[t].gram if what == "gram" else st64[t].gram,
                                   ours[t].mean if what == "mean" else st64[t].mean,
                                   ours[t].std if what == "std" else st64[t].std, st64[t].n_p)
                       for t in eng.style_taps}
                _, gx, _, _ = oracle_eval(O, x, po, masks, sx_override=mix)
                row[f"stats_only_{what}"] = rel(gx, gm)
            for t in eng.style_taps:
                r, o = st64[t], ours[t]
                dead64 = r.std < 1e-8
                deado = o.std < 1e-8
                rat = lambda st: np.where(st.std < 1e-8, 0.0, (st.std - po.style[t].std) / np.where(st.std < 1e-8, 1.0, st.std))
                row["tap_stats"][t].update({
                    "dead64": int(dead64.sum()), "dead_ours": int(deado.sum()),
                    "dead_mismatch": int((dead64 != deado).sum()),
                    "ratio_maxabs_diff": float(np.max(np.abs(rat(o) - rat(r)))),
                    "min_std64": float(r.std.min()), "n64": int(r.n_p), "n_ours": int(o.n_p),
                    "G_maxabs_rel": float(np.max(np.abs(o.gram - r.gram)) / np.max(np.abs(r.gram)))})
            print("     diag: " + json.dumps({k_: v for k_, v in row.items() if k_.startswith("stats_only_")}) + " "
                  + json.dumps({t: {k_: v for k_, v in d_.items() if k_ in ("dead64", "dead_ours", "dead_mismatch",
                                                                        "ratio_maxabs_diff", "min_std64", "n64",
                                                                        "n_ours", "G_maxabs_rel")}
                                for t, d_ in row["tap_stats"].items()}), flush=True)
        rows.append(row)
        print(f"[{k}] plain {row['plain']:.2e} (ref f32 {row['ref_f32_gap']:.2e}) arith {row['arith']:.2e} "
              f"bwd {row['bwd_with_our_stats']:.2e} stats {row['stats_only']:.2e} flips {nfl} "
              f"(tie {tie:.1e}) {per_fl} loss {row['loss_rel_f64']:.1e}", flush=True)
        print("     relu out: " + " ".join(f"{n_}:{v:.1e}" for n_, v in row["relu_out_rel"].items()), flush=True)
        print("     relu bias: " + " ".join(f"{n_}:{v:+.1e}" for n_, v in row["relu_out_bias"].items()), flush=True)
        print("     Gdiag bias: " + " ".join(f"{t}:{v['Gdiag_bias']:+.1e}" for t, v in row["tap_stats"].items()),
              flush=True)
        print("     taps: " + " ".join(f"{t}:G{v['G']:.1e}/dG{v['G_minus_Gref']:.1e}/sd{v['sd']:.1e}/"
                                        f"dsd{v['sd_minus_sdref']:.1e}/mu{v['mu']:.1e}"
                                        for t, v in row["tap_stats"].items()), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"lib": os.environ.get("SPST_LIB", "default"),
                       "env": {k_: v for k_, v in os.environ.items() if k_.startswith("SPST_")},
                       "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
