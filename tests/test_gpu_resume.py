"""Mid-scale resume: L-BFGS state in checkpoints.

The reference resumes only at scale boundaries (pipeline.py:199-205); here a run can also be
checkpointed every k iterations inside a scale, with the curvature history, and continued."""

import glob
import json
import os

import numpy as np
import pytest
import torch

import paper_2212_13459_b200 as spst
from paper_2212_13459_b200.lbfgs import LBFGSSnapshot
from paper_2212_13459_b200.pipeline import read_checkpoint

pytestmark = pytest.mark.gpu


def _rosen(z):
    x, y = z[0::2], z[1::2]
    f = float(np.sum((1 - x) ** 2 + 100 * (y - x ** 2) ** 2))
    g = np.empty_like(z)
    g[0::2] = -2 * (1 - x) - 400 * x * (y - x ** 2)
    g[1::2] = 200 * (y - x ** 2)
    return f, g


def _copy(sn):
    return LBFGSSnapshot(iteration=sn.iteration, x=sn.x.clone(), g=sn.g.clone(), loss=sn.loss,
                         s=[t.clone() for t in sn.s], y=[t.clone() for t in sn.y], rho=list(sn.rho), yy=list(sn.yy),
                         losses=list(sn.losses), grad_norms=list(sn.grad_norms))


def test_minimize_resume_is_bit_identical_on_a_host_objective():
    x0 = torch.tensor(np.tile([-1.2, 1.0], 8), dtype=torch.float64, device="cuda")
    cfg = spst.LBFGSConfig(history_size=4, max_iters=40)
    snaps = []
    x_full, tr_full = spst.minimize(_rosen, x0, cfg, snapshot=(7, lambda sn: snaps.append(_copy(sn))))
    assert [sn.iteration for sn in snaps] == [7, 14, 21, 28, 35]
    x_res, tr_res = spst.minimize(_rosen, torch.zeros_like(x0), cfg, resume=snaps[1])
    assert torch.equal(x_res, x_full)
    assert tr_res.losses == tr_full.losses
    # without the curvature history the continuation is a different trajectory
    bare = _copy(snaps[1])
    bare.s, bare.y, bare.rho, bare.yy = [], [], [], []
    x_bare, _ = spst.minimize(_rosen, torch.zeros_like(x0), cfg, resume=bare)
    assert not torch.equal(x_bare, x_full)


def test_pipeline_midscale_checkpoint_and_resume(tiny_spec, tmp_path):
    rng = np.random.default_rng(2)
    u = rng.random((64, 80, 3)).astype(np.float32)
    v = (0.5 + 0.4 * np.sin(np.arange(72)[None, :, None] / 3.0) * np.ones((60, 1, 3))).astype(np.float32)
    base = str(tmp_path / "run")
    kw = dict(n_scales=2, extractor=tiny_spec, mode="fast", block=32, margin=16, config_hash="cfgA")
    full = spst.multiscale_transfer(u, v, spst.RunConfig(checkpoint=base, checkpoint_every=10, **kw))
    sides = sorted(glob.glob(base + ".scale2.iter*.json"), key=lambda p: int(p.split(".iter")[1].split(".")[0]))
    assert sides, "no mid-scale checkpoints written"
    side = sides[len(sides) // 2]
    with open(side) as f:
        meta = json.load(f)
    assert meta["scales_done"] == 1 and meta["iteration"] > 0 and os.path.exists(os.path.join(tmp_path, meta["lbfgs"]))
    # no "scale" key: the reference's read_checkpoint (pipeline.py:151-163) cannot mistake a
    # partly optimised iterate for a finished scale
    assert "scale" not in meta
    done, x, snap = read_checkpoint(side, "cfgA", "f32", with_state=True)
    assert done == 1 and snap.iteration == meta["iteration"] and len(snap.s) > 0
    with pytest.raises(spst.ConfigError):  # the stateless (reference) form refuses a mid-scale sidecar
        read_checkpoint(side, "cfgA", "f32")
    with pytest.raises(spst.ConfigError):
        read_checkpoint(side, "otherB", "f32")
    resumed = spst.multiscale_transfer(u, v, spst.RunConfig(resume=side, **kw))
    # the engine re-derives its power-of-2 range exponents on resume: same trajectory to
    # fp32-class rounding, not bit-identical
    assert float(np.mean(np.abs(resumed - full))) <= 1e-4
