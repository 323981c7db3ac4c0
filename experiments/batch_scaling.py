#!/usr/bin/env python
"""NEXT-4: the batch-size hyper-parameter study of P:279-308 (Fig. 4, Fig. 5)
on a synthetic scene, run with the built step (GPU).

* Fig. 4 analogue ("Empirical Evidence of Independent Gradients"): at a fixed
  state, the batch-mean gradient of the diffuse-colour (SH DC) parameters over 32 random
  batches per batch size b; the inverse of the average per-parameter variance vs b (linear
  while gradients are uncorrelated, then a plateau).
* Fig. 5 analogue ("Empirical Testing of Proposed Scaling Rules"): from the same
  state with reset Adam moments, the cumulative diffuse-colour update after the same 32
  images, with batch size 1 (reference) and b in {4, 16, 32} under learning-rate rules
  {constant, sqrt, linear} (momentum scaled, Eq. 2) and momentum rules {scaled, unscaled}
  (sqrt learning rate, Eq. 1): cosine similarity to the b = 1 update and the norm ratio.

The kernel applies Eq. (1)-(2) from the batch size: lambda' = lambda sqrt(b), beta' = beta^b.
The alternatives are obtained by pre-compensating the arguments (constant: lambda/sqrt(b);
linear: lambda sqrt(b); unscaled momentum: beta^(1/b)).

Scene: 200k Gaussians of the C1 (garden-shaped) generator, 512x512 views; ground truth = the
scene rendered by the step's own forward; training starts from the scene with perturbed
diffuse colours.  Writes profiles/next4_batch_scaling.json.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
import paper_2406_18533_b200._lib as L  # noqa: E402
from paper_2406_18533_b200.engine import GrendelTrainer  # noqa: E402

DEV = torch.device("cuda", 0)
N, W, H, POOL = 200_000, 512, 512, 64


def render(ctx, p, cams):
    """Rendered images [b, H, W, 3] uint8 of the parameters p (forward only, through the ABI)."""
    b = len(cams)
    Wt, Ht = (W + 15) // 16, (H + 15) // 16
    dp = np.array([0, b * Wt * Ht], np.int64)
    idx = torch.empty(L.project_index_bytes(ctx, p.n, b), dtype=torch.uint8, device=DEV)
    try:
        cnt = L.project(ctx, p, cams, dp, None, 0, idx)
    except L.CapacityError as e:
        cnt = e.counts
    send = torch.empty((max(int(cnt.sum()), 1), L.RECORD_BYTES), dtype=torch.uint8, device=DEV)
    cnt = L.project(ctx, p, cams, dp, send, send.shape[0], idx)
    n = int(cnt.sum())
    rng = torch.empty(b * Wt * Ht + 1, dtype=torch.int32, device=DEV)
    try:
        npairs = L.bin_sort(ctx, send, n, cams, dp, None, 0, rng)
    except L.CapacityError as e:
        npairs = e.needed
    srt = torch.empty(max(npairs, 1), dtype=torch.int32, device=DEV)
    L.bin_sort(ctx, send, n, cams, dp, srt, npairs, rng)
    nb = b * Wt * Ht
    T = torch.empty(nb * 256, dtype=torch.float32, device=DEV)
    nl = torch.empty(nb * 256, dtype=torch.int32, device=DEV)
    rgb = torch.empty((nb, 3, 256), dtype=torch.float32, device=DEV)
    cost = torch.zeros(nb, dtype=torch.int64, device=DEV)
    L.render_fwd(ctx, send, srt, rng, cams, dp, (0, 0, 0), None, b, rgb, T, nl, None, None, cost, L.COST_WORK, None)
    a = rgb.cpu().numpy().reshape(b, Ht, Wt, 3, 16, 16).transpose(0, 1, 4, 2, 5, 3).reshape(b, Ht * 16, Wt * 16, 3)
    return np.clip(np.round(a[:, :H, :W] * 255), 0, 255).astype(np.uint8)


def dc_grad(tr):
    """The diffuse-colour gradient (SH plane 0 = (dc_r, dc_g, dc_b, sh1_r)) of the last step."""
    return tr.g.sh[0, :, :3].reshape(-1).double().cpu().numpy()


def dc(p):
    return p.sh[0, :, :3].reshape(-1).double().cpu().numpy()


def c_eye(k):
    """The C1 orbit (synth.cameras_garden) without its jitter: eye on a circle of radius 1.3."""
    a = 2 * np.pi * k / POOL
    return (1.3 * np.cos(a), 1.3 * np.sin(a), 0.4 + 0.3 * ((k * 7919) % POOL) / POOL)


def make(sc, noise):
    sh = sc.sh.copy()
    sh[:, 0, :] += noise
    return L.GaussianParams.from_arrays(sc.pos, sc.log_scale, sc.rot, sc.opac_logit, sh, DEV)


def main():
    sc = synth.scene_garden(N, seed=1)
    cams = [synth.look_at(c_eye(k), (0, 0, .25), (0, 0, 1), 0.8 * W, 0.8 * W, W, H, k) for k in range(POOL)]
    ctx = L.Context(0, 0, 1)
    true_p = L.GaussianParams.from_arrays(sc.pos, sc.log_scale, sc.rot, sc.opac_logit, sc.sh, DEV)
    gt = np.concatenate([render(ctx, true_p, cams[i:i + 8]) for i in range(0, POOL, 8)])
    gt_t = torch.from_numpy(gt).to(DEV)
    rng = np.random.default_rng(0)
    noise = rng.normal(0, 0.3, size=(N, 3)).astype(np.float32)
    out = {"scene": "C1 generator, %d Gaussians, %dx%d, pool %d" % (N, W, H, POOL), "fig4": {}, "fig5": {}}

    # ---- Fig. 4: inverse average per-parameter variance of batch-mean gradients
    for b in (1, 2, 4, 8, 16, 32):
        p = make(sc, noise)
        tr = GrendelTrainer(ctx, p, W, H, b, POOL, lr=(0.0,) * 6, rebalance=False)
        gs = []
        for trial in range(32):
            sel = rng.choice(POOL, b, replace=False)
            tr.step([cams[i] for i in sel], gt_t[torch.from_numpy(sel).to(DEV)])
            torch.cuda.synchronize()
            gs.append(dc_grad(tr))
        g = np.stack(gs)
        var = g.var(0).mean()
        out["fig4"][b] = {"inv_avg_var": float(1.0 / var), "sparsity": float((np.abs(g) > 0).mean())}
        print("fig4 b=%d 1/var=%.4g" % (b, 1.0 / var), flush=True)

    # ---- Fig. 5: cumulative diffuse-colour updates over the same 32 images
    order = rng.permutation(POOL)[:32]
    lr0 = (1.6e-4, 2.5e-3, 1.25e-4, 5e-2, 5e-3, 1e-3)

    def trajectory(b, lr_rule, mom_rule):
        p = make(sc, noise)
        start = dc(p)
        s = {"constant": 1.0 / np.sqrt(b), "sqrt": 1.0, "linear": np.sqrt(b)}[lr_rule]
        tr = GrendelTrainer(ctx, p, W, H, b, POOL, lr=tuple(x * s for x in lr0), rebalance=False)
        if mom_rule == "unscaled":
            tr.beta1, tr.beta2 = 0.9 ** (1.0 / b), 0.999 ** (1.0 / b)
        for k in range(0, 32, b):
            sel = order[k:k + b]
            tr.step([cams[i] for i in sel], gt_t[torch.from_numpy(sel).to(DEV)])
        torch.cuda.synchronize()
        return dc(tr.p) - start

    ref = trajectory(1, "sqrt", "scaled")
    for b in (4, 16, 32):
        for lr_rule, mom_rule in (("constant", "scaled"), ("sqrt", "scaled"), ("linear", "scaled"),
                                  ("sqrt", "unscaled")):
            d = trajectory(b, lr_rule, mom_rule)
            cos = float(d @ ref / (np.linalg.norm(d) * np.linalg.norm(ref)))
            ratio = float(np.linalg.norm(d) / np.linalg.norm(ref))
            out["fig5"]["b%d_%s_lr_%s_momentum" % (b, lr_rule, mom_rule)] = {"cosine": cos, "norm_ratio": ratio}
            print("fig5 b=%d lr=%s mom=%s cos=%.4f ratio=%.4f" % (b, lr_rule, mom_rule, cos, ratio), flush=True)
    path = os.path.join(ROOT, "profiles", "next4_batch_scaling.json")
    if len(sys.argv) > 1:
        path = sys.argv[1]
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
