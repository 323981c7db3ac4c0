#!/usr/bin/env python
"""Minimal step driver for ncu captures: the bench workload (or a reduced copy of it) through
GrendelTrainer, W warm-up steps then P steps.  ncu's kernel replay must save and restore
every buffer a kernel writes; the fused Adam kernel writes all parameters and moments
(8 GB at C2), so full-section captures use --views / --gaussians to shrink the footprint while
keeping the per-block and per-Gaussian work of the bench scene.

    python tools/prof_driver.py --config C2 --views 4 --gaussians 2800000 --warmup 2 --steps 1
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2406_18533_b200._lib as L  # noqa: E402
from paper_2406_18533_b200.engine import GrendelTrainer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--views", type=int, default=0)
    ap.add_argument("--gaussians", type=int, default=0)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--steps", type=int, default=1)
    a = ap.parse_args()
    cfg = dict(bench.CONFIGS[a.config])
    if a.gaussians:
        cfg["n"] = a.gaussians
    b = a.views or cfg["b"]
    dev = torch.device("cuda", 0)
    sc = bench.make_scene(cfg, 0, cfg["n"])
    from paper_2406_18533_b200.layout import reorder_scene
    sc = reorder_scene(sc)
    cams = bench.make_cameras(cfg)
    sched = bench.batches(dict(cfg, b=b), a.warmup + a.steps + 1) if cfg["seed"] != 4 else \
        bench.batches(cfg, a.warmup + a.steps + 1)
    W, H = cams[0].width, cams[0].height
    ctx = L.Context(0, 0, 1)
    p = L.GaussianParams.from_arrays(sc.pos, sc.log_scale, sc.rot, sc.opac_logit, sc.sh, dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(cfg["seed"] + 200)
    gt = torch.randint(0, 256, (b, H, W, 3), dtype=torch.uint8, device=dev, generator=gen)
    tr = GrendelTrainer(ctx, p, W, H, b, len(cams), device=dev)
    for k in range(a.warmup + a.steps):
        cams_k = [cams[i] for i in sched[k][:b]]
        tr.step(cams_k, gt, next_cams=[cams[i] for i in sched[k + 1][:b]])
    torch.cuda.synchronize()
    print("done", tr.last)


if __name__ == "__main__":
    main()
