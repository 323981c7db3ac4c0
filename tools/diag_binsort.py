"""Diagnostics (GPU box): bin_sort time per batch of the C2 schedule, device events and host
time, three repeats each, after projection (no training).  python tools/diag_binsort.py"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2406_18533_b200._lib as L  # noqa: E402
from paper_2406_18533_b200.engine import GrendelTrainer  # noqa: E402
from paper_2406_18533_b200.layout import reorder_scene  # noqa: E402

cfg = bench.CONFIGS["C2"]
dev = torch.device("cuda", 0)
ctx = L.Context(0, 0, 1)
scene = reorder_scene(bench.make_scene(cfg, 0, cfg["n"]))
cams = bench.make_cameras(cfg)
W, H = cams[0].width, cams[0].height
p = L.GaussianParams.from_arrays(scene.pos, scene.log_scale, scene.rot, scene.opac_logit, scene.sh, dev, 0)
sched = bench.batches(cfg, 16)
tr = GrendelTrainer(ctx, p, W, H, cfg["b"], len(cams), device=dev)
tr.reserve_for([[cams[i] for i in sched[k]] for k in range(16)])
for k in range(16):
    bc = [cams[i] for i in sched[k]]
    cnt = L.project(ctx, p, bc, tr.dp, tr.send.t, tr.send.cap, tr.bwd_index)
    n = int(cnt.sum())
    ts = []
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        e0.record()
        npairs = L.bin_sort(ctx, tr.send.t, n, bc, tr.dp, tr.sorted.t, tr.sorted.cap, tr.range.t)
        e1.record()
        torch.cuda.synchronize()
        ts.append((round(e0.elapsed_time(e1), 2), round(1000 * (time.perf_counter() - h0), 2)))
    print("batch %2d records %d pairs %d: %s" % (k, n, npairs, ts), flush=True)
