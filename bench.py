#!/usr/bin/env python
"""Benchmark: train views/s of the Grendel 3DGS training step on B200 (BASELINE.json metric
"train views/sec at 1/2/4/8 B200 (Rubble-shaped 4K); fwd+bwd raster ms/view").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl libgs|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

One step = the whole hot path (A1-A9: project, exchange, bin+sort, render fwd + fused L1,
render bwd, reverse exchange, transformation backward + Adam, rebalance) over one batch of b
views of a synthetic, seeded scene (synth/, recipe in DESIGN.md §3).  `value` is whole-job
views/s with inputs resident in HBM, timed by CUDA events on the step stream between a barrier
+ synchronize, max over ranks.  `e2e` repeats the timed loop through the same public API with
each step's ground-truth batch copied host(pinned)->device and the loss copied back.
Inputs (11.2M Gaussians x 3 states, 0.76 GB ground truth per batch) are far larger than L2.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

CONFIGS = {
    "C0": dict(workload="C0 tiny: 1,000 Gaussians, 64x64, batch 1", n=1000, b=1, pool=1, seed=0),
    "C1": dict(workload="Mip-NeRF360-garden-shaped: 5M Gaussians, 1920x1080, batch 4", n=5_000_000, b=4,
               pool=64, seed=1),
    "C2": dict(workload="Rubble-shaped: 11.2M Gaussians, 4591x3436, batch 16", n=11_200_000, b=16, pool=64,
               seed=2),
    "C3": dict(workload="Rubble-shaped 40.4M Gaussians, 4591x3436, batch 16", n=40_400_000, b=16, pool=64,
               seed=3),
    "C4": dict(workload="MatrixCity-shaped: 24M Gaussians, 1920x1080 street+aerial, batch 32", n=24_000_000,
               b=32, pool=128, seed=4),
}
METRIC = "train views/sec at 1/2/4/8 B200 (Rubble-shaped 4K); fwd+bwd raster ms/view"

# Roofline census (frozen): FP32-pipe lane-operations per evaluation.
CENSUS = dict(fwd_comp=13, fwd_skip=8, fwd_stop=9, bwd_contrib=41, bwd_skip=8)
# NEXT-1 D-SSIM census: lane-ops per pixel and channel of the separable
# evaluation without halo recomputation -- window sums of 5 products 11 taps each way
# (88 + 55), SSIM terms (30), 3 derivative maps filtered both ways (33 + 33), combination (10).
SSIM_OPS_PER_PIXEL = 3 * (88 + 55 + 30 + 33 + 33 + 10)


def make_scene(cfg, lo, hi):
    n, seed = cfg["n"], cfg["seed"]
    if cfg is CONFIGS["C0"]:
        return synth.scene_c0(seed).slice(lo, hi)
    fn = {1: synth.scene_garden, 2: synth.scene_rubble, 3: synth.scene_rubble, 4: synth.scene_city}[seed]
    return fn(n, seed, lo, hi)


def scene_extent(cams):
    """radius of the bounding sphere of the camera centres (c = -R^T t), x 1.1 as 3DGS."""
    cs = np.array([-np.asarray(c.R, np.float64).reshape(3, 3).T @ np.asarray(c.t, np.float64) for c in cams])
    centre = cs.mean(0)
    return 1.1 * float(np.linalg.norm(cs - centre, axis=1).max())


def make_cameras(cfg):
    seed = cfg["seed"]
    if seed == 0:
        return synth.cameras_c0()
    if seed in (2, 3):
        return synth.cameras_rubble(cfg["pool"], seed)
    if seed == 1:
        return synth.cameras_garden(cfg["pool"], seed)
    return synth.cameras_city(cfg["pool"], seed)


def batches(cfg, steps):
    if cfg["seed"] == 4:  # C4: 16 street + 16 aerial per batch
        half = cfg["pool"] // 2
        st = synth.batch_schedule(half, cfg["b"] // 2, steps, cfg["seed"])
        ae = synth.batch_schedule(half, cfg["b"] // 2, steps, cfg["seed"] + 1)
        return [s + [half + a for a in x] for s, x in zip(st, ae)]
    return synth.batch_schedule(cfg["pool"], cfg["b"], steps, cfg["seed"])


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.proc, self.lines, self.first = index, None, [], 0

    def mark(self):
        """Start of the timed region: only samples from here on count.  The sampler process is
        started before the warm-up steps, so nvidia-smi's NVML start-up (which can hold the
        driver for hundreds of ms on a fresh box) never lands inside the timed region."""
        self.first = len(self.lines)

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 15.0:  # NVML up before anything is timed
                time.sleep(0.05)
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        rows = []
        for ln in self.lines[self.first:]:
            f = [x.strip() for x in ln.split(",")]
            try:
                rows.append((float(f[0]), float(f[1]), f[3:7]))
            except Exception:
                pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [r[0] for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[2][k].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d, "measured (MEASURED_PEAKS.json)"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------------------- oracle arm

def cpu_info():
    """Host CPU model and logical CPU count (lscpu; os.cpu_count() if lscpu is missing)."""
    info = {"logical_cpus": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            k, _, v = ln.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core"):
                info[k.strip()] = v.strip()
    except Exception:
        pass
    return info


def _chunks(n, k):
    return [(n * i // k, n * (i + 1) // k) for i in range(k) if n * (i + 1) // k > n * i // k]


def oracle_sample(scene, cam, gt_img, threads=1, n_windows=16, win=64, adam_frac=1.0 / 16, seed=0):
    """One bounded sample of one view of the workload, run by the CPU oracle as it stands, on
    `threads` host threads (the C oracle releases the GIL; work is split into disjoint chunks
    whose results are concatenated in order -- the oracle's arithmetic is untouched).
    Sample: project ALL Gaussians for the view (O1-O9, measured as is); `n_windows` windows of
    `win` consecutive blocks, stratified over the view's block rows (window w starts at block
    ((w + 1/2) / n_windows) * blocks, shifted by `seed`): their lists (O11), render forward + L1
    + backward (O12-O15); the transformation backward of the records the windows touched (O16);
    Adam over a 1/16 slice of the Gaussians (O17).  Scaled: render to all blocks of the view,
    lists to one pass over the view's records (one window's list time), the transformation
    backward to all records of the view, Adam to all Gaussians (shared by the b views)."""
    import concurrent.futures as cf
    import oracle
    n = scene.n
    W, H = cam.width, cam.height
    Wt, Ht = (W + 15) // 16, (H + 15) // 16
    nblk = Wt * Ht
    ex = cf.ThreadPoolExecutor(max(1, threads))
    wall0 = time.perf_counter()
    cpu0 = time.process_time()
    # O1-O9 over Gaussian chunks (records of a chunk are in gid order, chunks concatenated in order)
    t0 = time.perf_counter()
    parts = list(ex.map(lambda lh: (lh[0], oracle.make_records(scene.slice(*lh), [cam], "parity")),
                        _chunks(n, max(1, threads))))
    vi = np.concatenate([r.vi + np.array([0, lo]) for lo, r in parts])
    recs = oracle.Records(np.concatenate([r.rec_f for _, r in parts]), np.concatenate([r.rec_i for _, r in parts]),
                          vi, np.concatenate([r.clamp for _, r in parts]))
    t1 = time.perf_counter()
    win = min(win, nblk)
    n_windows = max(1, min(n_windows, nblk // win))
    shift = (seed * 7919) % max(1, nblk // n_windows)
    starts = [min(int((w + 0.5) * nblk / n_windows) - win // 2 + shift, nblk - win) for w in range(n_windows)]
    starts = [max(0, s0) for s0 in starts]

    def window(b0):
        tl = time.perf_counter()
        off, ent = oracle.tile_lists(recs, b0, b0 + win, Wt, Ht)
        tr = time.perf_counter()
        f = oracle.render_fwd(recs, off, ent, b0, b0 + win, W, H, (0, 0, 0), gt_img[None], 1)
        g = oracle.render_bwd(recs, off, ent, b0, b0 + win, W, H, f["dl_dc"])
        touched = np.unique(ent)
        return tr - tl, time.perf_counter() - tr, touched, g[touched]

    wres = list(ex.map(window, starts))
    t2 = time.perf_counter()
    touched, inv = np.unique(np.concatenate([w[2] for w in wres]), return_inverse=True)
    grad = np.zeros((len(touched), 9))
    np.add.at(grad, inv, np.concatenate([w[3] for w in wres]))
    gidx = recs.vi[touched, 1]

    def pbwd(lh):
        lo, hi = lh
        sub = synth.Scene(scene.pos[gidx[lo:hi]], scene.log_scale[gidx[lo:hi]], scene.rot[gidx[lo:hi]],
                          scene.opac_logit[gidx[lo:hi]], scene.sh[gidx[lo:hi]])
        sel = oracle.Records(None, None, np.stack([np.zeros(hi - lo, np.int64), np.arange(hi - lo)], 1), None)
        return oracle.project_bwd(sub, [cam], sel, grad[lo:hi])

    list(ex.map(pbwd, _chunks(len(touched), max(1, threads))))
    t3 = time.perf_counter()
    m = max(1, int(n * adam_frac))

    def adam(lh):
        flat = oracle.flatten_params(scene.slice(*lh))
        return oracle.adam(flat, np.zeros_like(flat), np.zeros_like(flat), np.zeros_like(flat), 1e-3, batch=1, step=1)

    list(ex.map(adam, _chunks(m, max(1, threads))))
    t4 = time.perf_counter()
    ex.shutdown()
    sampled = n_windows * win
    proj = t1 - t0
    lists = float(np.mean([w[0] for w in wres]))  # one window's lists ~ one pass over the view's records
    rend = (t2 - t1) * nblk / sampled
    pb = (t3 - t2) * recs.n / max(len(touched), 1)
    adam_t = (t4 - t3) * n / m
    return dict(sec_per_view_est=proj + lists + rend + pb, adam_per_batch=adam_t, wall_s=t4 - wall0,
                cpu_s=time.process_time() - cpu0, threads=max(1, threads), blocks_sampled=sampled, windows=n_windows, win=win,
                parts=dict(project=proj, lists=lists, render=rend, proj_bwd=pb, adam=adam_t))


def cpu_views_per_s(sample, b):
    per_view = sample["sec_per_view_est"] + sample["adam_per_batch"] / b
    return 1.0 / per_view


SAMPLE_TEXT = ("one view: all Gaussians projected (O1-O9); %d blocks in %d windows of %d stratified over the "
               "view's block rows: lists (O11), render fwd + L1 + bwd (O12-O15), scaled to all blocks; the "
               "touched records' transformation backward (O16), scaled to all records; Adam over 1/16 of the "
               "Gaussians (O17), scaled and shared by the batch's b views")


def oracle_baseline(scene, cam, gt, b, seed=0):
    """The oracle on all host cores and on one thread (SURVEY §8(d) "Modes"), same sample."""
    ncpu = os.cpu_count() or 1
    s_all = oracle_sample(scene, cam, gt, threads=ncpu, seed=seed)
    s_one = oracle_sample(scene, cam, gt, threads=1, seed=seed)
    return {"value": cpu_views_per_s(s_all, b), "unit": "views/s", "cores": s_all["threads"], "kind": "oracle",
            "sample": SAMPLE_TEXT % (s_all["blocks_sampled"], s_all["windows"], s_all["win"])
                      + "; %.1f s wall on %d threads, %.1f s on 1" % (s_all["wall_s"], s_all["threads"],
                                                                      s_one["wall_s"]),
            "cpu": cpu_info(),
            "parts_s_per_view": {k: round(v, 3) for k, v in s_all["parts"].items()},
            "single_thread": {"value": cpu_views_per_s(s_one, b), "cores": 1,
                              "parts_s_per_view": {k: round(v, 3) for k, v in s_one["parts"].items()}}}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    scene = make_scene(cfg, 0, cfg["n"])
    cams = make_cameras(cfg)
    sched = batches(cfg, args.warmup + args.steps)
    times, samples = [], []
    ncpu = os.cpu_count() or 1
    for k in range(args.warmup + args.steps):
        cam = cams[sched[k][0]]
        gt = synth.gt_image(cfg["seed"], cam)
        t = time.perf_counter()
        s = oracle_sample(scene, cam, gt, threads=ncpu, seed=k)
        if k >= args.warmup:
            times.append(time.perf_counter() - t)
            samples.append(cpu_views_per_s(s, cfg["b"]))
    v = float(np.mean(samples))
    line = {"metric": METRIC, "value": v, "unit": "views/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * float(np.mean(times)), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": cfg["workload"], "global_batch": cfg["b"],
                       "parallelism": "oracle-cpu-%d-threads" % ncpu},
            "cpu_baseline": {"value": v, "unit": "views/s", "cores": ncpu, "kind": "oracle", "cpu": cpu_info(),
                             "sample": "per step: " + SAMPLE_TEXT % (s["blocks_sampled"], s["windows"], s["win"])},
            "e2e": {"value": v, "unit": "views/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- load-balance study

def run_virtual(args, cfg):
    """--virtual-ranks G: the E7 analogue (§3.2, §5.3) on one GPU.  The
    config's batch is split over G virtual ranks' pixel ranges (engine.VirtualGrendel); each
    rank's render fwd + bwd is timed with CUDA events; the ranks' max / mean time is the
    imbalance.  Compared: uniform division points (no rebalancing) against Algorithm 1 on
    MEASURED (SM cycles), WORK (evaluations) and PAPER_AVG (the rank's per-pixel average)
    costs, each from the same initial scene for `--epochs` passes over the camera pool; the
    first epoch fills the cost history ("after the first few" epochs) and is not
    reported."""
    import torch
    import paper_2406_18533_b200._lib as L
    from paper_2406_18533_b200.engine import DEFAULT_LR, VirtualGrendel
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    G = args.virtual_ranks
    cams = make_cameras(cfg)
    W, H = cams[0].width, cams[0].height
    per_epoch = len(cams) // cfg["b"]
    steps = per_epoch * args.epochs
    sched = batches(cfg, steps + 1)
    scene = make_scene(cfg, 0, cfg["n"])
    if not args.no_morton:
        from paper_2406_18533_b200.layout import reorder_scene
        scene = reorder_scene(scene)
    gen = torch.Generator(device=dev)
    gen.manual_seed(cfg["seed"] + 200)
    gt_pool = torch.randint(0, 256, (len(cams), H, W, 3), dtype=torch.uint8, device=dev, generator=gen)
    gt_batch = torch.empty((cfg["b"], H, W, 3), dtype=torch.uint8, device=dev)
    modes = [("uniform", L.COST_MEASURED, False), ("measured", L.COST_MEASURED, True),
             ("work", L.COST_WORK, True), ("paper_avg", L.COST_PAPER_AVG, True)]
    out = {}
    for name, cm, reb in modes:
        p = L.GaussianParams.from_arrays(scene.pos, scene.log_scale, scene.rot, scene.opac_logit, scene.sh, dev)
        lr = tuple(args.study_lr_scale * x for x in DEFAULT_LR)
        vg = VirtualGrendel(p, W, H, cfg["b"], len(cams), G, cost_mode=cm, rebalance=reb, device=dev, lr=lr)
        ratios, per_rank = [], []
        for k in range(steps):
            for i, j in enumerate(sched[k]):
                gt_batch[i].copy_(gt_pool[j])
            t = vg.step([cams[i] for i in sched[k]], gt_batch, [cams[i] for i in sched[k + 1]])
            if k >= per_epoch:
                ratios.append(float(t.max() / t.mean()))
                per_rank.append(t)
        pr = np.mean(per_rank, 0)
        out[name] = {"max_over_mean": round(float(np.mean(ratios)), 4),
                     "max_over_mean_per_step": [round(x, 3) for x in ratios],
                     "rank_ms_mean": [round(float(x), 3) for x in pr],
                     "raster_ms_per_step_max_rank": round(float(np.mean([t.max() for t in per_rank])), 3),
                     "final_dp": [int(x) for x in vg.dp]}
        print("%-10s imbalance %.3f  max-rank %.2f ms  ranks %s" % (name, out[name]["max_over_mean"],
              out[name]["raster_ms_per_step_max_rank"], out[name]["rank_ms_mean"]), file=sys.stderr, flush=True)
        del vg, p
        torch.cuda.empty_cache()
    line = {"study": "load_balance", "metric": "imbalance = max / mean over virtual ranks of render fwd+bwd time",
            "unit": "ratio", "higher_is_better": False, "n_gpus": 1, "virtual_ranks": G,
            "config": {"workload": cfg["workload"], "batch": cfg["b"], "epochs": args.epochs,
                       "lr_scale": args.study_lr_scale,
                       "reported": "epochs 2..%d (%d steps)" % (args.epochs, steps - per_epoch)},
            "data": "synthetic", "imbalance": out}
    print(json.dumps(line), flush=True)
    if args.json_out:
        with open(args.json_out, "w") as f:
            json.dump(line, f)
    return 0


# ----------------------------------------------------------------------------- libgs arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="libgs", choices=["libgs", "reference"])
    ap.add_argument("--cost-mode", default="paper_avg", choices=["measured", "work", "paper_avg"],
                    help="A9 cost estimate (N > 1): paper_avg = the rank's measured render time per pixel (P:210, "
                         "the best of the three in the --virtual-ranks study), measured = per-block SM cycles, "
                         "work = per-block walked entries")
    ap.add_argument("--no-rebalance", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-morton", action="store_true", help="keep the generator's (random) Gaussian order")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--breakdown-steps", type=int, default=5)
    ap.add_argument("--json-out", default=None)
    ap.add_argument("--densify", action="store_true",
                    help="NEXT-2: collect densification statistics every step and time one densify event at "
                         "the end (extra 'densify' object in the JSON line)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p"],
                    help="N > 1: grouped NCCL send/recv, or NEXT-3's exchanges fused into the projection and "
                         "render-backward kernels over peer memory (CUDA IPC / NVLink)")
    ap.add_argument("--loss", default="l1", choices=["l1", "ssim"],
                    help="l1: the hot-path loss (R11); ssim: L1 + D-SSIM, lambda 0.2 (NEXT-1)")
    ap.add_argument("--virtual-ranks", type=int, default=0,
                    help="load-balance study on one GPU: the config's batch over this many virtual ranks, "
                         "uniform DP vs Algorithm 1 on MEASURED / WORK / PAPER_AVG costs (an 'imbalance' line)")
    ap.add_argument("--epochs", type=int, default=3, help="--virtual-ranks: passes over the camera pool")
    ap.add_argument("--study-lr-scale", type=float, default=1.0,
                    help="--virtual-ranks: learning rates x this (0: parameters frozen, costs repeat exactly)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.virtual_ranks:
        return run_virtual(args, cfg)

    import torch
    import torch.distributed as dist
    import paper_2406_18533_b200._lib as L
    from paper_2406_18533_b200.engine import GrendelTrainer, event_ms, make_events

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        obj = [L.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = L.Context(local, rank, world, obj[0])
    else:
        ctx = L.Context(local, 0, 1)

    t_setup = time.perf_counter()
    n = cfg["n"]
    lo, hi = n * rank // world, n * (rank + 1) // world
    scene = make_scene(cfg, lo, hi)
    if not args.no_morton:
        from paper_2406_18533_b200.layout import reorder_scene
        scene = reorder_scene(scene)  # layout: Morton order within the rank's shard
    cams = make_cameras(cfg)
    W, H = cams[0].width, cams[0].height
    p = L.GaussianParams.from_arrays(scene.pos, scene.log_scale, scene.rot, scene.opac_logit, scene.sh, dev, lo)
    sched = batches(cfg, args.warmup + args.steps + args.breakdown_steps + args.steps + 2)
    # ground-truth pool on the device (uint8, i.i.d. uniform; only the L1 sign matters)
    gen = torch.Generator(device=dev)
    gen.manual_seed(cfg["seed"] + 200)
    gt_pool = torch.randint(0, 256, (len(cams), H, W, 3), dtype=torch.uint8, device=dev, generator=gen)
    gt_batch = torch.empty((cfg["b"], H, W, 3), dtype=torch.uint8, device=dev)
    cost_mode = {"measured": L.COST_MEASURED, "work": L.COST_WORK, "paper_avg": L.COST_PAPER_AVG}[args.cost_mode]
    tr = GrendelTrainer(ctx, p, W, H, cfg["b"], len(cams), cost_mode=cost_mode, rebalance=not args.no_rebalance,
                        device=dev, loss=args.loss, densify_stats=args.densify, exchange=args.exchange)
    stream = torch.cuda.current_stream()
    k_sched = [0]

    def batch_cams(k):
        return [cams[i] for i in sched[k]]

    def one_step(events=None, stats=False):
        k = k_sched[0]
        # the batch's ground truth: one contiguous device-to-device copy per view (cudaMemcpyAsync;
        # torch.index_select's gather kernel took ~1.8 ms for the 0.76 GB of a C2 batch)
        for i, j in enumerate(sched[k]):
            gt_batch[i].copy_(gt_pool[j])
        loss = tr.step(batch_cams(k), gt_batch, next_cams=batch_cams(k + 1), events=events, collect_stats=stats)
        k_sched[0] += 1
        return loss

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # size all buffers for every batch this run will use (setup, not timed)
    tr.reserve_for([batch_cams(k) for k in range(len(sched) - 1)])
    clocks = ClockSampler(local)
    if not os.environ.get("GS_NO_CLOCKS"):  # diagnostics: run without the nvidia-smi sampler
        clocks.start()
    for _ in range(args.warmup):
        one_step()
    setup_s = time.perf_counter() - t_setup

    # ---------------- timed region (device-resident inputs)
    # The step's host syncs (record and pair counts) leave the GPU idle while the host thread
    # is paused, and a full Python garbage collection landing there cost one step 5-40 ms at a
    # deterministic allocation count: collect and freeze the setup's objects, no automatic
    # collections while timing (what a training loop does).
    gc.collect()
    gc.freeze()
    gc.disable()
    barrier()
    clocks.mark()
    l0 = ctx.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    step_ev = []
    dbg = [] if os.environ.get("GS_BENCH_DEBUG") else None  # per-call events of every timed step
    for _ in range(args.steps):
        if dbg is not None:
            dbg.append(make_events())
            th0 = time.perf_counter()
        one_step(events=None if dbg is None else dbg[-1])
        if dbg is not None:
            dbg[-1]["host_ms"] = 1000.0 * (time.perf_counter() - th0)
            dbg[-1]["pairs"] = tr.last["n_pairs"]
        step_ev.append(torch.cuda.Event(enable_timing=True))
        step_ev[-1].record(stream)
    e1.record(stream)
    barrier()
    step_ms = [e0.elapsed_time(step_ev[0])] + [a.elapsed_time(b) for a, b in zip(step_ev, step_ev[1:])]
    print("timed steps (ms): " + " ".join("%.1f" % t for t in step_ms), file=sys.stderr, flush=True)
    if dbg is not None:
        for k, ev in enumerate(dbg):
            hm, npairs = ev.pop("host_ms"), ev.pop("pairs")
            print("step %d (batch %s, %d pairs, cap %d) host %.1f ms: %s" % (k, sched[args.warmup + k], npairs,
                                                                             tr.sorted.cap, hm,
                                                           {n: round(v, 2) for n, v in event_ms(ev).items()}),
                  file=sys.stderr, flush=True)
    clk = clocks.stop()
    launches = ctx.launch_count() - l0
    ms = e0.elapsed_time(e1)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    views = cfg["b"] * args.steps
    value = views / (ms_max / 1000.0)

    # ---------------- per-call breakdown + work counters (untimed pass)
    calls, call_lists = {}, {}
    stats = np.zeros(8, np.int64)
    counts = dict(n_send=0, n_recv=0, n_pairs=0, n_owned=0)
    # per-call times with the kernels of the timed region (no counters), then the same batches
    # again with the counting kernel variants for the work census (their times are not used)
    k_bd = k_sched[0]
    for _ in range(args.breakdown_steps):
        ev = make_events()
        one_step(events=ev)
        torch.cuda.synchronize()
        for kname, v in event_ms(ev).items():
            call_lists.setdefault(kname, []).append(v)
    # per call: the median over the breakdown steps, p10 / p90 reported beside it
    calls = {k: float(np.median(v)) for k, v in call_lists.items()}
    k_sched[0] = k_bd
    for _ in range(args.breakdown_steps):
        one_step(stats=True)
        torch.cuda.synchronize()
        stats += tr.stats.cpu().numpy() // 1
        for kname in counts:
            counts[kname] += tr.last[kname] / args.breakdown_steps
    stats = stats / args.breakdown_steps

    # ---------------- N > 1: exchange volumes, NVLink rates and raster imbalance
    multi = None
    if world > 1:
        sc_, rc_ = np.asarray(tr.last["send_counts"]), np.asarray(tr.last["recv_counts"])
        vec = torch.tensor([calls.get("exchange", 0.0), calls.get("exchange_grads", 0.0),
                            calls.get("render_fwd", 0.0) + calls.get("render_bwd", 0.0),
                            float(sc_.sum() - sc_[rank]), float(rc_.sum() - rc_[rank]), float(sc_.sum())],
                           dtype=torch.float64, device=dev)
        allv = [torch.zeros_like(vec) for _ in range(world)]
        dist.all_gather(allv, vec)
        a = torch.stack(allv).cpu().numpy()  # [rank][fwd_ms, rev_ms, raster_ms, sent, recvd, all sent]
        rb, gb = L.RECORD_BYTES, 4 * L.GRAD_FLOATS

        def rate(nbytes, ms):
            return [round(float(x) / (float(t) / 1e3) / 1e9, 2) if t > 0 else None for x, t in zip(nbytes, ms)]

        multi = {
            "forward_exchange": {"bytes_sent_remote": [int(x * rb) for x in a[:, 3]],
                                 "bytes_recv_remote": [int(x * rb) for x in a[:, 4]],
                                 "ms": [round(float(x), 4) for x in a[:, 0]],
                                 "GBps_sent_per_rank": rate(a[:, 3] * rb, a[:, 0]),
                                 "GBps_max_over_ranks": max([x for x in rate(a[:, 3] * rb, a[:, 0]) if x] or [0])},
            "reverse_exchange": {"bytes_sent_remote": [int(x * gb) for x in a[:, 4]],
                                 "ms": [round(float(x), 4) for x in a[:, 1]],
                                 "GBps_sent_per_rank": rate(a[:, 4] * gb, a[:, 1]),
                                 "GBps_max_over_ranks": max([x for x in rate(a[:, 4] * gb, a[:, 1]) if x] or [0])},
            "records_vs_dense_bound": round(float(a[:, 5].sum()) / (world * n * cfg["b"]), 5),
            "raster_ms_per_rank": [round(float(x), 3) for x in a[:, 2]],
            "raster_imbalance_max_over_mean": round(float(a[:, 2].max() / max(a[:, 2].mean(), 1e-9)), 4),
            "note": "per-call CUDA-event times of the breakdown steps on each rank's stream; bytes = records "
                    "(or 9-float gradients) exchanged with other ranks; dense bound = G x N records per view"}

    # ---------------- e2e: host (pinned) ground truth in, loss out, through the same API
    e2e = None
    if not args.no_e2e:
        gt_host = torch.empty((len(cams), H, W, 3), dtype=torch.uint8, pin_memory=True)
        gt_host.copy_(gt_pool.cpu())
        loss_host = torch.empty(1, dtype=torch.float64, pin_memory=True)
        # double-buffered ground truth: batch k+1 is copied host->device on a copy stream while
        # step k runs (every copy is inside the timed region; only the first is not overlapped)
        gt_bufs = [gt_batch, torch.empty_like(gt_batch)]
        copy_stream = torch.cuda.Stream(device=dev)
        copied = [torch.cuda.Event(), torch.cuda.Event()]
        freed = [torch.cuda.Event(), torch.cuda.Event()]

        def h2d(k, buf):
            with torch.cuda.stream(copy_stream):
                copy_stream.wait_event(freed[buf])
                for j, i in enumerate(sched[k]):
                    gt_bufs[buf][j].copy_(gt_host[i], non_blocking=True)
                copied[buf].record(copy_stream)

        for e in freed:
            e.record(stream)
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        k0 = k_sched[0]
        h2d(k0, 0)
        for s_ in range(args.steps):
            k = k_sched[0]
            buf = s_ % 2
            if s_ + 1 < args.steps:
                h2d(k + 1, 1 - buf)
            stream.wait_event(copied[buf])
            loss = tr.step(batch_cams(k), gt_bufs[buf], next_cams=batch_cams(k + 1))
            freed[buf].record(stream)
            loss_host.copy_(loss, non_blocking=True)
            k_sched[0] += 1
        f1.record(stream)
        barrier()
        ems = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e2e = {"value": views / (float(ems.item()) / 1000.0), "unit": "views/s",
               "h2d_bytes_per_step": int(cfg["b"] * H * W * 3), "d2h_bytes_per_step": 8}

    gc.enable()

    # ---------------- roofline of the dominant kernel
    pk, pk_src = peaks()
    sm_mhz = float(pk.get("sm_max_mhz", 1965.0))
    fp32_peak = 148 * 128 * sm_mhz * 1e6 / 1e12  # T lane-ops/s
    Efc, Efs, Estop, Eb, Ebc = stats[1], stats[2], stats[3], stats[4], stats[5]
    work = {
        "render_fwd": ("alu", (CENSUS["fwd_comp"] * Efc + CENSUS["fwd_skip"] * Efs + CENSUS["fwd_stop"] * Estop) / 1e12,
                       "T FP32-lane-op/s", fp32_peak),
        "render_bwd": ("alu", (CENSUS["bwd_contrib"] * Ebc + CENSUS["bwd_skip"] * (Eb - Ebc)) / 1e12,
                       "T FP32-lane-op/s", fp32_peak),
        "adam": ("hbm", (1416.0 * p.n + 36.0 * counts["n_send"]) / 1e9, "GB/s", float(pk.get("hbm_gbs", 6650.0))),
        "project": ("hbm", (236.0 * p.n + 56.0 * counts["n_send"]) / 1e9, "GB/s", float(pk.get("hbm_gbs", 6650.0))),
        "bin_sort": ("hbm", (28.0 * counts["n_pairs"] + 16.0 * counts["n_recv"]) / 1e9, "GB/s",
                     float(pk.get("hbm_gbs", 6650.0))),
        "loss": ("alu", SSIM_OPS_PER_PIXEL * 256.0 * counts["n_owned"] / 1e12, "T FP32-lane-op/s", fp32_peak),
    }
    dom = max((k for k in work if k in calls), key=lambda k: calls[k])
    bound, amount, unit, peak = work[dom]
    achieved = amount / (calls[dom] / 1000.0)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "dram_traffic.json")) as f:
            t = json.load(f).get(args.config, {}).get(dom)
            traffic = None if t is None else {"bytes_per_launch": t["bytes"], "source": t["source"]}
    except Exception:
        pass
    rooflines = {}
    for k, (bd, amt, un, pkv) in work.items():
        if k in calls and calls[k] > 0:
            a = amt / (calls[k] / 1000.0)
            rooflines[k] = {"bound": bd, "achieved": round(a, 3), "peak": pkv, "unit": un, "frac": round(a / pkv, 4),
                            "ms": round(calls[k], 3)}

    # ---------------- oracle baseline on the host cores (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        full = scene
        cam = batch_cams(0)[0]
        gt = gt_pool[sched[0][0]].cpu().numpy()
        cpu = oracle_baseline(full, cam, gt, cfg["b"])

    # ---------------- NEXT-2: one densify-and-prune event over the trained shard (after all
    # other measurements: it changes the shard), plus the per-step statistics kernel
    dens = None
    if args.densify:
        n_before = tr.p.n
        gen = torch.Generator(device=dev)
        gen.manual_seed(cfg["seed"] + 300)
        noise = torch.randn((n_before, 2, 3), dtype=torch.float32, device=dev, generator=gen)
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        w0.record()
        kc = tr.densify(L.densify_cfg(scene_extent=float(scene_extent(cams))), noise=noise, events=(d0, d1))
        w1.record()
        torch.cuda.synchronize()
        dms, wms = d0.elapsed_time(d1), w0.elapsed_time(w1)
        # algorithmic bytes: read p, m, v (3 x 240 B) + 3 statistics (12 B) + noise (24 B) per
        # Gaussian, write p, m, v of every output Gaussian (3 x 240 B)
        dbytes = 756.0 * n_before + 720.0 * int(kc[3])
        hbm = float(pk.get("hbm_gbs", 6650.0))
        dens = {"event_ms": round(dms, 3), "event_with_alloc_ms": round(wms, 3), "n_before": int(n_before),
                "counts": {
                    "kept": int(kc[0]), "clones": int(kc[1]), "children": int(kc[2]), "total": int(kc[3])},
                "stats_ms_per_step": round(calls.get("densify_stats", 0.0), 3),
                "roofline": {"bound": "hbm", "achieved": round(dbytes / (dms / 1000.0) / 1e9, 1), "peak": hbm,
                             "unit": "GB/s", "frac": round(dbytes / (dms / 1000.0) / 1e9 / hbm, 4)},
                "note": "event_ms: device time of the placing gs_densify call (classify, scan, write); "
                        "event_with_alloc_ms adds the size query and the new shard's allocation; statistics "
                        "from the timed steps of this run"}

    if rank == 0:
        raster_ms_view = (calls.get("render_fwd", 0) + calls.get("render_bwd", 0)) / cfg["b"]
        line = {"metric": METRIC, "value": round(value, 3), "unit": "views/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": cfg["workload"], "config_id": args.config, "global_batch": cfg["b"],
                           "image": [W, H], "gaussians": n, "parallelism": "gaussian+pixel x%d (Grendel)" % world,
                           "l2_policy": "inputs larger than L2 (params+Adam state %.1f GB, GT %.2f GB/step)" % (
                               3 * 240 * n / 1e9, cfg["b"] * W * H * 3 / 1e9),
                           "loss": "l1" if args.loss == "l1" else "l1+dssim(0.2)",
                           "cost_mode": args.cost_mode if world > 1 else "n/a (one rank)",
                           "rebalance": (not args.no_rebalance) if world > 1 else "n/a (one rank: DP = [0, B])",
                           "exchange": args.exchange if world > 1 else "none (one rank)",
                           "shard_layout": "random" if args.no_morton else "morton"},
                "raster_ms_per_view": round(raster_ms_view, 3),
                "calls_ms": {k: round(v, 3) for k, v in calls.items()},
                "calls_ms_p10_p90": {k: [round(float(np.percentile(v, 10)), 3), round(float(np.percentile(v, 90)), 3)]
                                     for k, v in call_lists.items()},
                "gpu_launches": int(launches),
                "roofline": {"bound": bound, "kernel": dom, "achieved": round(achieved, 3), "peak": peak,
                             "unit": unit, "frac": round(achieved / peak, 4), "traffic": traffic,
                             "peak_source": pk_src},
                "rooflines": rooflines,
                "work": {"E_f": int(stats[0]), "E_fc": int(Efc), "E_fs": int(Efs), "E_stop": int(Estop),
                         "E_b": int(Eb), "E_bc": int(Ebc), "records": int(counts["n_recv"]),
                         "pairs": int(counts["n_pairs"])},
                "clocks": clk, "e2e": e2e, "cpu_baseline": cpu, "setup_s": round(setup_s, 1)}
        if dens is not None:
            line["densify"] = dens
        if multi is not None:
            line["multi_gpu"] = multi
        s = json.dumps(line)
        print(s, flush=True)
        if args.json_out:
            with open(args.json_out, "w") as f:
                f.write(s + "\n")
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
