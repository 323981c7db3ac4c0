"""NEXT-2 oracle: adaptive density control (TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py).

Plain numpy, written from the paper and SPEC ("adaptive densification mechanism to add
Gaussians"; App. A.1 "whether their scale exceeds a threshold ... cloning or
splitting existing ones ... opacity reset techniques to remove redundant Gaussians"; P:501
App. A.3 "locally on the GPU that stores them") and the readings R13-R14 of
DESIGN.md.  Decisions that pick integers (which Gaussians are cloned / split / pruned) are
taken in fp32 against thresholds rounded once from fp64 (R14: the same precision as the
kernel, the task's rule for floating point deciding integers); new values are fp64.

Shard dictionaries: pos[n,3], log_scale[n,3], rot[n,4], opac_logit[n], sh[n,48] (the
gradient order of GROUP_SLICES), all numpy arrays.
"""
from __future__ import annotations

import math

import numpy as np

FIELDS = ("pos", "log_scale", "rot", "opac_logit", "sh")


def stats_from_record_grads(n, gid, grad_rec, radius, W, H, b):
    """S:366-373 accumulate: every record (Gaussian gid[r], one view) adds
    || b (W/2 dL/dmx, H/2 dL/dmy) || (R13: the NDC-space mean gradient of the per-image loss;
    the step's loss is the batch mean) to accum, 1 to denom, and raises max_radius."""
    accum = np.zeros(n)
    denom = np.zeros(n)
    max_radius = np.zeros(n)
    for r in range(len(gid)):
        i = int(gid[r])
        gx = b * (W / 2.0) * grad_rec[r, 0]
        gy = b * (H / 2.0) * grad_rec[r, 1]
        accum[i] += math.hypot(gx, gy)
        denom[i] += 1.0
        max_radius[i] = max(max_radius[i], radius[r])
    return accum, denom, max_radius


def thresholds(cfg):
    """R14: every threshold rounded once from fp64 to fp32."""
    f = np.float32
    return dict(grad=f(cfg["grad_thresh"]),
                log_split=f(math.log(cfg["percent_dense"] * cfg["scene_extent"])),
                logit_min_op=f(math.log(cfg["min_opacity"] / (1.0 - cfg["min_opacity"]))),
                max_screen=f(cfg["max_screen_size"]),
                log_big=f(math.log(0.1 * cfg["scene_extent"])),
                log_big_child=f(math.log(1.6 * 0.1 * cfg["scene_extent"])))


def _rotmat(q):
    w, x, y, z = q / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def densify(shard, m, v, accum, denom, max_radius, noise, cfg):
    """S:375-384 densify_and_prune, one event, in the 3DGS order: clones are appended, then the
    split children (first children of all split parents, then the second ones), the split
    parents are removed, and pruning applies to the result.  Returns (shard', m', v', counts)
    with counts = (kept originals, clones, children, total)."""
    th = thresholds(cfg)
    f32 = np.float32
    n = len(shard["pos"])
    a32 = np.asarray(accum, f32)
    d32 = np.asarray(denom, f32)
    avg = np.zeros(n, f32)
    nz = d32 > 0
    avg[nz] = a32[nz] / d32[nz]  # fp32 IEEE division
    sel = avg >= th["grad"]
    lmax = np.asarray(shard["log_scale"], f32).max(1)
    big = lmax > th["log_split"]
    clone, split = sel & ~big, sel & big
    logit = np.asarray(shard["opac_logit"], f32)
    low = logit < th["logit_min_op"]
    screen_on = th["max_screen"] > 0
    prune_orig = low | (screen_on & ((np.asarray(max_radius, f32) > th["max_screen"]) | (lmax > th["log_big"])))
    prune_clone = low | (screen_on & (lmax > th["log_big"]))
    prune_child = low | (screen_on & (lmax > th["log_big_child"]))
    keep_o = ~split & ~prune_orig
    keep_c = clone & ~prune_clone
    keep_k = split & ~prune_child

    out = {k: [] for k in FIELDS}
    om = {k: [] for k in FIELDS}
    ov = {k: [] for k in FIELDS}

    def push(src, i, st=None, zero_state=True, pos=None, log_scale=None):
        for k in FIELDS:
            val = np.array(src[k][i], np.float64)
            if k == "pos" and pos is not None:
                val = pos
            if k == "log_scale" and log_scale is not None:
                val = log_scale
            out[k].append(val)
            om[k].append(np.zeros_like(val) if zero_state else np.array(m[k][i], np.float64))
            ov[k].append(np.zeros_like(val) if zero_state else np.array(v[k][i], np.float64))

    for i in range(n):
        if keep_o[i]:
            push(shard, i, zero_state=False)
    for i in range(n):
        if keep_c[i]:
            push(shard, i)
    for t in range(2):
        for i in range(n):
            if keep_k[i]:
                ls = np.asarray(shard["log_scale"][i], np.float64)
                s = np.exp(ls)
                R = _rotmat(np.asarray(shard["rot"][i], np.float64))
                pos = np.asarray(shard["pos"][i], np.float64) + R @ (s * np.asarray(noise[i, t], np.float64))
                push(shard, i, pos=pos, log_scale=ls - math.log(1.6))
    n2 = len(out["pos"])
    pack = lambda d: {k: (np.array(d[k]) if n2 else np.zeros((0,) + np.shape(shard[k])[1:])) for k in FIELDS}
    counts = (int(keep_o.sum()), int(keep_c.sum()), int(2 * keep_k.sum()), n2)
    return pack(out), pack(om), pack(ov), counts


def opacity_reset(shard, m, v, max_opacity=0.01):
    """logits clamped to logit(max_opacity) (R14: in fp32, min(logit, threshold)),
    the opacity Adam moments zeroed."""
    thr = np.float32(math.log(max_opacity / (1.0 - max_opacity)))
    s2 = dict(shard)
    s2["opac_logit"] = np.minimum(np.asarray(shard["opac_logit"], np.float32), thr)
    m2, v2 = dict(m), dict(v)
    m2["opac_logit"] = np.zeros_like(m["opac_logit"])
    v2["opac_logit"] = np.zeros_like(v["opac_logit"])
    return s2, m2, v2


# ------------------------------------------------------------------ random redistribution

_M32 = 0xFFFFFFFF


def _fmix32(h):
    h ^= h >> 16
    h = (h * 0x85EBCA6B) & _M32
    h ^= h >> 13
    h = (h * 0xC2B2AE35) & _M32
    h ^= h >> 16
    return h


def feistel_half(N):
    k = 2
    while k < 64 and (1 << k) < N:
        k += 1
    return (k + (k & 1)) // 2


def perm(j, N, seed):
    """R15: the keyed bijection pi of [0, N) -- a 4-round Feistel network on the smallest even
    bit width covering N (round function: murmur3's 32-bit finaliser of the seed, the round and
    the right half), cycle-walked until the image falls in [0, N)."""
    s = (seed ^ (seed >> 32)) & _M32
    half = feistel_half(N)
    mask = (1 << half) - 1
    y = j
    while True:
        L, R = (y >> half) & mask, y & mask
        for r in range(4):
            f = _fmix32(s ^ ((r * 0x9E3779B9) & _M32) ^ _fmix32((R + 0x7F4A7C15 * (r + 1)) & _M32)) & mask
            L, R = R, L ^ f
        y = (L << half) | R
        if y < N:
            return y


def redistribute(shards, states_m, states_v, seed):
    """S:491-497 rebalance_gaussians: the concatenation of the rank shards (global index j) is
    reordered by pi and cut into G ranges [floor(dN/G), floor((d+1)N/G)).  Returns the new
    (shards, m, v) lists; Adam state travels with its Gaussian."""
    G = len(shards)
    cat = lambda ds: {k: np.concatenate([np.asarray(d[k]) for d in ds]) for k in FIELDS}
    allp, allm, allv = cat(shards), cat(states_m), cat(states_v)
    N = len(allp["pos"])
    order = np.empty(N, np.int64)
    for j in range(N):
        order[perm(j, N, seed)] = j  # new position pi(j) holds old element j
    out = []
    for d in range(G):
        lo, hi = d * N // G, (d + 1) * N // G
        idx = order[lo:hi]
        out.append(tuple({k: a[k][idx] for k in FIELDS} for a in (allp, allm, allv)))
    return [o[0] for o in out], [o[1] for o in out], [o[2] for o in out]
