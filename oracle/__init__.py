"""CPU oracle for the Grendel 3DGS training step (arXiv 2406.18533).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package.  It shares no code
with the CUDA library (paper_2406_18533_b200/, include/gs.h); the product path never
imports it.  The arithmetic lives in gs_oracle.c (plain C, fp32 membership chain + fp64
everything else, see its header); this module only marshals numpy arrays, and assembles
the single-partition definition of the step (SURVEY §8(c) "What the result is":
render the whole batch from the whole cloud, "changes where, never what").

Parity-unpinned parts (also listed in DESIGN.md §5): the MEASURED cost mode (hardware
timing; only DP-given-ET is pinned) and the SH sign convention (the paper is silent).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "gs_oracle.c")

FLAG_ALPHA, FLAG_T, FLAG_POWER, FLAG_OVERFLOW = 1, 2, 4, 16


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "gs_oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-std=c11",
                               "-fPIC", "-shared", "-o", _SO, _SRC, "-lm"])
    return _SO


class _Cam(C.Structure):
    _fields_ = [("R", C.c_float * 9), ("t", C.c_float * 3), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("width", C.c_int32), ("height", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.orc_exp_rn.restype = C.c_float
        _lib.orc_exp_rn.argtypes = [C.c_float]
        _lib.orc_division_points.restype = C.c_int
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _cam(cam) -> _Cam:
    c = _Cam()
    c.R[:] = [float(v) for v in np.asarray(cam.R, np.float32).reshape(-1)]
    c.t[:] = [float(v) for v in np.asarray(cam.t, np.float32).reshape(-1)]
    c.fx, c.fy, c.cx, c.cy = cam.fx, cam.fy, cam.cx, cam.cy
    c.width, c.height = cam.width, cam.height
    return c


def _f32(a):
    return np.ascontiguousarray(a, np.float32)


def _f64(a):
    return np.ascontiguousarray(a, np.float64)


def exp_rn(x: float) -> float:
    return float(np.float32(lib().orc_exp_rn(C.c_float(float(x)))))


def membership(scene, cam):
    """O1-O8 in fp32.  Returns dict of arrays over the scene's Gaussians."""
    n = scene.n
    out = dict(vis=np.zeros(n, np.int8), mx=np.zeros(n, np.float32), my=np.zeros(n, np.float32),
               depth=np.zeros(n, np.float32), cov=np.zeros((n, 3), np.float32),
               radius=np.zeros(n, np.int32), rect=np.zeros((n, 4), np.int32))
    c = _cam(cam)
    lib().orc_membership_f32(C.c_int64(n), _p(_f32(scene.pos)), _p(_f32(scene.log_scale)),
                             _p(_f32(scene.rot)), C.byref(c), _p(out["vis"]), _p(out["mx"]),
                             _p(out["my"]), _p(out["depth"]), _p(out["cov"]), _p(out["radius"]),
                             _p(out["rect"]))
    return out


PROJ_FIELDS = ["vis", "mx", "my", "depth", "a", "b", "c", "A", "B", "C", "opacity", "r", "g", "b_",
               "clamp", "radius"]


def project64(scene, cam):
    """O1-O9 in fp64: returns (out[n,16] in PROJ_FIELDS order, rect[n,4])."""
    n = scene.n
    out = np.zeros((n, 16), np.float64)
    rect = np.zeros((n, 4), np.int32)
    c = _cam(cam)
    lib().orc_project_f64(C.c_int64(n), _p(_f64(scene.pos)), _p(_f64(scene.log_scale)),
                          _p(_f64(scene.rot)), _p(_f64(scene.opac_logit)), _p(_f64(scene.sh)),
                          C.byref(c), _p(out), _p(rect))
    return out, rect


def exchange_sets(vis, rect, view, Wt, Ht, dp):
    """O10: destination bitmask per Gaussian for one view."""
    n = len(vis)
    mask = np.zeros(n, np.uint32)
    dp = np.ascontiguousarray(dp, np.int64)
    lib().orc_exchange_sets(C.c_int64(n), _p(np.ascontiguousarray(vis, np.int8)),
                            _p(np.ascontiguousarray(rect, np.int32)), C.c_int32(view), C.c_int32(Wt),
                            C.c_int32(Ht), C.c_int32(len(dp) - 1), _p(dp), _p(mask))
    return mask


class Records:
    """One record per visible (Gaussian, view) of the whole batch (the single-partition
    definition).  rec_f[:, :] = (mx, my, depth, A, B, C, opacity, r, g, b) fp64;
    rec_i = (gid, view, tx0, tx1, ty0, ty1); vi = (view, local index)."""

    def __init__(self, rec_f, rec_i, vi, clamp):
        self.rec_f, self.rec_i, self.vi, self.clamp = rec_f, rec_i, vi, clamp

    @property
    def n(self):
        return self.rec_f.shape[0]


def make_records(scene, cams, mode: str = "parity") -> Records:
    """mode='parity': mean2d, depth and the 2D covariance are the fp32 membership-chain
    values (R10: they decide tile membership and sort order, so they are defined in fp32);
    conic = inverse of that covariance computed in fp64 (O6), opacity and colour fp64 (O1, O9).
    mode='f64': every value fp64 (finite-difference pins)."""
    fs, is_, vis_, cl = [], [], [], []
    for v, cam in enumerate(cams):
        p64, rect64 = project64(scene, cam)
        if mode == "parity":
            mb = membership(scene, cam)
            vis = mb["vis"].astype(bool)
            cov = mb["cov"].astype(np.float64)
            a, b, c = cov[:, 0], cov[:, 1], cov[:, 2]
            det = a * c - b * b  # O6 (fp64)
            with np.errstate(divide="ignore", invalid="ignore"):
                A, B, Cc = c / det, -b / det, a / det
            mx, my, dep = mb["mx"].astype(np.float64), mb["my"].astype(np.float64), mb["depth"].astype(np.float64)
            rect = mb["rect"]
        else:
            vis = p64[:, 0] > 0
            mx, my, dep, A, B, Cc = (p64[:, k] for k in (1, 2, 3, 7, 8, 9))
            rect = rect64
        idx = np.nonzero(vis)[0]
        f = np.stack([mx, my, dep, A, B, Cc, p64[:, 10], p64[:, 11], p64[:, 12], p64[:, 13]], 1)[idx]
        i =np.stack([scene.gid_base + idx, np.full(len(idx), v), rect[idx, 0], rect[idx, 1],
                      rect[idx, 2], rect[idx, 3]], 1).astype(np.int64)
        fs.append(f)
        is_.append(i)
        vis_.append(np.stack([np.full(len(idx), v), idx], 1))
        cl.append(p64[idx, 14].astype(np.int32))
    return Records(np.ascontiguousarray(np.concatenate(fs)), np.ascontiguousarray(np.concatenate(is_)),
                   np.concatenate(vis_), np.concatenate(cl))


def tile_lists(recs: Records, b0, b1, Wt, Ht):
    """O11 lists for blocks [b0, b1): (offsets[nb+1], entries) with entries = record ids."""
    nb = b1 - b0
    off = np.zeros(nb + 1, np.int64)
    lib().orc_tile_lists(C.c_int64(recs.n), _p(recs.rec_f), _p(recs.rec_i), C.c_int64(b0),
                         C.c_int64(b1), C.c_int32(Wt), C.c_int32(Ht), _p(off), None)
    ent = np.zeros(max(int(off[-1]), 1), np.int64)
    lib().orc_tile_lists(C.c_int64(recs.n), _p(recs.rec_f), _p(recs.rec_i), C.c_int64(b0),
                         C.c_int64(b1), C.c_int32(Wt), C.c_int32(Ht), _p(off), _p(ent))
    return off, ent[: int(off[-1])]


# Decision margins (alpha_eps, t_eps, cond_eps, alpha_abs) of O12's two threshold decisions
# (gs_oracle.c orc_margins_t, DESIGN.md §2 R16): the first-order bound of the renderer's fp32
# exponent with cond_eps = u_r = 2^-24 per operation; alpha_eps = 1e-6 (the fp32 opacity),
# t_eps = 1e-6, alpha_abs = 1e-6 (ex2.approx: 1.44e-7 measured by gs_selftest_ex2, plus the
# opacity and product roundings).
MARGINS = (1e-6, 1e-6, 2.0 ** -24, 1e-6)


def render_fwd(recs, off, ent, b0, b1, W, H, bg=(0, 0, 0), gt=None, b_total=1, margins=MARGINS, max_paths=0):
    """O12/O13 over blocks [b0,b1).  gt: [n_views,H,W,3] uint8 or None.
    Nominal outputs (every decision on its exact side) plus, with max_paths > 0, every
    outcome path of the decisions within the margins of a threshold (path 0 = nominal):
    n_paths [nb,256], flips [nb,256,P] (uint64), path_c [nb,256,P,3], path_T, path_nl,
    path_counts [nb,256,P,4].  flags bit 16 marks a pixel with more than max_paths paths."""
    nb = b1 - b0
    P = int(max_paths)
    o = dict(c=np.zeros((nb, 256, 3)), T=np.zeros((nb, 256)), nlast=np.zeros((nb, 256), np.int32),
             flags=np.zeros((nb, 256), np.int32), counts=np.zeros((nb, 256, 4), np.int64),
             work=np.zeros(nb, np.int64), dl_dc=np.zeros((nb, 256, 3)) if gt is not None else None)
    if P > 0:
        o.update(n_paths=np.zeros((nb, 256), np.int32), flips=np.zeros((nb, 256, P), np.uint64),
                 path_c=np.zeros((nb, 256, P, 3)), path_T=np.zeros((nb, 256, P)),
                 path_nl=np.zeros((nb, 256, P), np.int32), path_counts=np.zeros((nb, 256, P, 4), np.int64))
    loss = C.c_double(0.0)
    bgv = np.asarray(bg, np.float64)
    gtp = np.ascontiguousarray(gt, np.uint8) if gt is not None else None
    ent = np.ascontiguousarray(ent, np.int64) if len(ent) else np.zeros(1, np.int64)
    mg = np.asarray(margins, np.float64)
    lib().orc_render_fwd(C.c_int64(recs.n), _p(recs.rec_f), _p(off), _p(ent), C.c_int64(b0),
                         C.c_int64(b1), C.c_int32(W), C.c_int32(H), _p(bgv), _p(gtp),
                         C.c_int32(b_total), _p(mg),
                         _p(o["c"]), _p(o["T"]),
                         _p(o["nlast"]), _p(o["flags"]), _p(o["counts"]), _p(o["work"]),
                         _p(o["dl_dc"]), C.byref(loss), C.c_int32(P),
                         *([_p(o[k]) for k in ("n_paths", "flips", "path_c", "path_T", "path_nl", "path_counts")]
                           if P > 0 else [None] * 6))
    o["loss"] = loss.value
    o["margins"] = tuple(margins)
    return o


def render_bwd(recs, off, ent, b0, b1, W, H, dl_dc, bg=(0, 0, 0), margins=MARGINS, flips=None):
    """O14/O15: returns grad_rec[n_rec, 9] = dL/d(mx,my,A,B,C,opacity,r,g,b); each pixel follows
    the outcome path flips[nb,256] of render_fwd (None: nominal)."""
    g = np.zeros((recs.n, 9))
    bgv = np.asarray(bg, np.float64)
    ent = np.ascontiguousarray(ent, np.int64) if len(ent) else np.zeros(1, np.int64)
    fl = np.ascontiguousarray(flips, np.uint64) if flips is not None else None
    lib().orc_render_bwd(C.c_int64(recs.n), _p(recs.rec_f), _p(off), _p(ent), C.c_int64(b0),
                         C.c_int64(b1), C.c_int32(W), C.c_int32(H), _p(bgv),
                         _p(np.ascontiguousarray(dl_dc, np.float64)), _p(np.asarray(margins, np.float64)),
                         _p(fl), _p(g))
    return g


def project_bwd(scene, cams, recs: Records, grad_rec):
    """O16 summed over views: returns grad[n, 59] = (pos3, log_scale3, rot4, logit1, sh48)."""
    n, nv = scene.n, len(cams)
    gv = np.zeros((nv, n, 9))
    gv[recs.vi[:, 0], recs.vi[:, 1]] = grad_rec
    out = np.zeros((n, 59))
    cam_arr = (_Cam * nv)(*[_cam(c) for c in cams])
    lib().orc_project_bwd(C.c_int64(n), _p(_f64(scene.pos)), _p(_f64(scene.log_scale)),
                          _p(_f64(scene.rot)), _p(_f64(scene.opac_logit)), _p(_f64(scene.sh)),
                          C.c_int32(nv), cam_arr, _p(gv), _p(out))
    return out


def adam(theta, m, v, g, lr, beta1=0.9, beta2=0.999, eps=1e-15, batch=1, step=1):
    """O17 in place on fp64 copies; returns (theta, m, v)."""
    th, mm, vv = (np.array(a, np.float64, copy=True).reshape(-1) for a in (theta, m, v))
    gg = np.ascontiguousarray(g, np.float64).reshape(-1)
    lib().orc_adam(C.c_int64(th.size), _p(th), _p(mm), _p(vv), _p(gg), C.c_double(lr),
                   C.c_double(beta1), C.c_double(beta2), C.c_double(eps), C.c_int32(batch),
                   C.c_int64(step))
    shp = np.shape(theta)
    return th.reshape(shp), mm.reshape(shp), vv.reshape(shp)


def division_points(et, G):
    """O18 (Algorithm 1): DP[G+1]."""
    et = np.ascontiguousarray(et, np.int64)
    dp = np.zeros(G + 1, np.int64)
    rc = lib().orc_division_points(_p(et) if et.size else None, C.c_int64(et.size), C.c_int32(G), _p(dp))
    if rc != 0:
        raise OverflowError("Algorithm 1 int64 guard")
    return dp


def costs_to_et(mode, dp, cost, npix):
    cost = np.ascontiguousarray(cost, np.int64)
    npix = np.ascontiguousarray(npix, np.int64)
    dp = np.ascontiguousarray(dp, np.int64)
    et = np.zeros_like(cost)
    lib().orc_costs_to_et(C.c_int32(mode), C.c_int64(cost.size), C.c_int32(dp.size - 1), _p(dp),
                          _p(cost), _p(npix), _p(et))
    return et


def next_et(hist, npix, rate_num, rate_den):
    """A9 step 3 (R17): ET of the next batch from history rows (-1: never rendered)."""
    hist = np.ascontiguousarray(hist, np.int64)
    npix = np.ascontiguousarray(npix, np.int64)
    et = np.zeros_like(hist)
    lib().orc_next_et(C.c_int64(hist.size), _p(hist), _p(npix), C.c_int64(int(rate_num)), C.c_int64(int(rate_den)),
                      _p(et))
    return et


def block_npix(W, H):
    """In-image pixels of each block of one W x H view (R18: partial edge blocks)."""
    Wt, Ht = (W + 15) // 16, (H + 15) // 16
    tx, ty = np.arange(Wt * Ht) % Wt, np.arange(Wt * Ht) // Wt
    return (np.minimum(16, W - 16 * tx) * np.minimum(16, H - 16 * ty)).astype(np.int64)


# ------------------------------------------------------------------ whole-step definition

GROUP_SLICES = {"pos": slice(0, 3), "scale": slice(3, 6), "rot": slice(6, 10),
                "opacity": slice(10, 11), "sh_dc": slice(11, 14), "sh_rest": slice(14, 59)}


def flatten_params(scene):
    return np.concatenate([scene.pos, scene.log_scale, scene.rot, scene.opac_logit[:, None],
                           scene.sh.reshape(scene.n, 48)], 1).astype(np.float64)


def render_batch(scene, cams, mode="parity", bg=(0, 0, 0), gt=None, max_paths=0, b0=None, b1=None):
    """Single-partition forward of the whole batch (all views share one image size)."""
    W, H = cams[0].width, cams[0].height
    Wt, Ht = (W + 15) // 16, (H + 15) // 16
    recs = make_records(scene, cams, mode)
    b0 = 0 if b0 is None else b0
    b1 = len(cams) * Wt * Ht if b1 is None else b1
    off, ent = tile_lists(recs, b0, b1, Wt, Ht)
    fwd = render_fwd(recs, off, ent, b0, b1, W, H, bg, gt, len(cams), max_paths=max_paths)
    return recs, off, ent, fwd


def block_to_image(arr, Wt, Ht, W, H, n_views):
    """Stitch block-major [nb,256,...] into [n_views,H,W,...] (test helper)."""
    tail = arr.shape[2:]
    a = arr.reshape(n_views, Ht, Wt, 16, 16, *tail)
    a = np.moveaxis(a, 3, 2).reshape(n_views, Ht * 16, Wt * 16, *tail)
    return a[:, :H, :W]


# ------------------------------------------------------------------ NEXT-1: L1 + D-SSIM

SSIM_LAMBDA = 0.2  # S:301 (the 3DGS default; the paper names both losses but not the mix)


def ssim_loss(img, gt, lam=SSIM_LAMBDA, want_grad=True):
    """One image: (loss, ssim_mean, grad[H,W,3] or None) of (1-lam) L1 + lam (1 - SSIM);
    img, gt float arrays [H,W,3] in [0,1] (gs_oracle.c orc_ssim_loss)."""
    img = np.ascontiguousarray(img, np.float64)
    gt = np.ascontiguousarray(gt, np.float64)
    H, W = img.shape[:2]
    loss, s = C.c_double(0), C.c_double(0)
    grad = np.zeros_like(img) if want_grad else None
    lib().orc_ssim_loss(C.c_int32(W), C.c_int32(H), _p(img), _p(gt), C.c_double(lam), C.byref(loss), C.byref(s),
                        _p(grad))
    return loss.value, s.value, grad


def ssim_loss_batch(imgs, gts, lam=SSIM_LAMBDA):
    """Batch of b images [b,H,W,3]: the step's loss = mean over images (as the L1 of O13
    divided by b), gradient [b,H,W,3] of that mean."""
    b = len(imgs)
    tot, grads = 0.0, []
    for i in range(b):
        l, _, g = ssim_loss(imgs[i], gts[i], lam)
        tot += l / b
        grads.append(g / b)
    return tot, np.stack(grads)
