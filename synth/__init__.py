"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no projection, compositing, loss,
gradients, Adam or Algorithm 1).  It only draws inputs: Gaussian parameter
clouds, pinhole cameras and ground-truth images, with the shapes, sizes and
value distributions of the paper's workloads (recipe restated in
DESIGN.md §3).  Random numbers come from numpy's counter-based Philox generator
keyed by (seed, stream, chunk) so that a scene is identical for every rank count
G: rank r can draw exactly its contiguous gid slice ("partitions the
Gaussians ... uniformly").

Parameterisation (the data model of P:92, "x_i, s_i, q_i, alpha_i, sh_i"):
  pos        [N,3] float32   world position x_i
  log_scale  [N,3] float32   s_i = exp(log_scale)
  rot        [N,4] float32   unnormalised quaternion (w, x, y, z)
  opac_logit [N]   float32   alpha_i = sigmoid(logit)
  sh         [N,16,3] float32 degree-3 real-SH coefficients, (l,m)-major, rgb inner
"""
from __future__ import annotations

import dataclasses
import math
import os

import numpy as np

CHUNK = 1 << 20  # gids per Philox chunk (scene independent of G)

# Philox stream ids: one independent stream per drawn quantity.
_S_POS, _S_SCALE, _S_ROT, _S_OPAC, _S_SH, _S_COMP = range(6)


def _rng(seed: int, stream: int, chunk: int) -> np.random.Generator:
    key = np.array([(seed & 0xFFFFFFFF) | (stream << 32), chunk], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


@dataclasses.dataclass
class Scene:
    pos: np.ndarray
    log_scale: np.ndarray
    rot: np.ndarray
    opac_logit: np.ndarray
    sh: np.ndarray
    gid_base: int = 0

    @property
    def n(self) -> int:
        return int(self.pos.shape[0])

    def slice(self, lo: int, hi: int) -> "Scene":
        return Scene(self.pos[lo:hi], self.log_scale[lo:hi], self.rot[lo:hi],
                     self.opac_logit[lo:hi], self.sh[lo:hi], self.gid_base + lo)


@dataclasses.dataclass
class Camera:
    """World->camera rotation R (rows = camera right, down, forward), translation t,
    pinhole intrinsics in pixels, image size and the id of its training image."""
    R: np.ndarray  # (3,3) float32
    t: np.ndarray  # (3,) float32
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    image_id: int = 0


# ----------------------------------------------------------------------------- cameras

def look_at(eye, target, up, fx, fy, width, height, image_id=0, cx=None, cy=None) -> Camera:
    """Look-at convention of SURVEY §8(d): f = normalize(target-eye),
    r = normalize(f x up) (up := +y if degenerate), d = f x r; rows (r, d, f); t = -R eye."""
    eye = np.asarray(eye, np.float64)
    f = np.asarray(target, np.float64) - eye
    f /= np.linalg.norm(f)
    r = np.cross(f, np.asarray(up, np.float64))
    if np.linalg.norm(r) < 1e-6:
        r = np.cross(f, np.array([0.0, 1.0, 0.0]))
    r /= np.linalg.norm(r)
    d = np.cross(f, r)
    R = np.stack([r, d, f]).astype(np.float32)
    t = (-(R.astype(np.float64) @ eye)).astype(np.float32)
    return Camera(R, t, float(fx), float(fy), float(width / 2 if cx is None else cx),
                  float(height / 2 if cy is None else cy), int(width), int(height), int(image_id))


def identity_camera(fx, fy, cx, cy, width, height, image_id=0) -> Camera:
    return Camera(np.eye(3, dtype=np.float32), np.zeros(3, np.float32), float(fx), float(fy),
                  float(cx), float(cy), int(width), int(height), int(image_id))


# ----------------------------------------------------------------------------- helpers

def _quat_z_to(n: np.ndarray, spin: np.ndarray) -> np.ndarray:
    """Quaternion (w,x,y,z) rotating local +z onto unit normal n, composed with a spin
    about local z.  Input drawing only (orientation of flat disks)."""
    z = np.array([0.0, 0.0, 1.0])
    axis = np.cross(np.broadcast_to(z, n.shape), n)
    s = np.linalg.norm(axis, axis=1)
    c = np.clip(n[:, 2], -1.0, 1.0)
    ang = np.arctan2(s, c)
    axis = np.where(s[:, None] > 1e-9, axis / np.maximum(s, 1e-30)[:, None], np.array([1.0, 0.0, 0.0]))
    qa = np.concatenate([np.cos(ang / 2)[:, None], np.sin(ang / 2)[:, None] * axis], axis=1)
    qs = np.stack([np.cos(spin / 2), np.zeros_like(spin), np.zeros_like(spin), np.sin(spin / 2)], 1)
    w1, x1, y1, z1 = qa.T
    w2, x2, y2, z2 = qs.T
    return np.stack([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2,
                     w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2,
                     w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2], 1)


def _surface_attrs(rng, pts, normals, d_loc, n):
    """Shared attribute recipe (SURVEY §8(d) 'Rules shared by C1-C4')."""
    pos = pts + normals * rng.normal(0.0, 0.002, (n, 1))
    ls = np.log(d_loc)[:, None] + rng.normal(0.0, 0.6, (n, 3))
    ls[:, 2] += math.log(0.1)  # flat disks: the local normal axis is thin
    rot = _quat_z_to(normals, rng.uniform(0, 2 * math.pi, n))
    mix = rng.random(n) < 0.8
    op = np.where(mix, rng.normal(4.0, 1.0, n), rng.normal(-2.0, 1.0, n))
    sh = np.empty((n, 16, 3))
    sh[:, 0, :] = rng.normal(0.0, 0.5, (n, 3))
    sh[:, 1:, :] = rng.normal(0.0, 0.05, (n, 15, 3))
    return pos, ls, rot, op, sh


def _finish(pos, ls, rot, op, sh, gid_base) -> Scene:
    return Scene(np.ascontiguousarray(pos, np.float32), np.ascontiguousarray(ls, np.float32),
                 np.ascontiguousarray(rot, np.float32), np.ascontiguousarray(op, np.float32),
                 np.ascontiguousarray(sh, np.float32), gid_base)


def _chunk_job(args):
    kind, seed, n_total, c = args
    g0, g1 = c * CHUNK, min((c + 1) * CHUNK, n_total)
    return _DRAW[kind](_rng(seed, _S_COMP, c), g0, g1, seed, n_total)


def _chunked(kind, seed, n_total, lo, hi) -> Scene:
    """Draw gids [lo, hi) chunk by chunk (each chunk from its own Philox key, so the result
    does not depend on how the range is split); chunks are drawn in parallel processes."""
    c0, c1 = lo // CHUNK, (hi + CHUNK - 1) // CHUNK
    jobs = [(kind, seed, n_total, c) for c in range(c0, c1)]
    if len(jobs) > 1:
        import concurrent.futures as cf
        import multiprocessing as mp
        # spawn, not fork: the caller may hold an initialised CUDA context (GPU tests, bench),
        # which a forked child must not touch
        with cf.ProcessPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1),
                                    mp_context=mp.get_context("spawn")) as ex:
            chunks = list(ex.map(_chunk_job, jobs))
    else:
        chunks = [_chunk_job(j) for j in jobs]
    parts = []
    for c, sc in zip(range(c0, c1), chunks):
        g0 = c * CHUNK
        g1 = g0 + sc.n
        parts.append(sc.slice(max(lo, g0) - g0, min(hi, g1) - g0))
    if not parts:
        z = np.zeros
        return Scene(z((0, 3), np.float32), z((0, 3), np.float32), z((0, 4), np.float32),
                     z((0,), np.float32), z((0, 16, 3), np.float32), lo)
    cat = lambda k: np.concatenate([getattr(p, k) for p in parts])
    return Scene(cat("pos"), cat("log_scale"), cat("rot"), cat("opac_logit"), cat("sh"), lo)


# ----------------------------------------------------------------------------- C0 tiny

def scene_c0(seed=0, n=1000, opaque=False) -> Scene:
    """C0 (exact): x ~ U([-2,2]^2 x [3,5]), log s = log 0.08 + N(0,0.4^2),
    q ~ N(0,I4), logit ~ N(0,2^2) (C0-opaque: N(4,1.5^2)), sh dc N(0,.5^2), rest N(0,.1^2)."""
    rng = _rng(seed, _S_POS, 0)
    pos = np.stack([rng.uniform(-2, 2, n), rng.uniform(-2, 2, n), rng.uniform(3, 5, n)], 1)
    ls = math.log(0.08) + rng.normal(0, 0.4, (n, 3))
    rot = rng.normal(0, 1, (n, 4))
    op = rng.normal(4, 1.5, n) if opaque else rng.normal(0, 2, n)
    sh = np.empty((n, 16, 3))
    sh[:, 0] = rng.normal(0, 0.5, (n, 3))
    sh[:, 1:] = rng.normal(0, 0.1, (n, 15, 3))
    return _finish(pos, ls, rot, op, sh, 0)


def cameras_c0(size=64, f=64.0):
    return [identity_camera(f, f, size / 2, size / 2, size, size, 0)]


# ----------------------------------------------------------------------------- C2 / C3 Rubble-shaped

def _terrain_h(x, y):
    return 0.04 * np.sin(6 * x) * np.cos(5 * y) + 0.02 * np.sin(23 * x + 3) * np.sin(19 * y)


def _terrain_n(x, y):
    hx = 0.24 * np.cos(6 * x) * np.cos(5 * y) + 0.46 * np.cos(23 * x + 3) * np.sin(19 * y)
    hy = -0.20 * np.sin(6 * x) * np.sin(5 * y) + 0.38 * np.sin(23 * x + 3) * np.cos(19 * y)
    n = np.stack([-hx, -hy, np.ones_like(x)], 1)
    return n / np.linalg.norm(n, axis=1, keepdims=True)


def scene_rubble(n_total=11_200_000, seed=2, lo=0, hi=None) -> Scene:
    """C2/C3 Rubble-shaped terrain over [-1,1]^2."""
    return _chunked("rubble", seed, n_total, lo, n_total if hi is None else hi)


def _draw_rubble(rng, g0, g1, seed, n_total):
    n = g1 - g0
    d_loc = math.sqrt(4.0 / n_total)
    x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    pts = np.stack([x, y, _terrain_h(x, y)], 1)
    return _finish(*_surface_attrs(rng, pts, _terrain_n(x, y), np.full(n, d_loc), n), g0)


def cameras_rubble(n_pool=64, seed=2, width=4591, height=3436):
    """Pool of aerial cameras: eye (U(-.5,.5), U(-.5,.5), U(.35,.6)), looking at a ground
    point offset horizontally by U(0,.7)*altitude, up=+z; fx=fy=0.9 W (P:330 4591x3436)."""
    rng = _rng(seed + 100, 0, 0)
    cams = []
    for k in range(n_pool):
        eye = np.array([rng.uniform(-.5, .5), rng.uniform(-.5, .5), rng.uniform(.35, .6)])
        ang, off = rng.uniform(0, 2 * math.pi), rng.uniform(0, .7) * eye[2]
        tgt = np.array([eye[0] + off * math.cos(ang), eye[1] + off * math.sin(ang), 0.0])
        cams.append(look_at(eye, tgt, (0, 0, 1), 0.9 * width, 0.9 * width, width, height, k))
    return cams


# ----------------------------------------------------------------------------- C1 garden-shaped

def scene_garden(n_total=5_000_000, seed=1, lo=0, hi=None) -> Scene:
    """C1: 45% ground disk r=1.6, 40% ellipsoid shell (.35,.35,.28) at (0,0,.3),
    15% background dome r=4."""
    return _chunked("garden", seed, n_total, lo, n_total if hi is None else hi)


def _draw_garden(rng, g0, g1, seed, n_total):
    areas = np.array([math.pi * 1.6 ** 2, 4 * math.pi * 0.33 ** 2, 2 * math.pi * 16.0])
    frac = np.array([0.45, 0.40, 0.15])
    d_comp = np.sqrt(areas / (frac * n_total))
    n = g1 - g0
    comp = np.searchsorted(np.cumsum(frac), rng.random(n), side="right").clip(0, 2)
    pts, nrm = np.zeros((n, 3)), np.zeros((n, 3))
    m = comp == 0
    r, th = 1.6 * np.sqrt(rng.random(m.sum())), rng.uniform(0, 2 * math.pi, m.sum())
    pts[m] = np.stack([r * np.cos(th), r * np.sin(th), np.zeros_like(r)], 1)
    nrm[m] = [0, 0, 1]
    m = comp == 1
    u = rng.normal(size=(m.sum(), 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    ax = np.array([.35, .35, .28])
    pts[m] = u * ax + [0, 0, .3]
    g = u / ax
    nrm[m] = g / np.linalg.norm(g, axis=1, keepdims=True)
    m = comp == 2
    u = rng.normal(size=(m.sum(), 3))
    u[:, 2] = np.abs(u[:, 2])
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    pts[m], nrm[m] = 4.0 * u, -u
    return _finish(*_surface_attrs(rng, pts, nrm, d_comp[comp], n), g0)




def cameras_garden(n_pool=64, seed=1, width=1920, height=1080):
    rng = _rng(seed + 100, 0, 0)
    cams = []
    for k in range(n_pool):
        a = 2 * math.pi * k / n_pool + rng.uniform(0, 0.05)
        eye = (1.3 * math.cos(a), 1.3 * math.sin(a), rng.uniform(.4, .7))
        cams.append(look_at(eye, (0, 0, .25), (0, 0, 1), 1536, 1536, width, height, k))
    return cams


# ----------------------------------------------------------------------------- C4 MatrixCity-shaped

_CITY = np.linspace(-0.95, 0.95, 20)


def _city_heights(seed):
    return _rng(seed, 7, 0).uniform(0.02, 0.12, (20, 20))


def scene_city(n_total=24_000_000, seed=4, lo=0, hi=None) -> Scene:
    """C4: 45% ground [-1,1]^2; 55% on the 5 faces of a 20x20 grid of box buildings
    (half-width .03, heights U(.02,.12))."""
    return _chunked("city", seed, n_total, lo, n_total if hi is None else hi)


def _draw_city(rng, g0, g1, seed, n_total):
    H = _city_heights(seed)
    hw = 0.03
    side = 2 * hw * H  # area of one side face per building
    top = (2 * hw) ** 2
    face_area = np.concatenate([np.repeat(side.reshape(-1, 1), 4, 1), np.full((400, 1), top)], 1)
    fa = face_area.reshape(-1)
    fcum = np.cumsum(fa) / fa.sum()
    d_ground = math.sqrt(4.0 / (0.45 * n_total))
    d_bld = math.sqrt(fa.sum() / (0.55 * n_total))

    n = g1 - g0
    ground = rng.random(n) < 0.45
    pts, nrm = np.zeros((n, 3)), np.zeros((n, 3))
    k = ground.sum()
    pts[ground] = np.stack([rng.uniform(-1, 1, k), rng.uniform(-1, 1, k), np.zeros(k)], 1)
    nrm[ground] = [0, 0, 1]
    m = ~ground
    k = m.sum()
    f = np.searchsorted(fcum, rng.random(k), side="right").clip(0, fa.size - 1)
    b, face = f // 5, f % 5
    bx, by = _CITY[b // 20], _CITY[b % 20]
    h = H.reshape(-1)[b]
    u, v = rng.uniform(-1, 1, k), rng.random(k)
    p = np.zeros((k, 3))
    q = np.zeros((k, 3))
    for fi, (nx, ny) in enumerate([(1, 0), (-1, 0), (0, 1), (0, -1)]):
        s = face == fi
        p[s, 0] = bx[s] + (nx * hw if nx else u[s] * hw)
        p[s, 1] = by[s] + (ny * hw if ny else u[s] * hw)
        p[s, 2] = v[s] * h[s]
        q[s] = [nx, ny, 0]
    s = face == 4
    p[s] = np.stack([bx[s] + u[s] * hw, by[s] + rng.uniform(-1, 1, s.sum()) * hw, h[s]], 1)
    q[s] = [0, 0, 1]
    pts[m], nrm[m] = p, q
    d = np.where(ground, d_ground, d_bld)
    return _finish(*_surface_attrs(rng, pts, nrm, d, n), g0)




def cameras_city(n_pool=128, seed=4, width=1920, height=1080):
    """64 street views (eye height .01 in a street canyon, looking along +-x, +1 deg pitch)
    then 64 aerial (altitude .5, oblique)."""
    rng = _rng(seed + 100, 0, 0)
    cams = []
    gaps = (_CITY[:-1] + _CITY[1:]) / 2
    for k in range(n_pool // 2):
        y = gaps[rng.integers(0, gaps.size)]
        x = rng.uniform(-0.9, 0.9)
        sgn = 1.0 if rng.random() < 0.5 else -1.0
        eye = (x, y, 0.01)
        tgt = (x + sgn, y, 0.01 + math.tan(math.radians(1.0)))
        cams.append(look_at(eye, tgt, (0, 0, 1), 1536, 1536, width, height, k))
    for k in range(n_pool // 2, n_pool):
        eye = np.array([rng.uniform(-.6, .6), rng.uniform(-.6, .6), 0.5])
        ang = rng.uniform(0, 2 * math.pi)
        tgt = (eye[0] + 0.4 * math.cos(ang), eye[1] + 0.4 * math.sin(ang), 0.0)
        cams.append(look_at(eye, tgt, (0, 0, 1), 1536, 1536, width, height, k))
    return cams


# ----------------------------------------------------------------------------- ground truth etc.

def gt_image(seed: int, cam: Camera) -> np.ndarray:
    """8-bit ground truth, i.i.d. uniform (only the sign of the L1 residual matters),
    [H, W, 3] uint8, stream seed+200+image_id."""
    rng = _rng(seed + 200 + cam.image_id, 0, 0)
    return rng.integers(0, 256, (cam.height, cam.width, 3), dtype=np.uint8)


def upstream_grad(seed: int, shape, scale=1.0) -> np.ndarray:
    """Seeded upstream dL/dpixel for render-backward parity (independent of the loss)."""
    return (_rng(seed, 9, 0).normal(0, 1, shape) * scale).astype(np.float32)


def adam_state(seed: int, n: int):
    """Random (grad, m, v) arrays of 60-float rows for the Adam-only parity tests."""
    rng = _rng(seed, 10, 0)
    g = rng.normal(0, 1e-3, (n, 60)).astype(np.float32)
    m = rng.normal(0, 1e-3, (n, 60)).astype(np.float32)
    v = (rng.random((n, 60)) * 1e-6).astype(np.float32)
    return g, m, v


def batch_schedule(n_pool: int, b: int, steps: int, seed: int):
    """Seeded permutation per epoch of the camera pool (P:99 random views, P:242 batching)."""
    out, perm, pos, epoch = [], None, n_pool, 0
    for _ in range(steps):
        batch = []
        while len(batch) < b:
            if pos >= n_pool:
                perm = _rng(seed + 300, 0, epoch).permutation(n_pool)
                pos, epoch = 0, epoch + 1
            batch.append(int(perm[pos]))
            pos += 1
        out.append(batch)
    return out


_DRAW = {"rubble": _draw_rubble, "garden": _draw_garden, "city": _draw_city}

CONFIGS = {
    "C0": dict(n=1000, b=1, size=(64, 64)),
    "C1": dict(n=5_000_000, b=4, size=(1920, 1080)),
    "C2": dict(n=11_200_000, b=16, size=(4591, 3436)),
    "C3": dict(n=40_400_000, b=16, size=(4591, 3436)),
    "C4": dict(n=24_000_000, b=32, size=(1920, 1080)),
}
