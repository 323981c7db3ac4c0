"""Pins of the oracle's decision margins (DESIGN.md §2 R16, gs_oracle.c orc_margins_t).

The oracle enumerates both outcomes of every skip / stop decision whose exact value lies
within the renderer's error bound of its threshold.  These tests check that claim directly:
an independent model of the renderer's documented arithmetic (include/gs.h record format and
the evaluation order R16 states -- written here from that description, sharing nothing with
the CUDA code) is run with every operation's result perturbed by an arbitrary relative error
within u_r = 2^-24 (random, and systematically biased both ways), and every pixel it produces
must be one of the oracle's enumerated outcome paths: n_last exact, T and colour within 1e-4.
A margin that is too narrow for the stated arithmetic fails here.  Scenes: the C0 parity
scenes and records of long thin Gaussians whose means lie far from the tile (the case the
reference-point evaluation exists for)."""
import math

import numpy as np
import pytest

import oracle
import synth

U_R = 2.0 ** -24
K = math.sqrt(0.5 / math.log(2.0))  # sqrt(0.5 log2 e): the record's factor prescale
EX2_ERR = 1.44e-7                    # ex2.approx max relative error (gs_selftest_ex2)


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


class Model:
    """The renderer's arithmetic with each operation's result x replaced by x (1 + d), |d| <= u_r
    (mode 'random': d uniform; '+' / '-': d = +-u_r, the worst alignment of a monotone chain;
    'rn': fp32 round to nearest)."""

    def __init__(self, mode, seed=0):
        self.mode = mode
        self.rng = np.random.default_rng(seed)

    def r(self, x):
        x = np.asarray(x, np.float64)
        if self.mode == "rn":
            return f32(x)
        if self.mode == "+":
            return x * (1 + U_R)
        if self.mode == "-":
            return x * (1 - U_R)
        return x * (1 + self.rng.uniform(-U_R, U_R, x.shape))


def record_fields(cov32, o64):
    """The record's fields from the fp32 covariance and the opacity (gs.h GS_RECORD_BYTES):
    the prescaled Cholesky factor of the conic as hi + lo (each rounded to nearest from fp64),
    the fp32 opacity and qmax = log2(255 o) rounded to nearest."""
    a, b, c = (cov32[:, k].astype(np.float64) for k in range(3))
    det = a * c - b * b
    sc, sd = np.sqrt(c), np.sqrt(det)
    L = np.stack([K * sc / sd, -K * b / (sd * sc), K / sc], 1)
    hi = f32(L)
    lo = f32(L - hi)
    o32 = f32(o64)
    qmax = f32(np.log2(255.0 * o32))
    return hi, lo, o32, qmax


def model_render(rec_f, mxy32, hi, lo, o32, qmax, rgb32, off, ent, b0, b1, W, H, m):
    """Model of k_render_fwd over blocks [b0, b1): per warp half (8x16 px) the exponent terms
    at the half's centre r in fp64 from hi + lo, rounded to fp32; per pixel (ex, ey0) = r - p of
    its first row, u0 = fma(h11, ex, fma(h21, ey0, u_ref)), three row steps u_j = u_{j-1} - 4 h21
    (likewise w), q = fma(u, u, w w); skip iff q > qmax; alpha = min(0.99f, o 2^-q) (ex2 error
    within EX2_ERR); T' = T (1 - alpha), stop if T' < 1e-4; C += alpha T c."""
    Wt = (W + 15) // 16
    nb = b1 - b0
    T_out = np.ones((nb, 256))
    nl_out = np.zeros((nb, 256), np.int32)
    C_out = np.zeros((nb, 256, 3))
    cap = float(np.float32(0.99))
    lane = np.arange(32)
    for kb in range(nb):
        beta = b0 + kb
        tx, ty = beta % Wt, beta // Wt
        L = ent[off[kb]:off[kb + 1]]
        for half in range(2):
            hx0, hy0 = tx * 16 + 8 * half, ty * 16
            rx, ry = hx0 + 3.5, hy0 + 7.5
            col = lane & 7
            y0 = lane >> 3
            ex = rx - (hx0 + col)
            ey0 = ry - (hy0 + y0)
            T = np.ones((32, 4))
            C = np.zeros((32, 4, 3))
            nl = np.zeros((32, 4), np.int32)
            live = np.ones((32, 4), bool)
            px = hx0 + col
            for j in range(4):
                live[:, j] &= (px < W) & (hy0 + y0 + 4 * j < H)
            for pos, e in enumerate(L):
                if not live.any():
                    break
                H64 = hi[e] + lo[e]
                dmx, dmy = mxy32[e, 0] - rx, mxy32[e, 1] - ry
                uref = f32(H64[0] * dmx + H64[1] * dmy)
                wref = f32(H64[2] * dmy)
                h11, h21, h22 = hi[e]
                t = m.r(h21 * ey0 + uref)
                u = m.r(h11 * ex + t)
                w = m.r(h22 * ey0 + wref)
                for j in range(4):
                    if j:
                        u = m.r(u - 4 * h21)
                        w = m.r(w - 4 * h22)
                    q = m.r(u * u + m.r(w * w))
                    comp = live[:, j] & (q <= qmax[e])
                    if not comp.any():
                        continue
                    g = 2.0 ** (-q) * (1 + m.rng.uniform(-EX2_ERR, EX2_ERR, q.shape) if m.mode == "random"
                                       else (1 + EX2_ERR if m.mode == "+" else 1 - EX2_ERR if m.mode == "-" else 1))
                    al = np.minimum(cap, m.r(o32[e] * g))
                    Tn = m.r(T[:, j] * m.r(1 - al))
                    stop = comp & (Tn < 1e-4)
                    live[:, j] &= ~stop
                    go = comp & ~stop
                    C[go, j] += (al[go] * T[go, j])[:, None] * rgb32[e][None, :]
                    T[go, j] = Tn[go]
                    nl[go, j] = pos + 1
            for j in range(4):
                p = (y0 + 4 * j) * 16 + 8 * half + col
                T_out[kb, p] = T[:, j]
                nl_out[kb, p] = nl[:, j]
                C_out[kb, p] = C[:, j]
    return T_out, nl_out, C_out


def check_covered(f, T, nl, C):
    P = f["flips"].shape[2]
    valid = np.arange(P)[None, None, :] < f["n_paths"][..., None]
    m = valid & (f["path_nl"] == nl[..., None]) & (np.abs(f["path_T"] - T[..., None]) <= 1e-4)
    m &= (np.abs(f["path_c"] - C[..., None, :]) <= 1e-4).all(-1)
    ok = m.any(-1)
    assert ok.all(), ("pixels outside the enumerated outcomes", np.argwhere(~ok)[:5].tolist())
    return int((f["n_paths"] > 1).sum())


def c0_case(seed, opaque):
    sc = synth.scene_c0(seed, opaque=opaque)
    cam = synth.cameras_c0()[0]
    recs = oracle.make_records(sc, [cam], "parity")
    mb = oracle.membership(sc, cam)
    idx = np.nonzero(mb["vis"])[0]
    hi, lo, o32, qmax = record_fields(mb["cov"][idx], recs.rec_f[:, 6])
    mxy = np.stack([mb["mx"][idx], mb["my"][idx]], 1).astype(np.float64)
    return recs, mxy, hi, lo, o32, qmax, f32(recs.rec_f[:, 7:10]), 64, 64, 0, 16


def thin_case(seed, n=60):
    """Long thin Gaussians (eigenvalues 0.3 .. 0.6 px^2 and 1e3 .. 3e4 px^2, random angle) whose
    means lie up to 300 px from a 2 x 2-block window, plus round ones; opacities up to 1."""
    rng = np.random.default_rng(seed)
    W = H = 32
    ang = rng.uniform(0, np.pi, n)
    lam1 = rng.uniform(1e3, 3e4, n)
    lam2 = rng.uniform(0.3, 0.6, n)
    round_ = rng.random(n) < 0.3
    lam1[round_] = rng.uniform(2, 30, round_.sum())
    lam2[round_] = lam1[round_] * rng.uniform(0.5, 1, round_.sum())
    cs, sn = np.cos(ang), np.sin(ang)
    a = lam1 * cs * cs + lam2 * sn * sn
    b = (lam1 - lam2) * cs * sn
    c = lam1 * sn * sn + lam2 * cs * cs
    cov32 = f32(np.stack([a, b, c], 1)).astype(np.float32)
    # mean on the long axis through a point of the window, up to 300 px away
    t = rng.uniform(-300, 300, n) * ~round_
    base = rng.uniform(0, 32, (n, 2))
    mxy = f32(base + t[:, None] * np.stack([cs, sn], 1))
    o = np.where(rng.random(n) < 0.3, rng.uniform(0.99, 1.0, n), rng.uniform(0.02, 0.99, n))
    A64, B64, C64 = cov32[:, 0].astype(np.float64), cov32[:, 1].astype(np.float64), cov32[:, 2].astype(np.float64)
    det = A64 * C64 - B64 * B64
    rec_f = np.zeros((n, 10))
    rec_f[:, 0:2] = mxy
    rec_f[:, 2] = rng.permutation(n) + 1.0
    rec_f[:, 3], rec_f[:, 4], rec_f[:, 5] = C64 / det, -B64 / det, A64 / det
    rec_f[:, 6] = o
    rec_f[:, 7:10] = rng.uniform(0, 1, (n, 3))
    rec_i = np.zeros((n, 6), np.int64)
    rec_i[:, 0] = np.arange(n)
    rec_i[:, 2], rec_i[:, 3], rec_i[:, 4], rec_i[:, 5] = 0, 1, 0, 1  # every record in every block
    recs = oracle.Records(rec_f, rec_i, None, None)
    hi, lo, o32, qmax = record_fields(cov32, o)
    return recs, mxy, hi, lo, o32, qmax, f32(rec_f[:, 7:10]), W, H, 0, 4


CASES = {"c0s0": lambda: c0_case(0, False), "c0s1": lambda: c0_case(1, False),
         "c0-opaque": lambda: c0_case(0, True), "thin0": lambda: thin_case(0), "thin1": lambda: thin_case(1)}


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("mode", ["rn", "random", "+", "-"])
def test_perturbed_arithmetic_within_enumerated_outcomes(case, mode):
    recs, mxy, hi, lo, o32, qmax, rgb32, W, H, b0, b1 = CASES[case]()
    Wt, Ht = (W + 15) // 16, (H + 15) // 16
    off, ent = oracle.tile_lists(recs, b0, b1, Wt, Ht)
    f = oracle.render_fwd(recs, off, ent, b0, b1, W, H, max_paths=64)
    T, nl, C = model_render(recs.rec_f, mxy, hi, lo, o32, qmax, rgb32, off, ent, b0, b1, W, H,
                            Model(mode, seed=hash((case, mode)) % 2 ** 32))
    n_multi = check_covered(f, T, nl, C)
    assert n_multi <= 0.02 * T.size


def test_less_accurate_arithmetic_is_caught():
    """The check has teeth: the same model with each operation's error scaled to 128 u_r (a
    renderer far less accurate than the one the margins describe) leaves the enumerated
    outcomes on the C0 scene (at 1x and 8x it stays inside: the margins' headroom)."""
    recs, mxy, hi, lo, o32, qmax, rgb32, W, H, b0, b1 = c0_case(0, False)
    off, ent = oracle.tile_lists(recs, b0, b1, 4, 4)
    f = oracle.render_fwd(recs, off, ent, b0, b1, W, H, max_paths=64)
    global U_R
    saved = U_R
    try:
        U_R = 128 * saved
        T, nl, C = model_render(recs.rec_f, mxy, hi, lo, o32, qmax, rgb32, off, ent, b0, b1, W, H, Model("+", 1))
        with pytest.raises(AssertionError):
            check_covered(f, T, nl, C)
    finally:
        U_R = saved
