"""Test helpers: drive libgs through the binding on one GPU, decode its outputs, and
compare with the oracle.  Nothing here computes any part of the method."""
from __future__ import annotations

import numpy as np

import oracle


RECORD_FLOATS = 16  # include/gs.h GS_RECORD_BYTES / 4
# sqrt(0.5 log2 e): the record's factor is the conic's Cholesky factor times this (gs.h)
L_PRESCALE = 0.84932180028801904272150283410289


def decode_records(rec_u8):
    """[n,64] uint8 tensor -> dict of numpy arrays (mx, my, depth, radius, prescaled factor hi/lo,
    opacity, rgb, qmax, gid, view)."""
    a = rec_u8.reshape(-1).view(dtype=__import__("torch").float32).reshape(-1, RECORD_FLOATS).cpu().numpy()
    meta = a[:, 15].view(np.uint32).astype(np.int64)
    return dict(mx=a[:, 0], my=a[:, 1], depth=a[:, 2], radius=a[:, 3], l11=a[:, 4], l21=a[:, 5], l22=a[:, 6],
                opacity=a[:, 7], rgb=a[:, 8:11], qmax=a[:, 11], l11_lo=a[:, 12], l21_lo=a[:, 13], l22_lo=a[:, 14],
                gid=meta >> 5, view=meta & 31, raw=a)


def conic_of(d):
    """conic (A, B, C) = L L^T from the record's double-float factor (test-side decode)."""
    l11 = (d["l11"].astype(np.float64) + d["l11_lo"]) / L_PRESCALE
    l21 = (d["l21"].astype(np.float64) + d["l21_lo"]) / L_PRESCALE
    l22 = (d["l22"].astype(np.float64) + d["l22_lo"]) / L_PRESCALE
    return np.stack([l11 * l11, l11 * l21, l21 * l21 + l22 * l22], 1)


def match_paths(fwd, T, nl, rgb, tol=1e-4, inside=None):
    """Every pixel of a GPU forward against the oracle's outcome paths (oracle.render_fwd with
    max_paths > 0): a pixel passes when one of its paths has the same n_last and T and colour
    within tol.  Returns (ok [nb,256] bool, flips [nb,256] uint64 of the first matching path
    (0 where none), n_multi = pixels with more than one path, n_overflow).  Pixels outside
    the image (inside False) must match path 0."""
    P = fwd["flips"].shape[2]
    valid = np.arange(P)[None, None, :] < fwd["n_paths"][..., None]
    m = valid & (fwd["path_nl"] == nl[..., None])
    m &= np.abs(fwd["path_T"] - T[..., None]) <= tol
    m &= (np.abs(fwd["path_c"] - rgb[..., None, :]) <= tol).all(-1)
    ok = m.any(-1)
    first = np.argmax(m, -1)
    flips = np.take_along_axis(fwd["flips"], first[..., None], -1)[..., 0]
    flips = np.where(ok, flips, 0).astype(np.uint64)
    n_multi = int((fwd["n_paths"] > 1).sum())
    n_over = int(((fwd["flags"] & 16) != 0).sum())
    return ok, flips, n_multi, n_over


def block_major(arr_flat, n_blocks, ch=None):
    a = arr_flat.cpu().numpy()
    if ch is None:
        return a[: n_blocks * 256].reshape(n_blocks, 256)
    return a[: n_blocks * ch * 256].reshape(n_blocks, ch, 256).transpose(0, 2, 1)


def grad_metric(got, ref):
    """SURVEY #31: per group, max|d| / max|ref| and ||d||_2 / ||ref||_2."""
    d = got - ref
    ninf = np.abs(ref).max() if ref.size else 0.0
    n2 = np.linalg.norm(ref)
    return (np.abs(d).max() / ninf if ninf > 0 else np.abs(d).max(),
            np.linalg.norm(d) / n2 if n2 > 0 else np.linalg.norm(d))


def oracle_rec_index(recs: "oracle.Records"):
    """(gid, view) -> oracle record index."""
    return {(int(g), int(v)): j for j, (g, v) in enumerate(recs.rec_i[:, :2])}
