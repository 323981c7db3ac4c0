"""Test helpers: drive libgs through the binding on one GPU, decode its outputs, and
compare with the oracle.  Nothing here computes any part of the method."""
from __future__ import annotations

import numpy as np

import oracle


def decode_records(rec_u8):
    """[n,48] uint8 tensor -> dict of numpy arrays (mx, my, depth, radius, L, opacity, rgb, gid, view)."""
    a = rec_u8.view(-1).view(dtype=__import__("torch").float32).reshape(-1, 12).cpu().numpy()
    meta = a[:, 11].view(np.uint32).astype(np.int64)
    return dict(mx=a[:, 0], my=a[:, 1], depth=a[:, 2], radius=a[:, 3], l11=a[:, 4], l21=a[:, 5], l22=a[:, 6],
                opacity=a[:, 7], rgb=a[:, 8:11], gid=meta >> 5, view=meta & 31, raw=a)


def conic_of(d):
    """conic (A, B, C) = L L^T from the record's Cholesky factor (test-side decode)."""
    l11, l21, l22 = d["l11"].astype(np.float64), d["l21"].astype(np.float64), d["l22"].astype(np.float64)
    return np.stack([l11 * l11, l11 * l21, l21 * l21 + l22 * l22], 1)


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
