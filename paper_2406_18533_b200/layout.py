"""Host-side data layout of a rank's Gaussian shard.

Within a shard the Gaussians are stored in Morton (Z-curve) order of their positions.  The
order is a layout choice, not part of the method: every kernel is order-independent except for
the (depth, gid) tie-break, and gid is simply the storage index.  It matters for SIMT
efficiency on B200: a warp's 32 Gaussians are then spatial neighbours, so the projection's
culling, the per-view chain rule of the backward and the record gathers of the renderer are
coherent within a warp, instead of every warp containing some visible Gaussian of every view.
Across ranks the shards stay uniform random subsets (contiguous ranges of a randomly ordered
cloud), which keeps the sparse all-to-all volumes balanced.
"""
from __future__ import annotations

import numpy as np


def _spread3(v: np.ndarray) -> np.ndarray:
    """Insert two zero bits between the 21 low bits of v (uint64)."""
    v = v & np.uint64(0x1FFFFF)
    v = (v | (v << np.uint64(32))) & np.uint64(0x1F00000000FFFF)
    v = (v | (v << np.uint64(16))) & np.uint64(0x1F0000FF0000FF)
    v = (v | (v << np.uint64(8))) & np.uint64(0x100F00F00F00F00F)
    v = (v | (v << np.uint64(4))) & np.uint64(0x10C30C30C30C30C3)
    v = (v | (v << np.uint64(2))) & np.uint64(0x1249249249249249)
    return v


def morton_order(pos: np.ndarray) -> np.ndarray:
    """Permutation sorting points [N,3] along a 63-bit Morton curve of their bounding box."""
    if len(pos) == 0:
        return np.zeros(0, np.int64)
    lo, hi = pos.min(0), pos.max(0)
    scale = (2 ** 21 - 1) / np.maximum(hi - lo, 1e-30)
    q = ((pos - lo) * scale).astype(np.uint64)
    code = _spread3(q[:, 0]) | (_spread3(q[:, 1]) << np.uint64(1)) | (_spread3(q[:, 2]) << np.uint64(2))
    return np.argsort(code, kind="stable")


def reorder_scene(scene):
    """Return the scene (synth.Scene-like) with its Gaussians in Morton order (same gid_base)."""
    perm = morton_order(np.asarray(scene.pos, np.float64))
    return type(scene)(scene.pos[perm], scene.log_scale[perm], scene.rot[perm], scene.opac_logit[perm],
                       scene.sh[perm], scene.gid_base)
