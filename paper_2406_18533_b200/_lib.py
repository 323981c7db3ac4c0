"""Thin ctypes binding of libgs (include/gs.h).  Argument marshalling only: every step of
the hot path runs in libgs's CUDA kernels; this module never computes any part of it and has
no fallback -- importing it fails loudly if libgs.so is missing.

Names mirror the C ABI without the ``gs_`` prefix.  Tensors are torch CUDA tensors (the
buffers the caller owns); host arrays are numpy / python ints.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# GS_LIB_VARIANT=<name> loads the in-tree A/B build libgs_<name>.so (tools/build_variant.sh)
LIB_PATH = os.path.join(_HERE, "libgs_%s.so" % os.environ["GS_LIB_VARIANT"] if os.environ.get("GS_LIB_VARIANT")
                        else "libgs.so")

GS_OK, GS_EINVAL, GS_ECAPACITY, GS_ENONFINITE, GS_ECUDA, GS_ENCCL, GS_ENOTSUP = range(7)
COST_MEASURED, COST_WORK, COST_PAPER_AVG = 0, 1, 2
ADAM_GRAD, ADAM_APPLY, ADAM_WRITE_GRAD = 1, 2, 4
RECORD_BYTES = 64
GRAD_FLOATS = 9


class GSError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("libgs status %d: %s" % (status, msg))
        self.status = status


class CapacityError(GSError):
    pass


class Camera(C.Structure):
    _fields_ = [("R", C.c_float * 9), ("t", C.c_float * 3), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("width", C.c_int32), ("height", C.c_int32),
                ("image_id", C.c_int32)]


class Params(C.Structure):
    _fields_ = [("pos_op", C.c_void_p), ("log_scale", C.c_void_p), ("rot", C.c_void_p),
                ("sh", C.c_void_p), ("n", C.c_int64), ("gid_base", C.c_int64)]


class DensifyCfg(C.Structure):
    _fields_ = [("grad_thresh", C.c_float), ("percent_dense", C.c_float), ("scene_extent", C.c_float),
                ("min_opacity", C.c_float), ("max_screen_size", C.c_float)]


class AdamHparams(C.Structure):
    _fields_ = [("lr", C.c_float * 6), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("batch", C.c_int32), ("step", C.c_int64)]


if not os.path.exists(LIB_PATH):
    raise ImportError("libgs.so not built (run __graft_entry__.build() or "
                      "python -m paper_2406_18533_b200.build); there is no CPU fallback")
_lib = C.CDLL(LIB_PATH)

_vp, _i64, _i32, _sz = C.c_void_p, C.c_int64, C.c_int32, C.c_size_t
_P64 = C.POINTER(C.c_int64)
_sig = {
    "gs_version": (C.c_int, []),
    "gs_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "gs_create": (C.c_int, [C.POINTER(_vp), C.c_int, C.c_int, C.c_int, C.c_char_p]),
    "gs_destroy": (None, [_vp]),
    "gs_last_error": (C.c_char_p, [_vp]),
    "gs_launch_count": (C.c_int64, [_vp]),
    "gs_check_finite": (C.c_int, [_vp, C.POINTER(Params), _P64, _vp]),
    "gs_project_index_bytes": (_sz, [_vp, _i64, C.c_int]),
    "gs_project": (C.c_int, [_vp, C.POINTER(Params), C.POINTER(Camera), C.c_int, _P64, _vp, _i64, _P64, _vp, _vp]),
    "gs_exchange": (C.c_int, [_vp, _vp, _P64, _vp, _i64, _P64, _P64, _vp]),
    "gs_bin_sort": (C.c_int, [_vp, _vp, _i64, C.POINTER(Camera), C.c_int, _P64, _vp, _i64, _vp, _P64, _vp]),
    "gs_render_fwd": (C.c_int, [_vp, _vp, _vp, _vp, C.POINTER(Camera), C.c_int, _P64, C.POINTER(C.c_float),
                                _vp, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp, C.c_int, _vp, _vp, _vp]),
    "gs_cull_words": (C.c_int64, [_i64, _i64]),
    "gs_render_bwd": (C.c_int, [_vp, _vp, _i64, _vp, _vp, C.POINTER(Camera), C.c_int, _P64,
                                C.POINTER(C.c_float), _vp, _vp, _vp, _vp, _vp, C.c_int, _vp, _vp, _vp]),
    "gs_exchange_grads": (C.c_int, [_vp, _vp, _P64, _P64, _vp, _vp]),
    "gs_adam_step": (C.c_int, [_vp, C.POINTER(Params), C.POINTER(Params), C.POINTER(Params), C.POINTER(Params),
                               C.POINTER(Camera), C.c_int, _P64, _vp, _vp, C.POINTER(AdamHparams), C.c_int, _vp]),
    "gs_rebalance": (C.c_int, [_vp, _vp, C.POINTER(Camera), C.c_int, _P64, _vp, _i64, C.c_int,
                               C.POINTER(Camera), C.c_int, _P64, _vp]),
    "gs_division_points": (C.c_int, [_P64, _i64, C.c_int, _P64]),
    "gs_rebalance_row": (C.c_int, [_vp, _vp, C.POINTER(Camera), C.c_int, _P64, _vp, _i64, C.c_int,
                                   C.POINTER(Camera), C.c_int, _P64, _vp]),
    "gs_exchange_plan": (C.c_int, [_P64, C.c_int, C.c_int, _P64, _P64]),
    "gs_halo_plan": (C.c_int, [_vp, C.POINTER(Camera), C.c_int, _P64, _P64, _i64, _P64]),
    "gs_halo_exchange": (C.c_int, [_vp, _vp, C.c_int, C.POINTER(Camera), C.c_int, _P64, _vp, _vp, _i64, _P64,
                                   _vp]),
    "gs_ssim_terms": (C.c_int, [_vp, _vp, _vp, _vp, _i64, _vp, C.POINTER(Camera), C.c_int, _P64, C.c_float,
                                C.c_int, _vp, _vp, _vp]),
    "gs_ssim_grad": (C.c_int, [_vp, _vp, _vp, _vp, _i64, _vp, _vp, C.POINTER(Camera), C.c_int, _P64, C.c_float,
                               C.c_int, _vp, _vp]),
    "gs_densify_stats": (C.c_int, [_vp, C.POINTER(Camera), C.c_int, _P64, _i64, _vp, _vp, _vp, C.c_int, _vp, _vp,
                                   _vp, _vp]),
    "gs_densify": (C.c_int, [_vp, C.POINTER(Params), C.POINTER(Params), C.POINTER(Params), _vp, _vp, _vp, _vp,
                             C.POINTER(DensifyCfg), C.POINTER(Params), C.POINTER(Params), C.POINTER(Params), _i64,
                             _P64, _vp]),
    "gs_opacity_reset": (C.c_int, [_vp, C.POINTER(Params), C.POINTER(Params), C.POINTER(Params), C.c_float, _vp]),
    "gs_redistribute_record_bytes": (C.c_int64, []),
    "gs_redistribute_pack": (C.c_int, [_vp, C.POINTER(Params), C.POINTER(Params), C.POINTER(Params), _i64,
                                       C.c_uint64, _vp, _i64, _P64, _vp]),
    "gs_redistribute_unpack": (C.c_int, [_vp, _vp, _i64, C.POINTER(Params), C.POINTER(Params), C.POINTER(Params),
                                         _vp]),
    "gs_redistribute": (C.c_int, [_vp, C.POINTER(Params), C.POINTER(Params), C.POINTER(Params), C.c_uint64, _vp,
                                  _i64, _vp, _i64, C.POINTER(Params), C.POINTER(Params), C.POINTER(Params), _P64,
                                  _P64, _vp]),
    # NEXT-3: peer-memory (NVLink) exchange
    "gs_p2p_offsets": (C.c_int, [_P64, C.c_int, C.c_int, _P64, _P64, _P64, _P64]),
    "gs_sym_alloc": (C.c_int, [_vp, C.c_int, _sz, C.POINTER(_vp), C.c_char_p]),
    "gs_ipc_open": (C.c_int, [_vp, C.c_char_p, C.POINTER(_vp)]),
    "gs_p2p_attach": (C.c_int, [_vp, C.POINTER(_vp), _P64, C.POINTER(_vp), _P64, C.POINTER(_vp)]),
    "gs_p2p_plan": (C.c_int, [_vp, _P64, _P64]),
    "gs_exchange_counts": (C.c_int, [_vp, _P64, _P64, _vp]),
    "gs_project_count": (C.c_int, [_vp, C.POINTER(Params), C.POINTER(Camera), C.c_int, _P64, _P64, _vp, _vp]),
    "gs_project_put": (C.c_int, [_vp, C.POINTER(Params), C.POINTER(Camera), C.c_int, _P64, _vp, _vp]),
    "gs_render_bwd_put": (C.c_int, [_vp, _vp, _i64, _vp, _vp, C.POINTER(Camera), C.c_int, _P64, _vp, _vp, _vp,
                                    _vp, C.c_int, _vp, _vp, _vp]),
    "gs_p2p_barrier": (C.c_int, [_vp, _vp]),
    "gs_p2p_status": (C.c_int, [_vp, _vp]),
    "gs_p2p_attach_counts": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_vp), _i64]),
    "gs_project_put_dev": (C.c_int, [_vp, C.POINTER(Params), C.POINTER(Camera), C.c_int, _P64, _vp, _vp]),
    "gs_p2p_counts": (C.c_int, [_vp, _P64, _P64]),
    "gs_p2p_put_costs": (C.c_int, [_vp, _vp, _P64, _vp]),
    "gs_selftest_ex2": (C.c_int, [_vp, C.c_float, C.c_float, C.POINTER(C.c_double), _vp]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def version() -> int:
    return _lib.gs_version()


def _ptr(t):
    """A torch tensor's device pointer, or a raw device pointer given as an int."""
    if t is None:
        return None
    return C.c_void_p(t) if isinstance(t, int) else C.c_void_p(t.data_ptr())


def _i64arr(vals):
    a = np.ascontiguousarray(np.asarray(vals, dtype=np.int64))
    return a, a.ctypes.data_as(_P64)


def cameras(cams) -> "C.Array":
    """Any objects with R (3x3), t (3), fx, fy, cx, cy, width, height, image_id."""
    arr = (Camera * len(cams))()
    for k, c in enumerate(cams):
        arr[k].R[:] = [float(x) for x in np.asarray(c.R, np.float32).reshape(-1)]
        arr[k].t[:] = [float(x) for x in np.asarray(c.t, np.float32).reshape(-1)]
        arr[k].fx, arr[k].fy, arr[k].cx, arr[k].cy = c.fx, c.fy, c.cx, c.cy
        arr[k].width, arr[k].height = c.width, c.height
        arr[k].image_id = int(getattr(c, "image_id", 0))
    return arr


def _stream(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


class Context:
    """One libgs context per rank (gs_create / gs_destroy)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None):
        self._h = C.c_void_p()
        st = _lib.gs_create(C.byref(self._h), device, rank, world, nccl_id)
        self.device, self.rank, self.world = device, rank, world
        self.has_comm = world > 1 and nccl_id is not None  # NCCL communicator (collective calls)
        if st != GS_OK:
            msg = self.last_error()
            _lib.gs_destroy(self._h)
            self._h = None
            raise GSError(st, msg)

    @property
    def handle(self):
        return self._h

    def launch_count(self) -> int:
        return int(_lib.gs_launch_count(self._h))

    def last_error(self) -> str:
        return (_lib.gs_last_error(self._h) or b"").decode()

    def check(self, st):
        if st == GS_OK:
            return
        cls = CapacityError if st == GS_ECAPACITY else GSError
        raise cls(st, self.last_error())

    def close(self):
        if self._h:
            _lib.gs_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = _lib.gs_nccl_unique_id(buf)
    if st != GS_OK:
        raise GSError(st, "gs_nccl_unique_id")
    return buf.raw


class GaussianParams:
    """Owner-side SoA float4 planes (include/gs.h gs_params) as torch CUDA tensors."""

    def __init__(self, pos_op, log_scale, rot, sh, gid_base=0):
        self.pos_op, self.log_scale, self.rot, self.sh = pos_op, log_scale, rot, sh
        self.gid_base = int(gid_base)

    @property
    def n(self):
        return int(self.pos_op.shape[0])

    def struct(self) -> Params:
        return Params(self.pos_op.data_ptr(), self.log_scale.data_ptr(), self.rot.data_ptr(),
                      self.sh.data_ptr(), self.n, self.gid_base)

    @classmethod
    def empty(cls, n, device, gid_base=0, zero=True):
        import torch
        f = torch.zeros if zero else torch.empty
        return cls(f((n, 4), dtype=torch.float32, device=device), f((n, 4), dtype=torch.float32, device=device),
                   f((n, 4), dtype=torch.float32, device=device), f((12, n, 4), dtype=torch.float32, device=device),
                   gid_base)

    @classmethod
    def from_arrays(cls, pos, log_scale, rot, opac_logit, sh, device, gid_base=0):
        """Pack numpy [N,3],[N,3],[N,4],[N],[N,16,3] into the float4 planes (layout only)."""
        import torch
        n = pos.shape[0]
        po = np.concatenate([pos, opac_logit[:, None]], 1).astype(np.float32)
        ls = np.concatenate([log_scale, np.zeros((n, 1), np.float32)], 1).astype(np.float32)
        shp = np.ascontiguousarray(np.asarray(sh, np.float32).reshape(n, 12, 4).transpose(1, 0, 2))
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(device)
        return cls(t(po), t(ls), t(rot), t(shp), gid_base)

    def to_flat(self) -> np.ndarray:
        """[N, 59] = (pos3, log_scale3, rot4, logit1, sh48), the oracle's gradient order."""
        po = self.pos_op.detach().cpu().numpy()
        ls = self.log_scale.detach().cpu().numpy()
        q = self.rot.detach().cpu().numpy()
        sh = self.sh.detach().cpu().numpy().transpose(1, 0, 2).reshape(self.n, 48)
        return np.concatenate([po[:, :3], ls[:, :3], q, po[:, 3:4], sh], 1)

    def zeros_like(self):
        return GaussianParams.empty(self.n, self.pos_op.device, self.gid_base)


# ----------------------------------------------------------------------------- calls

def check_finite(ctx, params, stream=None):
    bad = C.c_int64(-1)
    ps = params.struct()
    st = _lib.gs_check_finite(ctx.handle, C.byref(ps), C.byref(bad), _stream(stream))
    if st == GS_ENONFINITE:
        return int(bad.value)
    ctx.check(st)
    return -1


def project_index_bytes(ctx, n, n_views):
    return int(_lib.gs_project_index_bytes(ctx.handle, n, n_views))


def project(ctx, params, cams, dp, send_rec, send_cap, bwd_index, stream=None):
    """A1.  Returns send_counts (numpy int64[G]).  Raises CapacityError (counts in .counts)."""
    ca = cameras(cams)
    dpa, dpp = _i64arr(dp)
    cnt, cntp = _i64arr(np.zeros(ctx.world))
    ps = params.struct()
    st = _lib.gs_project(ctx.handle, C.byref(ps), ca, len(cams), dpp, _ptr(send_rec), send_cap, cntp,
                         _ptr(bwd_index), _stream(stream))
    if st == GS_ECAPACITY:
        e = CapacityError(st, ctx.last_error())
        e.counts = cnt.copy()
        raise e
    ctx.check(st)
    return cnt


def exchange(ctx, send_rec, send_counts, recv_rec, recv_cap, stream=None):
    """A2.  Returns (recv_counts int64[G], n_recv)."""
    sc, scp = _i64arr(send_counts)
    rc, rcp = _i64arr(np.zeros(ctx.world))
    nr = C.c_int64(0)
    st = _lib.gs_exchange(ctx.handle, _ptr(send_rec), scp, _ptr(recv_rec), recv_cap, rcp, C.byref(nr),
                          _stream(stream))
    if st == GS_ECAPACITY:
        e = CapacityError(st, ctx.last_error())
        e.needed = int(nr.value)
        raise e
    ctx.check(st)
    return rc, int(nr.value)


def bin_sort(ctx, recv_rec, n_recv, cams, dp, sorted_idx, pair_cap, tile_range, stream=None):
    """A3.  Returns n_pairs."""
    ca = cameras(cams)
    _, dpp = _i64arr(dp)
    npairs = C.c_int64(0)
    st = _lib.gs_bin_sort(ctx.handle, _ptr(recv_rec), n_recv, ca, len(cams), dpp, _ptr(sorted_idx), pair_cap,
                          _ptr(tile_range), C.byref(npairs), _stream(stream))
    if st == GS_ECAPACITY:
        e = CapacityError(st, ctx.last_error())
        e.needed = int(npairs.value)
        raise e
    ctx.check(st)
    return int(npairs.value)


def _bg(bg):
    a = (C.c_float * 3)(*[float(x) for x in (bg if bg is not None else (0, 0, 0))])
    return a


def render_fwd(ctx, recv_rec, sorted_idx, tile_range, cams, dp, bg, gt, b_loss, out_rgb, T_final, n_last,
               dL_dpix, loss_sum, tile_cost, cost_mode, stats, stream=None, cull=None):
    """A4.  cull: optional uint32 device buffer of cull_words() words the forward fills for
    render_bwd on the same lists."""
    ca = cameras(cams)
    _, dpp = _i64arr(dp)
    st = _lib.gs_render_fwd(ctx.handle, _ptr(recv_rec), _ptr(sorted_idx), _ptr(tile_range), ca, len(cams), dpp,
                            _bg(bg), _ptr(gt), int(b_loss), _ptr(out_rgb), _ptr(T_final), _ptr(n_last),
                            _ptr(dL_dpix), _ptr(loss_sum), _ptr(tile_cost), int(cost_mode), _ptr(stats),
                            _ptr(cull), _stream(stream))
    ctx.check(st)


def cull_words(n_pairs, n_owned):
    """Words of render_fwd's cull buffer for lists of n_pairs entries over n_owned blocks."""
    return int(_lib.gs_cull_words(int(n_pairs), int(n_owned)))


def render_bwd(ctx, recv_rec, n_recv, sorted_idx, tile_range, cams, dp, bg, dL_dpix, T_final, n_last,
               dL_drec, tile_cost, cost_mode, stats, stream=None, cull=None):
    """A5.  cull: the buffer render_fwd filled for these lists (None: the cull test runs here)."""
    ca = cameras(cams)
    _, dpp = _i64arr(dp)
    st = _lib.gs_render_bwd(ctx.handle, _ptr(recv_rec), int(n_recv), _ptr(sorted_idx), _ptr(tile_range), ca,
                            len(cams), dpp, _bg(bg), _ptr(dL_dpix), _ptr(T_final), _ptr(n_last), _ptr(dL_drec),
                            _ptr(tile_cost), int(cost_mode), _ptr(stats), _ptr(cull), _stream(stream))
    ctx.check(st)


def halo_plan(ctx, cams, dp):
    """NEXT-1: the rank's halo block ids (ascending numpy int64)."""
    ca = cameras(cams)
    _, dpp = _i64arr(dp)
    n = C.c_int64(0)
    st = _lib.gs_halo_plan(ctx.handle, ca, len(cams), dpp, None, 0, C.byref(n))
    if st == GS_ECAPACITY or (st == GS_OK and n.value > 0):
        ids = np.zeros(n.value, np.int64)
        st = _lib.gs_halo_plan(ctx.handle, ca, len(cams), dpp, ids.ctypes.data_as(_P64), n.value, C.byref(n))
        ctx.check(st)
        return ids
    ctx.check(st)
    return np.zeros(0, np.int64)


def halo_exchange(ctx, data, cams, dp, halo, halo_ids, stream=None):
    """NEXT-1 (collective): data [n_owned, fpb] f32 -> halo [cap, fpb], halo_ids [cap]; returns n_halo."""
    ca = cameras(cams)
    _, dpp = _i64arr(dp)
    n = C.c_int64(0)
    fpb = int(data[0].numel()) if data is not None and data.shape[0] else int(np.prod(halo.shape[1:]))
    cap = 0 if halo is None else min(halo.shape[0], halo_ids.shape[0])
    st = _lib.gs_halo_exchange(ctx.handle, _ptr(data), fpb, ca, len(cams), dpp, _ptr(halo), _ptr(halo_ids),
                               int(cap), C.byref(n), _stream(stream))
    if st == GS_ECAPACITY:
        e = CapacityError(st, ctx.last_error())
        e.needed = int(n.value)
        raise e
    ctx.check(st)
    return int(n.value)


def ssim_terms(ctx, out_rgb, halo_rgb, halo_ids, n_halo, gt, cams, dp, lam, b_loss, maps, loss_sum, stream=None):
    """NEXT-1 pass 1: SSIM statistics, loss share, derivative maps [n_owned, 3, 3, 256]."""
    ca = cameras(cams)
    _, dpp = _i64arr(dp)
    st = _lib.gs_ssim_terms(ctx.handle, _ptr(out_rgb), _ptr(halo_rgb), _ptr(halo_ids), int(n_halo), _ptr(gt), ca,
                            len(cams), dpp, C.c_float(lam), int(b_loss), _ptr(maps), _ptr(loss_sum),
                            _stream(stream))
    ctx.check(st)


def ssim_grad(ctx, maps, halo_maps, halo_ids, n_halo, out_rgb, gt, cams, dp, lam, b_loss, dL_dpix, stream=None):
    """NEXT-1 pass 2: dL/dpix of L1 + D-SSIM over the owned blocks."""
    ca = cameras(cams)
    _, dpp = _i64arr(dp)
    st = _lib.gs_ssim_grad(ctx.handle, _ptr(maps), _ptr(halo_maps), _ptr(halo_ids), int(n_halo), _ptr(out_rgb),
                           _ptr(gt), ca, len(cams), dpp, C.c_float(lam), int(b_loss), _ptr(dL_dpix), _stream(stream))
    ctx.check(st)


def densify_stats(ctx, cams, dp, n, bwd_index, send_rec, dL_dsend, b_loss, accum, denom, max_radius, stream=None):
    """NEXT-2: accumulate the densification statistics of one step (in place)."""
    ca = cameras(cams)
    _, dpp = _i64arr(dp)
    st = _lib.gs_densify_stats(ctx.handle, ca, len(cams), dpp, int(n), _ptr(bwd_index), _ptr(send_rec),
                               _ptr(dL_dsend), int(b_loss), _ptr(accum), _ptr(denom), _ptr(max_radius),
                               _stream(stream))
    ctx.check(st)


def densify_cfg(grad_thresh=0.0002, percent_dense=0.01, scene_extent=1.0, min_opacity=0.005, max_screen_size=0.0):
    return DensifyCfg(grad_thresh, percent_dense, scene_extent, min_opacity, max_screen_size)


def densify(ctx, p, m, v, accum, denom, max_radius, noise, cfg, stream=None, events=None):
    """NEXT-2: one densify-and-prune event; returns (p2, m2, v2, counts[4]) as new buffers.
    (A size query, the output allocation, then the placing call; `events` = (start, end)
    CUDA events recorded around the placing call.)"""
    ps, ms, vs = p.struct(), m.struct(), v.struct()
    counts = np.zeros(4, np.int64)
    e1, e2, e3 = (Params(None, None, None, None, 0, p.gid_base) for _ in range(3))
    st = _lib.gs_densify(ctx.handle, C.byref(ps), C.byref(ms), C.byref(vs), _ptr(accum), _ptr(denom),
                         _ptr(max_radius), _ptr(noise), C.byref(cfg), C.byref(e1), C.byref(e2), C.byref(e3), 0,
                         counts.ctypes.data_as(_P64), _stream(stream))
    if st not in (GS_OK, GS_ECAPACITY):
        ctx.check(st)
    n2 = int(counts[3])
    p2 = GaussianParams.empty(n2, p.pos_op.device, p.gid_base, zero=False)
    m2 = GaussianParams.empty(n2, p.pos_op.device, p.gid_base, zero=False)
    v2 = GaussianParams.empty(n2, p.pos_op.device, p.gid_base, zero=False)
    if n2 == 0:
        return p2, m2, v2, counts
    ps2, ms2, vs2 = p2.struct(), m2.struct(), v2.struct()
    if events is not None:
        events[0].record()
    st = _lib.gs_densify(ctx.handle, C.byref(ps), C.byref(ms), C.byref(vs), _ptr(accum), _ptr(denom),
                         _ptr(max_radius), _ptr(noise), C.byref(cfg), C.byref(ps2), C.byref(ms2), C.byref(vs2),
                         n2, counts.ctypes.data_as(_P64), _stream(stream))
    if events is not None:
        events[1].record()
    ctx.check(st)
    return p2, m2, v2, counts


def opacity_reset(ctx, p, m=None, v=None, max_opacity=0.01, stream=None):
    """NEXT-2: clamp opacities to max_opacity and zero their Adam moments."""
    ps = p.struct()
    ms = m.struct() if m is not None else None
    vs = v.struct() if v is not None else None
    st = _lib.gs_opacity_reset(ctx.handle, C.byref(ps), C.byref(ms) if ms else None, C.byref(vs) if vs else None,
                               C.c_float(max_opacity), _stream(stream))
    ctx.check(st)


def redistribute_record_bytes():
    return int(_lib.gs_redistribute_record_bytes())


def redistribute_pack(ctx, p, m, v, n_total, seed, stream=None):
    """NEXT-2: this rank's (index, p, m, v) records grouped by destination; returns (buf, counts)."""
    import torch
    ps, ms, vs = p.struct(), m.struct(), v.struct()
    counts = np.zeros(ctx.world, np.int64)
    rb = redistribute_record_bytes()
    buf = torch.empty((max(p.n, 1), rb), dtype=torch.uint8, device=p.pos_op.device)
    st = _lib.gs_redistribute_pack(ctx.handle, C.byref(ps), C.byref(ms), C.byref(vs), int(n_total),
                                   C.c_uint64(seed), _ptr(buf), p.n, counts.ctypes.data_as(_P64), _stream(stream))
    ctx.check(st)
    return buf, counts


def redistribute_unpack(ctx, recv_buf, n_recv, gid_base, device, stream=None):
    """NEXT-2: place received records; returns (p, m, v) of the new shard."""
    p2, m2, v2 = (GaussianParams.empty(n_recv, device, gid_base, zero=False) for _ in range(3))
    ps, ms, vs = p2.struct(), m2.struct(), v2.struct()
    st = _lib.gs_redistribute_unpack(ctx.handle, _ptr(recv_buf), int(n_recv), C.byref(ps), C.byref(ms),
                                     C.byref(vs), _stream(stream))
    ctx.check(st)
    return p2, m2, v2


def redistribute(ctx, p, m, v, seed, stream=None):
    """NEXT-2 (collective, world > 1): returns the new (p, m, v) shard (size query, then move)."""
    import torch
    rb = redistribute_record_bytes()
    dev = p.pos_op.device
    ps, ms, vs = p.struct(), m.struct(), v.struct()
    nt, no = C.c_int64(0), C.c_int64(0)
    q = [Params(None, None, None, None, 0, 0) for _ in range(3)]
    st = _lib.gs_redistribute(ctx.handle, C.byref(ps), C.byref(ms), C.byref(vs), C.c_uint64(seed), None, 0, None, 0,
                              *[C.byref(o) for o in q], C.byref(nt), C.byref(no), _stream(stream))
    ctx.check(st)
    n_out = int(no.value)
    sbuf = torch.empty((max(p.n, 1), rb), dtype=torch.uint8, device=dev)
    rbuf = torch.empty((max(n_out, 1), rb), dtype=torch.uint8, device=dev)
    new = [GaussianParams.empty(n_out, dev, 0, zero=False) for _ in range(3)]
    outs = [g.struct() for g in new]
    st = _lib.gs_redistribute(ctx.handle, C.byref(ps), C.byref(ms), C.byref(vs), C.c_uint64(seed), _ptr(sbuf), p.n,
                              _ptr(rbuf), n_out, *[C.byref(o) for o in outs], C.byref(nt), C.byref(no),
                              _stream(stream))
    ctx.check(st)
    for g, o in zip(new, outs):
        g.gid_base = int(o.gid_base)
    return tuple(new)


def exchange_grads(ctx, dL_drec, recv_counts, send_counts, dL_dsend, stream=None):
    """A6."""
    _, rcp = _i64arr(recv_counts)
    _, scp = _i64arr(send_counts)
    ctx.check(_lib.gs_exchange_grads(ctx.handle, _ptr(dL_drec), rcp, scp, _ptr(dL_dsend), _stream(stream)))


def adam_hparams(lr, batch, step, beta1=0.9, beta2=0.999, eps=1e-15) -> AdamHparams:
    h = AdamHparams()
    h.lr[:] = [float(x) for x in lr]
    h.beta1, h.beta2, h.eps, h.batch, h.step = beta1, beta2, eps, int(batch), int(step)
    return h


def adam_step(ctx, p, m, v, g, cams, dp, dL_dsend, bwd_index, hp, flags, stream=None):
    """A7 + A8."""
    ca = cameras(cams) if cams is not None else None
    n_views = len(cams) if cams is not None else 0
    _, dpp = _i64arr(dp if dp is not None else [0])
    st_ = [x.struct() if x is not None else None for x in (p, m, v, g)]
    refs = [C.byref(s) if s is not None else None for s in st_]
    st = _lib.gs_adam_step(ctx.handle, refs[0], refs[1], refs[2], refs[3], ca, n_views, dpp, _ptr(dL_dsend),
                           _ptr(bwd_index), C.byref(hp), int(flags), _stream(stream))
    ctx.check(st)


def rebalance(ctx, owned_tile_cost, cams, dp, history, n_images, cost_mode, next_cams, stream=None):
    """A9.  Returns dp_next (numpy int64[G+1])."""
    ca, na = cameras(cams), cameras(next_cams)
    _, dpp = _i64arr(dp)
    out, outp = _i64arr(np.zeros(ctx.world + 1))
    st = _lib.gs_rebalance(ctx.handle, _ptr(owned_tile_cost), ca, len(cams), dpp, _ptr(history), int(n_images),
                           int(cost_mode), na, len(next_cams), outp, _stream(stream))
    ctx.check(st)
    return out


def rebalance_row(ctx, cost_row, cams, dp, history, n_images, cost_mode, next_cams, stream=None):
    """A9's local part on the whole batch's cost row (no communication; virtual contexts).
    Returns dp_next (numpy int64[G+1])."""
    ca, na = cameras(cams), cameras(next_cams)
    _, dpp = _i64arr(dp)
    out, outp = _i64arr(np.zeros(ctx.world + 1))
    st = _lib.gs_rebalance_row(ctx.handle, _ptr(cost_row), ca, len(cams), dpp, _ptr(history), int(n_images),
                               int(cost_mode), na, len(next_cams), outp, _stream(stream))
    ctx.check(st)
    return out


def division_points(et, G):
    """Algorithm 1 (pure host function of libgs)."""
    a, ap = _i64arr(et)
    out, outp = _i64arr(np.zeros(G + 1))
    st = _lib.gs_division_points(ap if a.size else None, a.size, G, outp)
    if st != GS_OK:
        raise GSError(st, "gs_division_points")
    return out


def exchange_plan(counts, G, rank):
    a, ap = _i64arr(np.asarray(counts).reshape(-1))
    so, sop = _i64arr(np.zeros(G + 1))
    ro, rop = _i64arr(np.zeros(G + 1))
    st = _lib.gs_exchange_plan(ap, G, rank, sop, rop)
    if st != GS_OK:
        raise GSError(st, "gs_exchange_plan")
    return so, ro


# ------------------------------------------------------------------ NEXT-3 peer-memory exchange
SYM_RECV, SYM_DSEND, SYM_FLAGS, SYM_COUNTS, SYM_ROW = 0, 1, 2, 3, 4


def p2p_offsets(counts, G, rank):
    """Pure host plan arithmetic: (recv_seg[G+1], put_base[G], send_off[G+1], owner_off[G])."""
    cm, cmp_ = _i64arr(np.asarray(counts, np.int64).reshape(-1))
    out = [np.zeros(G + 1, np.int64), np.zeros(G, np.int64), np.zeros(G + 1, np.int64), np.zeros(G, np.int64)]
    st = _lib.gs_p2p_offsets(cmp_, G, rank, *[o.ctypes.data_as(_P64) for o in out])
    if st != GS_OK:
        raise GSError(st, "gs_p2p_offsets")
    return tuple(out)


def sym_alloc(ctx, which, nbytes):
    """Context-owned symmetric buffer: (device pointer int, 64-byte IPC handle)."""
    ptr = C.c_void_p()
    h = C.create_string_buffer(64)
    ctx.check(_lib.gs_sym_alloc(ctx.handle, int(which), int(nbytes), C.byref(ptr), h))
    return int(ptr.value), h.raw


def ipc_open(ctx, handle: bytes):
    ptr = C.c_void_p()
    ctx.check(_lib.gs_ipc_open(ctx.handle, handle, C.byref(ptr)))
    return int(ptr.value)


def p2p_attach(ctx, recv_ptrs, recv_caps, dsend_ptrs, dsend_caps, flag_ptrs):
    G = ctx.world
    arr = lambda ps: (C.c_void_p * G)(*[C.c_void_p(int(q)) for q in ps])  # noqa: E731
    _, rcp = rc = _i64arr(recv_caps)
    _, dcp = dc = _i64arr(dsend_caps)
    ctx.check(_lib.gs_p2p_attach(ctx.handle, arr(recv_ptrs), rcp, arr(dsend_ptrs), dcp, arr(flag_ptrs)))
    del rc, dc


def p2p_plan(ctx, counts):
    """Sets the G x G count matrix; returns n_recv.  CapacityError on every rank together."""
    cm, cmp_ = _i64arr(np.asarray(counts, np.int64).reshape(-1))
    nr = C.c_int64(0)
    st = _lib.gs_p2p_plan(ctx.handle, cmp_, C.byref(nr))
    if st == GS_ECAPACITY:
        e = CapacityError(st, ctx.last_error())
        e.needed = int(nr.value)
        raise e
    ctx.check(st)
    return int(nr.value)


def exchange_counts(ctx, send_counts, stream=None):
    """COLLECTIVE: the G x G count matrix (numpy int64 [G, G], row = source)."""
    sc, scp = _i64arr(send_counts)
    out = np.zeros(ctx.world * ctx.world, np.int64)
    ctx.check(_lib.gs_exchange_counts(ctx.handle, scp, out.ctypes.data_as(_P64), _stream(stream)))
    return out.reshape(ctx.world, ctx.world)


def project_count(ctx, params, cams, dp, bwd_index, stream=None):
    """Counting half of A1: send_counts (numpy int64[G])."""
    ca = cameras(cams)
    _, dpp = _i64arr(dp)
    cnt, cntp = _i64arr(np.zeros(ctx.world))
    ps = params.struct()
    ctx.check(_lib.gs_project_count(ctx.handle, C.byref(ps), ca, len(cams), dpp, cntp, _ptr(bwd_index),
                                    _stream(stream)))
    return cnt


def project_put(ctx, params, cams, dp, bwd_index, stream=None):
    """Writing half of A1 fused with A2: records straight into the destinations' buffers."""
    ca = cameras(cams)
    _, dpp = _i64arr(dp)
    ps = params.struct()
    ctx.check(_lib.gs_project_put(ctx.handle, C.byref(ps), ca, len(cams), dpp, _ptr(bwd_index), _stream(stream)))


def render_bwd_put(ctx, recv_rec, n_recv, sorted_idx, tile_range, cams, dp, dL_dpix, T_final, n_last, tile_cost,
                   cost_mode, stats, stream=None, recv_ptr=None, cull=None):
    """A5 fused with A6: gradient sums straight into the owners' dL/dsend buffers."""
    ca = cameras(cams)
    _, dpp = _i64arr(dp)
    rp = C.c_void_p(recv_ptr) if recv_ptr is not None else _ptr(recv_rec)
    ctx.check(_lib.gs_render_bwd_put(ctx.handle, rp, int(n_recv), _ptr(sorted_idx), _ptr(tile_range), ca,
                                     len(cams), dpp, _ptr(dL_dpix), _ptr(T_final), _ptr(n_last), _ptr(tile_cost),
                                     int(cost_mode), _ptr(stats), _ptr(cull), _stream(stream)))


def p2p_barrier(ctx, stream=None):
    ctx.check(_lib.gs_p2p_barrier(ctx.handle, _stream(stream)))


def p2p_status(ctx, stream=None):
    ctx.check(_lib.gs_p2p_status(ctx.handle, _stream(stream)))


def p2p_attach_counts(ctx, cmat_ptrs, row_ptrs, row_cap):
    """The G ranks' count-matrix buffers and cost-row buffers (row_cap int64 each; 0: none)."""
    G = ctx.world
    arr = lambda ps: (C.c_void_p * G)(*[C.c_void_p(int(q)) for q in ps])  # noqa: E731
    ctx.check(_lib.gs_p2p_attach_counts(ctx.handle, arr(cmat_ptrs), arr(row_ptrs) if row_cap else None,
                                        int(row_cap)))


def project_put_dev(ctx, params, cams, dp, bwd_index, stream=None):
    """A1 + A2 fused without a host sync: counts, device-side count exchange, records into the
    destinations' receive buffers (offsets from the device matrix).  Follow with p2p_counts."""
    ca = cameras(cams)
    _, dpp = _i64arr(dp)
    ps = params.struct()
    ctx.check(_lib.gs_project_put_dev(ctx.handle, C.byref(ps), ca, len(cams), dpp, _ptr(bwd_index),
                                      _stream(stream)))


def p2p_counts(ctx):
    """The count matrix of the last project_put_dev (event wait) and the plan it sets:
    (counts numpy int64 [G, G], n_recv).  CapacityError on every rank together."""
    G = ctx.world
    cm = np.zeros(G * G, np.int64)
    nr = C.c_int64(0)
    st = _lib.gs_p2p_counts(ctx.handle, cm.ctypes.data_as(_P64), C.byref(nr))
    if st == GS_ECAPACITY:
        e = CapacityError(st, ctx.last_error())
        e.needed = int(nr.value)
        e.counts = cm.reshape(G, G)
        raise e
    ctx.check(st)
    return cm.reshape(G, G), int(nr.value)


def p2p_put_costs(ctx, owned_cost, dp, stream=None):
    """This rank's owned cost segment into every rank's attached cost row."""
    _, dpp = _i64arr(dp)
    ctx.check(_lib.gs_p2p_put_costs(ctx.handle, _ptr(owned_cost), dpp, _stream(stream)))


def selftest_ex2(ctx, lo, hi, stream=None):
    """Max relative error of the renderer's ex2.approx over every fp32 in [lo, hi] (hi <= 0)."""
    r = C.c_double(0.0)
    ctx.check(_lib.gs_selftest_ex2(ctx.handle, C.c_float(lo), C.c_float(hi), C.byref(r), _stream(stream)))
    return r.value
