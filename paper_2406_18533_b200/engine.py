"""The training-step driver: one Grendel step per call (P:101-115 pipeline, P:190 mixed
parallelism, P:200-226 rebalancing), issuing the libgs C-ABI calls of CS1 in order on one
CUDA stream.  Buffers are torch CUDA tensors owned here and grown on GS_ECAPACITY.
This is the public API ``bench.py`` and the e2e measurement call.
"""
from __future__ import annotations

import math

import os

import numpy as np
import torch

from . import _lib as L

_DEBUG = bool(os.environ.get("GS_BENCH_DEBUG"))

# 3DGS default learning rates ("default hyperparameters from the 3DGS repository";
# values as S:349 lists them): pos, sh_dc, sh_rest, opacity, scale, rot
DEFAULT_LR = (1.6e-4, 2.5e-3, 1.25e-4, 5e-2, 5e-3, 1e-3)


def uniform_dp(B: int, G: int) -> np.ndarray:
    """Cold start: uniform block partition."""
    return np.array([g * B // G for g in range(G + 1)], np.int64)


class _Buf:
    """A growable torch buffer (capacity in elements of `row` shape)."""

    def __init__(self, device, dtype, row=(), cap=0):
        self.device, self.dtype, self.row, self.t, self.cap = device, dtype, tuple(row), None, 0
        if cap:
            self.ensure(cap)

    def ensure(self, n):
        if n > self.cap:
            cap = max(int(n * 1.5) + 1024, 1024)  # counts drift up during training (see gs_slot_get)
            self.t = torch.empty((cap,) + self.row, dtype=self.dtype, device=self.device)
            self.cap = cap
        return self.t


class GrendelTrainer:
    def __init__(self, ctx: L.Context, params: L.GaussianParams, width: int, height: int, n_views: int,
                 n_images: int, lr=DEFAULT_LR, cost_mode=L.COST_MEASURED, bg=(0.0, 0.0, 0.0),
                 rebalance=True, dp=None, device=None, split_adam=True, loss="l1", ssim_lambda=0.2,
                 densify_stats=False, exchange="nccl", count_gather="nccl", sync_free=True):
        self.ctx, self.p = ctx, params
        self.device = device or params.pos_op.device
        self.W, self.H, self.b = width, height, n_views
        self.Wt, self.Ht = (width + 15) // 16, (height + 15) // 16
        self.B = n_views * self.Wt * self.Ht
        self.G, self.rank = ctx.world, ctx.rank
        self.lr, self.cost_mode, self.bg, self.do_rebalance = tuple(lr), cost_mode, tuple(bg), rebalance
        self.beta1, self.beta2 = 0.9, 0.999  # before the Eq. (2) scaling beta^b the kernel applies
        if loss not in ("l1", "ssim"):
            raise ValueError("loss must be 'l1' or 'ssim' (L1 + D-SSIM, NEXT-1)")
        self.loss_kind, self.ssim_lambda = loss, float(ssim_lambda)
        # NEXT-3: "p2p" = the exchanges fused into the producing kernels over peer memory
        # (gs_project_put / gs_render_bwd_put, include/gs.h); "nccl" = grouped send/recv
        if exchange not in ("nccl", "p2p"):
            raise ValueError("exchange must be 'nccl' or 'p2p'")
        self.exchange_kind = exchange if ctx.world > 1 else "nccl"
        if self.exchange_kind == "p2p" and (loss != "l1" or densify_stats or any(bg)):
            raise ValueError("exchange='p2p' supports the L1 loss, black background, no densification statistics")
        self.p2p = None  # (recv_ptr, dsend_ptr, recv_cap, dsend_cap) once attached
        # p2p: the count matrix and the cost row exchanged on the devices (gs_project_put_dev,
        # gs_p2p_put_costs) instead of through the host (count_gather)
        self.sync_free = bool(sync_free)
        # which collective carries the G x G count matrix (G^2 int64): the context's NCCL
        # communicator, or torch.distributed's process group (contexts without one)
        self.count_gather = count_gather
        # NEXT-2: densification statistics (accum, denom, max screen radius) per owned Gaussian
        self.collect_densify = bool(densify_stats)
        self.dstats = self._new_stats(params.n) if densify_stats else None
        self.m, self.v = params.zeros_like(), params.zeros_like()
        # parameter-gradient buffer: gs_adam_step then runs backward and Adam as two passes
        # (faster than the fused single kernel on B200)
        self.g = params.zeros_like() if split_adam else None
        self.dp = uniform_dp(self.B, self.G) if dp is None else np.asarray(dp, np.int64)
        self.history = torch.full((n_images, self.Wt * self.Ht), -1, dtype=torch.int64, device=self.device)
        self.n_images = n_images
        self.step_count = 0
        dev = self.device
        self.bwd_index = torch.empty(L.project_index_bytes(ctx, params.n, n_views), dtype=torch.uint8, device=dev)
        self.send = _Buf(dev, torch.uint8, (L.RECORD_BYTES,))
        self.recv = _Buf(dev, torch.uint8, (L.RECORD_BYTES,))
        self.sorted = _Buf(dev, torch.int32)
        self.range = _Buf(dev, torch.int32)
        self.cull = _Buf(dev, torch.int32)  # the forward's per-entry cull bits, reused by the backward
        self.T = _Buf(dev, torch.float32, (256,))
        self.nl = _Buf(dev, torch.int32, (256,))
        self.dpix = _Buf(dev, torch.float32, (3, 256))
        self.rgb = _Buf(dev, torch.float32, (3, 256))      # rendered owned blocks (D-SSIM loss)
        self.halo = _Buf(dev, torch.float32, (3, 256))     # other ranks' blocks within 10 px
        self.halo_ids = _Buf(dev, torch.int64)
        self.maps = _Buf(dev, torch.float32, (3, 3, 256))  # SSIM derivative maps of owned blocks
        self.halo_maps = _Buf(dev, torch.float32, (3, 3, 256))
        self.cost = _Buf(dev, torch.int64)
        self.drec = _Buf(dev, torch.float32, (L.GRAD_FLOATS,))
        self.dsend = _Buf(dev, torch.float32, (L.GRAD_FLOATS,))
        self.loss = torch.zeros(1, dtype=torch.float64, device=dev)
        self.stats = torch.zeros(8, dtype=torch.int64, device=dev)
        self.last = {}

    def reserve_for(self, batches):
        """Size every growable buffer (and libgs's scratch) for the given camera batches by
        running their projection and binning once (setup, outside any timed region)."""
        saved = self.dp.copy()
        for cams in batches:
            cap = self.send.cap
            while True:
                try:
                    cnt = L.project(self.ctx, self.p, cams, self.dp, self.send.t, cap, self.bwd_index)
                    break
                except L.CapacityError as e:
                    self.send.ensure(int(e.counts.sum()))
                    cap = self.send.cap
            n = int(cnt.sum())
            self.drec.ensure(n), self.dsend.ensure(n), self.recv.ensure(n if self.G > 1 else 0)
            if self.G == 1:
                no = self.n_owned
                self.range.ensure(no + 1)
                while True:
                    try:
                        L.bin_sort(self.ctx, self.send.t, n, cams, self.dp, self.sorted.t, self.sorted.cap,
                                   self.range.t)
                        break
                    except L.CapacityError as e:
                        self.sorted.ensure(e.needed)
        no = self.B  # a rank may own up to every block after rebalancing
        self.T.ensure(no), self.nl.ensure(no), self.dpix.ensure(no), self.cost.ensure(no), self.range.ensure(no + 1)
        if self.loss_kind == "ssim":
            self.rgb.ensure(no), self.maps.ensure(no)
        self.dp = saved
        torch.cuda.synchronize()

    def _new_stats(self, n):
        return tuple(torch.zeros(max(n, 1), dtype=torch.float32, device=self.device) for _ in range(3))

    def densify(self, cfg=None, noise=None, generator=None, events=None):
        """NEXT-2: one densify-and-prune event on this rank's shard (local).  noise:
        N(0,1) draws [n, 2, 3] for split children (drawn here from `generator` if None).
        Replaces the parameters, Adam state and index buffers; returns the counts
        (kept, clones, children, total)."""
        if self.dstats is None:
            raise RuntimeError("construct the trainer with densify_stats=True")
        cfg = cfg if cfg is not None else L.densify_cfg()
        n = self.p.n
        if noise is None:
            noise = torch.randn((n, 2, 3), dtype=torch.float32, device=self.device, generator=generator)
        p2, m2, v2, counts = L.densify(self.ctx, self.p, self.m, self.v, *self.dstats, noise, cfg, events=events)
        if self.G > 1:
            # the shards changed size: the rank's global base is the exclusive prefix of the new
            # sizes (contiguous gid ranges), agreed through torch.distributed
            import torch.distributed as dist
            sizes = [None] * self.G
            dist.all_gather_object(sizes, int(p2.n))
            base = int(sum(sizes[: self.rank]))
            p2.gid_base = m2.gid_base = v2.gid_base = base
        self._replace_shard(p2, m2, v2)
        return counts

    def opacity_reset(self, max_opacity=0.01):
        """NEXT-2: opacity reset."""
        L.opacity_reset(self.ctx, self.p, self.m, self.v, max_opacity)

    def _replace_shard(self, p, m, v):
        self.p, self.m, self.v = p, m, v
        if self.g is not None:
            self.g = p.zeros_like()
        self.bwd_index = torch.empty(L.project_index_bytes(self.ctx, p.n, self.b), dtype=torch.uint8,
                                     device=self.device)
        if self.dstats is not None:
            self.dstats = self._new_stats(p.n)

    def _halo(self, data, buf, cams, dp, st):
        """Other ranks' blocks within the D-SSIM window reach (world > 1; collective).  The
        halo size is known locally (gs_halo_plan, host only), so the buffers are grown before
        the collective call: no rank can fail it alone."""
        if self.G == 1:
            return 0
        need = len(L.halo_plan(self.ctx, cams, dp))
        buf.ensure(need), self.halo_ids.ensure(need)
        return L.halo_exchange(self.ctx, data, cams, dp, buf.t, self.halo_ids.t, st)

    def _p2p_setup(self, recv_cap, dsend_cap):
        """COLLECTIVE (every rank, same capacities): symmetric buffers, IPC handles exchanged
        through torch.distributed, peers opened and attached (NEXT-3)."""
        import torch.distributed as dist
        ctx, G = self.ctx, self.G
        rp, rh = L.sym_alloc(ctx, L.SYM_RECV, recv_cap * L.RECORD_BYTES)
        dp_, dh = L.sym_alloc(ctx, L.SYM_DSEND, dsend_cap * L.GRAD_FLOATS * 4)
        fp, fh = L.sym_alloc(ctx, L.SYM_FLAGS, G * 8)
        # sync-free forward (gs_project_put_dev): the count matrices and the batch cost rows
        cp, ch = L.sym_alloc(ctx, L.SYM_COUNTS, G * G * 8)
        wp, wh = L.sym_alloc(ctx, L.SYM_ROW, self.B * 8)
        allh = [None] * G
        dist.all_gather_object(allh, (rh, dh, fh, ch, wh))
        own = (rp, dp_, fp, cp, wp)
        ptrs = [[own[k] if g == self.rank else L.ipc_open(ctx, allh[g][k]) for g in range(G)] for k in range(5)]
        L.p2p_attach(ctx, ptrs[0], [recv_cap] * G, ptrs[1], [dsend_cap] * G, ptrs[2])
        L.p2p_attach_counts(ctx, ptrs[3], ptrs[4], self.B)
        self.p2p = (rp, dp_, recv_cap, dsend_cap)
        self.p2p_row = wp

    def _p2p_exchange_dev(self, cams, dp, st):
        """A1 + A2 fused without a host round trip between counting and writing: the count
        matrix is exchanged on the devices, the records written at offsets computed from it,
        and the host reads the matrix while they are being written.  On a capacity shortfall
        (every rank sees it together) the buffers grow and the projection runs again."""
        ctx = self.ctx
        if self.p2p is None:
            self._p2p_setup(1 << 16, 1 << 16)
        while True:
            L.project_put_dev(ctx, self.p, cams, dp, self.bwd_index, st)
            L.p2p_barrier(ctx, st)  # records visible to their destinations
            try:
                C, n_recv = L.p2p_counts(ctx)
                break
            except L.CapacityError as e:
                n_in, n_out = e.counts.sum(0), e.counts.sum(1)
                self._p2p_setup(max(int(n_in.max() * 1.25) + 1024, self.p2p[2]),
                                max(int(n_out.max() * 1.25) + 1024, self.p2p[3]))
        return C[self.rank].copy(), C[:, self.rank].copy(), n_recv

    def _p2p_exchange(self, cams, dp, st):
        """A1 + A2 fused: count, all-gather the count matrix, put the records into the
        destinations' receive buffers, barrier.  Returns (send_counts, recv_counts, n_recv)."""
        ctx = self.ctx
        send_counts = L.project_count(ctx, self.p, cams, dp, self.bwd_index, st)
        if self.count_gather == "nccl":
            C = L.exchange_counts(ctx, send_counts, st)
        else:
            import torch.distributed as dist
            rows = [None] * self.G
            dist.all_gather_object(rows, [int(x) for x in send_counts])
            C = np.array(rows, np.int64)
        n_in, n_out = C.sum(0), C.sum(1)
        if self.p2p is None or n_in.max() > self.p2p[2] or n_out.max() > self.p2p[3]:
            self._p2p_setup(int(n_in.max() * 1.25) + 1024, int(n_out.max() * 1.25) + 1024)
        n_recv = L.p2p_plan(ctx, C)
        L.project_put(ctx, self.p, cams, dp, self.bwd_index, st)
        L.p2p_barrier(ctx, st)
        return send_counts, C[:, self.rank].copy(), n_recv

    def _gather_cost_row(self, dp, no):
        """The whole batch's cost row from every rank's owned segment (torch.distributed
        all-gather of equal-size padded segments; what gs_rebalance's NCCL allgatherv does)."""
        import torch.distributed as dist
        seg = int(max(dp[g + 1] - dp[g] for g in range(self.G)))
        mine = torch.zeros(max(seg, 1), dtype=torch.int64, device=self.device)
        mine[:no].copy_(self.cost.t[:no])
        parts = [torch.zeros_like(mine) for _ in range(self.G)]
        if dist.get_backend() == "gloo":  # gloo: host tensors
            mine_h = mine.cpu()
            parts_h = [torch.zeros_like(mine_h) for _ in range(self.G)]
            dist.all_gather(parts_h, mine_h)
            parts = [x.to(self.device) for x in parts_h]
        else:
            dist.all_gather(parts, mine)
        return torch.cat([parts[g][: int(dp[g + 1] - dp[g])] for g in range(self.G)])

    @property
    def n_owned(self):
        return int(self.dp[self.rank + 1] - self.dp[self.rank])

    def step(self, cams, gt, next_cams=None, stream=None, events=None, collect_stats=False):
        """One training step on the batch `cams` (len == n_views) with ground truth `gt`
        (uint8 CUDA tensor [n_views, H, W, 3]).  Returns the loss tensor (device, fp64).
        events: optional dict name -> (start, end) torch.cuda.Event pairs to record per call."""
        ctx, dp, st = self.ctx, self.dp, stream
        ev = events if events is not None else {}

        def rec(name, k):
            if name in ev:
                ev[name][k].record(torch.cuda.current_stream() if st is None else st)

        self.step_count += 1
        p2p = self.exchange_kind == "p2p"
        # A1 project (retry on capacity)
        rec("project", 0)
        cap = self.send.cap
        if p2p and self.sync_free:  # NEXT-3, counts exchanged on the devices
            send_counts, recv_counts, n_recv = self._p2p_exchange_dev(cams, dp, st)
        elif p2p:  # NEXT-3: projection writes straight into the destinations (A1 + A2 fused)
            send_counts, recv_counts, n_recv = self._p2p_exchange(cams, dp, st)
        while not p2p:
            try:
                send_counts = L.project(ctx, self.p, cams, dp, self.send.t, cap, self.bwd_index, st)
                break
            except L.CapacityError as e:
                cap = int(e.counts.sum())
                self.send.ensure(cap)
                cap = self.send.cap
        rec("project", 1)
        n_send = int(send_counts.sum())
        # A2 exchange
        rec("exchange", 0)
        if p2p:
            recv_t = self.p2p[0]
        elif self.G == 1:
            recv_t, recv_counts, n_recv = self.send.t, send_counts.copy(), n_send
        else:
            while True:
                try:
                    recv_counts, n_recv = L.exchange(ctx, self.send.t, send_counts, self.recv.t, self.recv.cap, st)
                    break
                except L.CapacityError as e:
                    self.recv.ensure(e.needed)
            recv_t = self.recv.t
        rec("exchange", 1)
        # A3 bin + sort
        rec("bin_sort", 0)
        no = self.n_owned
        self.range.ensure(no + 1)
        while True:
            try:
                n_pairs = L.bin_sort(ctx, recv_t, n_recv, cams, dp, self.sorted.t, self.sorted.cap,
                                     self.range.t, st)
                break
            except L.CapacityError as e:
                if _DEBUG:
                    print("engine: pair capacity %d < %d, growing" % (self.sorted.cap, e.needed), flush=True)
                self.sorted.ensure(e.needed)
        rec("bin_sort", 1)
        # A4 render forward + fused L1
        self.T.ensure(no), self.nl.ensure(no), self.dpix.ensure(no), self.cost.ensure(no)
        self.cull.ensure(L.cull_words(n_pairs, no))
        self.drec.ensure(n_recv), self.dsend.ensure(n_send)
        self.cost.t[:no].zero_()
        self.loss.zero_()
        stats = None
        if collect_stats:
            self.stats.zero_()
            stats = self.stats
        # PAPER_AVG ("the per-GPU average of measured time"): the rank's render time from
        # CUDA events, spread over its pixels by gs_rebalance; the kernels' counters are unused
        paper_avg = self.cost_mode == L.COST_PAPER_AVG
        cost_t = None if paper_avg else self.cost.t
        if paper_avg:
            self._pa_ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            self._pa_ev[0].record(torch.cuda.current_stream() if st is None else st)
        rec("render_fwd", 0)
        if self.loss_kind == "l1":  # L1 fused into the forward's epilogue (O13)
            L.render_fwd(ctx, recv_t, self.sorted.t, self.range.t, cams, dp, self.bg, gt, self.b, None, self.T.t,
                         self.nl.t, self.dpix.t, self.loss, cost_t, self.cost_mode, stats, st, cull=self.cull.t)
        else:
            self.rgb.ensure(no)
            L.render_fwd(ctx, recv_t, self.sorted.t, self.range.t, cams, dp, self.bg, None, self.b, self.rgb.t,
                         self.T.t, self.nl.t, None, None, cost_t, self.cost_mode, stats, st, cull=self.cull.t)
        rec("render_fwd", 1)
        if self.loss_kind == "ssim":  # NEXT-1: L1 + D-SSIM in two passes around halo exchanges
            rec("loss", 0)
            self.maps.ensure(no)
            n_halo = self._halo(self.rgb.t, self.halo, cams, dp, st)
            L.ssim_terms(ctx, self.rgb.t, self.halo.t, self.halo_ids.t, n_halo, gt, cams, dp, self.ssim_lambda,
                         self.b, self.maps.t, self.loss, st)
            n_halo = self._halo(self.maps.t, self.halo_maps, cams, dp, st)
            L.ssim_grad(ctx, self.maps.t, self.halo_maps.t, self.halo_ids.t, n_halo, self.rgb.t, gt, cams, dp,
                        self.ssim_lambda, self.b, self.dpix.t, st)
            rec("loss", 1)
        # A5 render backward
        rec("render_bwd", 0)
        if p2p:  # A5 + A6 fused: gradient sums reduced straight into the owners' buffers
            L.render_bwd_put(ctx, recv_t, n_recv, self.sorted.t, self.range.t, cams, dp, self.dpix.t, self.T.t,
                             self.nl.t, cost_t, self.cost_mode, stats, st, cull=self.cull.t)
        else:
            L.render_bwd(ctx, recv_t, n_recv, self.sorted.t, self.range.t, cams, dp, self.bg, self.dpix.t,
                         self.T.t, self.nl.t, self.drec.t, cost_t, self.cost_mode, stats, st, cull=self.cull.t)
        rec("render_bwd", 1)
        if paper_avg:
            self._pa_ev[1].record(torch.cuda.current_stream() if st is None else st)
        # A6 reverse exchange
        rec("exchange_grads", 0)
        if p2p:
            # the owned cost segment rides on the same barrier (A9's all-gather, sync-free form)
            row_put = self.sync_free and self.do_rebalance and next_cams is not None and not paper_avg
            if row_put:
                L.p2p_put_costs(ctx, self.cost.t, dp, st)
            L.p2p_barrier(ctx, st)
            dsend = self.p2p[1]
        elif self.G == 1:
            dsend = self.drec.t
        else:
            L.exchange_grads(ctx, self.drec.t, recv_counts, send_counts, self.dsend.t, st)
            dsend = self.dsend.t
        rec("exchange_grads", 1)
        if self.collect_densify:  # NEXT-2 statistics from this step's record gradients
            rec("densify_stats", 0)
            L.densify_stats(ctx, cams, dp, self.p.n, self.bwd_index, self.send.t, dsend, self.b, *self.dstats, st)
            rec("densify_stats", 1)
        # A7 + A8 transformation backward + Adam
        rec("adam", 0)
        hp = L.adam_hparams(self.lr, self.b, self.step_count, self.beta1, self.beta2)
        L.adam_step(ctx, self.p, self.m, self.v, self.g, cams, dp, dsend, self.bwd_index, hp,
                    L.ADAM_GRAD | L.ADAM_APPLY, st)
        rec("adam", 1)
        # A9 rebalance for the next batch
        rec("rebalance", 0)
        # one rank owns every block (DP = [0, B]): there is nothing to balance
        if self.do_rebalance and next_cams is not None and self.G > 1:
            if paper_avg:  # the rank's measured render time (ns) into its first owned block
                self._pa_ev[1].synchronize()
                ns = int(self._pa_ev[0].elapsed_time(self._pa_ev[1]) * 1e6)
                if no:
                    self.cost.t[:no].zero_()
                    self.cost.t[0] = ns
            if p2p and self.sync_free:  # the row is already on this device (p2p_put_costs)
                if paper_avg:
                    L.p2p_put_costs(ctx, self.cost.t, dp, st)
                    L.p2p_barrier(ctx, st)
                self.dp = L.rebalance_row(ctx, self.p2p_row, cams, dp, self.history, self.n_images,
                                          self.cost_mode, next_cams, st)
            elif ctx.has_comm:
                self.dp = L.rebalance(ctx, self.cost.t, cams, dp, self.history, self.n_images, self.cost_mode,
                                      next_cams, st)
            else:  # processes without a communicator (IPC exchange): the row through torch.distributed
                self.dp = L.rebalance_row(ctx, self._gather_cost_row(dp, no), cams, dp, self.history, self.n_images,
                                          self.cost_mode, next_cams, st)
        rec("rebalance", 1)
        self.last = dict(n_send=n_send, n_recv=n_recv, n_pairs=n_pairs, send_counts=send_counts,
                         recv_counts=recv_counts, n_owned=no)
        return self.loss


def make_events(names=("project", "exchange", "bin_sort", "render_fwd", "loss", "render_bwd", "exchange_grads",
                       "densify_stats", "adam", "rebalance")):
    return {n: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for n in names}


def event_ms(events):
    out = {}
    for n, (s, e) in events.items():
        try:
            out[n] = s.elapsed_time(e)
        except (RuntimeError, ValueError):  # not recorded this step (e.g. "loss" with the fused L1)
            pass
    return out


def position_lr(step, lr_init=1.6e-4, lr_final=1.6e-6, max_steps=30000, extent=1.0):
    """Host-side exponential position-lr schedule, log-linear interpolation."""
    t = min(max(step / max(max_steps, 1), 0.0), 1.0)
    return extent * math.exp(math.log(lr_init) * (1 - t) + math.log(lr_final) * t)


class VirtualGrendel:
    """G ranks' pixel partition simulated on one GPU (the load-balancing study, §3.2,
    the paper's Fig. E7 analogue): every rank is a world-G context without a communicator.  One
    owner context projects all Gaussians into G destination buckets (A1 + A2: rank r's receive
    buffer is bucket r of the owner's send buffer), each virtual rank bins and renders its DP
    range (A3-A5, timed separately with CUDA events), the record gradients land in the owner's
    send order (A6: rank r's rows are a slice of dL/dsend), the owner runs A7 + A8, and A9 runs
    Algorithm 1 on the whole batch's cost row (gs_rebalance_row; the row is the ranks' owned
    segments side by side, what gs_rebalance's all-gather assembles).  Per step it returns each
    rank's render fwd + bwd time: imbalance = max / mean over ranks."""

    def __init__(self, params: L.GaussianParams, width: int, height: int, n_views: int, n_images: int, G: int,
                 cost_mode=L.COST_MEASURED, rebalance=True, lr=DEFAULT_LR, device=None):
        self.p, self.G, self.b = params, G, n_views
        self.W, self.H = width, height
        self.Wt, self.Ht = (width + 15) // 16, (height + 15) // 16
        self.B = n_views * self.Wt * self.Ht
        self.cost_mode, self.do_rebalance, self.lr = cost_mode, rebalance, tuple(lr)
        dev = self.device = device or params.pos_op.device
        self.owner = L.Context(dev.index or 0, 0, G)
        self.ranks = [L.Context(dev.index or 0, r, G) for r in range(G)]
        self.dp = uniform_dp(self.B, G)
        self.m, self.v, self.g = params.zeros_like(), params.zeros_like(), params.zeros_like()
        self.history = torch.full((n_images, self.Wt * self.Ht), -1, dtype=torch.int64, device=dev)
        self.n_images = n_images
        self.bwd_index = torch.empty(L.project_index_bytes(self.owner, params.n, n_views), dtype=torch.uint8,
                                     device=dev)
        self.send = _Buf(dev, torch.uint8, (L.RECORD_BYTES,))
        self.dsend = _Buf(dev, torch.float32, (L.GRAD_FLOATS,))
        self.sorted = _Buf(dev, torch.int32)
        self.cull = _Buf(dev, torch.int32)
        self.range = _Buf(dev, torch.int32, (), self.B + 1)
        self.T = _Buf(dev, torch.float32, (256,), self.B)
        self.nl = _Buf(dev, torch.int32, (256,), self.B)
        self.dpix = _Buf(dev, torch.float32, (3, 256), self.B)
        self.row = torch.zeros(self.B, dtype=torch.int64, device=dev)
        self.loss = torch.zeros(1, dtype=torch.float64, device=dev)
        self.step_count = 0

    def step(self, cams, gt, next_cams=None):
        """One step; returns [G] render fwd + bwd milliseconds of each virtual rank."""
        dp = self.dp
        self.step_count += 1
        while True:
            try:
                counts = L.project(self.owner, self.p, cams, dp, self.send.t, self.send.cap, self.bwd_index)
                break
            except L.CapacityError as e:
                self.send.ensure(int(e.counts.sum()))
        off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        self.dsend.ensure(int(off[-1]))
        self.row.zero_()
        self.loss.zero_()
        ms = []
        for r, ctx in enumerate(self.ranks):
            n_recv = int(off[r + 1] - off[r])
            no = int(dp[r + 1] - dp[r])
            recv = self.send.t[off[r]:]
            while True:
                try:
                    n_pairs = L.bin_sort(ctx, recv, n_recv, cams, dp, self.sorted.t, self.sorted.cap, self.range.t)
                    break
                except L.CapacityError as e:
                    self.sorted.ensure(e.needed)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            # PAPER_AVG: the rank's measured render time, spread by gs_rebalance_row over
            # its pixels; the kernels' per-block counters are not used
            cost = None if self.cost_mode == L.COST_PAPER_AVG else (self.row[dp[r]:] if no else self.row)
            self.cull.ensure(L.cull_words(n_pairs, no))
            e0.record()
            L.render_fwd(ctx, recv, self.sorted.t, self.range.t, cams, dp, (0, 0, 0), gt, self.b, None, self.T.t,
                         self.nl.t, self.dpix.t, self.loss, cost, self.cost_mode, None, cull=self.cull.t)
            L.render_bwd(ctx, recv, n_recv, self.sorted.t, self.range.t, cams, dp, (0, 0, 0), self.dpix.t,
                         self.T.t, self.nl.t, self.dsend.t[off[r]:], cost, self.cost_mode, None, cull=self.cull.t)
            e1.record()
            ms.append((e0, e1))
        ms_r = None
        if self.cost_mode == L.COST_PAPER_AVG:
            torch.cuda.synchronize()
            ms_r = np.array([a.elapsed_time(b) for a, b in ms])
            for r in range(self.G):
                if dp[r + 1] > dp[r]:
                    self.row[int(dp[r])] = int(ms_r[r] * 1e6)  # ns
        if any(self.lr):
            hp = L.adam_hparams(self.lr, self.b, self.step_count)
            L.adam_step(self.owner, self.p, self.m, self.v, self.g, cams, dp, self.dsend.t, self.bwd_index, hp,
                        L.ADAM_GRAD | L.ADAM_APPLY)
        if self.do_rebalance and next_cams is not None:
            self.dp = L.rebalance_row(self.owner, self.row, cams, dp, self.history, self.n_images, self.cost_mode,
                                      next_cams)
        torch.cuda.synchronize()
        return ms_r if ms_r is not None else np.array([a.elapsed_time(b) for a, b in ms])
