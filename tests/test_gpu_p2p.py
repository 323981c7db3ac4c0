"""NEXT-3 parity: the peer-memory exchange -- gs_project_put (records written straight into
the destinations' receive buffers), gs_render_bwd_put (gradient sums added straight into the
owners' dL/dsend buffers) and gs_p2p_barrier -- over G virtual ranks of one process on one GPU
(the kernels address the peers' buffers exactly as they address NVLink-mapped ones), against
the copy transport of tests/test_gpu_parity.py (each bucket moved to its rank, ascending source
rank, P:190 / S:474):
  bit-exact  every rank's receive buffer (order and bytes);
  float-add  owners' dL/dsend against the gathered record gradients (only the order of the
             float reductions differs: max |diff| <= 1e-6 * max |g|).
"""
import time

import numpy as np
import pytest
import torch

import synth
from tests.test_gpu_parity import DEV, Run, params_of

L = pytest.importorskip("paper_2406_18533_b200._lib")

pytestmark = pytest.mark.gpu


def _scene(G, seed):
    sc = synth.scene_c0(seed)
    cams = synth.cameras_c0()
    gt = synth.gt_image(seed, cams[0])[None]
    W, H = cams[0].width, cams[0].height
    B = len(cams) * ((W + 15) // 16) * ((H + 15) // 16)
    rng = np.random.default_rng(100 + G)
    dp = np.concatenate([[0], np.sort(rng.integers(0, B + 1, G - 1)), [B]]).astype(np.int64)
    bounds = [sc.n * s // G for s in range(G + 1)]
    return sc, cams, gt, dp, bounds


def _render_put(ctx, recv, n_recv, cams, dp, gt):
    """bin_sort + render_fwd (fused L1 -> dL/dpix) + render_bwd_put on one rank's buffer."""
    r = ctx.rank
    no = int(dp[r + 1] - dp[r])
    rng_ = torch.empty(no + 1, dtype=torch.int32, device=DEV)
    try:
        npairs = L.bin_sort(ctx, recv, n_recv, cams, dp, None, 0, rng_)
    except L.CapacityError as e:
        npairs = e.needed
    srt = torch.empty(max(npairs, 1), dtype=torch.int32, device=DEV)
    L.bin_sort(ctx, recv, n_recv, cams, dp, srt, npairs, rng_)
    T = torch.empty(max(no, 1) * 256, dtype=torch.float32, device=DEV)
    nl = torch.empty(max(no, 1) * 256, dtype=torch.int32, device=DEV)
    rgb = torch.empty(max(no, 1) * 768, dtype=torch.float32, device=DEV)
    dpix = torch.zeros(max(no, 1) * 768, dtype=torch.float32, device=DEV)
    loss = torch.zeros(1, dtype=torch.float64, device=DEV)
    cost = torch.zeros(max(no, 1), dtype=torch.int64, device=DEV)
    L.render_fwd(ctx, recv, srt, rng_, cams, dp, (0, 0, 0), torch.from_numpy(gt).to(DEV), len(cams), rgb, T, nl,
                 dpix, loss, cost, L.COST_WORK, None)
    L.render_bwd_put(ctx, recv, n_recv, srt, rng_, cams, dp, dpix, T, nl, cost, L.COST_WORK, None)
    return rgb


@pytest.mark.parametrize("G,seed", [(2, 0), (3, 1), (4, 2)])
def test_p2p_exchange_equals_copy_transport(G, seed):
    sc, cams, gt, dp, bounds = _scene(G, seed)
    bg = (0, 0, 0)
    # reference: local projection into send buffers, buckets moved by copy, local backward
    owners = [Run(sc.slice(bounds[s], bounds[s + 1]), cams, bg, gt, world=G, rank=s, dp=dp) for s in range(G)]
    C = np.stack([o.send_counts for o in owners])
    recv_ref, drec_ref = [], []
    for r in range(G):
        parts = []
        for s in range(G):
            off = np.concatenate([[0], np.cumsum(owners[s].send_counts)])
            parts.append(owners[s].send[off[r]:off[r + 1]])
        recv = torch.cat(parts)
        recv_ref.append(recv)
        rr = Run(sc.slice(0, 1), cams, bg, gt, world=G, rank=r, dp=dp)
        rr.render(recv if len(recv) else torch.empty((1, L.RECORD_BYTES), dtype=torch.uint8, device=DEV), len(recv))
        drec_ref.append(rr.drec[:len(recv)].clone())
    dsend_ref = [torch.zeros((int(C[s].sum()), 9), dtype=torch.float32, device=DEV) for s in range(G)]
    for r in range(G):
        seg, _, _, own = L.p2p_offsets(C, G, r)
        for s in range(G):
            k = int(seg[s + 1] - seg[s])
            dsend_ref[s][own[s]:own[s] + k] = drec_ref[r][seg[s]:seg[s + 1]]

    # peer-memory path: fresh contexts, buffers attached as each other's peers
    ctxs = [L.Context(0, r, G) for r in range(G)]
    ps = [params_of(sc.slice(bounds[r], bounds[r + 1])) for r in range(G)]
    idx = [torch.empty(L.project_index_bytes(ctxs[r], ps[r].n, len(cams)), dtype=torch.uint8, device=DEV)
           for r in range(G)]
    cnt = np.stack([L.project_count(ctxs[r], ps[r], cams, dp, idx[r]) for r in range(G)])
    np.testing.assert_array_equal(cnt, C)
    n_in = C.sum(0)
    recv = [torch.full((int(n_in[r]) + 7, L.RECORD_BYTES), 0xAB, dtype=torch.uint8, device=DEV) for r in range(G)]
    dsend = [torch.full((int(C[r].sum()) + 1, 9), float("nan"), dtype=torch.float32, device=DEV) for r in range(G)]
    flags = [torch.zeros(G, dtype=torch.int64, device=DEV) for _ in range(G)]
    for r in range(G):
        L.p2p_attach(ctxs[r], [t.data_ptr() for t in recv], [t.shape[0] for t in recv],
                     [t.data_ptr() for t in dsend], [t.shape[0] for t in dsend], [t.data_ptr() for t in flags])
    n_recv = [L.p2p_plan(ctxs[r], C) for r in range(G)]
    assert n_recv == [int(x) for x in n_in]
    for r in range(G):
        L.project_put(ctxs[r], ps[r], cams, dp, idx[r])
    streams = [torch.cuda.Stream() for _ in range(G)]
    torch.cuda.synchronize()
    for r in range(G):  # concurrent on separate streams: every rank's kernel waits for all
        L.p2p_barrier(ctxs[r], streams[r])
    torch.cuda.synchronize()
    for r in range(G):
        L.p2p_status(ctxs[r])
        assert torch.equal(recv[r][:n_recv[r]], recv_ref[r]), r
        assert bool((recv[r][n_recv[r]:] == 0xAB).all())  # nothing written past the plan
    for r in range(G):
        _render_put(ctxs[r], recv[r], n_recv[r], cams, dp, gt)
    torch.cuda.synchronize()
    for r in range(G):
        L.p2p_barrier(ctxs[r], streams[r])
    torch.cuda.synchronize()
    for s in range(G):
        L.p2p_status(ctxs[s])
        n = int(C[s].sum())
        got, want = dsend[s][:n], dsend_ref[s]
        assert torch.isfinite(got).all()  # every row zeroed by project_put, then reduced into
        scale = float(want.abs().max()) if n else 1.0
        assert float((got - want).abs().max()) <= 1e-6 * max(scale, 1e-30), s
        assert torch.isnan(dsend[s][n:]).all()  # untouched past the plan


def test_p2p_barrier_times_out_instead_of_hanging():
    """A rank whose peer never arrives: the kernel gives up after ~4 s and the status says so."""
    G = 2
    ctxs = [L.Context(0, r, G) for r in range(G)]
    flags = [torch.zeros(G, dtype=torch.int64, device=DEV) for _ in range(G)]
    bufs = [torch.zeros(1, L.RECORD_BYTES, dtype=torch.uint8, device=DEV) for _ in range(G)]
    gr = [torch.zeros(1, 9, dtype=torch.float32, device=DEV) for _ in range(G)]
    for c in ctxs:
        L.p2p_attach(c, [b.data_ptr() for b in bufs], [1, 1], [g.data_ptr() for g in gr], [1, 1],
                     [f.data_ptr() for f in flags])
    t0 = time.time()
    L.p2p_barrier(ctxs[0])
    with pytest.raises(L.GSError):
        L.p2p_status(ctxs[0])
    assert time.time() - t0 < 60
    # rank 1 arrives late: its barrier completes at once (rank 0's flag already published)
    L.p2p_barrier(ctxs[1])
    L.p2p_status(ctxs[1])


def test_p2p_plan_capacity_fails_everywhere():
    G = 2
    ctxs = [L.Context(0, r, G) for r in range(G)]
    bufs = [torch.zeros(4, L.RECORD_BYTES, dtype=torch.uint8, device=DEV) for _ in range(G)]
    gr = [torch.zeros(4, 9, dtype=torch.float32, device=DEV) for _ in range(G)]
    fl = [torch.zeros(G, dtype=torch.int64, device=DEV) for _ in range(G)]
    for c in ctxs:
        L.p2p_attach(c, [b.data_ptr() for b in bufs], [4, 3], [g.data_ptr() for g in gr], [4, 4],
                     [f.data_ptr() for f in fl])
    C = np.array([[1, 2], [1, 2]])  # rank 1 receives 4 > 3
    for c in ctxs:
        with pytest.raises(L.CapacityError):
            L.p2p_plan(c, C)


def test_sym_alloc_exports_ipc_handles():
    ctx = L.Context(0, 0, 2)
    p0, h0 = L.sym_alloc(ctx, L.SYM_RECV, 1 << 20)
    p1, h1 = L.sym_alloc(ctx, L.SYM_FLAGS, 64)
    assert p0 and p1 and len(h0) == 64 and len(h1) == 64 and h0 != h1
    p0b, _ = L.sym_alloc(ctx, L.SYM_RECV, 1 << 10)  # no shrink, same buffer
    assert p0b == p0
