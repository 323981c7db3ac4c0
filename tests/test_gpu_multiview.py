"""A7 + A8 at batch size b > 1 ("Gaussian transformation backward ... distributed the
same way as the Gaussian transformation forward"; P:242-253 batching, Eq. 1-2): the fused
transformation backward reads each Gaussian's returned record gradients through the
backward index (per-Gaussian (view, destination) bitmask + per-CTA bucket bases) and sums
the chain rule O16 over the views of the batch.  Checked here through the C ABI:

* a C0-shaped scene seen by b = 4 and b = 8 cameras, Gaussians sharded over G = 1 and 3
  virtual owners and pixels over G ranks by DP cuts inside views, every bucket moved and
  every record gradient returned by the test (the transport), parameter gradients of every
  owner against oracle.project_bwd summed over the views, the oracle's render backward
  following the outcome path each GPU pixel took; b = 8, G = 3 includes Gaussians with more
  than 8 records (several listing rounds of k_bwd_adam, views split across a round);
* the full C2 bench configuration (11.2M Gaussians, 16 views of 4591x3436, G = 1, the
  trainer's own step): 2,000 sampled Gaussians' parameter gradients against the oracle's O16
  from the kernel's record gradients of all their (Gaussian, view) records.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.gsutil import block_major, decode_records, grad_metric, match_paths

L = pytest.importorskip("paper_2406_18533_b200._lib")
pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def cams_multi(b):
    rng = np.random.default_rng(b)
    out = []
    for v in range(b):
        eye = (rng.uniform(-0.25, 0.25), rng.uniform(-0.25, 0.25), rng.uniform(-0.2, 0.2))
        out.append(synth.look_at(eye, (rng.uniform(-0.1, 0.1), rng.uniform(-0.1, 0.1), 4.0), (0, -1, 0),
                                 64, 64, 64, 64, image_id=v))
    return out


def dp_inside_views(b, G, seed):
    """G - 1 cuts at random blocks strictly inside views (so views are split between ranks)."""
    rng = np.random.default_rng(seed)
    B = 16 * b
    cuts = np.sort(rng.choice([k for k in range(1, B) if k % 16 not in (0,)], G - 1, replace=False))
    return np.concatenate([[0], cuts, [B]]).astype(np.int64)


def group_check(pg_k, pg_or, what):
    for name, sl in oracle.GROUP_SLICES.items():
        e_inf, e_2 = grad_metric(pg_k[:, sl], pg_or[:, sl])
        assert e_inf <= 1e-3 and e_2 <= 1e-3, (what, name, e_inf, e_2)


@pytest.mark.parametrize("b,G", [(4, 1), (4, 3), (8, 1), (8, 3)])
def test_param_grads_multiview_virtual_ranks(b, G):
    from tests.test_gpu_parity import Run
    sc = synth.scene_c0(b + G)
    cams = cams_multi(b)
    bg = (0.2, 0.5, 0.8) if G == 3 else (0.0, 0.0, 0.0)
    B = 16 * b
    dp = dp_inside_views(b, G, b * 10 + G) if G > 1 else np.array([0, B], np.int64)
    up = synth.upstream_grad(40 + b, (B, 256, 3)).astype(np.float32)
    # owners: projection of their contiguous gid ranges (one rank per virtual context)
    bounds = [sc.n * s // G for s in range(G + 1)]
    owners = [Run(sc.slice(bounds[s], bounds[s + 1]), cams, bg, None, world=G, rank=s, dp=dp) for s in range(G)]
    send_off = [np.concatenate([[0], np.cumsum(o.send_counts)]) for o in owners]
    # renderers: receive each owner's bucket (ascending source rank), render fwd + bwd
    rr, recv_off = [], []
    for r in range(G):
        parts = [owners[s].send[send_off[s][r]:send_off[s][r + 1]] for s in range(G)]
        recv = torch.cat(parts) if sum(len(p) for p in parts) else torch.empty((1, L.RECORD_BYTES), dtype=torch.uint8,
                                                                               device=DEV)
        n = sum(len(p) for p in parts)
        run = Run(sc.slice(0, 1), cams, bg, None, world=G, rank=r, dp=dp)
        run.render(recv, n, upstream=up[dp[r]:dp[r + 1]])
        rr.append(run)
        recv_off.append(np.concatenate([[0], np.cumsum([len(p) for p in parts])]))
    # reverse transport: owner s's dL/dsend in its send order (destination-major)
    pg_k = []
    hp = L.adam_hparams((1e-3,) * 6, b, 1)
    for s in range(G):
        rows = [rr[d].drec[recv_off[d][s]:recv_off[d][s + 1]] for d in range(G)]
        dsend = torch.cat(rows) if sum(len(x) for x in rows) else torch.zeros((1, 9), device=DEV)
        gbuf = owners[s].p.zeros_like()
        L.adam_step(owners[s].ctx, owners[s].p, None, None, gbuf, cams, dp, dsend, owners[s].idx, hp,
                    L.ADAM_GRAD | L.ADAM_WRITE_GRAD)
        torch.cuda.synchronize()
        pg_k.append(gbuf.to_flat())
    pg_k = np.concatenate(pg_k)
    # oracle: the single-partition definition of the whole batch
    recs = oracle.make_records(sc, cams, "parity")
    off, ent = oracle.tile_lists(recs, 0, B, 4, 4)
    fwd = oracle.render_fwd(recs, off, ent, 0, B, 64, 64, bg, None, b, max_paths=64)
    T = np.concatenate([block_major(x.T, x.no) for x in rr])
    nl = np.concatenate([block_major(x.nl, x.no) for x in rr])
    rgb = np.concatenate([block_major(x.rgb, x.no, 3) for x in rr])
    ok, flips, n_multi, _ = match_paths(fwd, T, nl, rgb)
    assert ok.all(), int((~ok).sum())
    g_or = oracle.render_bwd(recs, off, ent, 0, B, 64, 64, up.astype(np.float64), bg, flips=flips)
    pg_or = oracle.project_bwd(sc, cams, recs, g_or)
    group_check(pg_k, pg_or, (b, G))
    # records per Gaussian (sum over views of its destination count), as the owners sent them
    per_g = np.zeros(sc.n, np.int64)
    for s in range(G):
        d = decode_records(owners[s].send[: owners[s].n_send])
        np.add.at(per_g, d["gid"], 1)
    print("b=%d G=%d: max records per Gaussian %d, Gaussians with > 8: %d, multi-outcome pixels %d" %
          (b, G, per_g.max(), int((per_g > 8).sum()), n_multi))
    assert per_g.max() >= b  # some Gaussian is seen by every view
    if (b, G) == (8, 3):
        assert (per_g > 8).sum() > 0  # several listing rounds of k_bwd_adam (kListCap = 8)


def test_full_c2_param_grads_sampled():
    """The bench configuration through the trainer's step (G = 1, b = 16): the parameter
    gradients the split Adam pass wrote (trainer.g, computed before the update) for 2,000
    sampled Gaussians against the oracle's O16 from the kernel's record gradients."""
    from paper_2406_18533_b200.engine import GrendelTrainer
    sc = synth.scene_rubble(11_200_000)
    pool = synth.cameras_rubble(64)
    cams = [pool[i] for i in synth.batch_schedule(64, 16, 1, 2)[0]]
    W, H = cams[0].width, cams[0].height
    gt = np.stack([synth.gt_image(2, c) for c in cams])
    ctx = L.Context(0, 0, 1)
    p = L.GaussianParams.from_arrays(sc.pos, sc.log_scale, sc.rot, sc.opac_logit, sc.sh, DEV, sc.gid_base)
    tr = GrendelTrainer(ctx, p, W, H, 16, 64, cost_mode=L.COST_WORK, rebalance=False)
    tr.step(cams, torch.from_numpy(gt).to(DEV))
    torch.cuda.synchronize()
    n_send = tr.last["n_send"]
    d = decode_records(tr.send.t[:n_send])
    drec = tr.drec.t[:n_send].cpu().numpy().astype(np.float64)
    # 2,000 Gaussians among those with records, at least half of them seen in several views
    rng = np.random.default_rng(5)
    gids, cnt = np.unique(d["gid"], return_counts=True)
    multi = gids[cnt > 1]
    pick = np.unique(np.concatenate([rng.choice(multi, 1000, replace=False),
                                     rng.choice(gids, 1000, replace=False)]))
    sel = np.isin(d["gid"], pick)
    local = {int(g): k for k, g in enumerate(pick)}
    sub = synth.Scene(sc.pos[pick], sc.log_scale[pick], sc.rot[pick], sc.opac_logit[pick], sc.sh[pick])
    vi = np.stack([d["view"][sel], [local[int(g)] for g in d["gid"][sel]]], 1)
    pg_or = oracle.project_bwd(sub, cams, oracle.Records(None, None, vi, None), drec[sel])
    idx = torch.from_numpy(pick).to(DEV)
    g = tr.g
    pg_k = L.GaussianParams(g.pos_op[idx], g.log_scale[idx], g.rot[idx], g.sh[:, idx]).to_flat()
    print("sampled %d Gaussians, %d records, max views per Gaussian %d" % (len(pick), int(sel.sum()), cnt.max()))
    group_check(pg_k, pg_or, "C2")


def test_fused_adam_equals_split():
    """gs_adam_step with and without a gradient buffer (the fused single kernel and the split
    backward + elementwise pass) make the same update on a multi-view step (b = 4, G = 3)."""
    from tests.test_gpu_parity import Run
    b, G = 4, 3
    sc = synth.scene_c0(11)
    cams = cams_multi(b)
    B = 16 * b
    dp = dp_inside_views(b, G, 77)
    owner = Run(sc, cams, (0, 0, 0), None, world=G, rank=0, dp=dp)
    dsend = torch.from_numpy(synth.upstream_grad(3, (max(owner.n_send, 1), 9)).astype(np.float32) * 1e-3).to(DEV)
    hp = L.adam_hparams((1.6e-4, 2.5e-3, 1.25e-4, 5e-2, 5e-3, 1e-3), b, 2)
    outs = []
    for split in (True, False):
        p = L.GaussianParams(owner.p.pos_op.clone(), owner.p.log_scale.clone(), owner.p.rot.clone(),
                             owner.p.sh.clone())
        m, v = p.zeros_like(), p.zeros_like()
        m.pos_op.fill_(1e-3), v.pos_op.fill_(1e-6)
        g = p.zeros_like() if split else None
        L.adam_step(owner.ctx, p, m, v, g, cams, dp, dsend, owner.idx, hp, L.ADAM_GRAD | L.ADAM_APPLY)
        torch.cuda.synchronize()
        outs.append((p.to_flat(), m.to_flat(), v.to_flat()))
    for a, c in zip(outs[0], outs[1]):
        np.testing.assert_allclose(a, c, rtol=1e-5, atol=1e-7 * max(1.0, np.abs(a).max()))
