"""NEXT-1 parity: the fused L1 + D-SSIM kernel (gs_loss_ssim) against the oracle's
orc_ssim_loss (fp64, direct window sums), the halo plan against brute force, and the
partitioned (virtual-rank) evaluation against the single-rank one, bit for bit."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


def _L():
    import paper_2406_18533_b200._lib as L
    return L


def _cams(W, H, b):
    return [synth.identity_camera(64.0, 64.0, W / 2, H / 2, W, H) for _ in range(b)]


def _images(W, H, b, seed):
    rng = np.random.default_rng(seed)
    # smooth-ish rendered images plus noise (SSIM terms away from their flat-region extremes)
    yy, xx = np.mgrid[0:H, 0:W]
    base = 0.5 + 0.3 * np.sin(xx[None, :, :, None] / 7.0 + np.arange(3) + np.arange(b)[:, None, None, None])
    img = np.clip(base + 0.15 * rng.standard_normal((b, H, W, 3)), 0, 1).astype(np.float32)
    gt = np.clip(np.round((img + 0.2 * rng.standard_normal(img.shape)) * 255), 0, 255).astype(np.uint8)
    return img, gt


def _to_blocks(img, Wt, Ht):
    b, H, W, _ = img.shape
    pad = np.zeros((b, Ht * 16, Wt * 16, 3), np.float32)
    pad[:, :H, :W] = img
    blk = pad.reshape(b, Ht, 16, Wt, 16, 3).transpose(0, 1, 3, 5, 2, 4).reshape(b * Ht * Wt, 3, 256)
    return np.ascontiguousarray(blk)


def _from_blocks(blk, Wt, Ht, W, H, b):
    a = blk.reshape(b, Ht, Wt, 3, 16, 16).transpose(0, 1, 4, 2, 5, 3).reshape(b, Ht * 16, Wt * 16, 3)
    return a[:, :H, :W]


def _terms(ctx, rgb_blocks, gt, cams, dp, lam):
    """Pass 1 on rank ctx.rank: halo of rendered blocks taken from rgb_blocks (all blocks)."""
    L = _L()
    r = ctx.rank
    lo, hi = int(dp[r]), int(dp[r + 1])
    ids = L.halo_plan(ctx, cams, dp)
    own = torch.from_numpy(rgb_blocks[lo:hi]).to(DEV)
    halo = torch.from_numpy(np.ascontiguousarray(rgb_blocks[ids])).to(DEV) if len(ids) else None
    hid = torch.from_numpy(ids).to(DEV) if len(ids) else None
    maps = torch.zeros((hi - lo, 3, 3, 256), dtype=torch.float32, device=DEV)
    loss = torch.zeros(1, dtype=torch.float64, device=DEV)
    L.ssim_terms(ctx, own, halo, hid, len(ids), torch.from_numpy(gt).to(DEV), cams, dp, lam, len(cams), maps, loss)
    torch.cuda.synchronize()
    return maps.cpu().numpy(), float(loss.item())


def _grad(ctx, all_maps, rgb_blocks, gt, cams, dp, lam):
    """Pass 2 on rank ctx.rank: halo of maps taken from all_maps (every block's maps)."""
    L = _L()
    r = ctx.rank
    lo, hi = int(dp[r]), int(dp[r + 1])
    ids = L.halo_plan(ctx, cams, dp)
    maps = torch.from_numpy(np.ascontiguousarray(all_maps[lo:hi])).to(DEV)
    hm = torch.from_numpy(np.ascontiguousarray(all_maps[ids])).to(DEV) if len(ids) else None
    hid = torch.from_numpy(ids).to(DEV) if len(ids) else None
    own = torch.from_numpy(rgb_blocks[lo:hi]).to(DEV)
    dpix = torch.zeros((hi - lo, 3, 256), dtype=torch.float32, device=DEV)
    L.ssim_grad(ctx, maps, hm, hid, len(ids), own, torch.from_numpy(gt).to(DEV), cams, dp, lam, len(cams), dpix)
    torch.cuda.synchronize()
    return dpix.cpu().numpy()


def _run_ranks(blocks, gt, cams, dp, lam):
    L = _L()
    G = len(dp) - 1
    ctxs = [L.Context(0, r, G) for r in range(G)]
    res = [_terms(ctxs[r], blocks, gt, cams, dp, lam) for r in range(G)]
    all_maps = np.concatenate([m for m, _ in res])
    dpix = np.concatenate([_grad(ctxs[r], all_maps, blocks, gt, cams, dp, lam) for r in range(G)])
    return dpix, sum(l for _, l in res), all_maps


@pytest.mark.parametrize("W,H,b,lam", [(64, 64, 1, 0.2), (75, 50, 2, 0.2), (150, 97, 1, 1.0), (41, 37, 2, 0.0)])
def test_loss_ssim_matches_oracle(W, H, b, lam):
    L = _L()
    Wt, Ht = (W + 15) // 16, (H + 15) // 16
    img, gt = _images(W, H, b, seed=W + H)
    cams = _cams(W, H, b)
    dp = np.array([0, b * Wt * Ht], np.int64)
    dpix, loss, _ = _run_ranks(_to_blocks(img, Wt, Ht), gt, cams, dp, lam)
    lo, go = oracle.ssim_loss_batch(img.astype(np.float64), gt.astype(np.float64) / 255.0, lam)
    gk = _from_blocks(dpix, Wt, Ht, W, H, b)
    assert abs(loss - lo) <= 2e-6 * abs(lo) + 1e-9, (loss, lo)
    # fp32 window sums against fp64: the SSIM part of the gradient carries ~1e-6 relative
    # error of its scale; the L1 sign part is exact except where |x - y| is at fp32 rounding
    scale = np.abs(go).max()
    err = np.abs(gk - go)
    assert err.max() <= 2e-4 * scale, (err.max(), scale)
    pad = _from_blocks(dpix, Wt, Ht, Wt * 16, Ht * 16, b)
    assert np.all(pad[:, H:] == 0) and np.all(pad[:, :, W:] == 0)  # outside the image


def test_halo_plan_bruteforce():
    L = _L()
    rng = np.random.default_rng(5)
    W, H, b = 100, 70, 3
    Wt, Ht = (W + 15) // 16, (H + 15) // 16
    B = b * Wt * Ht
    cams = _cams(W, H, b)
    for _ in range(20):
        G = int(rng.integers(2, 6))
        cuts = np.sort(rng.choice(np.arange(1, B), G - 1, replace=False))
        dp = np.concatenate([[0], cuts, [B]]).astype(np.int64)
        for r in range(G):
            ctx = L.Context(0, r, G)
            got = L.halo_plan(ctx, cams, dp)
            lo, hi = dp[r], dp[r + 1]
            want = set()
            for beta in range(lo, hi):
                v, l = divmod(beta, Wt * Ht)
                y, x = divmod(l, Wt)
                for dy in (-1, 0, 1):
                    for dx in (-1, 0, 1):
                        nx, ny = x + dx, y + dy
                        if (dx or dy) and 0 <= nx < Wt and 0 <= ny < Ht:
                            nb = v * Wt * Ht + ny * Wt + nx
                            if not lo <= nb < hi:
                                want.add(nb)
            assert list(got) == sorted(want)


def test_partition_equals_single_rank():
    L = _L()
    W, H, b, lam = 90, 70, 2, 0.2
    Wt, Ht = (W + 15) // 16, (H + 15) // 16
    B = b * Wt * Ht
    img, gt = _images(W, H, b, seed=9)
    cams = _cams(W, H, b)
    blocks = _to_blocks(img, Wt, Ht)
    d1, l1, m1 = _run_ranks(blocks, gt, cams, np.array([0, B], np.int64), lam)
    dp = np.array([0, 7, 23, 24, B], np.int64)  # uneven, a one-block rank, a seam inside a row
    d4, l4, m4 = _run_ranks(blocks, gt, cams, dp, lam)
    assert np.array_equal(m4, m1) and np.array_equal(d4, d1)  # same arithmetic per pixel: bitwise
    assert abs(l4 - l1) <= 1e-12 * abs(l1)


def test_trainer_step_with_ssim_loss():
    """GrendelTrainer(loss='ssim') on C0: the step's loss equals the oracle's L1 + D-SSIM of the
    oracle's rendering (up to the renderer's fp32 tolerance), and dL/dpix feeds the backward."""
    L = _L()
    from paper_2406_18533_b200.engine import GrendelTrainer
    sc = synth.scene_c0(0)
    cams = synth.cameras_c0()
    gt = synth.gt_image(0, cams[0])[None]
    p = L.GaussianParams.from_arrays(sc.pos, sc.log_scale, sc.rot, sc.opac_logit, sc.sh, DEV)
    tr = GrendelTrainer(L.Context(0, 0, 1), p, 64, 64, 1, 1, cost_mode=L.COST_WORK, loss="ssim")
    loss = tr.step(cams, torch.from_numpy(gt).to(DEV), next_cams=cams)
    torch.cuda.synchronize()
    _, _, _, fwd = oracle.render_batch(sc, cams, "parity", (0, 0, 0), None)
    img = oracle.block_to_image(fwd["c"], 4, 4, 64, 64, 1)
    lo, _ = oracle.ssim_loss_batch(img, gt.astype(np.float64) / 255.0, 0.2)
    assert abs(loss.item() - lo) <= 1e-4 * lo, (loss.item(), lo)
    assert torch.count_nonzero(tr.drec.t[: tr.last["n_recv"]]) > 0


def test_full_size_c2_view_crops():
    """The loss kernels at the bench's image size (one 4591x3436 C2 view, 61,705 blocks, the
    launch configuration bench.py times), checked on crops the oracle can evaluate exactly:
    dL/dpix at a pixel depends on the image within 10 pixels, so the oracle run on a crop
    grown by 10 pixels (or clipped at a real image border, where both sides zero-pad) is exact
    on the crop.  Crops: the four corners (partial blocks at the right/bottom edges) and
    random interior windows."""
    L = _L()
    W, H, b, lam = 4591, 3436, 1, 0.2
    Wt, Ht = (W + 15) // 16, (H + 15) // 16
    rng = np.random.default_rng(11)
    yy, xx = np.mgrid[0:H, 0:W]
    img = np.clip(0.5 + 0.3 * np.sin(xx / 9.0)[..., None] * np.cos(yy / 13.0)[..., None]
                  + 0.1 * rng.standard_normal((H, W, 3)), 0, 1).astype(np.float32)[None]
    gt = np.clip(np.round((img + 0.15 * rng.standard_normal(img.shape)) * 255), 0, 255).astype(np.uint8)
    cams = _cams(W, H, b)
    dpix, loss, _ = _run_ranks(_to_blocks(img, Wt, Ht), gt, cams, np.array([0, Wt * Ht], np.int64), lam)
    g = _from_blocks(dpix, Wt, Ht, W, H, b)[0]
    crops = [(0, 0), (0, W - 40), (H - 40, 0), (H - 40, W - 40)]
    crops += [(int(rng.integers(10, H - 60)), int(rng.integers(10, W - 60))) for _ in range(4)]
    norm = 3.0 * W * H * b
    for (r0, c0) in crops:
        r1, c1 = r0 + 40, c0 + 40
        R0, C0, R1, C1 = max(r0 - 10, 0), max(c0 - 10, 0), min(r1 + 10, H), min(c1 + 10, W)
        x = img[0, R0:R1, C0:C1].astype(np.float64)
        y = gt[0, R0:R1, C0:C1].astype(np.float64) / 255.0
        _, _, go = oracle.ssim_loss(x, y, lam)
        # the oracle normalises by the crop's pixel count: rescale to the view's
        go = go * (3.0 * x.shape[0] * x.shape[1]) / norm
        want = go[r0 - R0:r1 - R0, c0 - C0:c1 - C0]
        got = g[r0:r1, c0:c1]
        scale = np.abs(want).max()
        assert np.abs(got - want).max() <= 2e-4 * scale, ((r0, c0), np.abs(got - want).max(), scale)
