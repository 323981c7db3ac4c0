"""NEXT-2 GPU parity: gs_densify / gs_opacity_reset / gs_densify_stats (through the C ABI)
against oracle/densify.py on the same seeded inputs.  Decisions (which Gaussians are kept,
cloned, split, pruned, and the output order) bit-exact; copied values exact; computed values
(children's positions and log-scales, fp32 vs fp64) within 1e-5 relative."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import densify as D
from tests.gsutil import grad_metric

L = pytest.importorskip("paper_2406_18533_b200._lib")
pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _shard(n, rng):
    ls = np.where(rng.random((n, 1)) < 0.5, -6.0, -3.0) + 0.3 * rng.normal(size=(n, 3))
    return dict(pos=rng.normal(size=(n, 3)).astype(np.float32), log_scale=ls.astype(np.float32),
                rot=rng.normal(size=(n, 4)).astype(np.float32),
                opac_logit=rng.normal(0.0, 3.0, size=n).astype(np.float32),
                sh=rng.normal(size=(n, 48)).astype(np.float32))


def _gp(sh):
    n = len(sh["pos"])
    return L.GaussianParams.from_arrays(sh["pos"], sh["log_scale"], sh["rot"], sh["opac_logit"],
                                        sh["sh"].reshape(n, 16, 3), DEV)


def _flat(d):
    return np.concatenate([d["pos"], d["log_scale"], d["rot"], np.asarray(d["opac_logit"])[:, None], d["sh"]], 1)


@pytest.mark.parametrize("max_screen", [0.0, 12.0])
def test_densify_matches_oracle(max_screen):
    rng = np.random.default_rng(7)
    n = 4000
    sh, m, v = _shard(n, rng), _shard(n, rng), _shard(n, rng)
    accum = rng.exponential(0.0004, n).astype(np.float32)
    denom = rng.integers(0, 4, n).astype(np.float32)
    maxr = rng.integers(0, 30, n).astype(np.float32)
    noise = rng.normal(size=(n, 2, 3)).astype(np.float32)
    cfg = dict(grad_thresh=0.0002, percent_dense=0.01, scene_extent=4.0, min_opacity=0.005,
               max_screen_size=max_screen)
    out, om, ov, cnt = D.densify(sh, m, v, accum, denom, maxr, noise, cfg)
    assert cnt[1] > 0 and cnt[2] > 0 and cnt[0] < n  # every branch exercised
    ctx = L.Context(0, 0, 1)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    p2, m2, v2, kc = L.densify(ctx, _gp(sh), _gp(m), _gp(v), t(accum), t(denom), t(maxr), t(noise),
                               L.densify_cfg(**cfg))
    torch.cuda.synchronize()
    assert tuple(int(x) for x in kc) == cnt
    gk, go = p2.to_flat(), _flat(out)
    n_copy = cnt[0] + cnt[1]
    np.testing.assert_array_equal(gk[:n_copy], go[:n_copy].astype(np.float32))  # copies: exact
    np.testing.assert_array_equal(gk[n_copy:, 6:], go[n_copy:, 6:].astype(np.float32))  # children's rot/opacity/SH
    np.testing.assert_allclose(gk[n_copy:, :6], go[n_copy:, :6], rtol=1e-5, atol=1e-5)
    for k, o in ((m2, om), (v2, ov)):  # Adam state: survivors keep it, new Gaussians start at zero
        np.testing.assert_array_equal(k.to_flat(), _flat(o).astype(np.float32))


def test_opacity_reset_matches_oracle():
    rng = np.random.default_rng(8)
    sh, m, v = _shard(1000, rng), _shard(1000, rng), _shard(1000, rng)
    ctx = L.Context(0, 0, 1)
    p, mg, vg = _gp(sh), _gp(m), _gp(v)
    L.opacity_reset(ctx, p, mg, vg, 0.01)
    torch.cuda.synchronize()
    s2, m2, v2 = D.opacity_reset(sh, m, v, 0.01)
    np.testing.assert_array_equal(p.to_flat(), _flat(s2).astype(np.float32))
    np.testing.assert_array_equal(mg.to_flat(), _flat(m2).astype(np.float32))
    np.testing.assert_array_equal(vg.to_flat(), _flat(v2).astype(np.float32))


def test_stats_match_oracle_backward():
    """gs_densify_stats reads the step's record gradients through the backward index: against
    the oracle's render backward of the same C0 step (each pixel on the outcome path the GPU
    forward took, as in test_param_grads_and_adam)."""
    from tests.test_gpu_parity import Run, matched
    sc = synth.scene_c0(0)
    cams = synth.cameras_c0()
    recs, off, ent, fwd = oracle.render_batch(sc, cams, "parity", (0, 0, 0), None, 64)
    run = Run(sc, cams, (0, 0, 0), None)
    up = synth.upstream_grad(12, (16, 256, 3)).astype(np.float64) * 1e-3
    run.render(run.send, run.n_send, upstream=up.astype(np.float32))
    flips, _ = matched(run, fwd, "c0s0")
    n = sc.n
    acc, den, mr = (torch.zeros(n, dtype=torch.float32, device=DEV) for _ in range(3))
    L.densify_stats(run.ctx, cams, run.dp, n, run.idx, run.send, run.drec, 1, acc, den, mr)
    torch.cuda.synchronize()
    g_or = oracle.render_bwd(recs, off, ent, 0, 16, run.W, run.H, up.astype(np.float32).astype(np.float64),
                             (0, 0, 0), flips=flips)
    mb = oracle.membership(sc, cams[0])
    rad = mb["radius"][recs.vi[:, 1]].astype(np.float64)
    oa, od, orr = D.stats_from_record_grads(n, recs.rec_i[:, 0], g_or, rad, run.W, run.H, 1)
    np.testing.assert_array_equal(den.cpu().numpy(), od.astype(np.float32))
    np.testing.assert_array_equal(mr.cpu().numpy(), orr.astype(np.float32))
    e_inf, e_2 = grad_metric(acc.cpu().numpy()[:, None], oa[:, None])
    assert e_inf <= 1e-3 and e_2 <= 1e-3, (e_inf, e_2)


def test_redistribution_virtual_ranks_match_oracle():
    """gs_redistribute_pack / _unpack on virtual ranks (the test moves the records between
    them, as NCCL does in gs_redistribute): new shards bit-identical to the oracle's."""
    rng = np.random.default_rng(9)
    sizes = [1500, 200, 3100]
    G, N = len(sizes), sum(sizes)
    shards = [_shard(n, rng) for n in sizes]
    ms = [_shard(n, rng) for n in sizes]
    vs = [_shard(n, rng) for n in sizes]
    seed = 424242
    bases = np.concatenate([[0], np.cumsum(sizes)])
    packed = []
    for r in range(G):
        ctx = L.Context(0, r, G)
        p, m, v = _gp(shards[r]), _gp(ms[r]), _gp(vs[r])
        for g in (p, m, v):
            g.gid_base = int(bases[r])
        buf, counts = L.redistribute_pack(ctx, p, m, v, N, seed)
        torch.cuda.synchronize()
        off = np.concatenate([[0], np.cumsum(counts)])
        packed.append([buf[off[d]:off[d + 1]] for d in range(G)])
    new_o, nm_o, nv_o = D.redistribute(shards, ms, vs, seed)
    for d in range(G):
        ctx = L.Context(0, d, G)
        recv = torch.cat([packed[r][d] for r in range(G)])
        lo = d * N // G
        p2, m2, v2 = L.redistribute_unpack(ctx, recv, recv.shape[0], lo, DEV)
        torch.cuda.synchronize()
        assert p2.n == len(new_o[d]["pos"]) and p2.gid_base == lo
        for got, want in ((p2, new_o[d]), (m2, nm_o[d]), (v2, nv_o[d])):
            np.testing.assert_array_equal(got.to_flat(), _flat(want).astype(np.float32))
