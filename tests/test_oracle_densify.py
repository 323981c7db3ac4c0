"""Pins of the densification oracle (NEXT-2; S:361-416 examples and invariants)."""
import math

import numpy as np

from oracle import densify as D

CFG = dict(grad_thresh=0.0002, percent_dense=0.01, scene_extent=2.0, min_opacity=0.005, max_screen_size=0.0)


def _shard(n, rng, ls=-5.0):
    return dict(pos=rng.normal(size=(n, 3)), log_scale=np.full((n, 3), ls) + 0.1 * rng.normal(size=(n, 3)),
                rot=rng.normal(size=(n, 4)), opac_logit=rng.normal(2.0, 0.5, size=n), sh=rng.normal(size=(n, 48)))


def _state(sh, rng):
    return {k: rng.normal(size=np.shape(a)) for k, a in sh.items()}


def test_stats_examples():
    # an invisible Gaussian keeps zero statistics; norms 0.1 and 0.3 average 0.2
    W, H, b = 64, 32, 2
    g = np.array([[0.1 / (b * W / 2), 0.0], [0.0, 0.3 / (b * H / 2)]])
    acc, den, rad = D.stats_from_record_grads(3, np.array([1, 1]), g, np.array([2.0, 5.0]), W, H, b)
    assert acc[0] == 0 and den[0] == 0 and rad[0] == 0 and acc[2] == 0
    assert abs(acc[1] / den[1] - 0.2) < 1e-15 and rad[1] == 5.0


def test_zero_gradients_only_prune():
    rng = np.random.default_rng(0)
    sh = _shard(200, rng)
    sh["opac_logit"][:17] = -8.0  # alpha < 0.005
    m, v = _state(sh, rng), _state(sh, rng)
    z = np.zeros(200)
    out, om, ov, cnt = D.densify(sh, m, v, z, z, z, rng.normal(size=(200, 2, 3)), CFG)
    assert cnt == (183, 0, 0, 183)
    np.testing.assert_array_equal(out["pos"], sh["pos"][17:])
    np.testing.assert_array_equal(om["sh"], m["sh"][17:])  # survivors keep their Adam state


def test_one_small_selected_gaussian_is_cloned():
    rng = np.random.default_rng(1)
    sh = _shard(10, rng, ls=-6.0)  # max scale << 0.01 * extent
    m, v = _state(sh, rng), _state(sh, rng)
    acc = np.zeros(10)
    den = np.zeros(10)
    acc[4], den[4] = 0.001, 2.0  # avg 0.0005 >= 0.0002
    out, om, ov, cnt = D.densify(sh, m, v, acc, den, np.zeros(10), rng.normal(size=(10, 2, 3)), CFG)
    assert cnt == (10, 1, 0, 11)
    np.testing.assert_array_equal(out["pos"][:10], sh["pos"])  # parent preserved
    for k in D.FIELDS:
        np.testing.assert_array_equal(out[k][10], np.asarray(sh[k][4], np.float64))
        assert not np.any(om[k][10]) and not np.any(ov[k][10])  # fresh Adam state


def test_split_children_distribution():
    # children sampled from the parent's distribution: mean within 3 sigma / sqrt(n)
    rng = np.random.default_rng(2)
    n = 1000
    sh = dict(pos=np.tile([0.3, -0.2, 1.0], (n, 1)), log_scale=np.tile(np.log([0.05, 0.02, 0.01]), (n, 1)),
              rot=np.tile([0.9, 0.1, -0.3, 0.2], (n, 1)), opac_logit=np.zeros(n), sh=np.zeros((n, 48)))
    m, v = _state(sh, rng), _state(sh, rng)
    noise = rng.normal(size=(n, 2, 3))
    out, _, _, cnt = D.densify(sh, m, v, np.ones(n), np.ones(n), np.zeros(n), noise, CFG)
    assert cnt == (0, 0, 2 * n, 2 * n)  # every parent split and removed
    R = D._rotmat(np.array([0.9, 0.1, -0.3, 0.2]))
    local = (out["pos"] - sh["pos"][0]) @ R  # back to the parent's frame
    sd = np.array([0.05, 0.02, 0.01])
    assert np.all(np.abs(local.mean(0)) < 3 * sd / math.sqrt(2 * n))
    assert np.all(np.abs(local.std(0) / sd - 1) < 0.1)
    np.testing.assert_allclose(out["log_scale"], np.tile(np.log([0.05, 0.02, 0.01]) - math.log(1.6), (2 * n, 1)))


def test_lower_threshold_densifies_more():
    rng = np.random.default_rng(3)
    sh = _shard(500, rng, ls=-4.0)
    sh["log_scale"][::2] = -9.0
    m, v = _state(sh, rng), _state(sh, rng)
    acc, den = rng.exponential(0.0003, 500), rng.integers(1, 4, 500).astype(float)
    noise = rng.normal(size=(500, 2, 3))
    prev = -1
    for t in (0.001, 0.0005, 0.0002, 0.0001, 0.00001):
        cnt = D.densify(sh, m, v, acc, den, np.zeros(500), noise, dict(CFG, grad_thresh=t))[3]
        dens = cnt[1] + cnt[2] // 2
        assert dens >= prev
        prev = dens


def test_opacity_reset():
    sig = lambda x: 1 / (1 + np.exp(-x))
    logit = np.array([math.log(0.9 / 0.1), math.log(0.005 / 0.995)])
    sh = dict(pos=np.zeros((2, 3)), log_scale=np.zeros((2, 3)), rot=np.zeros((2, 4)), opac_logit=logit,
              sh=np.zeros((2, 48)))
    s2, m2, v2 = D.opacity_reset(sh, sh, sh)
    assert abs(sig(float(s2["opac_logit"][0])) - 0.01) < 1e-7  # 0.9 -> 0.01
    assert s2["opac_logit"][1] == np.float32(logit[1])  # already below: unchanged
    assert not np.any(m2["opac_logit"]) and not np.any(v2["opac_logit"])


def test_redistribution_permutation_is_a_bijection():
    for N in (1, 2, 3, 7, 64, 100, 1000, 4097):
        for seed in (0, 12345, 2 ** 40 + 7):
            img = sorted(D.perm(j, N, seed) for j in range(N))
            assert img == list(range(N))


def test_redistribution_sizes_and_multiset():
    # sizes {10, 2} -> {6, 6}; multiset of Gaussians (with their Adam state) unchanged
    rng = np.random.default_rng(4)
    sizes = [(10, 2), (5, 5, 5), (1, 0, 30, 2)]
    for sz in sizes:
        shards = [_shard(n, rng) for n in sz]
        ms = [{k: a[k] * 2 for k in a} for a in shards]
        vs = [{k: a[k] * 3 for k in a} for a in shards]
        new, nm, nv = D.redistribute(shards, ms, vs, seed=99)
        ns = [len(s["pos"]) for s in new]
        assert sum(ns) == sum(sz) and max(ns) - min(ns) <= 1
        key = lambda ds: sorted(map(tuple, np.concatenate([d["sh"] for d in ds]).round(12)))
        assert key(new) == key(shards)
        for s, m_, v_ in zip(new, nm, nv):  # state travels with its Gaussian
            np.testing.assert_array_equal(m_["pos"], s["pos"] * 2)
            np.testing.assert_array_equal(v_["sh"], s["sh"] * 3)
    assert [len(s["pos"]) for s in D.redistribute([_shard(10, rng), _shard(2, rng)], [_shard(10, rng), _shard(2, rng)],
                                                  [_shard(10, rng), _shard(2, rng)], 1)[0]] == [6, 6]
