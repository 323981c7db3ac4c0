"""The C-ABI library loads on a CPU-only host and exports every function include/gs.h
declares; host-only entry points work without a GPU."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "gs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gs_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared()
    for n in ("gs_project", "gs_exchange", "gs_bin_sort", "gs_render_fwd", "gs_render_bwd",
              "gs_exchange_grads", "gs_adam_step", "gs_rebalance"):
        assert n in names


def test_library_exports_every_declared_symbol():
    import paper_2406_18533_b200._lib as L
    lib = ctypes.CDLL(L.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True).stdout
    for n in declared():
        assert re.search(r"\bT %s\b" % n, out), n


def test_library_is_sm100a():
    import paper_2406_18533_b200._lib as L
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_only_calls():
    import paper_2406_18533_b200._lib as L
    assert L.version() >= 100
    rng = np.random.default_rng(1)
    for _ in range(300):
        B, G = int(rng.integers(0, 200)), int(rng.integers(1, 33))
        et = rng.integers(0, 10_000, B) * (rng.random(B) < 0.6)
        np.testing.assert_array_equal(L.division_points(et, G), oracle.division_points(et, G))
    so, ro = L.exchange_plan(np.array([[1, 2, 0], [3, 4, 5], [0, 0, 7]]), 3, 1)
    assert list(so) == [0, 3, 7, 12] and list(ro) == [0, 2, 6, 6]
    with pytest.raises(L.GSError):
        L.division_points([-1, 2], 2)


def test_cull_words_cover_every_staged_word():
    """gs_cull_words: the forward stores the keep ballot of list entries 32k..32k+31 of block lb
    and half h at word 2 (range[lb] / 32 + lb + k) + h (gs_render.cu k_render_fwd); every word
    a block's list can need (including the round's second word of a 64-entry staging round
    that starts inside the list) lies below gs_cull_words(n_pairs, n_owned), and no two blocks
    share a word."""
    import paper_2406_18533_b200._lib as L
    rng = np.random.default_rng(7)
    for trial in range(200):
        n_owned = int(rng.integers(1, 60))
        lens = rng.integers(0, 300, n_owned) * (rng.random(n_owned) < 0.8)
        rng_ = np.concatenate([[0], np.cumsum(lens)])
        n_pairs = int(rng_[-1])
        words = L.cull_words(n_pairs, n_owned)
        used = set()
        for lb in range(n_owned):
            beg, ln = int(rng_[lb]), int(lens[lb])
            for k in range((ln + 31) // 32):  # words written: entries 32k < len
                for h in (0, 1):
                    w = 2 * (beg // 32 + lb + k) + h
                    assert w < words, (trial, lb, k, w, words)
                    assert w not in used
                    used.add(w)
    assert L.cull_words(0, 0) == 2 and L.cull_words(-1, 3) == 0
