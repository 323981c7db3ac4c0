"""Debug helper (GPU box): find pixels where the kernel's n_last differs from the oracle's in
the city_aerial window case and print the oracle's evaluation trace around the decision."""
import sys
import os
import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa
import synth  # noqa
from tests.gsutil import block_major  # noqa
from tests.test_gpu_scale import _window_case  # noqa

sc, cam = synth.scene_city(4_000_000), synth.cameras_city(128)[70]
c = _window_case(sc, cam, lo_frac=0.5)
no = c["no"]
nl = block_major(c["nl"], no)
T = block_major(c["T"], no)
f = c["fwd"]
bad = np.argwhere((nl != f["nlast"]) & ((f["flags"] & 3) == 0))
print("mismatches", len(bad))
for kb, p in bad[:2]:
    print("block", kb, "pixel", p, "kernel nl", nl[kb, p], "oracle nl", f["nlast"][kb, p], "flags", f["flags"][kb, p],
          "T k/o", T[kb, p], f["T"][kb, p])
    beta = c["lo"] + kb
    tx, ty = beta % c["Wt"], beta // c["Wt"]
    px, py = tx * 16 + p % 16, ty * 16 + p // 16
    ent = c["ent"][c["off"][kb]:c["off"][kb + 1]]
    rec = c["recs"].rec_f[ent]
    dx, dy = rec[:, 0] - px, rec[:, 1] - py
    power = -0.5 * (rec[:, 3] * dx * dx + rec[:, 5] * dy * dy) - rec[:, 4] * dx * dy
    alpha = np.minimum(0.99, rec[:, 6] * np.exp(power))
    Tc = 1.0
    lo_, hi_ = min(nl[kb, p], f["nlast"][kb, p]) - 6, max(nl[kb, p], f["nlast"][kb, p]) + 2
    for k in range(len(ent)):
        a = alpha[k]
        if a < 1 / 255:
            if lo_ <= k <= hi_:
                print("  k=%d skip alpha*255=%.9f" % (k, a * 255))
            continue
        Tn = Tc * (1 - a)
        if lo_ <= k <= hi_ or Tn < 1e-4:
            print("  k=%d alpha=%.6g alpha*255=%.9f T'=%.9g" % (k, a, a * 255, Tn))
        if Tn < 1e-4:
            break
        Tc = Tn

# kernel-side emulation (float32) of the skip test for the first unflagged mismatch
from tests.gsutil import decode_records  # noqa
f32 = np.float32
if len(bad):
    kb, p = bad[0]
    beta = c["lo"] + kb
    tx, ty = beta % c["Wt"], beta // c["Wt"]
    x, y = p % 16, p // 16
    y0 = (y // 4) * 4
    j = y - y0
    px, py0 = f32(tx * 16 + x), f32(ty * 16 + y0)
    d = decode_records(c["recv"][: c["n_recv"]])
    srt = c["sorted"][: c["npairs"]].cpu().numpy().view(np.uint32)
    rng = c["range"].cpu().numpy()
    lst = srt[rng[kb]:rng[kb + 1]]
    K = f32(0.84932180028801907)
    lo_ = min(nl[kb, p], f["nlast"][kb, p]) - 6
    for k in range(max(0, lo_), min(len(lst), max(nl[kb, p], f["nlast"][kb, p]) + 2)):
        r = lst[k]
        l11, l21, l22, o = f32(d["l11"][r]) * K, f32(d["l21"][r]) * K, f32(d["l22"][r]) * K, f32(d["opacity"][r])
        dx = f32(f32(d["mx"][r]) - px)
        dy0 = f32(f32(d["my"][r]) - py0)
        u = f32(f32(l11 * dx) + f32(l21 * dy0))
        w = f32(l22 * dy0)
        for _ in range(j):
            u = f32(u - l21)
            w = f32(w - l22)
        q = f32(f32(u * u) + f32(w * w))
        qmax = f32(np.log2(f32(255 * o)))
        print("  kernel-emul k=%d q=%.7g qmax=%.7g alpha*255=%.9f  comp=%s  (L=%.4g %.4g %.4g, o=%.4g, dx=%.3f dy=%.3f)" % (
            k, q, qmax, 255 * o * 2.0 ** (-float(q)), q <= qmax, l11, l21, l22, o, dx, dy0 - j))
