"""Offline model of the aggregation's chunk work (reads gpurun_out/meta_c5.npz
from tools/dump_meta.py): cells searched vs cells processed by the
lockstep-chain kernel (G lanes per chain, 2*PPL*G-cell absolute chunks, the
warp looping over the union of its 32/G chains' chunk ranges)."""
import sys

import numpy as np

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/meta_c5.npz"
z = np.load(path)
keys = sorted({k.rsplit("_", 1)[0] for k in z.files})


def chains(fam, H, W):
    """pixel index arrays (chain, step) for the forward sweep, -1 = off."""
    if fam == "H":
        ys, xs = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
        return ys * W + xs
    if fam == "V":
        ys, xs = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
        return (ys * W + xs).T
    n = W + H - 1
    out = -np.ones((n, H), dtype=np.int64)
    for c in range(n):
        for y in range(H):
            x = (c - (H - 1)) + y if fam == "D1" else c - y
            if 0 <= x < W:
                out[c, y] = y * W + x
    return out


for G, PPL in ((4, 4), (8, 4), (4, 2), (2, 4)):
    CWc = 2 * PPL * G   # cells per chunk
    NG = 32 // G
    tot = {}
    for k in keys:
        lo = z[k + "_lo"].astype(np.int64)
        hi = z[k + "_hi"].astype(np.int64)
        H, W = lo.shape
        lo_f, hi_f = lo.ravel(), hi.ravel()
        useful = (hi_f - lo_f + 1).sum()
        for fam in ("H", "V", "D1", "D2"):
            P = chains(fam, H, W)
            nc, L = P.shape
            pad = (-nc) % NG
            P = np.concatenate([P, -np.ones((pad, L), dtype=np.int64)])
            Pw = P.reshape(-1, NG, L)
            off = Pw < 0
            clo = np.where(off, 1 << 20, (lo_f[np.maximum(Pw, 0)] >> 1) * 2 // CWc)
            chi = np.where(off, -1, (hi_f[np.maximum(Pw, 0)] >> 1) * 2 // CWc)
            own = np.where(off, 0, chi - clo + 1).sum() * CWc
            u = chi.max(1) - clo.min(1) + 1
            u = np.where(u > 0, u, 0)
            union = u.sum() * CWc * NG
            steps = (~off).any(1).sum()
            t = tot.setdefault(fam, [0, 0, 0, 0])
            t[0] += useful
            t[1] += own
            t[2] += union
            t[3] += steps
    print(f"G={G} PPL={PPL} chunk={CWc} cells")
    for fam, (us, own, un, st) in tot.items():
        print(f"  {fam:2s} useful {us/1e6:8.1f} M  own-chunks {own/us:5.2f}x  union {un/us:5.2f}x  warp-steps {st/1e3:8.1f} k")
