"""Per-item view of CTA 0's trace (run scripts/trace_attend.py first, which saves the raw
buffer): item width, tiles, local flag, softmax cycles per tile."""
import numpy as np
import torch  # noqa: F401
a = np.load("gpurun_out/trace_raw.npy")
t0 = a[0, 0]
items = a[2048:2048 + 64]
n = 0
for i, r in enumerate(items):
    if r[10] <= 0:
        break
    w, nt, loc = r[13], r[14], r[15]
    sm = a[n:n + nt, 8] - a[n:n + nt, 7]
    iv = np.diff(a[n:n + nt + 1, 1]) if n + nt < len(a) else np.array([0])
    print(f"item {i:3d} w={w} nt={nt:2d} local={loc} start={a[n, 1] - t0:8d} softmax/tile med {np.median(sm):6.0f} "
          f"interval med {np.median(iv):6.0f}")
    n += nt
# softmax phases of warp 2 (columns: 7 s_full seen, 4 after tcgen05.ld, 13 after the
# cross-warp barrier, 14 after the PV wait, 15 after stmatrix, 8 arrive)
n = 0
print("item w nt | ld  fwd+bar  red+bcast  lazy+exp  pvwait  stmatrix  fence+arrive  (median cycles)")
for i, r in enumerate(items[:24]):
    if r[10] <= 0:
        break
    nt = r[14]
    seg = a[n:n + nt]
    d = lambda x, y: np.median(seg[:, y] - seg[:, x])
    print(f"{i:3d} {r[13]} {nt:2d} | {d(7, 4):5.0f} {d(4, 13):7.0f} {d(13, 9):9.0f} {d(9, 10):8.0f} {d(10, 14):7.0f} {d(14, 15):8.0f} {d(15, 8):9.0f}")
    n += nt
