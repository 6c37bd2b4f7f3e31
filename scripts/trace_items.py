"""Per-item view of CTA 0's trace (run scripts/trace_attend.py first, which saves the raw
buffer): item width, tiles, local flag, softmax cycles per tile, and the softmax phases of
warp 2 per tile (7 s_full seen, 4 after tcgen05.ld, 9 after the max / lazy decision,
10 after exp + packing, 14 after the PV wait (+ rescale), 15 after stmatrix, 8 arrive)."""
import numpy as np

a = np.load("gpurun_out/trace_raw.npy")
t0 = a[0, 0]
items = a[2048:2048 + 64]
n = 0
print("item  w nt loc   start | per tile (median): ld  max  exp  pvwait  stsm  arrive | total  interval")
for i, r in enumerate(items):
    if r[10] <= 0:
        break
    w, nt, loc = r[13], r[14], r[15]
    seg = a[n:n + nt]
    d = lambda x, y: np.median(seg[:, y] - seg[:, x])
    nxt = a[n + nt, 1] if n + nt < len(a) and a[n + nt, 1] > 0 else a[n + nt - 1, 1]
    print(f"{i:4d} {w:2d} {nt:2d} {loc:3d} {a[n, 1] - t0:8d} | {d(7, 4):5.0f} {d(4, 9):5.0f} {d(9, 10):5.0f} "
          f"{d(10, 14):6.0f} {d(14, 15):5.0f} {d(15, 8):6.0f} | {d(7, 8):5.0f} {(nxt - a[n, 1]) / nt:8.0f}")
    n += nt
