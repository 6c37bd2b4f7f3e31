"""Summarise an ncu `--page source --csv --print-source sass` dump: samples by opcode and
the hottest instructions with their dominant stall reasons.
    python scripts/sass_hot.py gpurun_out/sass_<tag>.csv [lo_addr hi_addr]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
lo = int(sys.argv[2], 16) if len(sys.argv) > 3 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 62
tot = 0
by_op = collections.Counter()
by_op_n = collections.Counter()
hot = []
base = int(data[0][0], 16)
for r in data:
    if len(r) < len(hdr):
        continue
    a = int(r[0], 16) - base
    if not (lo <= a < hi):
        continue
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    n = int(r[ix["Instructions Executed"]] or 0)
    op = r[1].strip().split()[0] if r[1].strip() else "?"
    if op.startswith("@"):
        op = r[1].strip().split()[1]
    op = op.split(".")[0]
    tot += s
    by_op[op] += s
    by_op_n[op] += n
    st = sorted(((int(r[ix[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    hot.append((s, a, r[1].strip()[:60], n, st))
print("total samples", tot)
for op, s in by_op.most_common(25):
    print(f"{op:12s} {s:7d} {100 * s / max(tot, 1):5.1f}%  executed {by_op_n[op]}")
print()
for s, a, src, n, st in sorted(hot, reverse=True)[:45]:
    print(f"{a:#07x} {s:6d} {n:9d} {src:60s} {st}")
