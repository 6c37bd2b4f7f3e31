"""Warp-stall samples of attend_kernel by warp role and reason, from an ncu source page
(`ncu -i X.ncu-rep --page source --csv --print-source sass`) and the in-tree libtaper.so's
line table (nvdisasm -gi; the report must come from the same build).
    python scripts/stalls_by_role.py <sass.csv>"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2605_06914_b200", "csrc", "attention.cu")


def line_map():
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2605_06914_b200", "libtaper.so")],
                   cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.startswith("attention")][0]
    out = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
    lines = out.splitlines()
    i0 = [i for i, l in enumerate(lines) if l.startswith(".text._ZN5taper13attend_kernel")][0]
    cur, amap = None, {}
    for l in lines[i0 + 1:]:
        if l.startswith(".text."):
            break
        if "//##" in l:
            locs = re.findall(r'attention\.cu", line (\d+)', l)
            if locs:
                cur = int(locs[-1])
        m = re.search(r"/\*([0-9a-f]{4,6})\*/", l)
        if m:
            amap[int(m.group(1), 16)] = cur
    return amap


def roles():
    """Source line ranges of the warp-role branches of attend_kernel."""
    src = open(SRC).read().splitlines()
    marks = []
    for i, l in enumerate(src, 1):
        if "=== item scheduler" in l: marks.append((i, "scheduler (warp 11)"))
        if "=== TMA producers" in l: marks.append((i, "TMA producers (warps 0, 10)"))
        if "=== MMA issuer" in l: marks.append((i, "MMA issuer (warp 1)"))
        if "=== softmax / O correction" in l: marks.append((i, "softmax (warps 2-5, 12-15)"))
        if "=== epilogue (128 threads" in l: marks.append((i, "epilogue (warps 6-9)"))
    end = [i for i, l in enumerate(src, 1) if l.startswith("__global__ void __launch_bounds__(kMergeThreads")][0]
    return marks, end


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[2:] if len(r) >= len(hdr)]
    base = int(data[0][0], 16)
    amap = line_map()
    marks, end = roles()
    scols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]

    def role(ln):
        if ln is None:
            return "other"
        r = "prologue / epilogue of the kernel"
        for i, name in marks:
            if ln >= i:
                r = name
        return r if ln < end else "other"
    agg = collections.defaultdict(collections.Counter)
    for r in data:
        ln = amap.get(int(r[0], 16) - base)
        for c in scols:
            agg[role(ln)][c[6:]] += int(r[ix[c]] or 0)
    tot = sum(sum(c.values()) for c in agg.values())
    print(f"total stall samples {tot}")
    print("| role | share of samples | top reasons (share of the role's samples) |")
    print("|---|---|---|")
    for name, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values())):
        n = sum(c.values())
        top = ", ".join(f"{k} {100 * v / n:.0f} %" for k, v in c.most_common(5))
        print(f"| {name} | {100 * n / tot:.1f} % | {top} |")


if __name__ == "__main__":
    main()
