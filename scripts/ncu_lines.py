"""Per-source-line warp-stall samples of one ncu report (needs -lineinfo and
--import-source on at capture time).

    python scripts/ncu_lines.py gpurun_out/prof_<tag>.ncu-rep [top_n] [line_lo line_hi]

Prints the hottest source lines of attention.cu with their sample counts and the three
largest stall reasons, and the totals per line range (e.g. one warp role's code)."""
import csv
import io
import subprocess
import sys


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    lines = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in lines if r and r[0] == "Line No")
    res = []
    for r in lines:
        if len(r) != len(hdr) or not r[0].isdigit():
            continue
        res.append(dict(zip(range(len(hdr)), r)))
    return hdr, res


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    hdr, res = rows(rep)
    ix = {h: i for i, h in enumerate(hdr)}
    samp = ix["Warp Stall Sampling (All Samples)"]
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(int(r[samp] or 0) for r in res)
    print(f"total samples {tot}")
    res.sort(key=lambda r: -int(r[samp] or 0))
    for r in res[:top]:
        n = int(r[samp] or 0)
        st = sorted(((int(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
        print(f"{r[0]:>5} {n:7d} {100 * n / tot:5.1f}%  " + " ".join(f"{k}={v}" for v, k in st if v)
              + "  | " + r[1].strip()[:70])
    if len(sys.argv) > 4:
        lo, hi = int(sys.argv[3]), int(sys.argv[4])
        sub = [r for r in res if lo <= int(r[0]) <= hi]
        n = sum(int(r[samp] or 0) for r in sub)
        agg = {hdr[i][6:]: sum(int(r[i] or 0) for r in sub) for i in stall_cols}
        print(f"lines {lo}-{hi}: {n} samples ({100 * n / tot:.1f}%)",
              sorted(((v, k) for k, v in agg.items() if v), reverse=True)[:6])


if __name__ == "__main__":
    main()
