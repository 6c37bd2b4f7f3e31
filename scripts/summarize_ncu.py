"""Summarise ncu outputs (launch list CSV + one `--set full` report) into profiles/.

    python scripts/summarize_ncu.py <tag> [bench_json]

Reads gpurun_out/launches_<tag>.csv and gpurun_out/prof_attend_<tag>.ncu-rep, writes
profiles/<tag>_launches.csv (our kernels only), profiles/<tag>_attend_metrics.csv and
profiles/<tag>_summary.md.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg", "smsp__cycles_active.avg",
    "gpc__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second",
]


def launches(tag):
    path = os.path.join(OUT, f"launches_{tag}.csv")
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    idx = {h: i for i, h in enumerate(hdr)}
    keep = [hdr]
    per = collections.defaultdict(list)
    unit = ""
    for r in rows[hi + 1:]:
        if len(r) < len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[idx["Kernel Name"]].split("(")[0]
        if not any(k in name for k in ("admit_kernel", "attend_kernel", "merge_kernel")):
            continue
        keep.append(r)
        unit = r[idx["Metric Unit"]]
        per[name].append(float(r[idx["Metric Value"]].replace(",", "")))
    with open(os.path.join(PROF, f"{tag}_launches.csv"), "w", newline="") as f:
        csv.writer(f).writerows(keep)
    return per, unit


def full_metrics(tag):
    rep = os.path.join(OUT, f"prof_attend_{tag}.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for i, h in enumerate(hdr):
        if h in METRICS:
            out[h] = (vals[i], units[i])
    with open(os.path.join(PROF, f"{tag}_attend_metrics.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["metric", "value", "unit"])
        for k in METRICS:
            if k in out:
                w.writerow([k, out[k][0], out[k][1]])
    return out


def main():
    tag = sys.argv[1]
    bench = json.load(open(sys.argv[2])) if len(sys.argv) > 2 else None
    os.makedirs(PROF, exist_ok=True)
    per, unit = launches(tag)
    m = full_metrics(tag)
    scale = 1e-3 if unit == "ns" else (1.0 if unit == "us" else 1e-6 if unit == "ps" else 1.0)
    total = sum(sum(v) for v in per.values())
    lines = [f"# ncu summary — {tag}", "",
             "Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, our kernels "
             "only; cold-cache and serialised, so compare shares, not absolutes):", "",
             "| kernel | launches | mean us | share of our GPU time |", "|---|---|---|---|"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v) * scale:.1f} | {sum(v) / total * 100:.1f} % |")
    lines += ["", "`attend_kernel`, one `ncu --set full` capture (layer of config c2):", "",
              "| metric | value |", "|---|---|"]
    for k in METRICS:
        if k in m:
            lines.append(f"| {k} | {m[k][0]} {m[k][1]} |")
    if "dram__bytes_read.sum" in m and bench:
        alg = bench["roofline"]["bytes_per_launch"]
        rd = float(m["dram__bytes_read.sum"][0].replace(",", ""))
        wr = float(m["dram__bytes_write.sum"][0].replace(",", ""))
        mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
        rd *= mult.get(m["dram__bytes_read.sum"][1], 1)
        wr *= mult.get(m["dram__bytes_write.sum"][1], 1)
        lines += ["", f"DRAM traffic per launch {rd + wr:.4g} B (read {rd:.4g}, write {wr:.4g}) vs "
                      f"algorithmic {alg:.4g} B -> ratio {(rd + wr) / alg:.3f}."]
        json.dump({"workload": bench["config"]["workload"].split(":")[0], "kernel": "attend_kernel",
                   "bytes_per_launch": rd + wr, "read_bytes": rd, "write_bytes": wr,
                   "algorithmic_bytes": alg,
                   "source": f"profiles/{tag}_attend_metrics.csv (ncu --set full, one launch)"},
                  open(os.path.join(PROF, "attend_traffic.json"), "w"), indent=1)
    if bench:
        lines += ["", "Bench line of the same build:", "", "```", json.dumps(bench)[:3000], "```"]
    open(os.path.join(PROF, f"{tag}_summary.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:40]))


if __name__ == "__main__":
    main()
