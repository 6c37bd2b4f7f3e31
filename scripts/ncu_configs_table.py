"""Table of the targeted ncu metrics of one attend_kernel launch per config
(scripts/gpu_ncu_configs.sh <tag>) against the algorithmic bytes of the same launch
(bench.py roofline.bytes_per_launch).  python scripts/ncu_configs_table.py <tag> name=bench.json ..."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
alg = {}
for a in sys.argv[2:]:
    k, _, f = a.partition("=")
    try:
        alg[k] = float(a.split("=", 1)[1]) if f.replace(".", "").isdigit() else \
            json.loads(open(f).read().strip().splitlines()[-1])["roofline"]["bytes_per_launch"]
    except Exception as e:
        print("skip", a, e, file=sys.stderr)
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
print(f"| config | time µs | DRAM read GB | algorithmic GB | read / algorithmic | algorithmic TB/s | "
      f"frac of {peak:.0f} GB/s | tensor pipe | L2 hit | SM clock GHz |")
print("|---|---|---|---|---|---|---|---|---|---|")
for name in sorted(alg):
    path = os.path.join(ROOT, "gpurun_out", f"ncu_cfg_{tag}_{name}.csv")
    m = {}
    for r in csv.reader(open(path)):
        if len(r) > 3 and r[-3] in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                    "lts__t_sector_hit_rate.pct", "gpc__cycles_elapsed.avg.per_second",
                                    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"):
            m[r[-3]] = float(r[-1].replace(",", ""))
    t = m["gpu__time_duration.sum"] * 1e-9
    rd = m["dram__bytes_read.sum"]
    a = alg[name]
    print(f"| {name} | {t * 1e6:.1f} | {rd / 1e9:.3f} | {a / 1e9:.3f} | {rd / a:.3f} | {a / t / 1e12:.2f} | "
          f"{a / t / 1e9 / peak:.2f} | {m['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed']:.1f} % | "
          f"{m['lts__t_sector_hit_rate.pct']:.1f} % | {m['gpc__cycles_elapsed.avg.per_second'] / 1e9:.2f} |")
