"""Dev tool: capture CTA 0's pipeline timeline of attend_kernel on one C2 layer and print
per-tile intervals (clock64 cycles).  Usage (GPU box): python scripts/trace_attend.py [cfg]"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import scripts._tracelib  # noqa: E402,F401  (TAPER_TRACE build)
from paper_2605_06914_b200 import taper as T  # noqa: E402

EV = ["tma_issue", "mma_full", "qk_commit", "pv_pfull", "pv_ofree", "pv_commit", "mma_qfull",
      "sm_sfull", "sm_arrive", "ep_start", "ep_ofull", "ep_end"]


def main():
    global _fn
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    h = int(sys.argv[2]) if len(sys.argv) > 2 else 8  # KV heads of the rank (8 / G)
    b = synth.config_batch(cfg, seed=0)
    lay = synth.make_layout(b, 64, np.random.default_rng(1), 1)
    db = T.DeviceBatch.from_host(b)
    adm = T.DeviceAdmission.empty(b.n_req, b.n_slot)
    ws = torch.empty(T.taper_workspace_size(b.n_req, b.n_slot, h, T.max_chunk_slots(
        b.req_shared_len, b.req_slot_off, b.slot_local_len)), dtype=torch.uint8, device="cuda")
    T.taper_admit(db, (12.0, 0.03, 2e-5), "eager", 0.8, adm, h, ws)
    g = torch.Generator(device="cuda").manual_seed(0)
    shape = (lay.num_pages, h, 64, 128)
    k = torch.randn(shape, generator=g, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(shape, generator=g, device="cuda", dtype=torch.bfloat16)
    rpo, rp, spo, sp = T.page_tables_to_device(lay)
    kv = T.DeviceKV(k, v, rpo, rp, spo, sp)
    q = torch.randn((b.n_slot, 8 * h, 128), generator=g, device="cuda", dtype=torch.bfloat16)
    out = torch.empty_like(q)
    for _ in range(3):
        T.taper_decode_attention(db, adm, kv, q, out, None, 1 / math.sqrt(128), ws)
    cap = 3200
    tr = torch.zeros(cap * 16, dtype=torch.int64, device="cuda")
    T.taper_set_trace_buffer(tr, cap)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    T.taper_decode_attention(db, adm, kv, q, out, None, 1 / math.sqrt(128), ws)
    e1.record()
    torch.cuda.synchronize()
    T.taper_set_trace_buffer(None)
    clocks_under_load(lambda: T.taper_decode_attention(db, adm, kv, q, out, None,
                                                         1 / math.sqrt(128), ws))
    print(f"layer time {e0.elapsed_time(e1) * 1e3:.1f} us")
    cta = tr.view(cap, 16).cpu().numpy()[3000:3000 + 148, :3].astype(np.int64)
    g0 = cta[:, 0].min()
    print("per-CTA (us): start min/max %.1f/%.1f, first TMA median %.1f, end min/median/max %.1f/%.1f/%.1f" % (
        (cta[:, 0].min() - g0) / 1e3, (cta[:, 0].max() - g0) / 1e3, np.median(cta[:, 2] - g0) / 1e3,
        (cta[:, 1].min() - g0) / 1e3, np.median(cta[:, 1] - g0) / 1e3, (cta[:, 1].max() - g0) / 1e3))
    ctaf = tr.view(cap, 16).cpu().numpy()[3000:3000 + 148].astype(np.int64)
    for e, name in ((5, "prologue done"), (11, "epoch loaded (acquire)"), (12, "header loaded"),
                    (13, "first descriptor loaded"), (6, "first record resolved (early)"), (8, "grid dependency"),
                    (9, "first Q load issued"), (2, "first K/V TMA issued"), (10, "first Q landed (MMA)")):
        v = ctaf[:, e]
        if (v > 0).any():
            print(f"  CTA start -> {name}: median {np.median(v[v > 0] - ctaf[v > 0, 0]) / 1e3:.2f} us")
    cta5 = tr.view(cap, 16).cpu().numpy()[3000:3000 + 148, :5].astype(np.int64)
    if cta5[:, 4].any():  # built with -DTAPER_TRACE_ITEMS: items / tiles per CTA
        end = (cta5[:, 1] - g0) / 1e3
        o = np.argsort(end)
        print("CTA end us / items / tiles, 10 earliest:", [(round(end[i], 1), int(cta5[i, 3]), int(cta5[i, 4])) for i in o[:10]])
        print("10 latest:", [(round(end[i], 1), int(cta5[i, 3]), int(cta5[i, 4])) for i in o[-10:]])
        print("tiles per CTA min/median/max", cta5[:, 4].min(), np.median(cta5[:, 4]), cta5[:, 4].max(),
              "corr(end, tiles) %.2f" % np.corrcoef(end, cta5[:, 4])[0, 1])
    a = tr.view(cap, 16).cpu().numpy()
    np.save("gpurun_out/trace_raw.npy", a)
    n = int((a[:, 1] > 0).sum())
    a = a[:n].astype(np.int64)
    t0 = a[0, 0]
    a = np.where(a > 0, a - t0, -1)
    np.save("gpurun_out/trace.npy", a)
    print("tiles", n, "total cycles", a[n - 1, 5])
    d = np.diff(a[:, 1])
    print("mma_full interval: median", np.median(d), "mean", d.mean())
    for name, (x, y) in {"tma->full": (0, 1), "full->qkcommit": (1, 2), "qk->sm_sfull": (2, 7),
                         "sm_sfull->arrive": (7, 8), "arrive->pv_pfull": (8, 3),
                         "pfull->pvcommit": (3, 5)}.items():
        dd = a[:, y] - a[:, x]
        ok = (a[:, x] >= 0) & (a[:, y] >= 0)
        print(f"{name:18s} median {np.median(dd[ok]):8.0f} mean {dd[ok].mean():8.0f}")
    full = tr.view(cap, 16).cpu().numpy().astype(np.int64)
    ep = np.where(full[2048:2048 + 40] > 0, full[2048:2048 + 40] - t0, -1)
    it = full[2048:2048 + 12].astype(np.int64)
    rel = lambda v: int(v - t0) if v > 0 else -1
    print("per item (cycles rel.): sm_start sm_rowsum sm_ofree sm_mlarrive ep_start ep_end | w nt local")
    for i in range(12):
        r = it[i]
        if r[0] <= 0:
            break
        print(i, [rel(r[e]) for e in (0, 1, 2, 3, 10, 11)], "|", int(r[13]), int(r[14]), int(r[15]))
    print("epilogue per item: ofull->ml, ml->xdone, xdone->bar, bar->stores(w8), stores->end")
    for i in range(12):
        r = ep[i]
        print(i, r[12] - r[10], r[13] - r[12], r[14] - r[13], r[15] - r[14], r[11] - r[15])
    arr = a[:, [8, 9, 10, 11]]
    ok = (arr > 0).all(1)
    lag = arr[ok] - arr[ok].min(1, keepdims=True)
    print("softmax arrive lag per warp (2,3,4,5): median", np.median(lag, 0), "mean", lag.mean(0))
    print("slowest warp histogram", np.bincount(arr[ok].argmax(1), minlength=4))
    print("producer: top(15) kempty-ok(0) K-issued(12) vempty-ok(13) V-issued(14)")
    for i in range(1, 12):
        r = a[i]
        print(i, r[15], r[0] - r[15], r[12] - r[0], r[13] - r[12], r[14] - r[13], "next top", a[i + 1][15] - r[14])
    print("first 40 tiles (cycles rel.):")
    FIRST40 = True
    print("   n " + " ".join(f"{e[:9]:>9s}" for e in EV))
    for i in range(min(40, n)):
        print(f"{i:4d} " + " ".join(f"{x:9d}" for x in a[i, :12]))


def clocks_under_load(fn, seconds=3.0):
    """Run fn() back to back for ~seconds while sampling nvidia-smi every 50 ms."""
    import subprocess, time
    q = ("clocks.sm,clocks.mem,power.draw,clocks_event_reasons.sw_power_cap,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.hw_power_brake_slowdown,temperature.gpu")
    proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                             "-lms", "50", "-i", "0"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    t_end = time.time() + seconds
    n = 0
    while time.time() < t_end:
        for _ in range(20):
            fn()
        n += 20
    torch.cuda.synchronize()
    time.sleep(0.2)
    proc.terminate()
    lines = proc.stdout.read().strip().splitlines()
    print(f"{n} launches; nvidia-smi samples (sm MHz, mem MHz, W, pwr_cap, hw_slow, sw_therm, pwr_brake, C):")
    for ln in lines[len(lines) // 3: len(lines) // 3 + 12]:
        print("   ", ln)


if __name__ == "__main__":
    main()
