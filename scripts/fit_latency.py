"""NEXT-1: fit the step-latency model T(S) = a + b n + c L (App. C.1,
PAPER.md L314-341) by ordinary least squares on this kernel's own timings, for both
readings of L_context: per sequence (the paper's; every admitted branch counts its whole
context) and per request (cascade-aware; each prefix once -- what the kernel reads).

Grid: R requests x fanout f x prefix Lsh (+ local lengths ~ U{1..256}), all branches
admitted (Eager).  T(S) per point = one taper_admit + 64 x taper_decode_attention, timed
back to back with CUDA events (8 distinct KV layer buffers, cycled).  Writes
gpurun_out/latency_model_b200.json (committed as profiles/) and prints a summary.  GPU box only.
    python scripts/fit_latency.py [--quick]
"""
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2605_06914_b200 import taper as T  # noqa: E402

LAYERS = 64


def time_point(R, fan, lsh, rng, n_pools=8, calls=48):
    fans = [fan] * R
    loc = rng.integers(1, 257, size=R * fan).tolist()
    b = synth.make_batch([lsh] * R, fans, loc, 1e9, 0.0, rng=rng)
    lay = synth.make_layout(b, 64, rng, 1)
    db = T.DeviceBatch.from_host(b)
    adm = T.DeviceAdmission.empty(b.n_req, b.n_slot)
    ws = torch.empty(T.taper_workspace_size(b.n_req, b.n_slot, 8, T.max_chunk_slots(
        b.req_shared_len, b.req_slot_off, b.slot_local_len)), dtype=torch.uint8, device="cuda")
    model = (12.0, 0.03, 2e-5)
    g = torch.Generator(device="cuda").manual_seed(R * 1000 + fan)
    shape = (lay.num_pages, 8, 64, 128)
    rpo, rp, spo, sp = T.page_tables_to_device(lay)
    pools = []
    for _ in range(n_pools):
        k = torch.randn(shape, generator=g, device="cuda", dtype=torch.bfloat16)
        v = torch.randn(shape, generator=g, device="cuda", dtype=torch.bfloat16)
        pools.append(T.DeviceKV(k, v, rpo, rp, spo, sp))
    q = torch.randn((b.n_slot, 64, 128), generator=g, device="cuda", dtype=torch.bfloat16)
    out = torch.empty_like(q)
    sc = 1 / math.sqrt(128)
    for i in range(4):
        T.taper_admit(db, model, "eager", 0.8, adm, 8, ws)
        T.taper_decode_attention(db, adm, pools[i % n_pools], q, out, None, sc, ws)
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    for _ in range(16):
        T.taper_admit(db, model, "eager", 0.8, adm, 8, ws)
    e1.record()
    for i in range(calls):
        T.taper_decode_attention(db, adm, pools[i % n_pools], q, out, None, sc, ws)
    e2.record()
    torch.cuda.synchronize()
    admit_ms = e0.elapsed_time(e1) / 16
    layer_ms = e1.elapsed_time(e2) / calls
    n = b.n_slot
    L_seq = int(np.sum(np.repeat(b.req_shared_len, fans)) + np.sum(b.slot_local_len))
    L_req = int(np.sum(b.req_shared_len) + np.sum(b.slot_local_len))
    del pools
    torch.cuda.empty_cache()
    return {"R": R, "fanout": fan, "Lsh": lsh, "n": n, "L_per_sequence": L_seq,
            "L_per_request": L_req, "admit_ms": admit_ms, "layer_ms": layer_ms,
            "T_ms": admit_ms + LAYERS * layer_ms}


def ols(pts, key):
    X = np.array([[1.0, p["n"], p[key]] for p in pts])
    y = np.array([p["T_ms"] for p in pts])
    coef, *_ = np.linalg.lstsq(X, y, rcond=None)
    pred = X @ coef
    ss_res = float(np.sum((y - pred) ** 2))
    ss_tot = float(np.sum((y - y.mean()) ** 2))
    rel = np.abs(y - pred) / y
    return {"a_ms": float(coef[0]), "b_ms_per_seq": float(coef[1]), "c_ms_per_token": float(coef[2]),
            "r2": 1.0 - ss_res / ss_tot, "rmse_ms": math.sqrt(ss_res / len(y)),
            "max_rel_err": float(rel.max()), "median_rel_err": float(np.median(rel))}


def main():
    quick = "--quick" in sys.argv
    rng = np.random.default_rng(0)
    Rs = [8, 32] if quick else [4, 8, 16, 32, 64]
    fans = [1, 4] if quick else [1, 2, 4, 8]
    lshs = [1024, 8192] if quick else [512, 2048, 4096, 8192]
    pts = []
    for R in Rs:
        for fan in fans:
            for lsh in lshs:
                if R * lsh > 64 * 8192 or R * fan > 4096:
                    continue
                p = time_point(R, fan, lsh, rng)
                pts.append(p)
                print(f"R={R:3d} f={fan} Lsh={lsh:5d}  n={p['n']:4d} Lseq={p['L_per_sequence']:8d} "
                      f"Lreq={p['L_per_request']:8d}  layer {p['layer_ms'] * 1e3:7.1f} us  "
                      f"T {p['T_ms']:7.2f} ms", flush=True)
    fit_seq = ols(pts, "L_per_sequence")
    fit_req = ols(pts, "L_per_request")
    res = {"model": "T(S) = a + b n + c L  (App. C.1 L316); T = admit + 64 attention calls",
           "timing": "CUDA events, back to back, 48 calls over 8 KV buffers per point",
           "per_sequence": fit_seq, "per_request": fit_req, "points": pts,
           "gpu": torch.cuda.get_device_name(0)}
    out_dir = os.path.join(ROOT, "gpurun_out")  # merged back by gpurun; copy into profiles/
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "latency_model_b200.json"), "w") as f:
        json.dump(res, f, indent=1)
    for name, fit in (("per_sequence", fit_seq), ("per_request", fit_req)):
        print(f"{name:13s} a={fit['a_ms']:.4g} ms  b={fit['b_ms_per_seq']:.4g} ms/seq  "
              f"c={fit['c_ms_per_token']:.4g} ms/token  R^2={fit['r2']:.5f}  "
              f"rmse={fit['rmse_ms']:.3f} ms  max rel err={fit['max_rel_err']:.3f}")


if __name__ == "__main__":
    main()
