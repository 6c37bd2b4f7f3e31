"""NEXT-1: the paper's profiling grid for T(S) = a + b n + c L (App. C.1,
PAPER.md L316, "Fitting" L337: "500 profiling steps across a 20 x 25 grid of batch sizes
(1-512) and context lengths (128-8192) ... fit (a, b, c) via ordinary least squares"),
on this library's own step on one B200, with the Table-3 analog: MAPE per load regime
(batch 1-64, 64-256, 256-512) on a held-out fifth of the grid.

Grid point (n, Lctx): n sequences of context Lctx -- half serial requests (prefix Lctx),
half the branches of 4-way parallel requests (prefix Lctx - local, local ~ U{1..Lctx/8}).
T = one taper_admit + 64 x taper_decode_attention (Eager; no FFN -- this library has no
weights), CUDA-event timed over KV pools cycled like 64 layers (enough distinct pools that
the cycle exceeds L2).  Both readings of L_context are fitted: per sequence (the paper's)
and per request (cascade-aware, what the kernel reads).

    python scripts/fit_latency_grid.py [--out gpurun_out/latency_grid_b200.json]   (GPU box)
"""
import argparse
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

BATCH = np.unique(np.round(np.geomspace(1, 512, 22)).astype(int))  # 20 sizes
CTX = np.unique((np.round(np.geomspace(128, 8192, 25) / 16) * 16).astype(int))
LAYERS = 64
REGIMES = {"low (1-64)": (1, 64), "medium (64-256)": (65, 256), "high (256-512)": (257, 512)}


def compose(n, ctx, rng):
    n_par = 4 * (n // 8)           # branches of 4-way parallel requests
    n_ser = n - n_par
    shared, fans, loc = [], [], []
    for _ in range(n_ser):
        shared.append(ctx); fans.append(1); loc.append(0)
    for _ in range(n_par // 4):
        ll = rng.integers(1, max(2, ctx // 8) + 1, size=4)
        shared.append(max(1, ctx - int(ll.max()))); fans.append(4); loc += [int(x) for x in ll]
    return synth.make_batch(shared, fans, loc, 1e9, 0.0, rng=rng)


def counts(b):
    off = b.req_slot_off
    n = b.n_slot
    L_seq = int(sum(b.req_shared_len[r] * (off[r + 1] - off[r]) for r in range(b.n_req)) +
                b.slot_local_len.sum())
    L_req = int(b.req_shared_len.sum() + b.slot_local_len.sum())
    return n, L_seq, L_req


def time_point(b, rng, calls=16):
    lay = synth.make_layout(b, 64, rng, 1)
    db = T.DeviceBatch.from_host(b)
    adm = T.DeviceAdmission.empty(b.n_req, b.n_slot)
    ws = torch.empty(T.taper_workspace_size(b.n_req, b.n_slot, 8, T.max_chunk_slots(
        b.req_shared_len, b.req_slot_off, b.slot_local_len)), dtype=torch.uint8, device="cuda")
    pool_bytes = 2 * lay.num_pages * 8 * 64 * 128 * 2
    n_pools = int(min(LAYERS, max(2, math.ceil(300e6 / pool_bytes))))
    shape = (lay.num_pages, 8, 64, 128)
    g = torch.Generator(device="cuda").manual_seed(int(rng.integers(1 << 30)))
    rpo, rp, spo, sp = T.page_tables_to_device(lay)
    pools = [T.DeviceKV(torch.randn(shape, generator=g, device="cuda", dtype=torch.bfloat16),
                        torch.randn(shape, generator=g, device="cuda", dtype=torch.bfloat16),
                        rpo, rp, spo, sp) for _ in range(n_pools)]
    q = torch.randn((b.n_slot, 64, 128), generator=g, device="cuda", dtype=torch.bfloat16)
    out = torch.empty_like(q)
    sc = 1 / math.sqrt(128)
    model = (12.0, 0.03, 2e-5)
    for i in range(4):
        T.taper_admit(db, model, "eager", 0.8, adm, 8, ws)
        T.taper_decode_attention(db, adm, pools[i % n_pools], q, out, None, sc, ws)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    for _ in range(8):
        T.taper_admit(db, model, "eager", 0.8, adm, 8, ws)
    e[1].record()
    for i in range(calls):
        T.taper_decode_attention(db, adm, pools[i % n_pools], q, out, None, sc, ws)
    e[2].record()
    torch.cuda.synchronize()
    admit_ms = e[0].elapsed_time(e[1]) / 8
    layer_ms = e[1].elapsed_time(e[2]) / calls
    del pools
    return admit_ms + LAYERS * layer_ms, admit_ms, layer_ms, n_pools


def fit(X, y):
    coef, *_ = np.linalg.lstsq(X, y, rcond=None)
    return coef


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "latency_grid_b200.json"))
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    rng = np.random.default_rng(args.seed)
    pts = []
    for n in BATCH:
        for ctx in CTX:
            b = compose(int(n), int(ctx), rng)
            nn, Ls, Lr = counts(b)
            t, a_ms, l_ms, npools = time_point(b, rng)
            pts.append({"n": nn, "ctx": int(ctx), "L_per_sequence": Ls, "L_per_request": Lr,
                        "T_ms": t, "admit_ms": a_ms, "layer_ms": l_ms, "kv_pools": npools})
        print(f"batch {n}: {len(pts)} points, last T = {pts[-1]['T_ms']:.2f} ms", flush=True)
    y = np.array([p["T_ms"] for p in pts])
    n = np.array([p["n"] for p in pts], float)
    held = np.random.default_rng(args.seed + 1).random(len(pts)) < 0.2  # held-out fifth
    res = {"grid": {"batch_sizes": BATCH.tolist(), "context_lengths": CTX.tolist(),
                    "points": len(pts), "held_out": int(held.sum())},
           "model": "T(S) = a + b n + c L (App. C.1 L316); T = admit + 64 attention calls, no FFN"}
    for name in ("per_sequence", "per_request"):
        L = np.array([p[f"L_{name}"] for p in pts], float)
        X = np.c_[np.ones(len(y)), n, L]
        a, bb, c = fit(X[~held], y[~held])
        pred = a + bb * n + c * L
        ape = np.abs(pred - y) / y
        reg = {k: float(100 * ape[held & (n >= lo) & (n <= hi)].mean())
               for k, (lo, hi) in REGIMES.items() if (held & (n >= lo) & (n <= hi)).any()}
        res[name] = {"a_ms": float(a), "b_ms_per_seq": float(bb), "c_ms_per_token": float(c),
                     "heldout_mape_pct": float(100 * ape[held].mean()),
                     "heldout_mape_pct_by_regime": reg,
                     "train_mape_pct": float(100 * ape[~held].mean()),
                     "r2": float(1 - ((pred - y) ** 2).sum() / ((y - y.mean()) ** 2).sum())}
        print(name, json.dumps(res[name]), flush=True)
    res["points"] = pts
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
