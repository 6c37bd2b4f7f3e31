"""Dev tool: wall-clock anatomy of one C2 layer call (attend + merge) inside a back-to-back
sequence: event times vs. per-CTA globaltimer spans.  Usage (GPU box): python scripts/gaps.py"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import scripts._tracelib  # noqa: E402,F401  (TAPER_TRACE build)
from paper_2605_06914_b200 import taper as T  # noqa: E402


def main():
    b = synth.config_batch("c2", seed=0)
    lay = synth.make_layout(b, 64, np.random.default_rng(1), 1)
    db = T.DeviceBatch.from_host(b)
    adm = T.DeviceAdmission.empty(b.n_req, b.n_slot)
    ws = torch.empty(T.taper_workspace_size(b.n_req, b.n_slot, 8, T.max_chunk_slots(
        b.req_shared_len, b.req_slot_off, b.slot_local_len)), dtype=torch.uint8, device="cuda")
    T.taper_admit(db, (12.0, 0.03, 2e-5), "eager", 0.8, adm, 8, ws)
    g = torch.Generator(device="cuda").manual_seed(0)
    shape = (lay.num_pages, 8, 64, 128)
    k = torch.randn(shape, generator=g, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(shape, generator=g, device="cuda", dtype=torch.bfloat16)
    rpo, rp, spo, sp = T.page_tables_to_device(lay)
    kv = T.DeviceKV(k, v, rpo, rp, spo, sp)
    q = torch.randn((b.n_slot, 64, 128), generator=g, device="cuda", dtype=torch.bfloat16)
    out = torch.empty_like(q)
    call = lambda: T.taper_decode_attention(db, adm, kv, q, out, None, 1 / math.sqrt(128), ws)
    for _ in range(5):
        call()
    cap = 4000
    tr = torch.zeros(cap * 16, dtype=torch.int64, device="cuda")
    for rep in range(3):
        for _ in range(6):
            call()
        T.taper_set_trace_buffer(tr, cap)
        call()
        T.taper_set_trace_buffer(None)
        for _ in range(2):
            call()
        torch.cuda.synchronize()
        a = tr.view(cap, 16).cpu().numpy().astype(np.int64)
        at = a[3000:3148, :3]
        mt = a[3200:3200 + b.n_slot, :2]
        mt = mt[mt[:, 0] > 0]
        t0 = at[:, 0].min()
        print(f"rep {rep}: attend CTA start {0:.1f}..{(at[:, 0].max() - t0) / 1e3:.1f} us, "
              f"first TMA median {(np.median(at[:, 2]) - t0) / 1e3:.1f}, end min/med/max "
              f"{(at[:, 1].min() - t0) / 1e3:.1f}/{(np.median(at[:, 1]) - t0) / 1e3:.1f}/"
              f"{(at[:, 1].max() - t0) / 1e3:.1f}; merge CTAs {len(mt)} start min/max "
              f"{(mt[:, 0].min() - t0) / 1e3:.1f}/{(mt[:, 0].max() - t0) / 1e3:.1f} end max "
              f"{(mt[:, 1].max() - t0) / 1e3:.1f} us")
        tr.zero_()
    # back-to-back per-layer time from events over 20 calls
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        call()
    e1.record()
    torch.cuda.synchronize()
    print(f"back-to-back per call: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
    prof = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(20)]
    for pe in prof:
        for e in pe:
            e.record()
    e0.record()
    for i in range(20):
        T.taper_set_profile_events(prof[i])
        call()
    T.taper_set_profile_events(None)
    e1.record()
    torch.cuda.synchronize()
    att = np.mean([p[0].elapsed_time(p[1]) for p in prof]) * 1e3
    mer = np.mean([p[1].elapsed_time(p[2]) for p in prof]) * 1e3
    print(f"with 3 events per call: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us (attend {att:.1f}, merge {mer:.1f})")
    pools = [kv]
    for i in range(7):
        k2 = torch.randn(shape, generator=g, device="cuda", dtype=torch.bfloat16)
        v2 = torch.randn(shape, generator=g, device="cuda", dtype=torch.bfloat16)
        pools.append(T.DeviceKV(k2, v2, rpo, rp, spo, sp))
    e0.record()
    for i in range(24):
        T.taper_decode_attention(db, adm, pools[i % 8], q, out, None, 1 / math.sqrt(128), ws)
    e1.record()
    torch.cuda.synchronize()
    print(f"8 distinct KV pools, per call: {e0.elapsed_time(e1) / 24 * 1e3:.1f} us")


if __name__ == "__main__":
    main()
