"""Dev tool (GPU box): globaltimer timeline across two PDL-chained attention calls (C2 one
rank of G by default): call 1's attend CTA ends and merge CTA ends, call 2's attend CTA
starts, grid-dependency resolution and first TMA.  python scripts/trace_chain.py [cfg] [h]"""
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
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    h = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    b = synth.config_batch(cfg, seed=0)
    lay = synth.make_layout(b, 64, np.random.default_rng(1), 1)
    db = T.DeviceBatch.from_host(b)
    adm = T.DeviceAdmission.empty(b.n_req, b.n_slot)
    ws = torch.empty(T.taper_workspace_size(b.n_req, b.n_slot, h, T.max_chunk_slots(
        b.req_shared_len, b.req_slot_off, b.slot_local_len)), dtype=torch.uint8, device="cuda")
    T.taper_admit(db, (12.0, 0.03, 2e-5), "eager", 0.8, adm, h, ws)
    g = torch.Generator(device="cuda").manual_seed(0)
    shape = (lay.num_pages, h, 64, 128)
    rpo, rp, spo, sp = T.page_tables_to_device(lay)
    kvs = [T.DeviceKV(torch.randn(shape, generator=g, device="cuda", dtype=torch.bfloat16),
                      torch.randn(shape, generator=g, device="cuda", dtype=torch.bfloat16), rpo, rp, spo, sp)
           for _ in range(3)]
    q = torch.randn((b.n_slot, 8 * h, 128), generator=g, device="cuda", dtype=torch.bfloat16)
    out = torch.empty_like(q)
    sc = 1 / math.sqrt(128)
    for i in range(6):
        T.taper_decode_attention(db, adm, kvs[i % 3], q, out, None, sc, ws)
    cap = 3600
    bufs = [torch.zeros(cap * 16, dtype=torch.int64, device="cuda") for _ in range(2)]
    torch.cuda.synchronize()
    T.taper_decode_attention(db, adm, kvs[0], q, out, None, sc, ws)  # keeps the chain busy
    for i in range(2):
        T.taper_set_trace_buffer(bufs[i], cap)
        T.taper_decode_attention(db, adm, kvs[1 + i], q, out, None, sc, ws)
    T.taper_set_trace_buffer(None)
    torch.cuda.synchronize()
    a = [x.view(cap, 16).cpu().numpy().astype(np.int64) for x in bufs]
    att = [x[3000:3000 + 148] for x in a]
    mer = [x[3200:3200 + b.n_slot] for x in a]
    t0 = att[0][:, 0].min()
    us = lambda v: (v - t0) / 1e3
    for i in range(2):
        s, e = att[i][:, 0], att[i][:, 1]
        print(f"call {i}: attend CTA start min/med/max {us(s.min()):.1f}/{us(np.median(s)):.1f}/{us(s.max()):.1f}"
              f"  end min/med/max {us(e.min()):.1f}/{us(np.median(e)):.1f}/{us(e.max()):.1f}")
        for ev, name in ((8, "grid dependency"), (2, "first TMA"), (10, "first Q landed")):
            v = att[i][:, ev]
            v = v[v > 0]
            if len(v):
                print(f"   {name}: min/med/max {us(v.min()):.1f}/{us(np.median(v)):.1f}/{us(v.max()):.1f}")
        ms, me = mer[i][:, 0], mer[i][:, 1]
        ok = (ms > 0) & (me > 0)
        if ok.any():
            print(f"   merge CTA start min/med/max {us(ms[ok].min()):.1f}/{us(np.median(ms[ok])):.1f}/{us(ms[ok].max()):.1f}"
                  f"  end min/med/max {us(me[ok].min()):.1f}/{us(np.median(me[ok])):.1f}/{us(me[ok].max()):.1f}")


if __name__ == "__main__":
    main()
