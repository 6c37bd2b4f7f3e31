"""Dev tool: back-to-back per-call time of taper_decode_attention on one C2 layer shape
(8 distinct KV pools, eager admission).  Prints the median of 5 x 32 calls in us.
The library is the one TAPER_LIB points to (default: the in-tree build)."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_06914_b200 import taper as T  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    n_pools = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    n_calls = int(sys.argv[3]) if len(sys.argv) > 3 else 32
    h = int(sys.argv[4]) if len(sys.argv) > 4 else 8  # KV heads of the rank (8 / G)
    b = synth.config_batch(cfg, seed=0)
    lay = synth.make_layout(b, 64, np.random.default_rng(1), 1,
                            contiguous=os.environ.get("LAYOUT") == "contig")
    db = T.DeviceBatch.from_host(b)
    adm = T.DeviceAdmission.empty(b.n_req, b.n_slot)
    # 2x the h = 1 bound: room for experimental finer splits (TAPER_CHUNK_MIN variants)
    ws = torch.empty(T.taper_workspace_size(b.n_req, b.n_slot, h, 2 * T.max_chunk_slots(
        b.req_shared_len, b.req_slot_off, b.slot_local_len)), dtype=torch.uint8, device="cuda")
    T.taper_admit(db, (12.0, 0.03, 2e-5), "eager", 0.8, adm, h, ws)
    assert int(adm.status.item()) == 0, T.taper_status_string(int(adm.status.item()))
    g = torch.Generator(device="cuda").manual_seed(0)
    shape = (lay.num_pages, h, 64, 128)
    rpo, rp, spo, sp = T.page_tables_to_device(lay)
    pools = []
    for _ in range(n_pools):
        k = torch.randn(shape, generator=g, device="cuda", dtype=torch.bfloat16)
        v = torch.randn(shape, generator=g, device="cuda", dtype=torch.bfloat16)
        pools.append(T.DeviceKV(k, v, rpo, rp, spo, sp))
    q = torch.randn((b.n_slot, 8 * h, 128), generator=g, device="cuda", dtype=torch.bfloat16)
    out = torch.empty_like(q)
    sc = 1 / math.sqrt(128)
    for i in range(n_pools):
        T.taper_decode_attention(db, adm, pools[i], q, out, None, sc, ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # INTERLEAVE=1: a foreign kernel between calls (as the projections / MLP of a real layer
    # would be), so the attend prologue cannot overlap the previous merge via PDL; the tiny
    # kernel's own time (~2 us) is included
    inter = os.environ.get("INTERLEAVE") == "1"
    dummy = torch.zeros(1024, device="cuda")
    ts = []
    for rep in range(5):
        e0.record()
        for i in range(n_calls):
            T.taper_decode_attention(db, adm, pools[i % n_pools], q, out, None, sc, ws)
            if inter:
                dummy.add_(1.0)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / n_calls * 1e3)
    print(" ".join(f"{t:.1f}" for t in ts), f"median {np.median(ts):.1f}")


if __name__ == "__main__":
    main()
