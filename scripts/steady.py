"""Dev tool: steady-state (power-capped) per-call time of taper_decode_attention on C2:
~4 s of back-to-back calls over 8 KV pools while nvidia-smi samples clocks / power; reports
the per-call time of the last 2 s and the median SM clock / board power there."""
import math
import os
import subprocess
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_06914_b200 import taper as T  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    b = synth.config_batch(cfg, seed=0)
    lay = synth.make_layout(b, 64, np.random.default_rng(1), 1)
    db = T.DeviceBatch.from_host(b)
    adm = T.DeviceAdmission.empty(b.n_req, b.n_slot)
    ws = torch.empty(T.taper_workspace_size(b.n_req, b.n_slot, 8, T.max_chunk_slots(
        b.req_shared_len, b.req_slot_off, b.slot_local_len)), dtype=torch.uint8, device="cuda")
    T.taper_admit(db, (12.0, 0.03, 2e-5), "eager", 0.8, adm, 8, ws)
    g = torch.Generator(device="cuda").manual_seed(0)
    shape = (lay.num_pages, 8, 64, 128)
    rpo, rp, spo, sp = T.page_tables_to_device(lay)
    pools = []
    for _ in range(8):
        k = torch.randn(shape, generator=g, device="cuda", dtype=torch.bfloat16)
        v = torch.randn(shape, generator=g, device="cuda", dtype=torch.bfloat16)
        pools.append(T.DeviceKV(k, v, rpo, rp, spo, sp))
    q = torch.randn((b.n_slot, 64, 128), generator=g, device="cuda", dtype=torch.bfloat16)
    out = torch.empty_like(q)
    sc = 1 / math.sqrt(128)
    call = lambda i: T.taper_decode_attention(db, adm, pools[i % 8], q, out, None, sc, ws)
    for i in range(16):
        call(i)
    torch.cuda.synchronize()
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-lms", "100", "-i", "0"], stdout=subprocess.PIPE, text=True)
    t_start = time.time()
    i = 0
    while time.time() - t_start < 2.0:  # warm to the power cap
        for _ in range(40):
            call(i)
            i += 1
        torch.cuda.synchronize()
    t_meas = time.time()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 0
    while time.time() - t_meas < 2.0:
        for _ in range(40):
            call(i)
            i += 1
            n += 1
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    t_end = time.time()
    smi.terminate()
    lines = smi.stdout.read().strip().splitlines()
    # samples of the measured window (~last 2 s at 100 ms)
    samp = np.array([[float(x) for x in ln.split(",")] for ln in lines[-18:-2]])
    print(f"{e0.elapsed_time(e1) / n * 1e3:.1f} us/call  sm {np.median(samp[:, 0]):.0f} MHz  "
          f"{np.median(samp[:, 1]):.0f} W")


if __name__ == "__main__":
    main()
