"""Dev tool (GPU box): event-timed latency of one taper_admit call (median of 200 back-to-back
calls) per config, policy and utility kind; admission is latency-bound, so it
is reported as time.  usage: python scripts/admit_time.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_06914_b200 import taper as T  # noqa: E402

MODEL = (12.0, 0.03, 2e-5)
for cfg in ("c2", "c5"):
    b = synth.config_batch(cfg, seed=0, slack_min_ms=0.0)
    rng = np.random.default_rng(0)
    db0 = T.DeviceBatch.from_host(b)
    adm = T.DeviceAdmission.empty(b.n_req, b.n_slot)
    ws = torch.empty(T.taper_workspace_size(b.n_req, b.n_slot, 8, T.max_chunk_slots(
        b.req_shared_len, b.req_slot_off, b.slot_local_len)), dtype=torch.uint8, device="cuda")
    T.taper_admit(db0, MODEL, "off", 0.8, adm, 8, ws)
    T0 = float(adm.diag[0].item())
    T.taper_admit(db0, MODEL, "eager", 0.8, adm, 8, ws)
    Te = float(adm.diag[2].item())
    b.req_slack_ms = T0 + 0.5 * (Te - T0) / 0.8 + rng.uniform(0, 20, b.n_req)  # partial regime
    db = T.DeviceBatch.from_host(b)
    K = int(np.diff(b.req_slot_off).max())
    tables = {"linear (sort+scan)": None,
              "concave table (literal loop)": torch.as_tensor(
                  synth.utility_table(rng, b.n_req, K, "concave")).cuda()}
    for pol in ("off", "eager", "taper"):
        for name, u in tables.items():
            if pol != "taper" and u is not None:
                continue
            f = lambda: T.taper_admit(db, MODEL, pol, 0.8, adm, 8, ws, utility=u)
            for _ in range(10):
                f()
            ts = []
            for _ in range(200):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); f(); e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            n = int(adm.n_adm.item())
            print(f"{cfg} R={b.n_req} S={b.n_slot} {pol:6s} {name:30s} median {np.median(ts):7.1f} us"
                  f"  p90 {np.percentile(ts, 90):7.1f} us  admitted {n}")
