"""Test-side plumbing: build a case from synth, run the CUDA path through the C ABI,
and compare with the oracle.  Holds no method arithmetic."""
from __future__ import annotations

import math

import numpy as np
import torch

import oracle
import synth

TOL_ABS, TOL_REL = 2e-3, 1e-2  # BASELINE.json north_star; allclose reading [C-att-5]


class Case:
    def __init__(self, batch, page=64, h_kv=8, seed=0, variant="flat", local_capacity=None,
                 layout_seed=1, device_kv=False):
        self.batch = batch
        self.h_kv = h_kv
        self.layout = synth.make_layout(batch, page, np.random.default_rng(layout_seed),
                                        spare_pages=1, local_capacity=local_capacity)
        # device_kv: draw the pools on the GPU (full-size configs: tens of GB of bf16) and
        # keep a host copy for the oracle; the GPU run then uses the device pools as drawn
        self.kv_dev = None
        if device_kv:
            kd, vd = synth.make_kv(self.layout.num_pages, h_kv, page, 128, seed, device="cuda")
            self.kv_dev = (kd, vd)
            self.k, self.v = kd.cpu(), vd.cpu()
        else:
            self.k, self.v = synth.make_kv(self.layout.num_pages, h_kv, page, 128, seed)
        gain = 4.0 if variant == "peaked" else 1.0
        self.q = synth.make_q(batch.n_slot, 8 * h_kv, 128, seed, gain)
        if variant == "sink":
            synth.plant_sink(self.k, self.q, batch, self.layout)
        self.scale = 1.0 / math.sqrt(128)

    # ------------------------------------------------------------- CUDA path
    def run_gpu(self, model=(12.0, 0.03, 2e-5), policy="eager", rho=0.8, cap=2, heads=None,
                with_lse=True):
        from paper_2605_06914_b200 import taper as T
        b = self.batch
        dev = "cuda"
        g0, g1 = (0, self.h_kv) if heads is None else heads
        h = g1 - g0
        db = T.DeviceBatch.from_host(b, dev)
        adm = T.DeviceAdmission.empty(b.n_req, b.n_slot, dev)
        ws_bytes = T.taper_workspace_size(b.n_req, b.n_slot, h,
                                          T.max_chunk_slots(b.req_shared_len, b.req_slot_off,
                                                            b.slot_local_len, b.seg_len))
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        T.taper_admit(db, model, policy, rho, adm, h, ws, cap)
        rpo, rp, spo, sp = T.page_tables_to_device(self.layout, dev)
        spg = None
        if self.layout.seg_page_off is not None:
            spg = torch.as_tensor(np.concatenate([self.layout.seg_page_off, [0]]).astype(np.int32)).to(dev)
        if self.kv_dev is not None and (g0, g1) == (0, self.h_kv):
            kd, vd = self.kv_dev
        else:
            kd, vd = self.k[:, g0:g1].contiguous().to(dev), self.v[:, g0:g1].contiguous().to(dev)
        kv = T.DeviceKV(kd, vd, rpo, rp, spo, sp, spg)
        q = self.q[:, 8 * g0:8 * g1].contiguous().to(dev)
        out = torch.full_like(q, float("nan"))
        lse = torch.full((b.n_slot, 8 * h), float("nan"), device=dev) if with_lse else None
        T.taper_decode_attention(db, adm, kv, q, out, lse, self.scale, ws)
        torch.cuda.synchronize()
        return adm, out.cpu(), (lse.cpu() if with_lse else None)

    # ------------------------------------------------------------- oracle
    def run_oracle(self, slots, qheads):
        b, lay = self.batch, self.layout
        return oracle.attention(b.req_slot_off, b.req_shared_len, b.slot_local_len,
                                lay.req_page_off, lay.req_pages, lay.slot_page_off,
                                lay.slot_pages, self.k, self.v, self.q, slots, qheads,
                                self.scale, b.slot_seg_off, b.seg_len, lay.seg_page_off)


# C-att-5 diagnostics of every comparison (max abs error, max relative error over |r| >= 1e-3,
# worst bound use), written by tests/conftest.py to gpurun_out/parity_diagnostics.json
DIAGNOSTICS: list[dict] = []


def assert_close(gpu: np.ndarray, ref: np.ndarray, what=""):
    """Pass iff every element satisfies |x - r| <= 2e-3 + 1e-2 |r| [C-att-5]."""
    gpu = np.asarray(gpu, np.float64)
    err = np.abs(gpu - ref)
    bound = TOL_ABS + TOL_REL * np.abs(ref)
    big = np.abs(ref) >= 1e-3
    DIAGNOSTICS.append({
        "what": what, "elements": int(err.size),
        "max_abs": float(np.nanmax(err)) if err.size else 0.0,
        "max_rel": float(np.nanmax(err[big] / np.abs(ref[big]))) if big.any() else 0.0,
        "max_bound_use": float(np.nanmax(err / bound)) if err.size else 0.0})
    bad = ~(err <= bound)
    if bad.any():
        i = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {bad.sum()} elements out of tolerance; first at {tuple(i)}: "
                             f"gpu={gpu[tuple(i)]!r} ref={ref[tuple(i)]!r} "
                             f"max_abs={err.max():.3e}")
    return float(err.max())
