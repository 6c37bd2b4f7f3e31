"""NEXT-2 closed loop on the GPU (scripts/closed_loop.py): every step of a synthetic trace is
admitted by the device taper_admit AND by the literal Alg. 1 oracle,
which must agree bit for bit on the admitted set and on T(S) -- along a trajectory the
admission itself drives (the realised step time feeds the next step's slack).  The step
clock is the App. C.1 linear model (L316) so the trajectory is deterministic.  The
no-replanning ablation (Table 1) hands its composed mask to taper_build_work."""
import importlib.util
import os
import sys

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_spec = importlib.util.spec_from_file_location("closed_loop", os.path.join(ROOT, "scripts", "closed_loop.py"))
CL = importlib.util.module_from_spec(_spec)
sys.modules["closed_loop"] = CL
_spec.loader.exec_module(CL)

MODEL = (0.707 + CL.REST[0], 0.0107 + CL.REST[1], 4.07e-5)


def _gpu_drivers(stats):
    from paper_2605_06914_b200 import taper as T
    ws = torch.empty(T.taper_workspace_size(T.TAPER_MAX_SLOTS, T.TAPER_MAX_SLOTS, 8, 1 << 14),
                     dtype=torch.uint8, device="cuda")
    state = {}

    def admit_fn(b, policy, rho, model):
        kind, cap = CL.POLICY_ARGS[policy]
        db = T.DeviceBatch.from_host(b)
        adm = T.DeviceAdmission.empty(b.n_req, b.n_slot)
        T.taper_admit(db, model, kind, rho, adm, 8, ws, cap, ctx="per_request")
        mask = adm.slot_admitted.cpu().numpy()[:b.n_slot].astype(bool)
        t_s = float(adm.diag[2].item())
        o = oracle.admit(b.req_shared_len, b.req_slot_off, b.req_slack_ms, b.slot_local_len,
                         model, kind, cap, rho, ctx="per_request")
        assert int(adm.status.item()) == 0
        assert np.array_equal(mask, o.slot_admitted.astype(bool)), stats["steps"]
        assert np.float64(t_s).tobytes() == np.float64(o.T_S).tobytes()
        assert (adm.req_width.cpu().numpy()[:b.n_req] >= 1).all()  # every request advances
        stats["steps"] += 1
        state["db"], state["adm"] = db, adm
        return mask, t_s

    def set_mask(b, mask):
        state["adm"].slot_admitted[:b.n_slot].copy_(torch.from_numpy(mask.astype(np.uint8)))
        T.taper_build_work(state["db"], state["adm"], 8, ws)
        assert int(state["adm"].n_adm.item()) == int(mask.sum())
        stats["rebuilt"] += 1

    def step_fn(b, mask):
        return MODEL[0] + MODEL[1] * int(mask.sum()) + MODEL[2] * CL.context_per_request(b, mask)

    return admit_fn, step_fn, set_mask


@pytest.mark.parametrize("policy,ablation", [("taper", None), ("taper", "noreplan"), ("cap2", None)])
def test_closed_loop_device_admission_equals_oracle_every_step(policy, ablation):
    stats = {"steps": 0, "rebuilt": 0}
    admit_fn, step_fn, set_mask = _gpu_drivers(stats)
    r = CL.run(policy, admit_fn, step_fn, 220, seed=4, model=MODEL, ablation=ablation,
               set_mask=set_mask)
    assert stats["steps"] >= 200
    assert r["finished"] > 5 and 0.0 <= r["attainment"] <= 1.0
    if ablation == "noreplan":
        assert stats["rebuilt"] > 0
