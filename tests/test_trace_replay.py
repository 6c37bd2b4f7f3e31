"""Config 4 (BASELINE.json configs[3]): 1000-step trace replay with per-step admission
under a varying slack schedule (low / high / moderate load, P385 regime proportions).
CPU: the oracle's TAPER behaves like the paper's regimes (P206-210).  GPU: taper_admit
is bit-exact against the oracle on every step for IRP-Off, IRP-Eager and TAPER."""
import numpy as np
import pytest
import torch

import oracle
import synth

MODEL, RHO = (12.0, 0.03, 2e-5), 0.8


def _slack(tr, b):
    off = oracle.admit(b.req_shared_len, b.req_slot_off, b.req_slack_ms + 1e9, b.slot_local_len,
                       MODEL, "off")
    eag = oracle.admit(b.req_shared_len, b.req_slot_off, b.req_slack_ms + 1e9, b.slot_local_len,
                       MODEL, "eager")
    x = tr.slack_x()
    b.req_slack_ms = b.req_slack_ms + off.T0 + x * (eag.T_S - off.T0) / RHO


def test_replay_regimes_oracle():
    tr = synth.TraceReplay(seed=1)
    rate = []
    for step in range(1000):
        b = tr.batch()
        _slack(tr, b)
        a = oracle.admit(b.req_shared_len, b.req_slot_off, b.req_slack_ms, b.slot_local_len,
                         MODEL, "taper", 2, RHO)
        assert (a.req_width >= 1).all() and a.T_S <= a.budget  # P128, P136
        opp = b.n_slot - b.n_req
        rate.append((a.req_width.sum() - b.n_req) / max(opp, 1))
        tr.advance(a.slot_admitted)
    rate = np.array(rate)
    low, high, mod = rate[:400].mean(), rate[400:650].mean(), rate[650:].mean()
    # P206-210: ~100 % admission at low load, contracts under stress, partial recovery
    assert low > 0.95 and high < 0.3 and high < mod < low


@pytest.mark.gpu
@pytest.mark.parametrize("policy", ["off", "eager", "taper"])
def test_replay_gpu_bit_exact(policy):
    from paper_2605_06914_b200 import taper as T
    tr = synth.TraceReplay(seed=2)
    ws = torch.empty(T.taper_workspace_size(T.TAPER_MAX_SLOTS, T.TAPER_MAX_SLOTS, 8, 8192),
                     dtype=torch.uint8, device="cuda")
    for step in range(1000):
        b = tr.batch()
        _slack(tr, b)
        o = oracle.admit(b.req_shared_len, b.req_slot_off, b.req_slack_ms, b.slot_local_len,
                         MODEL, policy, 2, RHO)
        db = T.DeviceBatch.from_host(b)
        adm = T.DeviceAdmission.empty(b.n_req, b.n_slot)
        T.taper_admit(db, MODEL, policy, RHO, adm, 8, ws)
        g_adm = adm.slot_admitted.cpu().numpy()[:b.n_slot]
        assert (g_adm == o.slot_admitted).all(), step
        d = adm.diag.cpu().numpy()
        assert d.tobytes() == np.array([o.T0, o.budget, o.T_S, o.E, o.min_slack]).tobytes(), step
        tr.advance(o.slot_admitted)
