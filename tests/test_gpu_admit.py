"""GPU parity of taper_admit against the literal Alg. 1 oracle: bit-exact widths,
admitted sets, T0 / budget / T(S) / E / min-slack fp64 bits, adm_list and status."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


def _gpu_admit(b, model, policy, rho, cap=2, h=8, ctx="per_sequence", utility=None):
    from paper_2605_06914_b200 import taper as T
    db = T.DeviceBatch.from_host(b)
    adm = T.DeviceAdmission.empty(b.n_req, b.n_slot)
    ws = torch.empty(T.taper_workspace_size(b.n_req, b.n_slot, h,
                                            T.max_chunk_slots(b.req_shared_len, b.req_slot_off, b.slot_local_len)),
                     dtype=torch.uint8, device="cuda")
    u = None if utility is None else torch.as_tensor(utility, dtype=torch.float64).cuda()
    T.taper_admit(db, model, policy, rho, adm, h, ws, cap, ctx=ctx, utility=u)
    torch.cuda.synchronize()
    return adm


def _compare(b, model, policy, rho, cap=2, ctx="per_sequence", utility=None):
    g = _gpu_admit(b, model, policy, rho, cap, ctx=ctx, utility=utility)
    o = oracle.admit(b.req_shared_len, b.req_slot_off, b.req_slack_ms, b.slot_local_len, model,
                     policy, cap, rho, utility=utility, ctx=ctx)
    R, S = b.n_req, b.n_slot
    np.testing.assert_array_equal(g.req_width.cpu().numpy()[:R], o.req_width)
    np.testing.assert_array_equal(g.slot_admitted.cpu().numpy()[:S], o.slot_admitted)
    d = g.diag.cpu().numpy()
    ref = np.array([o.T0, o.budget, o.T_S, o.E, o.min_slack])
    assert d.tobytes() == ref.tobytes(), (d, ref)  # bit-exact fp64
    n_adm = int(g.n_adm.item())
    assert n_adm == int(o.slot_admitted.sum())
    np.testing.assert_array_equal(g.adm_list.cpu().numpy()[:n_adm], np.flatnonzero(o.slot_admitted))
    st = int(g.status.item())
    assert (st & 1) == (o.status & 1) and (st & ~(1 | 4 | 32)) == 0, st
    # TAPER_STATUS_EMPTY_CONTEXT iff some admitted slot has Lsh_r + Lloc_s = 0 [C-att-4]
    req = np.searchsorted(b.req_slot_off, np.arange(S), side="right") - 1
    empty = (o.slot_admitted.astype(bool) & (b.req_shared_len[req] == 0) & (b.slot_local_len == 0)).any()
    assert bool(st & 32) == bool(empty), st
    return o


@pytest.mark.parametrize("ctx", ["per_sequence", "per_request"])
@pytest.mark.parametrize("policy", ["off", "cap", "eager", "taper"])
def test_random_small_batches(policy, ctx):
    rng = np.random.default_rng(42)
    for i in range(300):
        b = synth.random_small_batch(rng, max_req=12, max_fanout=6, max_local=50)
        model = (rng.uniform(0, 20), rng.uniform(1e-3, 0.1), rng.uniform(1e-5, 1e-2))
        _compare(b, model, policy, float(rng.uniform(0.05, 1.0)), cap=int(rng.integers(1, 6)),
                 ctx=ctx)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c5"])
@pytest.mark.parametrize("x", [-0.5, 0.0, 0.3, 0.7, 2.0])
def test_config_batches_all_regimes(name, x):
    # slack placed relative to T0 and T_eager: ms = T0 + x (T_eager - T0) / rho
    model, rho = (12.0, 0.03, 2e-5), 0.8
    b = synth.config_batch(name, seed=3, slack_min_ms=0.0)
    o_off = oracle.admit(b.req_shared_len, b.req_slot_off, b.req_slack_ms + 1e9, b.slot_local_len,
                         model, "off")
    o_eag = oracle.admit(b.req_shared_len, b.req_slot_off, b.req_slack_ms + 1e9, b.slot_local_len,
                         model, "eager")
    ms = o_off.T0 + x * (o_eag.T_S - o_off.T0) / rho
    b.req_slack_ms = ms + np.random.default_rng(1).uniform(0, 20, size=b.n_req)
    b.req_slack_ms[0] = ms
    for pol in ("off", "eager", "taper", "cap"):
        o = _compare(b, model, pol, rho, cap=2)
        if pol == "taper":
            frac = (o.req_width.sum() - b.n_req) / max(1, b.n_slot - b.n_req)
            if x <= 0:
                assert frac == 0
            if x >= 1.0:
                assert frac == 1.0


def test_many_ties_and_capacity_limits():
    rng = np.random.default_rng(5)
    # all branches equal length -> ties resolved by (r, slot)
    b = synth.make_batch([100] * 50, [5] * 50, [7] * 250, 30.0, 5.0, rng=rng)
    _compare(b, (5.0, 0.05, 0.001), "taper", 0.5)
    # maximum size: 4096 slots
    fan = np.full(1024, 4)
    b = synth.make_batch(rng.integers(0, 32768, 1024), fan, rng.integers(0, 512, 4096), 40.0, 20.0,
                         rng=rng)
    for pol in ("taper", "cap", "eager"):
        _compare(b, (12.0, 0.03, 2e-5), pol, 0.8, cap=3)


def test_empty_inputs_and_empty_request():
    b = synth.make_batch([], [], [], 10.0, 0.0)
    g = _gpu_admit(b, (3.0, 0.1, 0.01), "taper", 0.8)
    assert g.diag.cpu().numpy()[0] == 3.0 and int(g.n_adm.item()) == 0
    b = synth.make_batch([10, 20], [0, 2], [1, 2], 50.0, 0.0)
    b.req_slack_ms[:] = [5.0, 50.0]
    o = _compare(b, (1.0, 0.1, 0.01), "eager", 0.8)
    assert o.status == 1


def test_invalid_arguments_rejected():
    from paper_2605_06914_b200 import taper as T
    b = synth.config_batch("c1")
    with pytest.raises(T.TaperError, match="rho"):
        _gpu_admit(b, (1.0, 0.1, 0.01), "taper", 0.0)
    with pytest.raises(T.TaperError, match="monotone"):
        _gpu_admit(b, (1.0, 0.0, 0.01), "taper", 0.8)
    with pytest.raises(T.TaperError, match="monotone"):
        _gpu_admit(b, (1.0, 0.1, -1.0), "taper", 0.8)


# ---------------------------------------------------------------- non-linear utilities
# Sec. 3.4 (L142) "pluggable utility interface"; Alg. 1 line 15 (L167).  The device runs
# Alg. 1's loop literally for a utility table; it must match the literal oracle bit for bit.

@pytest.mark.parametrize("ctx", ["per_sequence", "per_request"])
@pytest.mark.parametrize("kind", ["concave", "weighted", "plateau", "linear"])
def test_utility_tables_match_oracle(kind, ctx):
    rng = np.random.default_rng(7)
    for i in range(200):
        b = synth.random_small_batch(rng, max_req=14, max_fanout=7, max_local=50)
        K = int(rng.integers(2, 9))  # short tables exercise the flat extension
        util = synth.utility_table(rng, b.n_req, K, kind)
        model = (rng.uniform(0, 20), rng.uniform(1e-3, 0.1), rng.uniform(1e-5, 1e-2))
        _compare(b, model, "taper", float(rng.uniform(0.05, 1.0)), ctx=ctx, utility=util)


def test_linear_table_equals_sort_scan_path():
    """u_r(k) = k as a table (literal loop on the device) == utility=NULL (sort + scan):
    two device formulations of Alg. 1 that share no code past the candidate keys."""
    rng = np.random.default_rng(11)
    for name in ("c2", "c5"):
        b = synth.config_batch(name, seed=2, slack_min_ms=0.0)
        b.req_slack_ms = 40.0 + rng.uniform(0, 20, size=b.n_req)
        K = int(np.diff(b.req_slot_off).max()) + 1
        lin = synth.utility_table(rng, b.n_req, K, "linear")
        for rho in (0.2, 0.5, 0.8, 1.0):
            g1 = _gpu_admit(b, (12.0, 0.03, 2e-5), "taper", rho, utility=lin)
            g2 = _gpu_admit(b, (12.0, 0.03, 2e-5), "taper", rho)
            assert torch.equal(g1.slot_admitted, g2.slot_admitted)
            assert g1.diag.cpu().numpy().tobytes() == g2.diag.cpu().numpy().tobytes()


@pytest.mark.parametrize("kind", ["concave", "weighted"])
def test_utility_config_batches(kind):
    """Config-sized batches (c2: 64 requests; c5: 256 requests, ~390 candidates), every
    regime of the budget, bit-exact against the literal oracle."""
    rng = np.random.default_rng(13)
    for name in ("c2", "c5"):
        b = synth.config_batch(name, seed=4, slack_min_ms=0.0)
        util = synth.utility_table(rng, b.n_req, 17, kind)
        for base in (10.0, 30.0, 45.0, 80.0):
            b.req_slack_ms = base + rng.uniform(0, 20, size=b.n_req)
            _compare(b, (12.0, 0.03, 2e-5), "taper", 0.8, utility=util)


@pytest.mark.parametrize("R", [1024, 2048])
def test_utility_max_capacity(R):
    """4096 slots; R = 2048 gives every admission thread two requests (kOwn > 1)."""
    rng = np.random.default_rng(17)
    fan = np.full(R, 4096 // R)
    b = synth.make_batch(rng.integers(0, 32768, R), fan, rng.integers(0, 512, 4096), 40.0, 20.0,
                         rng=rng)
    util = synth.utility_table(rng, b.n_req, 4, "concave")
    _compare(b, (12.0, 0.03, 2e-5), "taper", 0.8, utility=util)


def test_utility_stride_validated():
    from paper_2605_06914_b200 import taper as T
    b = synth.config_batch("c1")
    with pytest.raises(T.TaperError, match="utility_stride"):
        _gpu_admit(b, (1.0, 0.1, 0.01), "taper", 0.8, utility=np.zeros((b.n_req, 1)))
