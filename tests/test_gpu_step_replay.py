"""Config 4 (BASELINE.json configs[3]) through the whole decode step on the GPU.

For 240 TraceReplay steps (330-569: the end of the low-load regime and most of the high-load
one; the earlier steps advance the trace on the host), every step
enqueues taper_admit -> taper_append_kv -> taper_decode_attention back to back on ONE
workspace and ONE stream while the batch state, the page tables and the admitted set change
from step to step.  Nothing synchronises the host between a step's calls, and step t + 1 is
enqueued before step t is checked, so a stale hand-off between the admission and the
attention (the attention kernel resolves its first work item before its grid dependency
resolves, include/taper.h "Ordering contract") or between two steps would show up here.
Checks per step: the admission bit-exact vs the literal Alg. 1 oracle,
and sampled (slot, Q head) outputs vs the fp64 oracle on the cache as the appends of
steps 0..t left it ([C-att-3]: the current token is the last position of the context).
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.helpers import assert_close
from tests.test_trace_replay import MODEL, RHO, _slack

pytestmark = pytest.mark.gpu

FIRST, N_STEPS = 330, 240  # GPU steps FIRST .. FIRST + N_STEPS - 1 (low load ends at 400)
PAGE = 64


def _append_rows(b, lay, mask):
    """(slot, page, row) of each admitted slot's current token [C-att-3] (test-side)."""
    off = b.req_slot_off
    rows = []
    for s in np.flatnonzero(mask):
        r = int(np.searchsorted(off, s, side="right") - 1)
        if b.slot_local_len[s] > 0:
            t = int(b.slot_local_len[s]) - 1
            page = lay.slot_pages[lay.slot_page_off[s] + t // PAGE]
        else:
            t = int(b.req_shared_len[r]) - 1
            page = lay.req_pages[lay.req_page_off[r] + t // PAGE]
        rows.append((int(s), int(page), t % PAGE))
    return rows


@pytest.mark.parametrize("policy", ["taper"])
def test_step_replay_admit_append_attend(policy):
    from paper_2605_06914_b200 import taper as T
    tr = synth.TraceReplay(seed=4)
    # the whole trajectory first (host): batches, slack, oracle admissions; the GPU's
    # admission must equal the oracle's, so the oracle's drives the replay
    steps = []
    for t in range(FIRST + N_STEPS):
        b = tr.batch()
        _slack(tr, b)
        o = oracle.admit(b.req_shared_len, b.req_slot_off, b.req_slack_ms, b.slot_local_len,
                         MODEL, policy, 2, RHO)
        if t >= FIRST:
            steps.append((b, o))
        tr.advance(o.slot_admitted)
    need = max(int(((b.req_shared_len.astype(np.int64) + PAGE - 1) // PAGE).sum()
                   + ((b.slot_local_len.astype(np.int64) + PAGE - 1) // PAGE).sum())
               for b, _ in steps)
    P = need + 8
    R_max = max(b.n_req for b, _ in steps)
    S_max = max(b.n_slot for b, _ in steps)
    dev = "cuda"
    stream = torch.cuda.Stream()
    k_host, v_host = synth.make_kv(P, 8, PAGE, 128, seed=11)  # the host mirror of the pools
    kd, vd = k_host.to(dev), v_host.to(dev)
    cs = max(T.max_chunk_slots(b.req_shared_len, b.req_slot_off, b.slot_local_len) for b, _ in steps)
    ws = torch.empty(T.taper_workspace_size(R_max, S_max, 8, cs), dtype=torch.uint8, device=dev)
    adm = T.DeviceAdmission.empty(R_max, S_max, dev)
    # device copies of the changing batch state / page tables (max sizes, written in place)
    dbuf = {k: torch.zeros(n, dtype=dt, device=dev) for k, n, dt in
            [("lsh", R_max, torch.int32), ("off", R_max + 1, torch.int32),
             ("slack", R_max, torch.float64), ("lloc", S_max, torch.int32),
             ("rpo", R_max + 1, torch.int32), ("rp", P, torch.int32),
             ("spo", S_max + 1, torch.int32), ("sp", P, torch.int32)]}
    g = torch.Generator().manual_seed(5)
    pending = []  # enqueued, unchecked steps

    def enqueue(t):
        b, o = steps[t]
        R, S = b.n_req, b.n_slot
        need_t = int(((b.req_shared_len.astype(np.int64) + PAGE - 1) // PAGE).sum()
                     + ((b.slot_local_len.astype(np.int64) + PAGE - 1) // PAGE).sum())
        # a fresh random page assignment of the whole pool every step
        lay = synth.make_layout(b, PAGE, np.random.default_rng(1000 + t), spare_pages=P - need_t)
        assert lay.num_pages == P
        host = {"lsh": b.req_shared_len, "off": b.req_slot_off, "slack": b.req_slack_ms,
                "lloc": b.slot_local_len, "rpo": lay.req_page_off, "rp": lay.req_pages,
                "spo": lay.slot_page_off, "sp": lay.slot_pages}
        pinned = {k: torch.as_tensor(np.ascontiguousarray(v)).pin_memory() for k, v in host.items()}
        k_new = torch.randn((S, 8, 128), generator=g).bfloat16()
        v_new = torch.randn((S, 8, 128), generator=g).bfloat16()
        q = synth.make_q(S, 64, 128, seed=t)
        pin_x = [k_new.pin_memory(), v_new.pin_memory(), q.pin_memory()]
        with torch.cuda.stream(stream):
            for k, v in pinned.items():
                dbuf[k][:v.numel()].copy_(v, non_blocking=True)
            kn, vn, qd = (x.to(dev, non_blocking=True) for x in pin_x)
            db = T.DeviceBatch(dbuf["lsh"][:R], dbuf["off"][:R + 1], dbuf["slack"][:R],
                               dbuf["lloc"][:S])
            kv = T.DeviceKV(kd, vd, dbuf["rpo"][:R + 1], dbuf["rp"], dbuf["spo"][:S + 1], dbuf["sp"])
            T.taper_admit(db, MODEL, policy, RHO, adm, 8, ws, 2, stream=stream)
            T.taper_append_kv(db, adm, kv, kn, vn, stream=stream)
            out = torch.full((S, 64, 128), float("nan"), dtype=torch.bfloat16, device=dev)
            T.taper_decode_attention(db, adm, kv, qd, out, None, 128 ** -0.5, ws, stream=stream)
            res = {"mask": adm.slot_admitted[:S].to("cpu", non_blocking=True),
                   "diag": adm.diag.to("cpu", non_blocking=True),
                   "status": adm.status.to("cpu", non_blocking=True),
                   "out": out.to("cpu", non_blocking=True)}
            ev = torch.cuda.Event()
            ev.record(stream)
        pending.append((t, lay, k_new, v_new, q, res, ev, pinned, pin_x, (kn, vn, qd, out)))

    def check(item):
        t, lay, k_new, v_new, q, res, ev, *_ = item
        b, o = steps[t]
        ev.synchronize()
        assert int(res["status"][0]) == 0, (t, T.taper_status_string(int(res["status"][0])))
        mask = res["mask"].numpy()
        assert (mask == o.slot_admitted).all(), t
        d = res["diag"].numpy()
        assert d.tobytes() == np.array([o.T0, o.budget, o.T_S, o.E, o.min_slack]).tobytes(), t
        for s, page, row in _append_rows(b, lay, mask):  # the mirror takes step t's appends
            k_host[page, :, row] = k_new[s]
            v_host[page, :, row] = v_new[s]
        rng = np.random.default_rng(t)
        adm_slots = np.flatnonzero(mask)
        slots = np.sort(rng.choice(adm_slots, min(6, len(adm_slots)), replace=False))
        es, eh = np.repeat(slots, 2), np.tile(rng.choice(64, 2, replace=False), len(slots))
        ref, _ = oracle.attention(b.req_slot_off, b.req_shared_len, b.slot_local_len,
                                  lay.req_page_off, lay.req_pages, lay.slot_page_off,
                                  lay.slot_pages, k_host, v_host, q, es, eh)
        assert_close(res["out"][es, eh].float().numpy(), ref, f"step {t}")
        assert torch.isfinite(res["out"][adm_slots].float()).all(), t
        na = np.flatnonzero(mask == 0)
        assert torch.isnan(res["out"][na].float()).all(), t  # non-admitted slots untouched

    rates = []
    for t in range(N_STEPS):
        enqueue(t)
        if len(pending) > 2:  # step t-2 is checked while t-1 and t are in flight
            check(pending.pop(0))
        b, o = steps[t]
        rates.append((o.slot_admitted.sum() - b.n_req) / max(b.n_slot - b.n_req, 1))
    while pending:
        check(pending.pop(0))
    rates = np.array(rates)
    # the replay crossed the regimes: full admission at low load, partial under stress
    n_low = 400 - FIRST
    assert rates[:n_low].mean() > 0.9 and rates[n_low:].mean() < 0.5
    # and the final device pools equal the mirror (every append landed, nothing else moved)
    torch.cuda.synchronize()
    assert torch.equal(kd.cpu(), k_host) and torch.equal(vd.cpu(), v_host)
