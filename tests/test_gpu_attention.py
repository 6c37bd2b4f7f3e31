"""GPU parity of taper_decode_attention (tcgen05 shared-prefix kernel + local split-K +
LSE merge) against the fp64 oracle, element by element, plus the closed forms and the
invariances the paper fixes (Lemma 1 / visibility rule, GQA mapping, KV-head sharding)."""
import numpy as np
import pytest
import torch

import synth
from tests.helpers import Case, assert_close

pytestmark = pytest.mark.gpu


def _check_all(case, adm, out, lse, heads=range(64), what=""):
    b = case.batch
    adm_slots = np.flatnonzero(adm.slot_admitted.cpu().numpy()[:b.n_slot])
    es, eh = np.meshgrid(adm_slots, np.asarray(list(heads)), indexing="ij")
    es, eh = es.ravel(), eh.ravel()
    ref, ref_lse = case.run_oracle(es, eh)
    got = out[es, eh].float().numpy()
    m = assert_close(got, ref, what)
    if lse is not None:
        np.testing.assert_allclose(lse[es, eh].numpy(), ref_lse, atol=2e-3, rtol=1e-4,
                                   err_msg=what + " lse")
    return m


@pytest.mark.parametrize("w1", [1, 2, 4])
def test_c1_tiny_all_widths(w1):
    b = synth.config_batch("c1", seed=0)
    case = Case(b)
    policy = {1: "off", 2: "cap", 4: "eager"}[w1]
    adm, out, lse = case.run_gpu(policy=policy, cap=2)
    assert adm.req_width.cpu().tolist()[:2] == [1, w1]
    _check_all(case, adm, out, lse, what=f"c1 w={w1}")
    # non-admitted slots are not written
    na = np.flatnonzero(adm.slot_admitted.cpu().numpy()[:b.n_slot] == 0)
    assert torch.isnan(out[na]).all()


@pytest.mark.parametrize("variant", ["flat", "peaked", "sink"])
@pytest.mark.parametrize("page", [16, 32, 64, 128])
def test_multi_chunk_ragged(variant, page):
    # prefixes spanning several 4096-token chunks with ragged tails, up to 16 branches
    # (128 stacked rows), serial requests, local lengths crossing page boundaries
    rng = np.random.default_rng(11)
    lsh = [2500, 1, 64, 4095, 4097, 9000, 0, 700]
    fan = [16, 1, 3, 1, 5, 2, 4, 9]
    loc = []
    for r, f in enumerate(fan):
        loc += ([0] if f == 1 else rng.integers(1, 300, size=f).tolist())
    if lsh[6] == 0:
        loc[sum(fan[:6]):sum(fan[:7])] = [5, 1, 70, 129]
    b = synth.make_batch(lsh, fan, loc, 1e3, 0.0, rng=rng)
    case = Case(b, page=page, seed=3, variant=variant)
    adm, out, lse = case.run_gpu(policy="eager")
    _check_all(case, adm, out, lse, what=f"{variant} page={page}")


def test_single_key_exact_and_equal_keys():
    b = synth.make_batch([1, 0, 37], [1, 1, 3], [0, 1, 0, 0, 0], 1e3, 0.0)
    case = Case(b)
    adm, out, _ = case.run_gpu(policy="eager")
    # request 0: one key -> o = bf16(v0) exactly; request 1: one local key
    for s, r in ((0, 0), (1, 1)):
        if r == 0:
            page, row = case.layout.req_pages[case.layout.req_page_off[0]], 0
        else:
            page, row = case.layout.slot_pages[case.layout.slot_page_off[1]], 0
        for hq in range(64):
            assert torch.equal(out[s, hq], case.v[page, hq // 8, row]), (s, hq)


def test_gqa_mapping_constant_v():
    b = synth.config_batch("c1", seed=1)
    case = Case(b)
    for g in range(8):
        case.v[:, g] = float(g)
    adm, out, _ = case.run_gpu(policy="eager")
    for s in range(b.n_slot):
        for hq in range(64):
            assert (out[s, hq].float() == hq // 8).all()


def test_schedule_invariance_bitwise():
    # Lemma 1 / Table 7 analog: a slot's output bits do not depend on co-admitted siblings
    b = synth.config_batch("c2", seed=2)
    case = Case(b, seed=2)
    adm_e, out_e, _ = case.run_gpu(policy="eager", with_lse=False)
    adm_c, out_c, _ = case.run_gpu(policy="cap", cap=2, with_lse=False)
    adm_o, out_o, _ = case.run_gpu(policy="off", with_lse=False)
    both = (adm_e.slot_admitted.cpu().numpy()[:b.n_slot] & adm_c.slot_admitted.cpu().numpy()[:b.n_slot]).astype(bool)
    assert torch.equal(out_e[both], out_c[both])
    proto = adm_o.slot_admitted.cpu().numpy()[:b.n_slot].astype(bool)
    assert torch.equal(out_e[proto], out_o[proto])


def test_kv_head_sharding():
    """Multi-GPU partition: the per-rank head slices of G = 2, 4, 8
    concatenated match the oracle; ranks with the same prefix split (taper_chunk_tokens:
    h = 1 and h = 2 both use 1024-token chunks) give bitwise-identical heads, and every
    slice equals the same heads of a one-GPU run with that h (a rank's result does not
    depend on which other heads exist)."""
    b = synth.config_batch("c2", seed=4)
    case = Case(b, seed=4)
    adm, full, _ = case.run_gpu(policy="eager", with_lse=False)
    cats = {}
    for G in (2, 4, 8):
        h = 8 // G
        parts = [case.run_gpu(policy="eager", heads=(g * h, (g + 1) * h), with_lse=False)[1]
                 for g in range(G)]
        cats[G] = torch.cat(parts, dim=1)
        _check_all(case, adm, cats[G], None, heads=[0, 13, 38, 63], what=f"G={G}")
    assert torch.equal(cats[4], cats[8])  # h = 2 and h = 1: same 1024-token split


def test_c2_full_size_sampled():
    # BASELINE.json configs[1] at full size, the launch configuration bench.py times;
    # every admitted slot x 4 sampled Q heads against the oracle
    b = synth.config_batch("c2", seed=0)
    case = Case(b, seed=0)
    adm, out, lse = case.run_gpu(policy="eager")
    rng = np.random.default_rng(0)
    heads = sorted(rng.choice(64, 4, replace=False).tolist())
    _check_all(case, adm, out, lse, heads=heads, what="c2")


@pytest.mark.parametrize("policy", ["taper", "cap"])
def test_partial_admission_outputs(policy):
    b = synth.config_batch("c2", seed=5, slack_min_ms=26.0)
    case = Case(b, seed=5)
    adm, out, lse = case.run_gpu(policy=policy, rho=0.8)
    n = int(adm.n_adm.item())
    assert b.n_req <= n < b.n_slot
    _check_all(case, adm, out, lse, heads=[0, 9, 63], what=policy)


@pytest.mark.parametrize("page", [16, 32, 64])
def test_garbage_past_sequence_end(page):
    """Token slots of the pool past every segment's end (the tail of its last page, spare
    pages) hold NaN: a partial tile must never let them reach O (P = 0 there, but
    0 * NaN = NaN), and the result must still match the oracle, which reads valid tokens
    only."""
    rng = np.random.default_rng(5)
    lsh = [100, 1, 64, 1000, 65, 2049]
    fan = [3, 1, 2, 5, 1, 8]
    loc = rng.integers(1, 140, size=sum(fan)).tolist()
    b = synth.make_batch(lsh, fan, loc, 1e3, 0.0, rng=rng)
    case = Case(b, page=page, seed=9)
    lay = case.layout
    valid = np.zeros((lay.num_pages, page), bool)

    def mark(pages, n_tok):
        for j, pg in enumerate(pages):
            valid[pg, : max(0, min(page, n_tok - j * page))] = True

    for r in range(b.n_req):
        mark(lay.req_pages[lay.req_page_off[r]:lay.req_page_off[r + 1]], int(b.req_shared_len[r]))
    for s in range(b.n_slot):
        mark(lay.slot_pages[lay.slot_page_off[s]:lay.slot_page_off[s + 1]], int(b.slot_local_len[s]))
    bad = torch.from_numpy(~valid)
    assert bad.any()
    case.k[bad.nonzero(as_tuple=True)[0], :, bad.nonzero(as_tuple=True)[1]] = float("nan")
    case.v[bad.nonzero(as_tuple=True)[0], :, bad.nonzero(as_tuple=True)[1]] = float("nan")
    adm, out, lse = case.run_gpu(policy="eager")
    adm_slots = np.flatnonzero(adm.slot_admitted.cpu().numpy()[:b.n_slot])
    assert torch.isfinite(out[adm_slots]).all()
    _check_all(case, adm, out, lse, what=f"nan tail page={page}")


# ------------------------------------------------------------ multi-segment local context
# Reduce steps (Sec. 3.1): the slot's local context is several segments (the
# finished branches' h_i (+) y_i in canonical order, then z), each in its own pages.

@pytest.mark.parametrize("variant", ["flat", "peaked"])
@pytest.mark.parametrize("page", [16, 64])
def test_reduce_segments_small(variant, page):
    rng = np.random.default_rng(21)
    b = synth.make_batch([300, 0, 70, 4100, 5], [1, 1, 3, 1, 2], [0] * 8, 1e3, 0.0, rng=rng)
    segs = [[17, 64, 1, 130], [1, 63, 65], [5], [200], [77], [1500, 3, 40, 2200], [], [9, 9]]
    b = synth.with_segments(b, segs)
    case = Case(b, page=page, seed=6, variant=variant)
    adm, out, lse = case.run_gpu(policy="eager")
    _check_all(case, adm, out, lse, what=f"segments {variant} page={page}")


def test_reduce_batch_sampled():
    """Reduce-step mix at the C2 prefix size (4096): serial, parallel-phase and reduce-phase
    requests (2-10 branch segments + z); every admitted slot x 4 sampled heads."""
    b = synth.reduce_batch(seed=3)
    case = Case(b, seed=3)
    adm, out, lse = case.run_gpu(policy="eager")
    heads = [0, 17, 42, 63]
    _check_all(case, adm, out, lse, heads=heads, what="reduce mix")


def test_segments_not_summing_to_local_length_flagged():
    from paper_2605_06914_b200 import taper as T
    b = synth.make_batch([64, 32], [1, 2], [0, 0, 0], 1e3, 0.0)
    b = synth.with_segments(b, [[10, 20], [5], [7]])
    b.seg_len = b.seg_len.copy()
    b.seg_len[1] = 21  # slot 0: 10 + 21 != 30
    db = T.DeviceBatch.from_host(b)
    adm = T.DeviceAdmission.empty(b.n_req, b.n_slot)
    ws = torch.empty(T.taper_workspace_size(2, 3, 8, 64), dtype=torch.uint8, device="cuda")
    T.taper_admit(db, (1.0, 0.1, 0.01), "eager", 0.8, adm, 8, ws)
    assert int(adm.status.item()) & T.TAPER_STATUS_BAD_LENGTH
    assert int(adm.n_adm.item()) == 0


def test_max_slots_capacity():
    """TAPER_MAX_SLOTS: 1024 requests x 4 branches = 4096 slots with short ragged contexts
    (thousands of work items); sampled slots x heads against the oracle, every admitted
    slot written."""
    rng = np.random.default_rng(31)
    R = 1024
    b = synth.make_batch(rng.integers(0, 300, R), np.full(R, 4), rng.integers(1, 90, 4 * R),
                         1e3, 0.0, rng=rng)
    case = Case(b, seed=8)
    adm, out, lse = case.run_gpu(policy="eager")
    assert int(adm.n_adm.item()) == 4096
    assert torch.isfinite(out.float()).all()
    slots = np.sort(rng.choice(4096, 96, replace=False))
    es, eh = np.repeat(slots, 2), np.tile([5, 60], len(slots))
    ref, ref_lse = case.run_oracle(es, eh)
    assert_close(out[es, eh].float().numpy(), ref, "max slots")


# ------------------------------------------------------------ KV append of the current token
@pytest.mark.parametrize("segmented", [False, True])
def test_append_kv_places_current_token(segmented):
    """taper_append_kv writes each ADMITTED slot's new K/V row at the last position of its
    context ([C-att-3]): last local token (last non-empty segment) for a branch, last shared
    token for a serial request; every other pool row is untouched, and the attention that
    follows matches the oracle on the updated cache."""
    from paper_2605_06914_b200 import taper as T
    rng = np.random.default_rng(41)
    b = synth.make_batch([70, 5, 130, 64], [1, 2, 2, 1], [0, 3, 64, 9, 1, 0], 1e3, 0.0, rng=rng)
    if segmented:
        b = synth.with_segments(b, [[], [1, 2], [64], [4, 5, 0], [1], []])
    b.req_slack_ms[:] = 1e3
    case = Case(b, page=16, seed=2)
    lay, ps = case.layout, 16
    dev = "cuda"
    db = T.DeviceBatch.from_host(b, dev)
    adm = T.DeviceAdmission.empty(b.n_req, b.n_slot, dev)
    ws = torch.empty(T.taper_workspace_size(b.n_req, b.n_slot, 8, 64), dtype=torch.uint8, device=dev)
    T.taper_admit(db, (1.0, 0.1, 1e-3), "off", 0.8, adm, 8, ws)  # protected slots only
    rpo, rp, spo, sp = T.page_tables_to_device(lay, dev)
    spg = None if lay.seg_page_off is None else \
        torch.as_tensor(np.concatenate([lay.seg_page_off, [0]]).astype(np.int32)).to(dev)
    k0, v0 = case.k.clone(), case.v.clone()
    kd, vd = case.k.to(dev), case.v.to(dev)
    kv = T.DeviceKV(kd, vd, rpo, rp, spo, sp, spg)
    g = torch.Generator().manual_seed(5)
    kn = torch.randn((b.n_slot, 8, 128), generator=g).bfloat16()
    vn = torch.randn((b.n_slot, 8, 128), generator=g).bfloat16()
    T.taper_append_kv(db, adm, kv, kn.to(dev), vn.to(dev))
    torch.cuda.synchronize()
    assert int(adm.status.item()) == 0
    mask = adm.slot_admitted.cpu().numpy()[:b.n_slot].astype(bool)
    assert 0 < mask.sum() < b.n_slot
    exp_k, exp_v = k0.clone(), v0.clone()
    off = b.req_slot_off
    for s in np.flatnonzero(mask):  # expected position, test-side
        r = int(np.searchsorted(off, s, side="right") - 1)
        if b.slot_local_len[s] > 0:
            if segmented:
                segs = [q for q in range(b.slot_seg_off[s], b.slot_seg_off[s + 1]) if b.seg_len[q] > 0]
                q = segs[-1]
                t = int(b.seg_len[q]) - 1
                page = lay.slot_pages[lay.seg_page_off[q] + t // ps]
            else:
                t = int(b.slot_local_len[s]) - 1
                page = lay.slot_pages[lay.slot_page_off[s] + t // ps]
        else:
            t = int(b.req_shared_len[r]) - 1
            page = lay.req_pages[lay.req_page_off[r] + t // ps]
        exp_k[page, :, t % ps] = kn[s]
        exp_v[page, :, t % ps] = vn[s]
    assert torch.equal(kd.cpu(), exp_k) and torch.equal(vd.cpu(), exp_v)
    # the step's attention on the updated cache
    case.k, case.v = exp_k, exp_v
    q = case.q.to(dev)
    out = torch.full_like(q, float("nan"))
    T.taper_decode_attention(db, adm, kv, q, out, None, case.scale, ws)
    torch.cuda.synchronize()
    _check_all(case, adm, out.cpu(), None, heads=[0, 21, 63], what="after append")


@pytest.mark.parametrize("heads", [(0, 3), (3, 8), (2, 7)])
def test_odd_head_counts(heads):
    """h_local need not divide 8 (the C ABI takes 1..8 heads): 3- and 5-head slices at an
    arbitrary head offset match the oracle (prefix split taper_chunk_tokens(Lsh, h))."""
    rng = np.random.default_rng(3)
    b = synth.make_batch([5000, 700, 64], [3, 1, 2], rng.integers(1, 200, 6).tolist(), 1e3, 0.0,
                         rng=rng)
    case = Case(b, page=64, seed=12)
    adm, out, lse = case.run_gpu(policy="eager", heads=heads)
    g0, g1 = heads
    sub = np.arange(8 * g0, 8 * g1)
    adm_slots = np.flatnonzero(adm.slot_admitted.cpu().numpy()[:b.n_slot])
    es, eh = np.meshgrid(adm_slots, np.arange(len(sub)), indexing="ij")
    es, eh = es.ravel(), eh.ravel()
    ref, _ = case.run_oracle(es, sub[eh])
    assert_close(out[es, eh].float().numpy(), ref, f"heads {heads}")


@pytest.mark.parametrize("name", ["c3", "c5"])
def test_full_size_one_rank_of_8_sampled(name):
    """BASELINE.json configs[2] / [4] at full size as one rank of the 8-GPU KV-head shard
    (h_local = 1, the launch configuration `bench.py --rank-of 8` times): sampled admitted
    slots x all 8 local Q heads against the oracle."""
    b = synth.config_batch(name, seed=1)
    case = Case(b, h_kv=1, seed=1)
    adm, out, lse = case.run_gpu(policy="eager")
    rng = np.random.default_rng(1)
    slots = np.sort(rng.choice(np.flatnonzero(adm.slot_admitted.cpu().numpy()[:b.n_slot]), 24,
                               replace=False))
    es, eh = np.repeat(slots, 8), np.tile(np.arange(8), len(slots))
    ref, ref_lse = case.run_oracle(es, eh)
    assert_close(out[es, eh].float().numpy(), ref, f"{name} rank of 8")
    np.testing.assert_allclose(lse[es, eh].numpy(), ref_lse, atol=2e-3, rtol=1e-4)


@pytest.mark.parametrize("name", ["c3", "c5"])
def test_full_size_h8_sampled(name):
    """BASELINE.json configs[2] / [4] at full size with all 8 KV heads on one GPU -- the launch
    configuration `bench.py --config c3 | c5` times (c3: 8-16 branches on 16-32k prefixes;
    c5: 256 requests, 1k-32k prefixes, ~11 GB of K/V): sampled admitted slots x 4 Q heads
    (one per pair of KV heads) against the oracle, every admitted slot finite."""
    b = synth.config_batch(name, seed=2)
    case = Case(b, h_kv=8, seed=2, device_kv=True)
    adm, out, lse = case.run_gpu(policy="eager")
    mask = adm.slot_admitted.cpu().numpy()[:b.n_slot]
    assert mask.all()
    assert torch.isfinite(out.float()).all()
    rng = np.random.default_rng(2)
    slots = np.sort(rng.choice(b.n_slot, 40, replace=False))
    heads = np.array([3, 20, 41, 62])
    es, eh = np.repeat(slots, len(heads)), np.tile(heads, len(slots))
    ref, ref_lse = case.run_oracle(es, eh)
    assert_close(out[es, eh].float().numpy(), ref, f"{name} h=8")
    np.testing.assert_allclose(lse[es, eh].numpy(), ref_lse, atol=2e-3, rtol=1e-4)


def test_branch_isolation_and_wide_schedule_invariance_bitwise():
    """Sec. 3.1 visibility rule / Lemma 1 on the GPU, bitwise: (a) perturbing the local KV of
    a slot's siblings leaves its output bits unchanged; (b) a 14-branch request admitted at
    width 14 (two branch groups of one chunk) or width 5 (one group) gives the common slots
    identical bits."""
    rng = np.random.default_rng(17)
    b = synth.make_batch([5000, 300], [14, 1], rng.integers(1, 300, 14).tolist() + [0], 1e3, 0.0,
                         rng=rng)
    case = Case(b, seed=4)
    adm_e, out_e, _ = case.run_gpu(policy="eager", with_lse=False)
    adm_c, out_c, _ = case.run_gpu(policy="cap", cap=5, with_lse=False)
    both = (adm_e.slot_admitted.cpu().numpy()[:b.n_slot] & adm_c.slot_admitted.cpu().numpy()[:b.n_slot]).astype(bool)
    assert both.sum() == 6
    assert torch.equal(out_e[both], out_c[both])
    # (a) perturb every sibling of slot 0 in its own local pages
    lay = case.layout
    for s in range(1, 14):
        for pg in lay.slot_pages[lay.slot_page_off[s]:lay.slot_page_off[s + 1]]:
            case.k[pg] = (case.k[pg].float() + 3.0).bfloat16()
            case.v[pg] = (case.v[pg].float() - 5.0).bfloat16()
    _, out_p, _ = case.run_gpu(policy="eager", with_lse=False)
    assert torch.equal(out_p[0], out_e[0])
    assert not torch.equal(out_p[1], out_e[1])


def test_build_work_from_broadcast_mask_matches_admit():
    """G > 1 path: every rank rebuilds its work list from rank 0's
    broadcast slot mask with taper_build_work.  From the mask alone it must reproduce
    taper_admit's adm_list / n_adm / widths and give bitwise the same attention output, also
    for a mask no policy of this batch would produce."""
    from paper_2605_06914_b200 import taper as T
    b = synth.config_batch("c2", seed=6, slack_min_ms=30.0)
    case = Case(b, seed=6)
    dev = "cuda"
    db = T.DeviceBatch.from_host(b, dev)
    ws = torch.empty(T.taper_workspace_size(b.n_req, b.n_slot, 8, T.max_chunk_slots(
        b.req_shared_len, b.req_slot_off, b.slot_local_len)), dtype=torch.uint8, device=dev)
    rpo, rp, spo, sp = T.page_tables_to_device(case.layout, dev)
    kv = T.DeviceKV(case.k.to(dev), case.v.to(dev), rpo, rp, spo, sp)
    q = case.q.to(dev)
    adm = T.DeviceAdmission.empty(b.n_req, b.n_slot, dev)
    T.taper_admit(db, (12.0, 0.03, 2e-5), "taper", 0.8, adm, 8, ws)
    out1 = torch.full_like(q, float("nan"))
    T.taper_decode_attention(db, adm, kv, q, out1, None, case.scale, ws)
    # a second admission object holding only the mask, as after ncclBroadcast
    adm2 = T.DeviceAdmission.empty(b.n_req, b.n_slot, dev)
    adm2.slot_admitted.copy_(adm.slot_admitted)
    ws.zero_()
    T.taper_build_work(db, adm2, 8, ws)
    out2 = torch.full_like(q, float("nan"))
    T.taper_decode_attention(db, adm2, kv, q, out2, None, case.scale, ws)
    torch.cuda.synchronize()
    n = int(adm.n_adm.item())
    assert 0 < n < b.n_slot and int(adm2.n_adm.item()) == n
    assert torch.equal(adm.adm_list[:n], adm2.adm_list[:n])
    assert torch.equal(adm.req_width, adm2.req_width)
    m = adm.slot_admitted.bool()[:b.n_slot].cpu()
    assert torch.equal(out1.cpu()[m], out2.cpu()[m])
    # an arbitrary mask (every request keeps >= 1 slot): parity with the oracle
    rng = np.random.default_rng(2)
    mask = (rng.random(b.n_slot) < 0.5).astype(np.uint8)
    mask[b.req_slot_off[:-1]] = 1
    adm3 = T.DeviceAdmission.empty(b.n_req, b.n_slot, dev)
    adm3.slot_admitted.copy_(torch.as_tensor(mask))
    T.taper_build_work(db, adm3, 8, ws)
    out3 = torch.full_like(q, float("nan"))
    T.taper_decode_attention(db, adm3, kv, q, out3, None, case.scale, ws)
    torch.cuda.synchronize()
    _check_all(case, adm3, out3.cpu(), None, heads=[3, 40], what="build_work mask")


@pytest.mark.parametrize("variant", ["flat", "peaked"])
def test_row_mode_widths_groups_and_invariance(variant):
    """Row mode (requests with >= 9 ready slots: 128 stacked rows on the MMA's M, P in TMEM,
    DESIGN.md Sec. 6; reading R-mode): 9 to 33 ready branches (one or three 16-branch groups
    per prefix chunk), ragged prefixes over several chunks, local segments crossing pages, and
    partial admission (Cap 1 / 2 / 5: a row item with 8-40 live rows of 128).  Every admitted
    row against the fp64 oracle, and the common slots bitwise equal across the admitted widths
    (Sec. 3.1 / Lemma 1: the mode depends on n_r, not on w_r)."""
    rng = np.random.default_rng(21)
    lsh = [5000, 300, 4097, 65, 1800, 9100]
    fan = [9, 13, 16, 17, 24, 33]
    loc = rng.integers(1, 400, size=sum(fan)).tolist()
    b = synth.make_batch(lsh, fan, loc, 1e3, 0.0, rng=rng)
    case = Case(b, page=64, seed=9, variant=variant)
    outs = {}
    for policy, cap in (("eager", 2), ("cap", 1), ("cap", 2), ("cap", 5)):
        adm, out, lse = case.run_gpu(policy=policy, cap=cap)
        mask = adm.slot_admitted.cpu().numpy()[:b.n_slot].astype(bool)
        _check_all(case, adm, out, lse, heads=range(0, 64, 3), what=f"row {variant} {policy}{cap}")
        outs[(policy, cap)] = (mask, out)
    m_e, o_e = outs[("eager", 2)]
    for key in (("cap", 1), ("cap", 2), ("cap", 5)):
        m, o = outs[key]
        both = torch.from_numpy(m & m_e)
        assert both.sum() > 0 and torch.equal(o[both], o_e[both]), key


def test_row_mode_one_rank_of_8_heads():
    """Row items on a rank holding one KV head (h = 1, 1024-token chunks at the batch size)
    match the same heads of the oracle."""
    rng = np.random.default_rng(23)
    b = synth.make_batch([3000, 12000], [11, 16], rng.integers(1, 300, size=27).tolist(), 1e3, 0.0, rng=rng)
    case = Case(b, seed=12)
    for g in (0, 5):
        adm, out, _ = case.run_gpu(policy="eager", heads=(g, g + 1), with_lse=False)
        slots = np.flatnonzero(adm.slot_admitted.cpu().numpy()[:b.n_slot])
        es, eh = np.repeat(slots, 8), np.tile(np.arange(8), len(slots))
        ref, _ = case.run_oracle(es, eh + 8 * g)
        assert_close(out[es, eh].float().numpy(), ref, f"row h=1 head {g}")
