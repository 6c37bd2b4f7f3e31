"""Pins for oracle_attention (oracle/taper_oracle.c) against what the paper and
the mathematics fix: an independent library routine (torch SDPA in fp64),
closed forms (single key, equal keys, GQA mapping via constant V), the cascade
identity (LSE merge of prefix and local partials == attention over the
concatenation), branch isolation (Sec. 3.1 visibility rule) and layout
invariance (page size)."""
import numpy as np
import pytest
import torch

import oracle
import synth


def _case(Lsh, fanouts, Lloc, page=16, h_kv=2, q_heads=16, d=32, seed=0, local_capacity=None):
    b = synth.make_batch(Lsh, fanouts, Lloc, 10.0, 0.0)
    lay = synth.make_layout(b, page, np.random.default_rng(seed), spare_pages=2,
                            local_capacity=local_capacity)
    k, v = synth.make_kv(lay.num_pages, h_kv, page, d, seed)
    q = synth.make_q(b.n_slot, q_heads, d, seed)
    return b, lay, k, v, q


def _gather(b, lay, pool, s, g):
    """Test-side materialisation of slot s's context for KV head g (torch indexing)."""
    off = b.req_slot_off
    r = int(np.searchsorted(off, s, side="right") - 1)
    page = lay.page_size
    rows = []
    for t in range(int(b.req_shared_len[r])):
        rows.append(pool[lay.req_pages[lay.req_page_off[r] + t // page], g, t % page])
    for t in range(int(b.slot_local_len[s])):
        rows.append(pool[lay.slot_pages[lay.slot_page_off[s] + t // page], g, t % page])
    return torch.stack(rows).double()


def _all_pairs(b, q_heads):
    es, eh = np.meshgrid(np.arange(b.n_slot), np.arange(q_heads), indexing="ij")
    return es.ravel(), eh.ravel()


def _run(b, lay, k, v, q, es, eh, scale=None):
    return oracle.attention(b.req_slot_off, b.req_shared_len, b.slot_local_len, lay.req_page_off,
                            lay.req_pages, lay.slot_page_off, lay.slot_pages, k, v, q, es, eh,
                            scale)


def test_matches_torch_sdpa_fp64():
    b, lay, k, v, q = _case([37, 70, 0], [1, 3, 2], [0, 5, 0, 17, 3, 9])
    es, eh = _all_pairs(b, q.shape[1])
    out, lse = _run(b, lay, k, v, q, es, eh)
    group = q.shape[1] // k.shape[1]
    for i, (s, hq) in enumerate(zip(es, eh)):
        K = _gather(b, lay, k, s, hq // group)
        V = _gather(b, lay, v, s, hq // group)
        qq = q[s, hq].double()
        ref = torch.nn.functional.scaled_dot_product_attention(
            qq[None, None, None], K[None, None], V[None, None])[0, 0, 0]
        np.testing.assert_allclose(out[i], ref.numpy(), rtol=1e-12, atol=1e-13)
        ref_lse = torch.logsumexp(K @ qq / np.sqrt(q.shape[2]), 0)
        assert abs(lse[i] - ref_lse.item()) < 1e-12


def test_single_key_returns_v0_exactly():
    b, lay, k, v, q = _case([1, 0], [1, 1], [0, 1])
    es, eh = _all_pairs(b, q.shape[1])
    out, lse = _run(b, lay, k, v, q, es, eh)
    for i, (s, hq) in enumerate(zip(es, eh)):
        V = _gather(b, lay, v, s, hq // 8)
        assert (out[i] == V[0].numpy()).all()


def test_equal_keys_give_mean_of_values():
    b, lay, k, v, q = _case([50], [2], [0, 13])
    k[:] = k[0, 0, 0]  # every key identical -> uniform softmax
    es, eh = _all_pairs(b, q.shape[1])
    out, lse = _run(b, lay, k, v, q, es, eh)
    for i, (s, hq) in enumerate(zip(es, eh)):
        V = _gather(b, lay, v, s, hq // 8)
        np.testing.assert_allclose(out[i], V.mean(0).numpy(), rtol=0, atol=1e-13)
        assert abs(lse[i] - (float(q[s, hq].double() @ k[0, 0, 0].double()) / np.sqrt(32)
                             + np.log(len(V)))) < 1e-12


def test_gqa_mapping_constant_v_per_head():
    # C-att-2: q head hq reads KV head hq // group.  Set V of KV head g to the constant g.
    b, lay, k, v, q = _case([40, 10], [1, 2], [0, 3, 4], h_kv=4, q_heads=32)
    for g in range(4):
        v[:, g] = float(g)
    es, eh = _all_pairs(b, 32)
    out, _ = _run(b, lay, k, v, q, es, eh)
    np.testing.assert_allclose(out, (eh // 8)[:, None] * np.ones((1, 32)), atol=1e-12)


def test_cascade_identity_lse_merge():
    # A8: merging the prefix-only and local-only partials by log-sum-exp equals
    # attention over the concatenation (the cascade kernel's contract).
    b, lay, k, v, q = _case([64, 33], [2, 3], [7, 1, 20, 0, 5])
    es, eh = _all_pairs(b, q.shape[1])
    full, lse_full = _run(b, lay, k, v, q, es, eh)
    # prefix-only: zero local lengths; local-only: zero shared lengths (same pages)
    import copy
    bp = copy.deepcopy(b)
    bp.slot_local_len = np.zeros_like(b.slot_local_len)
    bl = copy.deepcopy(b)
    bl.req_shared_len = np.zeros_like(b.req_shared_len)
    o1, l1 = _run(bp, lay, k, v, q, es, eh)
    has_loc = b.slot_local_len[es] > 0
    o2 = np.zeros_like(o1)
    l2 = np.full_like(l1, -np.inf)
    if has_loc.any():
        o2[has_loc], l2[has_loc] = _run(bl, lay, k, v, q, es[has_loc], eh[has_loc])
    lse = np.logaddexp(l1, l2)
    merged = np.exp(l1 - lse)[:, None] * o1 + np.exp(l2 - lse)[:, None] * o2
    np.testing.assert_allclose(merged, full, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(lse, lse_full, rtol=1e-13, atol=1e-13)


def test_branch_isolation_sibling_perturbation():
    # Sec. 3.1 visibility rule / Lemma 1: a branch never sees sibling tokens.
    b, lay, k, v, q = _case([48], [3], [10, 20, 30])
    es, eh = _all_pairs(b, q.shape[1])
    out, _ = _run(b, lay, k, v, q, es, eh)
    k2, v2 = k.clone(), v.clone()
    for s in (1, 2):  # perturb siblings of slot 0
        for p in lay.slot_pages[lay.slot_page_off[s]:lay.slot_page_off[s + 1]]:
            k2[p] += 3.0
            v2[p] -= 5.0
    out2, _ = _run(b, lay, k2, v2, q, es, eh)
    m0 = es == 0
    assert (out2[m0] == out[m0]).all()
    assert not np.allclose(out2[~m0], out[~m0])


def test_page_size_invariance():
    b = synth.make_batch([100, 7], [2, 1], [9, 40, 0], 10.0, 0.0)
    res = []
    for page in (8, 16, 64):
        lay = synth.make_layout(b, page, np.random.default_rng(page))
        k = torch.zeros((lay.num_pages, 1, page, 16), dtype=torch.bfloat16)
        v = torch.zeros_like(k)
        # write the same logical tokens into each layout
        g = torch.Generator().manual_seed(3)
        Ksh = [torch.randn(int(b.req_shared_len[r]), 16, generator=g).bfloat16() for r in range(2)]
        Kl = [torch.randn(int(b.slot_local_len[s]), 16, generator=g).bfloat16() for s in range(3)]
        for r in range(2):
            for t in range(int(b.req_shared_len[r])):
                p = lay.req_pages[lay.req_page_off[r] + t // page]
                k[p, 0, t % page] = Ksh[r][t]
                v[p, 0, t % page] = -Ksh[r][t]
        for s in range(3):
            for t in range(int(b.slot_local_len[s])):
                p = lay.slot_pages[lay.slot_page_off[s] + t // page]
                k[p, 0, t % page] = Kl[s][t]
                v[p, 0, t % page] = 2 * Kl[s][t]
        q = synth.make_q(3, 8, 16, 5)
        es, eh = _all_pairs(b, 8)
        res.append(_run(b, lay, k, v, q, es, eh)[0])
    assert (res[0] == res[1]).all() and (res[1] == res[2]).all()


def test_planted_dominant_key():
    # one key with logit gap >= D over all others -> o = v* + O(n e^{-D})
    b, lay, k, v, q = _case([30], [1], [0], d=32, q_heads=8, h_kv=1)
    qq = q[0, 0].double()
    p0 = lay.req_pages[0]
    k[p0, 0, 0] = (qq / qq.norm() * 120.0).bfloat16()  # logit ~ 120*|q|/sqrt(32)
    out, lse = _run(b, lay, k, v, q, [0], [0])
    K = _gather(b, lay, k, 0, 0)
    x = (K @ qq / np.sqrt(32)).numpy()
    gap = x[0] - np.max(x[1:])
    assert gap > 20
    V = _gather(b, lay, v, 0, 0).numpy()
    assert np.abs(out[0] - V[0]).max() <= 30 * np.exp(-gap) * np.abs(V).max() + 1e-15


def test_empty_context_is_an_error():
    b, lay, k, v, q = _case([0], [1], [0])
    with pytest.raises(ValueError):
        _run(b, lay, k, v, q, [0], [0])


# ------------------------------------------------------------ multi-segment local context
# Sec. 3.1 (L104-107): a reduce step attends to P (+) H (+) every branch's h_i (+) y_i in
# canonical order (+) z; each branch's KV stays in its own pages (local segments).

def _seg_case(page=16, seed=4):
    b = synth.make_batch([40, 0, 23], [1, 1, 2], [0, 0, 0, 0], 10.0, 0.0)
    b = synth.with_segments(b, [[5, 17, 1, 9], [33, 2], [], [16]])
    lay = synth.make_layout(b, page, np.random.default_rng(seed), spare_pages=2)
    k, v = synth.make_kv(lay.num_pages, 2, page, 32, seed)
    q = synth.make_q(b.n_slot, 16, 32, seed)
    return b, lay, k, v, q


def _run_seg(b, lay, k, v, q, es, eh):
    return oracle.attention(b.req_slot_off, b.req_shared_len, b.slot_local_len, lay.req_page_off,
                            lay.req_pages, lay.slot_page_off, lay.slot_pages, k, v, q, es, eh,
                            None, b.slot_seg_off, b.seg_len, lay.seg_page_off)


def test_segments_match_torch_sdpa_fp64():
    b, lay, k, v, q = _seg_case()
    es, eh = _all_pairs(b, 16)
    out, lse = _run_seg(b, lay, k, v, q, es, eh)
    page = lay.page_size
    for i, (s, hq) in enumerate(zip(es, eh)):
        g = hq // 8
        r = int(np.searchsorted(b.req_slot_off, s, side="right") - 1)
        rows_k, rows_v = [], []
        for t in range(int(b.req_shared_len[r])):
            p = lay.req_pages[lay.req_page_off[r] + t // page]
            rows_k.append(k[p, g, t % page]); rows_v.append(v[p, g, t % page])
        for qs in range(b.slot_seg_off[s], b.slot_seg_off[s + 1]):  # segments in order
            for t in range(int(b.seg_len[qs])):
                p = lay.slot_pages[lay.seg_page_off[qs] + t // page]
                rows_k.append(k[p, g, t % page]); rows_v.append(v[p, g, t % page])
        K, V = torch.stack(rows_k).double(), torch.stack(rows_v).double()
        qq = q[s, hq].double()
        ref = torch.nn.functional.scaled_dot_product_attention(
            qq[None, None, None], K[None, None], V[None, None])[0, 0, 0]
        np.testing.assert_allclose(out[i], ref.numpy(), rtol=1e-12, atol=1e-13)
        assert abs(lse[i] - torch.logsumexp(K @ qq / np.sqrt(32), 0).item()) < 1e-12


def test_segments_equal_contiguous_copy():
    """The same logical tokens in per-segment pages and copied into one contiguous local
    segment give bit-identical outputs (the segment walk only locates tokens)."""
    b, lay, k, v, q = _seg_case()
    import copy
    bc = copy.deepcopy(b)
    bc.slot_seg_off = None
    bc.seg_len = None
    lay_c = synth.make_layout(bc, lay.page_size, np.random.default_rng(9), spare_pages=2)
    kc = torch.zeros((lay_c.num_pages,) + tuple(k.shape[1:]), dtype=k.dtype)
    vc = torch.zeros_like(kc)
    ps = lay.page_size
    for r in range(b.n_req):
        for t in range(int(b.req_shared_len[r])):
            src = lay.req_pages[lay.req_page_off[r] + t // ps]
            dst = lay_c.req_pages[lay_c.req_page_off[r] + t // ps]
            kc[dst, :, t % ps] = k[src, :, t % ps]; vc[dst, :, t % ps] = v[src, :, t % ps]
    for s in range(b.n_slot):
        u = 0
        for qs in range(b.slot_seg_off[s], b.slot_seg_off[s + 1]):
            for t in range(int(b.seg_len[qs])):
                src = lay.slot_pages[lay.seg_page_off[qs] + t // ps]
                dst = lay_c.slot_pages[lay_c.slot_page_off[s] + u // ps]
                kc[dst, :, u % ps] = k[src, :, t % ps]; vc[dst, :, u % ps] = v[src, :, t % ps]
                u += 1
    es, eh = _all_pairs(b, 16)
    o1, l1 = _run_seg(b, lay, k, v, q, es, eh)
    o2, l2 = _run(bc, lay_c, kc, vc, q, es, eh)
    assert (o1 == o2).all() and (l1 == l2).all()


def test_segments_must_sum_to_local_length():
    b, lay, k, v, q = _seg_case()
    b.seg_len = b.seg_len.copy()
    b.seg_len[0] += 1
    with pytest.raises(ValueError):
        _run_seg(b, lay, k, v, q, np.array([0]), np.array([0]))


def test_threads_do_not_change_bits():
    """oracle.set_threads only spreads independent (slot, head) pairs over host cores: the
    results are bit-identical to the serial evaluation."""
    b = synth.config_batch("c1", seed=3)
    lay = synth.make_layout(b, 16, np.random.default_rng(2), spare_pages=1)
    k, v = synth.make_kv(lay.num_pages, 8, 16, 128, seed=3)
    q = synth.make_q(b.n_slot, 64, 128, seed=3)
    es, eh = np.meshgrid(np.arange(b.n_slot), np.arange(0, 64, 5), indexing="ij")
    args = (b.req_slot_off, b.req_shared_len, b.slot_local_len, lay.req_page_off, lay.req_pages,
            lay.slot_page_off, lay.slot_pages, k, v, q, es.ravel(), eh.ravel())
    oracle.set_threads(1)
    o1, l1 = oracle.attention(*args)
    try:
        oracle.set_threads(4)
        o4, l4 = oracle.attention(*args)
    finally:
        oracle.set_threads(1)
    assert o1.tobytes() == o4.tobytes() and l1.tobytes() == l4.tobytes()
