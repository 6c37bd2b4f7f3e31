"""Pins for the admission oracle (oracle/taper_oracle.c: oracle_T, oracle_budget,
oracle_admit, oracle_bruteforce) against what PAPER.md fixes.

Every pin is independent of the oracle's own code path: worked values printed in
tests/golden/admission_examples.json (cited), brute force over all subsets,
the knapsack reduction of App. B, hand-built instances whose answer follows
from the definitions, and invariants (Sec. 3.3 progress and budget safety).
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "admission_examples.json")))


def _batch(Lsh, fanouts, Lloc, slack):
    b = synth.make_batch(Lsh, fanouts, Lloc, 0.0, 0.0)
    b.req_slack_ms = np.asarray(slack, np.float64)
    return b


def _admit(b, model, policy="taper", rho=0.8, cap=2, utility=None):
    return oracle.admit(b.req_shared_len, b.req_slot_off, b.req_slack_ms, b.slot_local_len,
                        model, policy, cap, rho, utility)


# ---------------------------------------------------------------- golden values
@pytest.mark.parametrize("ex", GOLD["predict"])
def test_predict_golden(ex):
    assert oracle.T(*ex["model"], ex["n"], ex["L"]) == pytest.approx(ex["expect"], abs=1e-12)


@pytest.mark.parametrize("ex", GOLD["budget"])
def test_budget_golden(ex):
    assert oracle.budget(ex["T0"], ex["min_slack"], ex["rho"]) == pytest.approx(ex["expect"],
                                                                                abs=1e-12)


def test_budget_through_admit_golden():
    # T0 = 5 + 0.05*2 + 0.001*(2000+2900) = 10 ms ; slacks {40, 60} ; rho 0.8 -> 34 ms
    b = _batch([2000, 2900], [1, 1], [0, 0], [40.0, 60.0])
    a = _admit(b, (5, 0.05, 0.001))
    assert a.T0 == pytest.approx(10.0, abs=1e-12)
    assert a.budget == pytest.approx(GOLD["budget"][0]["expect"], abs=1e-12)
    assert a.min_slack == 40.0


def test_externality_golden():
    ex = GOLD["externality"][0]
    # baseline: r0 (200) + r1 (300) + r2's protected branch (Lsh 0 + Lloc 100) -> n=3, L=600;
    # Eager adds r2's second branch with 100 context tokens.
    b = _batch([200, 300, 0], [1, 1, 2], [0, 0, 100, 100], [50, 50, 50])
    a = _admit(b, ex["model"], "eager")
    assert a.T0 == pytest.approx(oracle.T(*ex["model"], ex["base_n"], ex["base_L"]), abs=1e-12)
    assert a.E == pytest.approx(ex["expect"], abs=1e-12)


def test_protected_composition_golden():
    ex = GOLD["protected"][0]
    # a=0, b=1000, c=1 makes (n, L) readable from T0 = 1000 n + L (L < 1000).
    b = _batch(ex["contexts"], [1, 1, 1], [0, 0, 0], [50, 50, 50])
    a = _admit(b, (0.0, 1000.0, 1.0), "off")
    assert a.T0 == 1000.0 * ex["expect_n"] + ex["expect_L"]
    assert list(a.req_width) == [1, 1, 1]


def test_knapsack_golden_bruteforce():
    ex = GOLD["knapsack"][0]
    # App. B reduction: one request per item, one opportunistic branch each.
    # With (a,b,c) = (1, .5, .5) a branch of dL tokens costs .5 + .5 dL ms (exact binary
    # fractions), so dL = 2w - 1 gives marginal cost w.  T_max = T0 + W via rho=1.
    costs = [w for w, _ in ex["items_cost_value"]]
    values = [v for _, v in ex["items_cost_value"]]
    local = []
    for w in costs:
        local += [0, 2 * w - 1]
    T0 = 1 + 0.5 * 3
    b = _batch([0, 0, 0], [2, 2, 2], local, [T0 + ex["W"]] * 3)
    util = np.array([[0.0, v] for v in values])
    best, mask, n_opp, bud = oracle.bruteforce(b.req_shared_len, b.req_slot_off, b.req_slack_ms,
                                               b.slot_local_len, (1, .5, .5), 1.0, util)
    assert bud == T0 + ex["W"]
    assert n_opp == 3
    assert best == ex["expect"]
    assert mask == 0b110  # items 2 and 3


# ---------------------------------------------------------------- hand-built instances
def test_fixed_policies_definitions():
    # App. D: Off w=1; C2 w=min(n,2); C5 w=min(n,5); Eager w=n_r.
    b = _batch([100], [4], [3, 1, 2, 0], [1e9])
    assert list(_admit(b, (1, .1, .01), "off").req_width) == [1]
    assert list(_admit(b, (1, .1, .01), "cap", cap=2).req_width) == [2]
    assert list(_admit(b, (1, .1, .01), "cap", cap=5).req_width) == [4]
    assert list(_admit(b, (1, .1, .01), "eager").req_width) == [4]
    # Cap picks the protected slot plus the next one in canonical order (smallest Lloc).
    adm = _admit(b, (1, .1, .01), "cap", cap=2).slot_admitted
    assert list(adm) == [0, 1, 0, 1]


def test_protected_is_canonical_first_and_ties_lowest_index():
    # equal local lengths -> lowest slot index is protected (SPEC L279 tie-break)
    b = _batch([10], [3], [5, 5, 5], [0.0])
    a = _admit(b, (1, .1, .01), "taper")
    assert list(a.slot_admitted) == [1, 0, 0]
    b = _batch([10], [3], [7, 2, 5], [0.0])
    assert list(_admit(b, (1, .1, .01), "off").slot_admitted) == [0, 1, 0]


def test_planner_admits_cheaper_branch_only():
    # Two requests, one opportunistic branch each, marginal costs 3 ms and 5 ms,
    # budget - T0 = 4 ms  ->  admit the 3 ms branch only (Alg. 1).
    model = (5, 0.05, 0.001)
    b = _batch([2950, 4950], [2, 2], [0, 0, 0, 0], [0, 0])
    T0 = oracle.T(*model, 2, 2950 + 4950)
    b.req_slack_ms[:] = T0 + 4.0 / 0.8
    a = _admit(b, model, "taper", 0.8)
    assert list(a.req_width) == [2, 1]
    assert a.T_S == pytest.approx(T0 + 3.0, abs=1e-9) and a.T_S <= a.budget


def test_planner_no_slack_protected_only():
    model = (5, 0.05, 0.001)
    b = _batch([1000, 1000], [3, 3], [1, 2, 3, 1, 2, 3], [0, 0])
    T0 = oracle.T(*model, 2, 2002)
    b.req_slack_ms[:] = T0  # budget = T0
    a = _admit(b, model)
    assert list(a.req_width) == [1, 1] and a.E == 0.0 and a.budget == a.T0
    b.req_slack_ms[:] = T0 - 100.0  # slack below T0: still progress (clamp)
    a = _admit(b, model)
    assert list(a.req_width) == [1, 1] and a.budget == a.T0


def test_planner_budget_allows_two_of_three():
    model = (5, 0.05, 0.001)  # branch cost 0.05 + 0.001*950 = 1 ms
    b = _batch([950], [4], [0, 0, 0, 0], [0])
    T0 = oracle.T(*model, 1, 950)
    b.req_slack_ms[:] = T0 + 2.5  # rho = 1 -> room for 2.5 ms
    a = _admit(b, model, rho=1.0)
    assert list(a.req_width) == [3]


def test_weighted_counterexample_half_remark_false():
    # C-adm-12: App. B's "within 1/2" remark does not hold for Alg. 1 with weights.
    # A: weight 2, cost 1 ms ; B: weight 100, cost 100 ms ; room 100 ms.
    model = (1, .5, .5)
    b = _batch([0, 0], [2, 2], [0, 1, 0, 199], [0, 0])
    T0 = oracle.T(*model, 2, 0)
    b.req_slack_ms[:] = T0 + 100.0
    util = np.array([[0.0, 2.0], [0.0, 100.0]])
    g = _admit(b, model, rho=1.0, utility=util)
    best, *_ = oracle.bruteforce(b.req_shared_len, b.req_slot_off, b.req_slack_ms,
                                 b.slot_local_len, model, 1.0, util)
    assert list(g.req_width) == [2, 1]  # greedy takes A (utility 2)
    assert best == 100.0                # optimum takes B
    # knapsack instance: greedy 7 vs optimum 8
    T0k = 1 + 0.5 * 3
    bk = _batch([0, 0, 0], [2, 2, 2], [0, 5, 0, 7, 0, 3], [T0k + 6] * 3)
    gk = _admit(bk, model, rho=1.0, utility=np.array([[0, 4.], [0, 5.], [0, 3.]]))
    assert list(gk.req_width) == [2, 1, 2]


# ---------------------------------------------------------------- properties on random batches
def _scan_admit(b, model, rho):
    """Independent restatement of the claim the GPU kernel rests on (DESIGN.md
    "Alg. 1 as sort + scan"): for linear utility, Alg. 1 admits candidates in
    (dL, r, slot) order while T(n0+m, L0+S_m) <= budget."""
    a_, b_, c_ = (float(x) for x in model)
    T = lambda n, L: (a_ + b_ * float(n)) + c_ * float(L)
    off, Lloc, Lsh = b.req_slot_off, b.slot_local_len, b.req_shared_len
    adm = np.zeros(b.n_slot, np.uint8)
    n0 = L0 = 0
    ms = np.inf
    cands = []
    for r in range(b.n_req):
        slots = sorted(range(off[r], off[r + 1]), key=lambda s: (Lloc[s], s))
        if not slots:
            continue
        adm[slots[0]] = 1
        n0 += 1
        L0 += int(Lsh[r]) + int(Lloc[slots[0]])
        ms = min(ms, b.req_slack_ms[r])
        cands += [(int(Lsh[r]) + int(Lloc[s]), r, s) for s in slots[1:]]
    T0 = T(n0, L0)
    budget = T0 + rho * max(0.0, ms - T0) if n0 else T0
    cands.sort()
    n, L = n0, L0
    for dL, r, s in cands:
        if T(n + 1, L + dL) > budget:
            break
        n, L = n + 1, L + dL
        adm[s] = 1
    return adm, T(n, L), budget


@pytest.mark.parametrize("seed", range(4))
def test_random_invariants_and_bruteforce(seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(150):
        b = synth.random_small_batch(rng, max_req=5, max_fanout=4, max_shared=2000, max_local=40)
        model = (rng.uniform(0, 20), rng.uniform(1e-3, 0.1), rng.uniform(1e-5, 1e-2))
        rho = float(rng.uniform(0.05, 1.0))
        a = _admit(b, model, "taper", rho)
        # Sec. 3.3: every active request advances exactly >= 1 token
        assert (a.req_width >= 1).all()
        # Sec. 3.3: T(S) <= T0 + rho B_t  (budget safety, E <= rho B_t)
        assert a.T_S <= a.budget
        assert a.E == a.T_S - a.T0
        # width bookkeeping
        off = b.req_slot_off
        for r in range(b.n_req):
            assert a.req_width[r] == a.slot_admitted[off[r]:off[r + 1]].sum()
        # App. B: linear utility -> greedy count equals the exhaustive optimum
        best, *_ = oracle.bruteforce(b.req_shared_len, b.req_slot_off, b.req_slack_ms,
                                     b.slot_local_len, model, rho)
        assert best == a.req_width.sum() - b.n_req
        # Alg. 1 literal loop == sorted scan (bit-exact T(S))
        adm, ts, bud = _scan_admit(b, model, rho)
        assert bud == a.budget
        assert (adm == a.slot_admitted).all()
        assert ts == a.T_S
        # evaluation-count bound: <= 2 evaluations per candidate per iteration
        n_cand0 = int(((off[1:] - off[:-1]) > 1).sum())
        grants = int(a.req_width.sum() - b.n_req)
        assert a.n_evals <= 2 * n_cand0 * (grants + 1)


def test_monotone_in_rho_and_slack():
    rng = np.random.default_rng(7)
    for _ in range(200):
        b = synth.random_small_batch(rng)
        model = (rng.uniform(0, 20), rng.uniform(1e-3, 0.1), rng.uniform(1e-5, 1e-2))
        prev = None
        for rho in (0.1, 0.3, 0.5, 0.8, 1.0):
            adm = _admit(b, model, "taper", rho).slot_admitted
            if prev is not None:
                assert (adm >= prev).all()  # superset as the budget grows
            prev = adm
        eager = _admit(b, model, "eager").slot_admitted
        off = _admit(b, model, "off").slot_admitted
        assert (prev <= eager).all() and (off <= prev).all()


def test_empty_request_is_flagged_and_skipped():
    b = _batch([10, 20], [0, 2], [1, 2], [5.0, 50.0])
    a = _admit(b, (1, .1, .01), "eager")
    assert a.status == 1
    assert list(a.req_width) == [0, 2]
    assert a.min_slack == 50.0  # inactive request does not count


def test_zero_requests():
    b = _batch([], [], [], [])
    a = _admit(b, (3, .1, .01))
    assert a.T0 == 3.0 and a.budget == 3.0 and a.min_slack == np.inf


# ---- cascade-aware context counting (reading R-ctx)

def test_per_request_worked_example():
    """One request, prefix 1000, branches Lloc 10/20/30/40, T = 1 + 0.1 n + 0.001 L (ms),
    rho = 1, min slack 3.5 ms (budget 3.5).  Worked by hand:
      T0 = 1 + 0.1 + 0.001 * 1010 = 2.11.
      per sequence: +20 -> L 2030, T 3.23 <= 3.5; +30 -> L 3060, T 4.36 > 3.5: width 2.
      per request:  +20 -> L 1030, T 2.23; +30 -> 1060, 2.36; +40 -> 1100, 2.50: width 4."""
    args = ([1000], [0, 4], [3.5], [10, 20, 30, 40], (1.0, 0.1, 0.001))
    seq = oracle.admit(*args, policy="taper", rho=1.0, ctx="per_sequence")
    req = oracle.admit(*args, policy="taper", rho=1.0, ctx="per_request")
    assert seq.req_width.tolist() == [2] and seq.slot_admitted.tolist() == [1, 1, 0, 0]
    assert req.req_width.tolist() == [4] and req.slot_admitted.tolist() == [1, 1, 1, 1]
    assert abs(seq.T_S - 3.23) < 1e-12 and abs(req.T_S - 2.50) < 1e-12
    assert abs(req.T0 - 2.11) < 1e-12 and req.T0 == seq.T0  # S0 counts each prefix once anyway


def test_per_request_eager_closed_form():
    """Eager admits every slot; per-request counting makes T(S) = a + b S + c (sum Lsh +
    sum Lloc) -- each prefix once -- checked against integers summed here."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        b = synth.random_small_batch(rng, max_req=6, max_fanout=5, max_local=80)
        o = oracle.admit(b.req_shared_len, b.req_slot_off, b.req_slack_ms, b.slot_local_len,
                         (2.0, 0.25, 0.5), "eager", ctx="per_request")
        n = int(b.n_slot)
        L = int(np.sum(b.req_shared_len)) + int(np.sum(b.slot_local_len))
        assert o.T_S == (2.0 + 0.25 * n) + 0.5 * L


def test_per_request_greedy_is_optimal_and_dominates():
    """Linear utility, costs additive in (n, L): cheapest-first is optimal under any
    monotone threshold (theorem), so greedy == brute force also for the
    cascade-aware count; and per-request admits a superset of per-sequence (every
    candidate is cheaper, the budget is the same)."""
    rng = np.random.default_rng(11)
    for _ in range(200):
        b = synth.random_small_batch(rng, max_req=5, max_fanout=4, max_shared=2000, max_local=40)
        model = (rng.uniform(0, 20), rng.uniform(1e-3, 0.1), rng.uniform(1e-5, 1e-2))
        rho = float(rng.uniform(0.1, 1.0))
        req = oracle.admit(b.req_shared_len, b.req_slot_off, b.req_slack_ms, b.slot_local_len,
                           model, "taper", rho=rho, ctx="per_request")
        seq = oracle.admit(b.req_shared_len, b.req_slot_off, b.req_slack_ms, b.slot_local_len,
                           model, "taper", rho=rho, ctx="per_sequence")
        best, _, n_opp, budget = oracle.bruteforce(b.req_shared_len, b.req_slot_off,
                                                   b.req_slack_ms, b.slot_local_len, model,
                                                   rho=rho, ctx="per_request")
        assert req.req_width.sum() - b.n_req == best
        assert req.T_S <= budget
        assert np.all(req.slot_admitted >= seq.slot_admitted)


@pytest.mark.parametrize("kind", ["concave", "weighted", "plateau"])
def test_nonlinear_utility_greedy_feasible_and_bounded_by_optimum(kind):
    """App. B (L290-305) with operator utilities (L142): the literal Alg. 1 must return a
    feasible allocation (T(S) <= budget, progress for every request) whose utility never
    exceeds the exhaustive optimum.  The ratio greedy / optimum is reported, not asserted
    >= 1/2: the Remark's factor does not hold for plain density greedy [C-adm-12]."""
    rng = np.random.default_rng(23)
    ratios = []
    for _ in range(300):
        b = synth.random_small_batch(rng, max_req=5, max_fanout=4, max_local=40)
        if b.n_slot - b.n_req > 14:
            continue
        util = synth.utility_table(rng, b.n_req, 4, kind)
        model = (rng.uniform(0, 5), rng.uniform(1e-2, 0.5), rng.uniform(1e-4, 1e-2))
        rho = float(rng.uniform(0.1, 1.0))
        g = _admit(b, model, rho=rho, utility=util)
        best, _, _, budget = oracle.bruteforce(b.req_shared_len, b.req_slot_off, b.req_slack_ms,
                                               b.slot_local_len, model, rho, util)
        assert g.T_S <= g.budget and g.budget == budget
        assert (g.req_width >= 1).all()
        got = sum(util[r, min(int(g.req_width[r]) - 1, util.shape[1] - 1)] for r in range(b.n_req))
        assert got <= best + 1e-9
        if best > 0:
            ratios.append(got / best)
    assert len(ratios) > 40 and min(ratios) > 0.0
